for g in 0 1 2 3 4 6 8 12; do
  RCPG_ALS_MAXG=$g timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e --no-scaling-config --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('G cap', $g, 'value', round(d['value'],4), 'als', round(d['passes']['als_iterations']['ms_per_step'],4), 'iters', d['iterations'], 'relerr', d['relerr'])"
done
for g in 0 4 8; do
  RCPG_ALS_MAXG=$g timeout 300 python bench.py --config C1 --no-cpu-baseline --no-e2e --no-scaling-config --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C1 G cap', $g, 'value', round(d['value'],4), 'als', round(d['passes']['als_iterations']['ms_per_step'],4), 'iters', d['iterations'], 'relerr', d['relerr'])"
done
