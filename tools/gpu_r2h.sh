#!/bin/bash
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 2>&1 | tail -5
for i in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-scaling-config 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', round(d['value'],3), d['iterations'], d['parity']['pass'], d['gpu_launches'], d['roofline']['frac'], d['e2e']['value'], {k: round(v['ms_per_step'],3) for k,v in d['passes'].items()})"
done
RCPG_NO_GRAPH=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-scaling-config --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 nograph', round(d['value'],3), d['gpu_launches'])"
for c in C1 C3 C4 C5; do
timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-scaling-config --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['value'],3), d['iterations'], d['gpu_launches'], d['roofline']['frac'], d['e2e']['value'])"
done
