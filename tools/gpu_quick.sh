#!/bin/bash
# quick loop: GPU tests (subset via $TESTS or all), then bench lines for $CFGS (default C2) with parity
TAG=${TAG:-quick}; O=gpurun_out/$TAG; mkdir -p $O
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
for c in ${CFGS:-C2}; do
  timeout 1500 python bench.py --config $c --no-scaling-config --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
  python - $O/bench_$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d['config']['workload'][:3], 'value', round(d['value'],4), 'frac', round(d['roofline']['frac'],3), 'parity', d.get('parity',{}).get('pass'), 'iters', d['iterations'])
print({k:round(v['ms_per_step'],3) for k,v in d['passes'].items()})
PY
done
