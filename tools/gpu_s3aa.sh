#!/bin/bash
for c in C4 C5 C3; do
  for p in "" general; do
    RCPG_ALS_PATH=$p timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-scaling-config > /tmp/b.json 2>/dev/null
    python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$c', '${p:-loop}', round(d['value'],2), d['iterations'], round(d['passes']['als_iterations']['ms_per_step'],3), d['relerr'])"
  done
done
