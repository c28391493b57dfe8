#!/bin/bash
run() {
  env "$@" timeout 600 python bench.py $CFG --steps 5 --warmup 3 --no-scaling-config --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['value'],3), d['iterations'], d['relerr'], {k: round(v['ms_per_step'],3) for k,v in d['passes'].items() if k in ('als_init','als_iterations')})"
}
run X=1
run RCPG_ALS_CLUSTER=0
CFG="--config C1" run X=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bcd.py -q -x 2>&1 | tail -2
