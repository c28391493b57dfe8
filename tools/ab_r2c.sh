#!/bin/bash
run() {
  env "$@" timeout 600 python bench.py $CFG --steps 5 --warmup 3 --no-scaling-config --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$CFG $*', round(d['value'],3), d['iterations'], d['relerr'], {k: round(v['ms_per_step'],3) for k,v in d['passes'].items() if k in ('relerr',)})"
}
run X=1
run RCPG_RESID_ROWS64=1
CFG="--config C1" run X=1
CFG="--config C1" run RCPG_RESID_ROWS64=1
timeout 900 python -m pytest tests/test_gpu_passes.py tests/test_gpu_fullsize.py -q -x -k "relative or C1 or C2" 2>&1 | tail -2
