#!/bin/bash
O=gpurun_out/${TAG:-s3f}; mkdir -p $O
./tools/microbench/gj_regs 2>&1 | head -9
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for c in C3 C5 C4; do
  RCPG_PROFILE_ALS=1 RCPG_PROFILE_LU=1 timeout 600 python tools/profile_step.py --config $c --warmup 0 > $O/prof_$c.log 2>&1; grep "rcpg als\]\|rcpg als grid\|iters" $O/prof_$c.log
done
bash tools/gpu_quick2.sh ${TAG:-s3f}_q notests
