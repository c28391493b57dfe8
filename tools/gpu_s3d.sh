#!/bin/bash
# LU phase profile (all stab_w calls) + ALS with the pinv on CTA 0 (GJ stamp) for C3, C5, C4
O=gpurun_out/s3d; mkdir -p $O
for c in C3 C5 C4; do
  RCPG_PROFILE_LU=1 timeout 600 python tools/profile_step.py --config $c --warmup 0 > $O/lu_$c.log 2>&1
  RCPG_PROFILE_ALS=1 RCPG_ALS_SPLIT=0 timeout 600 python tools/profile_step.py --config $c --warmup 0 > $O/als_$c.log 2>&1
done
for f in $O/*.log; do echo "== $f"; cat $f; done
