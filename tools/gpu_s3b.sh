#!/bin/bash
# phase profiles (ALS / QR / LU stamps) for C2, C3, C5
O=gpurun_out/s3b; mkdir -p $O
for c in C2 C3 C5 C4; do
  RCPG_PROFILE_ALS=1 RCPG_PROFILE_QR=1 RCPG_PROFILE_LU=1 timeout 600 python tools/profile_step.py --config $c > $O/prof_$c.log 2>&1
done
for f in $O/prof_*.log; do tail -n 12 $f; done
