#!/bin/bash
# ncu full captures of C2's LU kernels (resident 160000x30, onchip 400x30, cluster 12000x30)
O=gpurun_out/s3c; mkdir -p $O
for k in plu_resident plu_onchip plu_cluster cqr2_coop init_from_gram; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 0 -c 1 -o $O/C2_$k \
    python tools/profile_step.py --config C2 --warmup 0 > $O/ncu_$k.log 2>&1
done
ls -la $O
