#!/bin/bash
# ncu full captures of C2's LU kernels (resident 160000x30, onchip 400x30, cluster 12000x30);
# exported to CSV on the box (the .ncu-rep files are too large to bring back)
O=gpurun_out/s3c; mkdir -p $O; T=/tmp/s3c; mkdir -p $T
for k in plu_resident plu_onchip plu_cluster cqr2_coop init_from_gram; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 0 -c 1 -o $T/C2_$k \
    python tools/profile_step.py --config C2 --warmup 0 > $O/ncu_$k.log 2>&1
  ncu -i $T/C2_$k.ncu-rep --page details --csv > $O/C2_${k}_details.csv 2>/dev/null
  ncu -i $T/C2_$k.ncu-rep --page source --csv --print-source sass,cuda > $O/C2_${k}_source.csv 2>/dev/null
done
gzip -f $O/*_source.csv
ls -la $O
