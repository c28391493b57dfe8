#!/bin/bash
# launch lists (C2, C4) + full captures: omega (C4), residual_dmma (C2), residual_tc (C5), resident LU (C2)
O=gpurun_out/s3k; mkdir -p $O; T=/tmp/s3k; mkdir -p $T
for c in C2 C4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python tools/profile_step.py --config $c --warmup 0 > $O/launches_$c.log 2>&1
done
cap() {  # name config kernel-regex
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$3 -s 0 -c 1 -o $T/$1 \
    python tools/profile_step.py --config $2 --warmup 0 > $O/ncu_$1.log 2>&1
  ncu -i $T/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>/dev/null
  ncu -i $T/$1.ncu-rep --page source --csv --print-source sass,cuda 2>/dev/null | gzip > $O/$1_source.csv.gz
}
cap omega_C4 C4 omega_pairs
cap resid_C2 C2 residual_dmma
cap resid_C5 C5 residual_tc
cap hh_C5 C5 householder_cluster
ls -la $O
