#!/bin/bash
O=gpurun_out/s3p; mkdir -p $O; T=/tmp/s3p; mkdir -p $T
cap() {  # name config kernel-regex [skip]
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$3 -s ${4:-0} -c 1 -o $T/$1 \
    python tools/profile_step.py --config $2 --warmup 0 > $O/ncu_$1.log 2>&1
  ncu -i $T/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>/dev/null
  ncu -i $T/$1.ncu-rep --page source --csv --print-source sass,cuda 2>/dev/null | gzip > $O/$1_source.csv.gz
}
cap lucoop_C4 C4 plu_coop
cap als_C4 C4 als_loop
cap sketch_C3 C3 sketch_dmma_tma
ls -la $O
