#!/bin/bash
# ncu source-level captures of C2's latency kernels (ALS loop, init, residual, reg LU)
O=gpurun_out/ncu_c2; mkdir -p $O; T=/tmp/ncu_c2; mkdir -p $T
cap() {  # name config kernel-regex
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$3 -s 0 -c 1 -o $T/$1 \
    python tools/profile_step.py --config $2 --warmup 0 > $O/ncu_$1.log 2>&1
  ncu -i $T/$1.ncu-rep --page details --csv > $O/ncu_$1_details.csv 2>/dev/null
  ncu -i $T/$1.ncu-rep --page source --csv --print-source sass,cuda 2>/dev/null | gzip > $O/ncu_$1_source.csv.gz
  python tools/ncu_src_top.py $O/ncu_$1_source.csv.gz 40 > $O/ncu_$1_source_top.txt
}
cap C2_als C2 als_loop
cap C2_init C2 init_from_gram
cap C2_residual C2 residual_dmma
cap C2_reglu C2 plu_reg
ls -la $O
