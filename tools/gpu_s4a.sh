#!/bin/bash
# ncu source-level captures of the small-panel factorizations (C2's 400 x 30 LU / QR, 900 x 30, 12000 x 30 LU)
O=gpurun_out/s4a; mkdir -p $O
python tools/one_factor.py 0 400 30 1 > $O/plain.txt 2>&1
python tools/one_factor.py 1 400 30 1 >> $O/plain.txt 2>&1
python tools/one_factor.py 0 12000 30 1 >> $O/plain.txt 2>&1
for spec in "0 400 30 lu400" "1 400 30 qr400" "0 12000 30 lu12k"; do
  set -- $spec
  timeout 300 ncu --set full --import-source on --clock-control none -c 1 -k regex:'plu|householder|cqr' \
    -o $O/$4 python tools/one_factor.py $1 $2 $3 1 > $O/$4.log 2>&1
  ncu -i $O/$4.ncu-rep --page source --csv --print-source sass,cuda > $O/$4_src.csv 2>/dev/null
  ncu -i $O/$4.ncu-rep --page details --csv > $O/$4_details.csv 2>/dev/null
  python tools/ncu_src_top.py $O/$4_src.csv 30 > $O/$4_top.txt
  gzip -f $O/$4_src.csv; rm -f $O/$4.ncu-rep
done
