#!/bin/bash
# wave-tail probe: fp64 project pass (K = 400, l = 30) at 4.0 / 4.22 / 4.5 / 5.0 waves of 592 resident CTAs
O=gpurun_out/wave_tail; mkdir -p $O
for R in 151552 160000 170496 189440; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:project_dmma --csv --log-file $O/p_$R.csv \
    python tools/pass_bench.py project 1 400 $R 30 f64 3 > /dev/null 2>&1
  python - $O/p_$R.csv $R <<'PY'
import csv,sys
lines=[l for l in open(sys.argv[1]) if l.startswith('"')]
v=[float(x['Metric Value'])/1000 for x in csv.DictReader(lines)]
R=int(sys.argv[2]); print(R, 'tiles', (R+63)//64, 'waves', round((R+63)//64/592,2), 'us', v, 'ns/row', round(1000*min(v)/R,4))
PY
done
