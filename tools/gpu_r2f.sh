#!/bin/bash
# round-2 ncu launch lists (C2, C3 faithful) -- per-kernel device times, cold/serialised
O=gpurun_out/r2f; mkdir -p $O
for c in C2 C3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-scaling-config > $O/ncu_launches_$c.log 2>&1
  python tools/launch_summary.py $O/ncu_launches_$c.csv 30
done
