#!/bin/bash
# Round-2 measurements: bench lines C1-C5 (+ cpu_baseline / parity), the reference arm,
# ncu launch lists and full captures of the dominant pass kernels. Usage: bash tools/measure_round2.sh TAG
TAG=${1:-r2v1}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
for c in C1 C3 C4 C5; do
  timeout 1200 python bench.py --config $c --no-scaling-config > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err
for c in C2 C3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-scaling-config > $O/ncu_launches_$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sketch_dmma_tma -s 0 -c 1 -o $O/C2_sketch_full \
  python bench.py --config C2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-scaling-config > $O/ncu_full_C2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sketch_dmma_tma -s 0 -c 1 -o $O/C3_sketch_f32_full \
  python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-scaling-config > $O/ncu_full_C3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:plu_coop -s 0 -c 1 -o $O/C4_lu_full \
  python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-scaling-config > $O/ncu_full_C4.log 2>&1
ls -la $O
