#!/bin/bash
# Round measurements: tests, bench lines C1-C5 (+ cpu_baseline / parity),
# the reference arm, ncu launch lists and full captures (exported to CSV on the box).
TAG=${1:-r02s5}
O=gpurun_out/$TAG; mkdir -p $O; T=/tmp/$TAG; mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py --impl reference > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err
for c in C1 C3 C4 C5; do
  timeout 1500 python bench.py --config $c --no-scaling-config > $O/bench_$c.json 2> $O/bench_$c.err
done
for c in C2 C3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-scaling-config > $O/ncu_launches_$c.log 2>&1
done
cap() {  # name config kernel-regex
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$3 -s 0 -c 1 -o $T/$1 \
    python tools/profile_step.py --config $2 --warmup 0 > $O/ncu_$1.log 2>&1
  ncu -i $T/$1.ncu-rep --page details --csv > $O/ncu_$1_details.csv 2>/dev/null
  ncu -i $T/$1.ncu-rep --page source --csv --print-source sass,cuda 2>/dev/null | gzip > $O/ncu_$1_source.csv.gz
}
cap C2_sketch C2 sketch_dmma_tma
cap C3_sketch_f32 C3 sketch_dmma_tma
cap C2_resident_lu C2 plu_resident
cap C4_coop_lu C4 plu_coop
cap C5_residual_tc C5 residual_tc
cap C5_als C5 als_loop
ls -la $O
cap C2_als C2 als_loop
cap C2_init C2 init_from_gram
cap C2_residual C2 residual_dmma
cap C2_reglu C2 plu_reg
for n in C2_sketch C3_sketch_f32 C2_resident_lu C4_coop_lu C5_residual_tc C5_als C2_als C2_init C2_residual C2_reglu; do
  python tools/ncu_src_top.py $O/ncu_${n}_source.csv.gz 40 > $O/ncu_${n}_source_top.txt 2>/dev/null
done
for c in C2 C3; do python tools/launch_summary.py $O/ncu_launches_$c.csv > $O/ncu_launches_${c}_summary.txt 2>/dev/null; done
