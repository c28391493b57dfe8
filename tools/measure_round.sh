# Round measurements: bench lines for C1-C5 and the reference arm, ncu launch lists, one full
# capture of C2's dominant streamed-pass kernel. Usage: bash tools/measure_round.sh TAG
TAG=${1:-v4}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
for c in C2 C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err
for c in C2 C3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_launches_$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sketch_dmma_tma -s 0 -c 1 -o $O/C2_sketch_full \
  python bench.py --config C2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_full_C2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_pass_kernel -s 0 -c 1 -o $O/C3_tc_full \
  python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_full_C3.log 2>&1
