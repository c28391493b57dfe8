timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
for c in C2 C5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_x.json 2> gpurun_out/bench_${c}_x.err; done
