timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
for c in C3 C5 C4; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_${c}_tc.json 2> gpurun_out/bench_${c}_tc.err; done
