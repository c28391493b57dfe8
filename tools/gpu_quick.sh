# quick GPU check: factor/pass tests, factor timings, C2 bench (args: extra pytest -k filter)
timeout 600 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
python tools/bench_factor.py > gpurun_out/bf.txt 2>&1
RCPG_PROFILE_QR=1 python tools/one_factor.py 1 400 30 > gpurun_out/qr_prof.txt 2>&1
RCPG_PROFILE_QR=1 python tools/one_factor.py 1 1024 70 0 >> gpurun_out/qr_prof.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
RCPG_PROFILE_ALS=1 python tools/profile_step.py --config C2 > gpurun_out/als_prof.txt 2>&1
