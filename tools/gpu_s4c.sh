#!/bin/bash
# register LU: parity, times with / without, per-phase cycles (profiling build)
O=gpurun_out/s4c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "plu" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for env in "RCPG_LU_REG=0" "RCPG_LU_REG=1" "RCPG_LU_REG_RPT=2"; do
  echo "$env"; env $env timeout 300 python tools/lu_default_times.py
done 2>&1 | tee $O/times.txt
for spec in "400 30 1" "900 30 1" "12000 30 1" "1024 70 0" "128 48 0" "10000 80 0"; do
  RCPG_LIB=$PWD/paper_1703_09074_b200/librcpg_luprof.so timeout 60 python tools/one_factor.py 0 $spec 2>&1 | tail -1
done | tee $O/phases.txt
