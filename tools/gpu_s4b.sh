#!/bin/bash
# register-resident LU: parity of the LU paths, then plu_basis times with / without it
O=gpurun_out/s4b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "plu" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for env in "RCPG_LU_REG=0" "RCPG_LU_REG=1" "RCPG_LU_REG_RPT=2" "RCPG_LU_REG_CS=16"; do
  echo "$env"; env $env timeout 300 python tools/lu_default_times.py
done 2>&1 | tee $O/times.txt
