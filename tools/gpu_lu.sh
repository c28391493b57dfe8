timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "plu" > gpurun_out/pytest_lu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_lu.log
rm -f gpurun_out/lu_paths.txt
for p in "" onchip; do for s in "0 400 30" "0 100 20" "0 900 30" "0 128 48" "0 512 48" "0 1000 80" "0 1024 70"; do echo "path=$p $s: $(RCPG_LU_PATH=$p python tools/one_factor.py $s)" >> gpurun_out/lu_paths.txt; done; done
