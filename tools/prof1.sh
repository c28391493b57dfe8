set -x
python tools/bench_factor.py > gpurun_out/bf_default.txt 2>&1
for p in smem coop householder; do RCPG_QR_PATH=$p python tools/one_factor.py 1 400 30 >> gpurun_out/qr_paths.txt 2>&1; echo "^ $p 400" >> gpurun_out/qr_paths.txt; RCPG_QR_PATH=$p python tools/one_factor.py 1 1024 70 0 >> gpurun_out/qr_paths.txt 2>&1; echo "^ $p 1024x70 f32" >> gpurun_out/qr_paths.txt; done
RCPG_PROFILE_QR=1 python tools/one_factor.py 1 400 30 > gpurun_out/qr_prof.txt 2>&1
for t in 1 2 ; do RCPG_LU_TPR=$t python tools/one_factor.py 0 400 30 >> gpurun_out/lu_tpr.txt 2>&1; RCPG_LU_TPR=$t python tools/one_factor.py 0 900 30 >> gpurun_out/lu_tpr.txt 2>&1; done
RCPG_PROFILE_ALS=1 python tools/profile_step.py --config C2 > gpurun_out/als_prof.txt 2>&1
