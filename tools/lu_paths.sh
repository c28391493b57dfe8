# LU path timings (device time per call) on the C1/C2 panel shapes
rm -f gpurun_out/lu_paths.txt
for p in "" rcluster cluster resident; do for s in "0 400 30" "0 900 30" "0 12000 30" "0 160000 30" "0 100 20" "0 400 20"; do
  echo "path=$p $s: $(RCPG_LU_PATH=$p python tools/one_factor.py $s)" >> gpurun_out/lu_paths.txt; done; done
