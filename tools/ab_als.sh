for lib in "" "$PWD/paper_1703_09074_b200/librcpg_ab.so" ""; do
  echo "lib=$lib" >> gpurun_out/ab_als.txt
  RCPG_LIB=$lib RCPG_PROFILE_ALS=1 python tools/profile_step.py --config C4 2>&1 | tail -4 >> gpurun_out/ab_als.txt
  RCPG_LIB=$lib python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['passes']['als_iterations'])" >> gpurun_out/ab_als.txt
done
