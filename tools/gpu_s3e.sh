#!/bin/bash
O=gpurun_out/s3e; mkdir -p $O
./tools/microbench/gj_regs > $O/gj_regs.txt 2>&1
cat $O/gj_regs.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "als or bcd or fullsize or decompose" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for c in C2 C3 C5; do
  RCPG_PROFILE_ALS=1 timeout 600 python tools/profile_step.py --config $c --warmup 0 > $O/als_$c.log 2>&1; grep "rcpg als\]\|iters" $O/als_$c.log
done
bash tools/gpu_quick2.sh s3e_q notests
