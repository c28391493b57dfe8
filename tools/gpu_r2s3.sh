#!/bin/bash
# session-3 state check: GPU tests + default bench line
O=gpurun_out/s3a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
tail -3 $O/pytest_gpu.log
