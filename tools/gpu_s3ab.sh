#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/gpu_quick2.sh s3ab_q notests
echo "== no chunks"; RCPG_OMEGA_CHUNKS=1 bash tools/gpu_quick2.sh s3ab_q1 notests
