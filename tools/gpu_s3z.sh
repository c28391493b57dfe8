#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 300 python tools/lu_tag_ab.py 2>&1 | head -3
bash tools/gpu_quick2.sh s3z_q notests
