#!/bin/bash
O=gpurun_out/s3n; mkdir -p $O
echo "== tagged"; timeout 600 python tools/lu_tag_ab.py 2>&1 | tee $O/tag.txt
echo "== barrier"; RCPG_LU_BARRIER=1 timeout 600 python tools/lu_tag_ab.py 2>&1 | tee $O/bar.txt
