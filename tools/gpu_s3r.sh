#!/bin/bash
for lib in "" pf4m3 pf8m2 pf4m2; do
  L=""; [ -n "$lib" ] && L=$PWD/paper_1703_09074_b200/librcpg_$lib.so
  echo "lib=${lib:-default}"; RCPG_LIB=$L timeout 300 python tools/lu_coop_times.py
done
echo "cluster 256/512 default:"; timeout 300 python tools/lu_default_times.py
