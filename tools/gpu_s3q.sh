#!/bin/bash
for lib in "" "$PWD/paper_1703_09074_b200/librcpg_t512.so" "$PWD/paper_1703_09074_b200/librcpg_t1024.so"; do
  echo "lib=${lib:-default}"; RCPG_LIB=$lib timeout 300 python tools/lu_default_times.py
done
