#!/bin/bash
for t in "" 2 4; do echo "TPR=${t:-1}"; RCPG_LU_TPR=$t timeout 300 python tools/lu_default_times.py; done
for r in 128 256 512; do echo "HH_ROWS=$r"; RCPG_HH_ROWS=$r timeout 300 python - <<'PY'
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import paper_1703_09074_b200 as rcp
ctx = rcp.default_context()
out=[]
for dt, rows, cols in [(0, 10000, 80), (0, 1024, 70), (0, 1000, 80), (0, 128, 48)]:
    ms = C.c_double()
    st = ctx.lib.rcpg_bench_factor(ctx.h, dt, 1, rows, cols, 5, C.byref(ms))
    out.append(f"qr {rows}x{cols}: {ms.value*1e3:.1f}" if st == 0 else f"{rows}x{cols}: err{st}")
print(" | ".join(out))
PY
done
