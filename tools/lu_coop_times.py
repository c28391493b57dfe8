"""plu_basis device time of the grid (coop) LU on the big W panels."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_09074_b200 as rcp
ctx = rcp.default_context()
out = []
for dt, rows, cols in [(0, 8388608, 48), (0, 3145728, 48), (0, 1048576, 70), (0, 500000, 80), (0, 1179648, 48)]:
    ms = C.c_double()
    st = ctx.lib.rcpg_bench_factor(ctx.h, dt, 0, rows, cols, 3, C.byref(ms))
    out.append(f"{rows}x{cols}: {ms.value * 1e3:.0f}" if st == 0 else f"{rows}x{cols}: err{st}")
print(" | ".join(out), flush=True)
