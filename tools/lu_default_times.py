"""plu_basis device time on the default path for the panels the cluster LU serves."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_09074_b200 as rcp
ctx = rcp.default_context()
out = []
for dt, rows, cols in [(1, 12000, 30), (1, 900, 30), (1, 400, 30), (0, 1024, 70), (0, 4900, 70), (0, 6400, 80),
                       (0, 10000, 80), (0, 3072, 48), (0, 128, 48)]:
    ms = C.c_double()
    st = ctx.lib.rcpg_bench_factor(ctx.h, dt, 0, rows, cols, 5, C.byref(ms))
    out.append(f"{'f64' if dt else 'f32'} {rows}x{cols}: {ms.value * 1e3:.1f}" if st == 0 else f"{rows}x{cols}: err{st}")
print(" | ".join(out), flush=True)
