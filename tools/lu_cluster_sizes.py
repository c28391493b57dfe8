"""Device time of plu_basis on the cluster path by smallest cluster size tried (RCPG_LU_MINCS)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import paper_1703_09074_b200 as rcp
ctx = rcp.default_context()
for dt, rows, cols in [(0, 1024, 70), (0, 600, 80), (1, 700, 70), (0, 2048, 40)]:
    out = []
    for mcs in ["1", "2", "4", "8", "16"]:
        os.environ["RCPG_LU_MINCS"] = mcs
        ms = C.c_double()
        st = ctx.lib.rcpg_bench_factor(ctx.h, dt, 0, rows, cols, 5, C.byref(ms))
        out.append(f"cs>={mcs}: {ms.value*1e3:8.1f}" if st == 0 else f"cs>={mcs}: err{st}")
    print(("f64" if dt else "f32"), rows, cols, " | ".join(out))
