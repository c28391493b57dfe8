"""plu_basis device time on the SM-resident grid LU by target rows per CTA (RCPG_LU_RES_ROWS)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_09074_b200 as rcp  # noqa: E402
ctx = rcp.default_context()
for dt, rows, cols in [(1, 12000, 30), (0, 10000, 80), (1, 160000, 30), (0, 71680, 70), (0, 40000, 80), (0, 110592, 48)]:
    out = []
    for target in [None, "1024", "512", "256"]:
        if target:
            os.environ["RCPG_LU_RES_ROWS"] = target
        else:
            os.environ.pop("RCPG_LU_RES_ROWS", None)
        ms = C.c_double()
        st = ctx.lib.rcpg_bench_factor(ctx.h, dt, 0, rows, cols, 5, C.byref(ms))
        out.append(f"{target or 'default'}: {ms.value * 1e3:7.1f}" if st == 0 else f"{target}: err{st}")
    print(("f64" if dt else "f32"), rows, cols, " | ".join(out), flush=True)
