"""plu_basis device time: default path vs the SM-resident grid LU at several rows per CTA."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_09074_b200 as rcp
ctx = rcp.default_context()
for dt, rows, cols in [(1, 12000, 30), (0, 10000, 80), (0, 4096, 48), (0, 2048, 70), (1, 3000, 48)]:
    out = []
    for path, tr in [("", None), ("resident", None), ("resident", "256"), ("resident", "128")]:
        for k, v in (("RCPG_LU_PATH", path), ("RCPG_LU_RES_ROWS", tr)):
            if v: os.environ[k] = v
            else: os.environ.pop(k, None)
        ms = C.c_double()
        st = ctx.lib.rcpg_bench_factor(ctx.h, dt, 0, rows, cols, 5, C.byref(ms))
        out.append(f"{path or 'default'}{tr or ''}: {ms.value * 1e3:7.1f}" if st == 0 else f"{path}{tr}: err{st}")
    print(("f64" if dt else "f32"), rows, cols, " | ".join(out), flush=True)
