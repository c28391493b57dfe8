"""plu_basis device time: default path vs the SM-resident LU (tagged slots, and the
grid-barrier kernel with RCPG_LU_BARRIER=1) at several rows per CTA."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_09074_b200 as rcp
ctx = rcp.default_context()
for dt, rows, cols in [(1, 160000, 30), (1, 12000, 30), (1, 900, 30), (0, 71680, 70), (0, 40000, 80),
                       (0, 110592, 48), (0, 4900, 70), (0, 6400, 80), (0, 1024, 70)]:
    out = []
    for path, tr in [("", None), ("resident", None), ("resident", "256"), ("resident", "128"), ("resident", "64")]:
        for k, v in (("RCPG_LU_PATH", path), ("RCPG_LU_RES_ROWS", tr)):
            if v: os.environ[k] = v
            else: os.environ.pop(k, None)
        ms = C.c_double()
        st = ctx.lib.rcpg_bench_factor(ctx.h, dt, 0, rows, cols, 5, C.byref(ms))
        out.append(f"{path or 'default'}{tr or ''}: {ms.value * 1e3:7.1f}" if st == 0 else f"{path}{tr}: err{st}")
    print(("f64" if dt else "f32"), rows, cols, " | ".join(out), flush=True)
