"""plu_basis device time: default path vs an 8/16-CTA cluster for panels that fit one CTA."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_09074_b200 as rcp  # noqa: E402
ctx = rcp.default_context()
for dt, rows, cols in [(1, 400, 30), (1, 900, 30), (0, 1024, 48), (0, 512, 48), (0, 128, 48), (1, 12000, 30), (0, 10000, 80), (0, 4096, 48)]:
    out = []
    for path, mcs in [("", None), ("cluster", "4"), ("cluster", "8"), ("cluster", "16")]:
        for k, v in (("RCPG_LU_PATH", path), ("RCPG_LU_MINCS", mcs)):
            if v:
                os.environ[k] = v
            else:
                os.environ.pop(k, None)
        ms = C.c_double()
        st = ctx.lib.rcpg_bench_factor(ctx.h, dt, 0, rows, cols, 5, C.byref(ms))
        out.append(f"{path or 'default'}{mcs or ''}: {ms.value * 1e3:7.1f}" if st == 0 else f"{path}{mcs}: err{st}")
    print(("f64" if dt else "f32"), rows, cols, " | ".join(out), flush=True)
