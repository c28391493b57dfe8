"""Device time of the tall-skinny factorizations on their own (rcpg_bench_factor)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_09074_b200 as rcp  # noqa: E402

ctx = rcp.default_context()
for dt, dname in [(1, "f64"), (0, "f32")]:
    for kind, kname in [(0, "plu_basis"), (1, "thin_qr")]:
        for rows, cols in [(400, 30), (1024, 70), (128, 48), (512, 48), (10000, 80), (12000, 30), (160000, 30)]:
            ms = C.c_double()
            st = ctx.lib.rcpg_bench_factor(ctx.h, dt, kind, rows, cols, 5, C.byref(ms))
            print(f"{dname} {kname:9s} {rows:7d} x {cols:3d}: {ms.value * 1e3:9.1f} us" if st == 0 else f"err {st}")
