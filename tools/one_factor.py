import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_09074_b200 as rcp
ctx = rcp.default_context()
ms = C.c_double()
kind = int(sys.argv[1]); rows = int(sys.argv[2]); cols = int(sys.argv[3]); dt = int(sys.argv[4]) if len(sys.argv) > 4 else 1
print(ctx.lib.rcpg_bench_factor(ctx.h, dt, kind, rows, cols, 2, C.byref(ms)), ms.value * 1e3, "us")
