"""Time one streamed pass (sketch / projection) on a large mode view, device-side.

Usage: python tools/pass_bench.py [sketch|project] L I R cols [dtype] [reps]
Inputs are uploaded once through rcpg_stream_pass (so the H2D copy is outside the
kernel time); run under ncu for per-kernel durations, or read the printed
CUDA-event time of the whole call (which includes the copies).
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1703_09074_b200 as rcp  # noqa: E402


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "sketch"
    L, I, R, cols = (int(a) for a in sys.argv[2:6]) if len(sys.argv) > 5 else (1, 1024, 262144, 70)
    dtype = np.float32 if (len(sys.argv) <= 6 or sys.argv[6] == "f32") else np.float64
    reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
    rng = np.random.default_rng(0)
    x = rng.standard_normal((L, I, R), dtype=np.float32).astype(dtype)
    p = (rng.standard_normal((L, cols, R), dtype=np.float32) if kind == "sketch"
         else rng.standard_normal((I, cols), dtype=np.float32)).astype(dtype)
    for _ in range(reps):
        t = time.perf_counter()
        rcp.stream_pass(kind, x, p, cols)
        print(f"{kind} {L}x{I}x{R} cols={cols}: {1e3 * (time.perf_counter() - t):.2f} ms (incl. copies)")


if __name__ == "__main__":
    main()
