"""Repeated decompositions through the graph cache (debug aid)."""
import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import paper_1703_09074_b200 as rcp
import pyoracle as oracle
x, _ = oracle.random_lowrank([40, 36, 30], 4, 7, snr=3.0, noise_seed=7)
ctx = rcp.Context(0)
ctx.set_option("pass_timing", 1)
X = rcp.DeviceTensor.upload(x, ctx=ctx)
cs = oracle.derive_seed(5, oracle.stream_id(1))
g = rcp.DecomposeConfig(rank=4, tol=1e-8, max_iter=200, seed=5,
                        compress=rcp.CompressConfig(target_rank=4, oversampling=5, power_iterations=2, seed=cs))
for i in range(4):
    l0 = ctx.kernel_launches()
    try:
        m, t = rcp.decompose(X, g, ctx=ctx)
        print(i, t.iterations, t.final_relative_error, ctx.kernel_launches() - l0, m.weights[:2], flush=True)
    except Exception:
        traceback.print_exc()
print(ctx.pass_timings()[:6])
