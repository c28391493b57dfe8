"""One warm decompose of a BASELINE config (for ncu / compute-sanitizer runs)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1703_09074_b200 as rcp  # noqa: E402
from paper_1703_09074_b200 import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--warmup", type=int, default=1)
args = ap.parse_args()
cfg = synthetic.CONFIGS[args.config]
ctx = rcp.Context(0)
w, f = synthetic.model(cfg.kind, cfg.shape, cfg.rank, cfg.seed)
X = rcp.DeviceTensor.synth(cfg.shape, w, f, cfg.snr, cfg.seed, dtype=cfg.dtype, ctx=ctx)
cs = rcp.derive_seed(cfg.seed, rcp.stream_id(rcp.COMPRESS))
d = rcp.DecomposeConfig(rank=cfg.rank, tol=cfg.tol, max_iter=cfg.max_iter, seed=cfg.seed,
                        compress=rcp.CompressConfig(target_rank=cfg.rank, oversampling=cfg.oversampling,
                                                    power_iterations=cfg.power_iterations, seed=cs))
for _ in range(args.warmup + 1):
    m, t = rcp.decompose(X, d, ctx=ctx)
print("iters", t.iterations, "relerr", t.final_relative_error)
