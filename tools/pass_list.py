"""Every timed pass of one warm decompose of a BASELINE config, in call order.

Usage: python tools/pass_list.py [CFG] [--filter NAME]
Prints name, ms and algorithmic bytes of each pass instance (the bench's `passes`
block sums them by name).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1703_09074_b200 as rcp  # noqa: E402
from paper_1703_09074_b200 import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="C2")
ap.add_argument("--filter", default="")
args = ap.parse_args()
cfg = synthetic.CONFIGS[args.config]
ctx = rcp.Context(0)
ctx.set_option("pass_timing", 1)
w, f = synthetic.model(cfg.kind, cfg.shape, cfg.rank, cfg.seed)
X = rcp.DeviceTensor.synth(cfg.shape, w, f, cfg.snr, cfg.seed, dtype=cfg.dtype, ctx=ctx)
cs = rcp.derive_seed(cfg.seed, rcp.stream_id(rcp.COMPRESS))
d = rcp.DecomposeConfig(rank=cfg.rank, tol=cfg.tol, max_iter=cfg.max_iter, seed=cfg.seed,
                        compress=rcp.CompressConfig(target_rank=cfg.rank, oversampling=cfg.oversampling,
                                                    power_iterations=cfg.power_iterations, seed=cs))
rcp.decompose(X, d, ctx=ctx)
ctx.event_record(0)
rcp.decompose(X, d, ctx=ctx)
ctx.event_record(1)
ctx.synchronize()
call_ms = ctx.event_elapsed_ms(0, 1)
tot = 0.0
gaps = 0.0
offs = ctx.pass_offsets()
prev_end = None
for (name, ms, by), t0 in zip(ctx.pass_timings(), offs):
    tot += ms
    gap = 0.0 if prev_end is None else t0 - prev_end
    gaps += gap
    prev_end = t0 + ms
    if args.filter in name:
        print(f"{name:16s} {ms:9.3f} ms  {by / 1e6:10.1f} MB   gap before {gap * 1e3:7.1f} us")
print(f"total {tot:.3f} ms in passes, {gaps:.3f} ms between passes, span {prev_end:.3f} ms, call {call_ms:.3f} ms")
