"""Device time of repeated C2 decompositions with the per-pass timing events on / off."""
import sys
sys.path.insert(0, ".")
import paper_1703_09074_b200 as rcp
from paper_1703_09074_b200 import synthetic

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = synthetic.CONFIGS[name]
ctx = rcp.Context(0)
w, f = synthetic.model(cfg.kind, cfg.shape, cfg.rank, cfg.seed)
X = rcp.DeviceTensor.synth(cfg.shape, w, f, cfg.snr, cfg.seed, dtype=cfg.dtype, ctx=ctx)
cs = rcp.derive_seed(cfg.seed, rcp.stream_id(rcp.COMPRESS))
d = rcp.DecomposeConfig(rank=cfg.rank, tol=cfg.tol, max_iter=cfg.max_iter, seed=cfg.seed,
                        compress=rcp.CompressConfig(target_rank=cfg.rank, oversampling=cfg.oversampling,
                                                    power_iterations=cfg.power_iterations, seed=cs))
for rep in range(2):
    for on in (1, 0):
        ctx.set_option("pass_timing", on)
        for _ in range(4):
            rcp.decompose(X, d, ctx=ctx)
        ctx.synchronize()
        ctx.event_record(2)
        for _ in range(20):
            m, t = rcp.decompose(X, d, ctx=ctx)
        ctx.event_record(3)
        print(f"{name} pass_timing={on}: {ctx.event_elapsed_ms(2, 3) / 20:.4f} ms per decomposition, iters {t.iterations}")
