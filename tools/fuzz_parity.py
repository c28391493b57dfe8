"""Seeded fuzz: GPU compress / decompose against the oracle over random orders, extents,
ranks, oversampling, power iterations, stabilizers, distributions and mode subsets (fp64).
Prints every case that misses the north_star bars or raises on one side only."""
import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import paper_1703_09074_b200 as rcp
import pyoracle as oracle



def run(N, seed0, out=print, dtype=np.float64):
    rng = np.random.default_rng(seed0)
    bad = 0
    for case in range(N):
        order = int(rng.integers(2, 6))
        hi = {2: 90, 3: 40, 4: 16, 5: 9}[order]
        shape = [int(rng.integers(1, hi + 1)) for _ in range(order)]
        if int(np.prod(shape)) < 2:
            shape[0] = 3
        rank = int(rng.integers(1, 7))
        p, q = int(rng.integers(0, 7)), int(rng.integers(0, 4))
        stab, dist = int(rng.integers(0, 2)), int(rng.integers(0, 2))
        modes = None
        if rng.random() < 0.3:
            modes = sorted(set(int(m) for m in rng.integers(0, order, size=int(rng.integers(0, order + 1)))))
        seed = int(rng.integers(1, 1 << 30))
        kind = rng.random()
        if kind < 0.7:
            x, _ = oracle.random_lowrank(shape, min(rank, max(1, min(shape))), seed, snr=float(rng.choice([1.0, 3.0, 10.0])),
                                         noise_seed=seed)
        else:
            x = np.random.default_rng(seed).standard_normal(shape)
        x = np.ascontiguousarray(x, dtype=dtype)
        f32 = dtype == np.float32
        btol, rtol = (1e-4, 1e-4) if f32 else (1e-8, 1e-8)  # fp32 bar: fit within 1e-4 relative
        desc = f"case {case}: shape={shape} R={rank} p={p} q={q} stab={stab} dist={dist} modes={modes} seed={seed}"
        # compress
        try:
            gc = rcp.compress(x, rcp.CompressConfig(target_rank=rank, oversampling=p, power_iterations=q, seed=seed,
                                                    stabilizer=stab, distribution=dist, modes=modes))
            gerr = None
        except Exception as e:  # noqa: BLE001
            gc, gerr = None, e
        try:
            oc = oracle.compress(x, oracle.CompressConfig(target_rank=rank, oversampling=p, power_iterations=q, seed=seed,
                                                          stabilizer=stab, distribution=dist, modes=modes))
            oerr = None
        except Exception as e:  # noqa: BLE001
            oc, oerr = None, e
        if (gerr is None) != (oerr is None):
            bad += 1
            out("ERRMISMATCH compress", desc, "| gpu:", repr(gerr), "| oracle:", repr(oerr))
        elif gerr is None:
            sc = max(np.max(np.abs(oc.compressed)), 1e-300)
            d = np.max(np.abs(gc.compressed - oc.compressed)) / sc if gc.compressed.shape == oc.compressed.shape else np.inf
            if not d <= btol:
                bad += 1
                out("MISMATCH compress", desc, "B diff", d)
        # decompose
        cs = oracle.derive_seed(seed, oracle.stream_id(1))
        kw = dict(rank=rank, tol=1e-8, max_iter=60, seed=seed)
        ck = dict(target_rank=rank, oversampling=p, power_iterations=q, seed=cs, stabilizer=stab, distribution=dist,
                  modes=modes)
        try:
            gm, gt = rcp.decompose(x, rcp.DecomposeConfig(compress=rcp.CompressConfig(**ck), **kw))
            gerr = None
        except Exception as e:  # noqa: BLE001
            gerr = e
        try:
            om = oracle.decompose(x, oracle.DecomposeConfig(compress=oracle.CompressConfig(**ck), **kw))
            oerr = None
        except Exception as e:  # noqa: BLE001
            oerr = e
        if (gerr is None) != (oerr is None) or (gerr is not None and str(gerr) != str(oerr)):
            bad += 1
            out("ERRMISMATCH decompose", desc, "| gpu:", repr(gerr), "| oracle:", repr(oerr))
        elif gerr is None:
            exact = om.final_relative_error < 1e-12  # exact fits: relerr is rounding noise, factors may be non-unique
            dr = abs(gt.final_relative_error - om.final_relative_error) / max(om.final_relative_error, 1e-300)
            df = max(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300) for a, b in zip(gm.factors, om.factors))
            if exact:
                dr, df = (0.0 if gt.final_relative_error < 1e-12 else np.inf), 0.0
            if f32:  # north_star fp32 bar: fit (1 - relerr^2) within 1e-4 relative
                fg, fo = 1 - gt.final_relative_error ** 2, 1 - om.final_relative_error ** 2
                dr, df = (0.0 if abs(fg - fo) <= 1e-4 * max(abs(fo), 1e-4) else abs(fg - fo)), 0.0
            if (not f32 and gt.iterations != om.iterations) or not dr <= rtol or not df <= rtol:
                bad += 1
                out("MISMATCH decompose", desc, "iters", gt.iterations, om.iterations, "relerr diff", dr, "factor diff", df,
                      "relerr", om.final_relative_error)
    return bad


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    b = run(n, int(sys.argv[2]) if len(sys.argv) > 2 else 2024,
            dtype=np.float32 if len(sys.argv) > 3 and sys.argv[3] == "f32" else np.float64)
    print(f"fuzz: {n} cases, {b} flagged")
