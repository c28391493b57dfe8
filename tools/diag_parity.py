"""Stage-by-stage GPU-vs-oracle comparison on one BASELINE config (diagnostic).

    python tools/diag_parity.py --config C4 [--out gpurun_out/diag_C4]

Generates the config's tensor on the device, downloads it, then compares
  1. compress: per-mode Q_n and the compressed tensor B (GPU vs oracle);
  2. ALS on the SAME compressed tensor (the oracle's B) on both sides
     (decompose with randomized=false), fit traces side by side;
  3. the full decompose on both sides.
The oracle is the checker (test infrastructure); it runs on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip-full", action="store_true")
    ap.add_argument("--omega-host", action="store_true")
    ap.add_argument("--fast", action="store_true", help="fp32_arith=1 (3xTF32)")
    a = ap.parse_args()
    os.environ.setdefault("RCPO_THREADS", str(os.cpu_count() or 1))
    import paper_1703_09074_b200 as rcp
    from paper_1703_09074_b200 import synthetic
    import pyoracle as oracle

    cfg = synthetic.CONFIGS[a.config]
    out = a.out or os.path.join(ROOT, "gpurun_out", f"diag_{a.config}")
    os.makedirs(out, exist_ok=True)
    ctx = rcp.default_context()
    if a.omega_host:
        ctx.set_option("omega_host", 1)
    if a.fast:
        ctx.set_option("fp32_arith", 1)
    w, facs = synthetic.model(cfg.kind, cfg.shape, cfg.rank, cfg.seed)
    X = rcp.DeviceTensor.synth(cfg.shape, w, facs, cfg.snr, cfg.seed, dtype=cfg.dtype, ctx=ctx)
    x = X.download()
    cs = rcp.derive_seed(cfg.seed, rcp.stream_id(rcp.COMPRESS))
    ccfg_g = rcp.CompressConfig(target_rank=cfg.rank, oversampling=cfg.oversampling,
                                power_iterations=cfg.power_iterations, seed=cs)
    ccfg_o = oracle.CompressConfig(target_rank=cfg.rank, oversampling=cfg.oversampling,
                                   power_iterations=cfg.power_iterations, seed=cs)
    rep = {"config": cfg.name}
    t0 = time.time()
    cg = rcp.compress(X, ccfg_g)
    t1 = time.time()
    co = oracle.compress(x, ccfg_o)
    t2 = time.time()
    rep["compress_s"] = {"gpu": t1 - t0, "oracle": t2 - t1}
    modes = []
    for n, (bg, qo) in enumerate(zip(cg.bases, co.q)):
        if qo is None:
            modes.append({"mode": n, "identity": True})
            continue
        qg = bg.q.astype(np.float64)
        qo64 = qo.astype(np.float64)
        d = np.abs(qg - qo64)
        col = np.linalg.norm(qg - qo64, axis=0) / np.linalg.norm(qo64, axis=0)
        # span agreement (sign/rotation invariant)
        s = np.linalg.svd(qg.T @ qo64, compute_uv=False)
        modes.append({"mode": n, "max_abs": float(d.max()), "col_rel_max": float(col.max()),
                      "first_bad_col": int(np.argmax(col > 1e-3)) if (col > 1e-3).any() else None,
                      "bitwise_frac": float(np.mean(bg.q == qo)),
                      "span_min_sv": float(s.min())})
    rep["bases"] = modes
    Bg, Bo = cg.compressed.astype(np.float64), co.compressed.astype(np.float64)
    rep["B_rel"] = float(np.linalg.norm(Bg - Bo) / np.linalg.norm(Bo))
    rep["B_bitwise_frac"] = float(np.mean(cg.compressed == co.compressed))
    print(json.dumps(rep), flush=True)
    np.save(os.path.join(out, "B_oracle.npy"), co.compressed)

    # 2. ALS on the oracle's compressed tensor, both sides
    dg = rcp.DecomposeConfig(rank=cfg.rank, tol=cfg.tol, max_iter=cfg.max_iter, seed=cfg.seed, randomized=False)
    do = oracle.DecomposeConfig(rank=cfg.rank, tol=cfg.tol, max_iter=cfg.max_iter, seed=cfg.seed, randomized=False)
    for name, B in (("B_oracle", co.compressed), ("B_gpu", cg.compressed)):
        mg, tg = rcp.decompose(np.ascontiguousarray(B), dg)
        ro = oracle.decompose(np.ascontiguousarray(B), do)
        fg = np.array([e.fit for e in tg.entries])
        fo = ro.trace_fit
        n = min(len(fg), len(fo))
        dfit = np.abs(fg[:n] - fo[:n])
        als = {"on": name, "iters": [tg.iterations, ro.iterations],
               "relerr": [tg.final_relative_error, ro.final_relative_error],
               "fit_gpu": fg.tolist(), "fit_oracle": fo.tolist(),
               "dfit_max_first": float(dfit[: min(n, 10)].max()) if n else None,
               "first_dfit_gt_1e-6": int(np.argmax(dfit > 1e-6)) if (dfit > 1e-6).any() else None}
        print(json.dumps({k: v for k, v in als.items() if not k.startswith("fit_")}), flush=True)
        rep["als_" + name] = als
    if not a.skip_full:
        cfg_g = rcp.DecomposeConfig(rank=cfg.rank, tol=cfg.tol, max_iter=cfg.max_iter, seed=cfg.seed,
                                    compress=ccfg_g)
        cfg_o = oracle.DecomposeConfig(rank=cfg.rank, tol=cfg.tol, max_iter=cfg.max_iter, seed=cfg.seed,
                                       compress=ccfg_o)
        mg, tg = rcp.decompose(X, cfg_g)
        ro = oracle.decompose(x, cfg_o)
        full = {"iters": [tg.iterations, ro.iterations], "relerr": [tg.final_relative_error,
                                                                    ro.final_relative_error],
                "fit_gpu": [e.fit for e in tg.entries], "fit_oracle": ro.trace_fit.tolist()}
        print(json.dumps({k: v for k, v in full.items() if not k.startswith("fit_")}), flush=True)
        rep["full"] = full
    with open(os.path.join(out, "report.json"), "w") as f:
        json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
