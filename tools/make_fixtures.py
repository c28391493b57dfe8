"""Generate the full-size parity fixtures tests/golden/<cfg>_oracle.npz (run on a GPU box).

    python tools/make_fixtures.py C3 C4 C5 [--out tests/golden]

For each BASELINE config: the synthetic input is generated on the device
(rcpg_synth, deterministic), downloaded, digested (tests/golden_digest.py),
and decomposed by the oracle (the C++ restatement of the reference, all host
threads) with the bench's seeds. The fixture stores the oracle's weights,
factors, fit trace, relative error and iteration count plus the input digest,
so tests/test_gpu_fullsize.py can check the GPU against the reference's
algorithm on the identical input without re-running the multi-minute oracle.
The oracle is the checker here (test infrastructure), never the product.
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
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    os.environ.setdefault("RCPO_THREADS", str(os.cpu_count() or 1))
    import paper_1703_09074_b200 as rcp
    from paper_1703_09074_b200 import synthetic
    import pyoracle as oracle
    from golden_digest import digest
    import bench

    os.makedirs(a.out, exist_ok=True)
    for name in a.configs:
        cfg = synthetic.CONFIGS[name]
        ctx = rcp.default_context()
        w, facs = synthetic.model(cfg.kind, cfg.shape, cfg.rank, cfg.seed)
        X = rcp.DeviceTensor.synth(cfg.shape, w, facs, cfg.snr, cfg.seed, dtype=cfg.dtype, ctx=ctx)
        x = X.download()
        dg = digest(x)
        c = bench.configs(cfg, rcp)
        t0 = time.time()
        ref = oracle.decompose(x, bench._oracle_cfg(oracle, c))
        t_or = time.time() - t0
        rec = dict(weights=ref.weights, trace_fit=ref.trace_fit, relerr=np.float64(ref.final_relative_error),
                   iterations=np.int64(ref.iterations), converged=np.int64(ref.converged),
                   digest_sample=np.frombuffer(dg[0].encode(), dtype=np.uint8), digest_sum=np.float64(dg[1]),
                   meta=np.frombuffer(json.dumps({"config": bench.workload_str(cfg), "seeds": c,
                                                  "oracle_seconds": t_or,
                                                  "oracle_threads": os.environ["RCPO_THREADS"]}).encode(),
                                      dtype=np.uint8))
        for m, f in enumerate(ref.factors):
            rec[f"factor{m}"] = f
        np.savez_compressed(os.path.join(a.out, f"{name}_oracle.npz"), **rec)
        line = {"config": name, "oracle_s": t_or, "relerr": ref.final_relative_error, "iterations": ref.iterations}
        # the GPU on the same input, device Omega and host-evaluated Omega
        dcfg = rcp.DecomposeConfig(rank=c["rank"], tol=c["tol"], max_iter=c["max_iter"], seed=c["seed"],
                                   compress=rcp.CompressConfig(**c["compress"]))
        for omega_host in (0, 1):
            ctx.set_option("omega_host", omega_host)
            model, trace = rcp.decompose(X, dcfg, ctx=ctx)
            line[f"gpu_omega_host{omega_host}"] = bench.parity_record(cfg, model, trace, ref)
        ctx.set_option("omega_host", 0)
        X.free()
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
