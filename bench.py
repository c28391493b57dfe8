#!/usr/bin/env python
"""Benchmark of the B200-native rCP hot path (rcp::decompose, randomized ALS).

One step = one full rcp::decompose (randomized=true, method=als) of the
BASELINE.json workload (default C2: 400^3 fp64, rank 20, p=10, q=2, tol 1e-8,
max 200 iterations; synthetic input of that shape and distribution, generated
on the device). `value` = device time-to-solution per decomposition with the
tensor already in HBM (CUDA events on the library's stream, max over ranks);
`e2e` = the same through the C-ABI with the host tensor copied in (pinned)
and the model copied out inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

Multi-GPU: one process per GPU (torchrun; `--gpus N` without torchrun re-launches
itself under torch.distributed.run with N ranks). The configs BASELINE.json shards
(C3 along mode 3, C4 along mode 4, C5 along mode 1) are split in slabs and decomposed
collectively (strong scaling, value = the max over ranks of the
device time). C1 / C2 are single-GPU configs in BASELINE.json: at N > 1 every rank
decomposes its own tensor (replicas, weak scaling). The line carries
`scaling_config` (C3) and `scaling_config_C5`, the sharded configs timed the same
way at this N.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

STREAMED = ("sketch", "power_xtq", "power_xz", "project")
# Omega is generated into a panel before the sketch (SURVEY.md 8(d) counts its bytes as 0):
# when generated in line ("omega") its time is charged to the streamed passes; by default
# it is generated on a side stream concurrently with the input check ("omega_overlapped",
# off the critical path, not charged)
STREAMED_TIME = STREAMED + ("omega",)
# FP64 DMMA / DFMA peak measured on this pool's B200 by tools/microbench/fp64_peak.cu
# (not in MEASURED_PEAKS.json, which carries HBM and bf16 only)
FP64_PEAK_TFLOPS = 37.0


def streamed_flops(cfg) -> float:
    """Algorithmic flops of the streamed passes: 2 S_n l per pass,
    1 sketch + q X^T Q + q X Z + 1 projection per compressed mode, tensor shrinking."""
    shape = list(cfg.shape)
    total = 0.0
    for n in range(len(shape)):
        l = min(cfg.rank + cfg.oversampling, shape[n])
        if l >= shape[n]:
            continue
        S = float(np.prod(shape))
        total += (2 + 2 * cfg.power_iterations) * 2.0 * S * l
        shape[n] = l
    return total


def workload_str(cfg) -> str:
    """The config string both arms print (identical, so the driver's same_config holds)."""
    return (f"{cfg.name}: {'x'.join(map(str, cfg.shape))} rank {cfg.rank} p={cfg.oversampling} "
            f"q={cfg.power_iterations} tol={cfg.tol:g} max_iter={cfg.max_iter}")


def fms(w1, f1, w2, f2) -> float:
    """Factor match score: greedy |congruence| matching of components,
    mean over components of (1 - |dlambda| / max lambda) * prod_n |a_n . b_n|."""
    R = len(w1)
    score = np.ones((R, R))
    for a, b in zip(f1, f2):
        an = a / np.maximum(np.linalg.norm(a, axis=0), 1e-300)
        bn = b / np.maximum(np.linalg.norm(b, axis=0), 1e-300)
        score *= np.abs(an.T.astype(np.float64) @ bn.astype(np.float64))
    used, tot = set(), 0.0
    for i in range(R):
        j = next(j for j in np.argsort(-score[i]) if j not in used)
        used.add(j)
        lam = 1 - abs(float(w1[i]) - float(w2[j])) / max(abs(float(w1[i])), abs(float(w2[j])), 1e-300)
        tot += lam * score[i, j]
    return tot / R


def parity_record(cfg, model, trace, ref) -> dict:
    """GPU result vs the oracle on the same input (north_star bars): fp64 factors and relerr
    within 1e-8 relative with equal iteration counts; fp32 fit within 1e-4 relative and FMS >= 0.99."""
    fit_g = 1.0 - trace.final_relative_error ** 2
    fit_o = 1.0 - ref.final_relative_error ** 2
    rec = {"oracle_relerr": ref.final_relative_error, "gpu_relerr": trace.final_relative_error,
           "oracle_iterations": ref.iterations, "gpu_iterations": trace.iterations,
           "fit_rel_diff": abs(fit_g - fit_o) / abs(fit_o),
           "relerr_rel_diff": abs(trace.final_relative_error - ref.final_relative_error) / ref.final_relative_error,
           "fms": fms(model.weights, model.factors, ref.weights, ref.factors)}
    if cfg.dtype == np.float64:
        fd = max(float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b))
                 for a, b in zip(model.factors, ref.factors))
        rec["factor_rel_diff_max"] = fd
        rec["bar"] = "fp64: factors and relerr <= 1e-8 relative, equal iterations"
        rec["pass"] = bool(fd <= 1e-8 and rec["relerr_rel_diff"] <= 1e-8 and ref.iterations == trace.iterations)
    else:
        rec["bar"] = "fp32: fit <= 1e-4 relative, FMS >= 0.99"
        rec["pass"] = bool(rec["fit_rel_diff"] <= 1e-4 and rec["fms"] >= 0.99)
    return rec


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent decompositions instead of one sharded along the slab mode")
    ap.add_argument("--shard", action="store_true",
                    help="force the sharded path (NCCL communicator) also at N = 1")
    ap.add_argument("--no-scaling-config", action="store_true",
                    help="skip the scaling_config (C3) sub-record")
    ap.add_argument("--host-check", action="store_true",
                    help="launch / process-group / max-over-ranks plumbing only (no GPU work; CPU tests)")
    ap.add_argument("--fast-fp32", action="store_true",
                    help="fp32_arith = 1: 3xTF32 tcgen05 passes (not bit-faithful to the reference)")
    ap.add_argument("--omega-host", action="store_true",
                    help="Omega evaluated on the host and uploaded (bit-identical; slower)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_cmd(gpus: int, argv) -> list:
    """`bench.py --gpus N` outside torchrun: the same command under torch.distributed.run, N ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + list(argv)


class Dist:
    def __init__(self, world, rank, local):
        self.world, self.rank, self.local = world, rank, local
        self.pg = None
        if world > 1:
            import torch
            import torch.distributed as td
            if torch.cuda.is_available():
                torch.cuda.set_device(local)
                td.init_process_group("nccl", device_id=torch.device("cuda", local))
                self.dev = "cuda"
            else:  # host-side tests (gloo, world_size 2 on CPU)
                td.init_process_group("gloo")
                self.dev = "cpu"
            self.td, self.torch = td, torch

    def barrier(self):
        if self.world > 1:
            self.td.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def broadcast_bytes(self, b: bytes, root: int = 0) -> bytes:
        """Rank root's bytes on every rank (the NCCL unique id of the library's communicator)."""
        if self.world == 1:
            return b
        t = self.torch.tensor(list(b), dtype=self.torch.uint8, device=self.dev)
        self.td.broadcast(t, src=root)
        return bytes(t.cpu().tolist())

    def close(self):
        if self.world > 1:
            self.td.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            try:
                rows.append((float(p[0]), float(p[1]), float(p[2]), p[3:7]))
            except (ValueError, IndexError):
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [r for r in rows if r[2] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(loaded)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def profile_traffic(cfg_name):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get(cfg_name, {}).get("traffic_bytes_per_launch")
    except Exception:
        return None


def configs(cfg, rcp):
    seed = cfg.seed
    cs = rcp.derive_seed(seed, rcp.stream_id(rcp.COMPRESS))
    return dict(rank=cfg.rank, tol=cfg.tol, max_iter=cfg.max_iter, seed=seed,
                compress=dict(target_rank=cfg.rank, oversampling=cfg.oversampling,
                              power_iterations=cfg.power_iterations, seed=cs))


def run_reference(args, dist, cfg):
    """--impl reference: the reference's algorithm on the host cores (oracle
    port; the Eigen reference itself cannot be built here)."""
    if dist.rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    cores = os.cpu_count() or 1
    os.environ["RCPO_THREADS"] = str(cores)
    import pyoracle as oracle
    import paper_1703_09074_b200 as rcp
    x, _ = oracle.synth(cfg.kind, cfg.shape, cfg.rank, cfg.seed, cfg.snr, dtype=cfg.dtype) if cfg.kind != 1 else \
        oracle.random_lowrank(cfg.shape, cfg.rank, cfg.seed, snr=cfg.snr, noise_seed=cfg.seed)
    c = configs(cfg, rcp)
    ocfg = oracle.DecomposeConfig(rank=c["rank"], tol=c["tol"], max_iter=c["max_iter"], seed=c["seed"],
                                  compress=oracle.CompressConfig(**c["compress"]))
    times, res = [], None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        res = oracle.decompose(x, ocfg)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt * 1e3)
    ms = statistics.median(times)
    line = {
        "impl": "reference", "metric": "rCP time-to-solution", "value": ms, "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if cfg.dtype == np.float64 else "f32", "data": "synthetic",
        "config": {"workload": workload_str(cfg), "parallelism": "host threads"},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "port",
                         "sample": f"full {cfg.name} decompose per step (C++ oracle restatement, "
                                   f"std::thread x{cores}, -O3)"},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "relerr": res.final_relative_error, "iterations": res.iterations,
    }
    print(json.dumps(line), flush=True)


def _oracle_cfg(oracle, c):
    return oracle.DecomposeConfig(rank=c["rank"], tol=c["tol"], max_iter=c["max_iter"], seed=c["seed"],
                                  compress=oracle.CompressConfig(**c["compress"]))


def cpu_baseline(cfg, x_host, c):
    """The oracle (C++ restatement of the reference) on the box's host cores, all threads, on
    the downloaded input. Returns (record, oracle result) -- the result is also the parity check."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    cores = os.cpu_count() or 1
    os.environ["RCPO_THREADS"] = str(cores)
    import pyoracle as oracle
    t0 = time.perf_counter()
    res = oracle.decompose(x_host, _oracle_cfg(oracle, c))
    dt = (time.perf_counter() - t0) * 1e3
    rec = {"value": dt, "unit": "ms", "cores": cores, "kind": "port",
           "sample": f"1 full {cfg.name} decompose on the downloaded input (C++ oracle, std::thread x{cores}, "
                     f"-O3 no -march)",
           "relerr": res.final_relative_error, "iterations": res.iterations}
    return rec, res


SINGLE_WORKER = r"""
import os, sys, time, json
import numpy as np
sys.path.insert(0, sys.argv[1])
import pyoracle as oracle
x = np.load(sys.argv[2])
c = json.loads(sys.argv[3])
cfg = oracle.DecomposeConfig(rank=c["rank"], tol=c["tol"], max_iter=c["max_iter"], seed=c["seed"],
                             compress=oracle.CompressConfig(**c["compress"]))
t0 = time.perf_counter()
r = oracle.decompose(x, cfg)
print(json.dumps({"ms": (time.perf_counter() - t0) * 1e3, "relerr": r.final_relative_error,
                  "iterations": r.iterations}))
"""


def cpu_baseline_single(cfg, x_host, c):
    """Reference-faithful CPU number: the oracle with one
    thread (the reference's build has no OpenMP / threads), in a subprocess so the thread
    count is fresh. Only for inputs it finishes within a few minutes (C1, C2)."""
    if x_host.nbytes > 600e6:
        return {"value": None, "cores": 1, "skipped": "input above 600 MB: minutes of single-thread work"}
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        fn = os.path.join(d, "x.npy")
        np.save(fn, x_host)
        env = dict(os.environ, RCPO_THREADS="1")
        out = subprocess.run([sys.executable, "-c", SINGLE_WORKER, os.path.join(ROOT, "oracle"), fn, json.dumps(c)],
                             env=env, capture_output=True, text=True, timeout=600)
    if out.returncode != 0:
        return {"value": None, "cores": 1, "error": out.stderr[-300:]}
    r = json.loads(out.stdout.strip().splitlines()[-1])
    return {"value": r["ms"], "unit": "ms", "cores": 1, "kind": "port",
            "sample": f"1 full {cfg.name} decompose, oracle with 1 thread (-O3, no -march: the reference's build)",
            "relerr": r["relerr"], "iterations": r["iterations"]}


def lu_sweep_bytes(cfg) -> float:
    """Algorithmic HBM traffic of the faithful complete-pivoting LUs of the W = X_(n)^T Q panels
    (compress.hpp:127-132): at pivot k the trailing J x (l - k) panel is read
    once to find the next pivot, sum_k J (l - k) b bytes per LU, q LUs per compressed mode."""
    shape = list(cfg.shape)
    b = np.dtype(cfg.dtype).itemsize
    total = 0.0
    for n in range(len(shape)):
        l = min(cfg.rank + cfg.oversampling, shape[n])
        if l >= shape[n]:
            continue
        J = float(np.prod(shape)) / shape[n]
        total += cfg.power_iterations * J * b * l * (l + 1) / 2.0
        shape[n] = l
    return total


def binding_roofline(cfg, pass_ms, pass_bytes, steps, fast_fp32=False, traffic=None):
    """Roofline of the streamed passes against their binding roof.

    The passes run on the FP64 tensor cores (DMMA) for fp64 data and, in the default faithful
    fp32 arithmetic, for fp32 data too; at l = 30..80 their arithmetic intensity (2 l flops per
    element) puts them above the DMMA ridge, so the binding roof is the FP64 tensor pipe
    (bound "tensor", TFLOP/s); the fast 3xTF32 fp32 path (fp32_arith = 1) is HBM-bound.
    Both fractions are reported; `frac` is the binding one."""
    peak, peak_kind = measured_peaks()
    sm_ms, achieved, _, _ = pass_roofline(pass_ms, pass_bytes, steps)
    fl = streamed_flops(cfg)
    by = sum(pass_bytes.get(n, 0.0) for n in STREAMED) / steps
    hbm = {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak if peak else None,
           "peak_source": peak_kind}
    t_pipe, t_hbm = fl / (FP64_PEAK_TFLOPS * 1e12), by / (peak * 1e9)
    if not fast_fp32 and t_pipe >= t_hbm and sm_ms > 0:
        tf = fl * steps / (sm_ms / 1e3) / 1e12
        return {"bound": "tensor", "achieved": tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": tf / FP64_PEAK_TFLOPS, "traffic": traffic,
                "kernel": "streamed mode-n passes on the FP64 tensor cores (Omega + sketch / X^T Q / X Z / projection)",
                "peak_source": "own DMMA microbenchmark (tools/microbench/fp64_peak.cu, 37.0 TFLOP/s); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "flops_per_step": fl, "hbm": hbm}
    return dict(bound="hbm", achieved=achieved, peak=peak, unit="GB/s", frac=hbm["frac"], traffic=traffic,
                kernel="streamed mode-n passes (Omega + sketch / X^T Q / X Z / projection)", peak_source=peak_kind)


def pass_roofline(pass_ms, pass_bytes, steps):
    peak, peak_kind = measured_peaks()
    sm_ms = sum(pass_ms.get(n, 0.0) for n in STREAMED_TIME)
    sm_by = sum(pass_bytes.get(n, 0.0) for n in STREAMED)
    achieved = (sm_by / 1e9) / (sm_ms / 1e3) if sm_ms > 0 else 0.0
    return sm_ms, achieved, peak, peak_kind


PROFILED = {}  # instrumented step time of the last timed_decompositions call


def timed_decompositions(rcp, ctx, X, dcfg, steps, warmup, dist):
    """W untimed + K timed decompositions on the device; device time per step (max over ranks),
    per-pass times of the timed steps, launches, the last model."""
    ctx.set_option("pass_timing", 0)  # the library default: no instrumentation in the timed region
    for _ in range(warmup):
        model, trace = rcp.decompose(X, dcfg, ctx=ctx)
    ctx.synchronize()
    dist.barrier()
    l0 = ctx.kernel_launches()
    pass_ms, pass_bytes = {}, {}
    ctx.event_record(0)
    for _ in range(steps):
        model, trace = rcp.decompose(X, dcfg, ctx=ctx)
    ctx.event_record(1)
    total_ms = ctx.event_elapsed_ms(0, 1)
    ctx.synchronize()
    launches = ctx.kernel_launches() - l0
    dist.barrier()
    # Per-pass times (the roofline's kernel durations): the same steps again with the library's
    # per-pass CUDA events on. The ~60 event records cost 0.3 ms per decomposition (C2), so they
    # stay out of `value`; PROFILED["ms_per_step"] is the instrumented step time.
    ctx.set_option("pass_timing", 1)
    for _ in range(min(warmup, 2) + 1):  # (the option change drops the captured graph: call, capture, replay)
        rcp.decompose(X, dcfg, ctx=ctx)
    ctx.synchronize()
    ctx.event_record(4)
    for _ in range(steps):
        rcp.decompose(X, dcfg, ctx=ctx)
    ctx.event_record(5)
    PROFILED["ms_per_step"] = ctx.event_elapsed_ms(4, 5) / steps
    for name, ms, by in ctx.pass_timings():  # last profiled step
        pass_ms[name] = pass_ms.get(name, 0.0) + ms * steps
        pass_bytes[name] = pass_bytes.get(name, 0.0) + by * steps
    ctx.set_option("pass_timing", 0)
    dist.barrier()
    return dist.max(total_ms / steps), pass_ms, pass_bytes, launches, model, trace


def shard_mode(cfg) -> int:
    """The slab mode of the multi-GPU runs (BASELINE.json: C3 mode 3, C4 mode 4, C5 mode 1)."""
    return cfg.shard_mode if cfg.shard_mode >= 0 else len(cfg.shape) - 1


def shard_desc(cfg, world) -> str:
    return f"slab-sharded along mode {shard_mode(cfg) + 1} over {world} GPUs (NCCL)"


def make_tensor(rcp, synthetic, cfg, ctx, shard, world, rank):
    w, facs = synthetic.model(cfg.kind, cfg.shape, cfg.rank, cfg.seed)
    X = rcp.DeviceTensor.synth(cfg.shape, w, facs, cfg.snr, cfg.seed, dtype=cfg.dtype, ctx=ctx)
    sm = shard_mode(cfg)
    slo, shi = 0, cfg.shape[sm]
    if shard:
        slo, shi = rcp.slab_range(cfg.shape[sm], world, rank)
        Xs = X.slab(slo, shi, mode=sm)
        X.free()
        X = Xs
    return X, slo, shi


SHARDED_CONFIGS = ("C3", "C4", "C5")  # BASELINE.json: sharded at 1/2/4/8 GPUs


def scaling_record(args, dist, rcp, synthetic, ctx, world, rank, shard, name="C3"):
    """scaling_config: a config BASELINE.json shards (C3 along mode 3, C5 along mode 1: the
    largest sharded tensor of north_star's 1 -> 8 GPU target) device-timed at this N, with
    its streamed-pass roofline."""
    from paper_1703_09074_b200.synthetic import CONFIGS
    cfg = CONFIGS[name]
    X, _, _ = make_tensor(rcp, synthetic, cfg, ctx, shard, world, rank)
    c = configs(cfg, rcp)
    dcfg = rcp.DecomposeConfig(rank=c["rank"], tol=c["tol"], max_iter=c["max_iter"], seed=c["seed"],
                               compress=rcp.CompressConfig(**c["compress"]))
    steps = max(2, min(args.steps, 5))
    ms, pass_ms, pass_bytes, launches, model, trace = timed_decompositions(rcp, ctx, X, dcfg, steps, 1, dist)
    X.free()
    sm_ms, achieved, peak, peak_kind = pass_roofline(pass_ms, pass_bytes, steps)
    return {"workload": workload_str(cfg), "metric": "rCP time-to-solution", "value": ms, "unit": "ms",
            "n_gpus": world, "steps": steps, "warmup": 1, "higher_is_better": False,
            "scaling": "strong" if shard else "weak",
            "parallelism": (shard_desc(cfg, world) if shard else "single GPU"),
            "gpu_launches": int(launches),
            "roofline": binding_roofline(cfg, pass_ms, pass_bytes, steps, fast_fp32=ctx.get_option("fp32_arith") == 1),
            "passes_ms": {n: pass_ms[n] / steps for n in pass_ms},
            "relerr": trace.final_relative_error, "iterations": trace.iterations}


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        sys.exit(subprocess.run(spawn_cmd(args.gpus, sys.argv[1:])).returncode)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch one rank per GPU)")
    # stdout carries exactly one JSON line: NCCL's INFO log (communicator lines) goes to stderr
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    dist = Dist(world, rank, local)
    if args.host_check:
        m = dist.max(float(rank))
        if rank == 0:
            print(json.dumps({"host_check": True, "world": world, "max_rank": m}), flush=True)
        dist.close()
        return
    from paper_1703_09074_b200.synthetic import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, dist, cfg)
        dist.close()
        return

    import paper_1703_09074_b200 as rcp
    from paper_1703_09074_b200 import synthetic
    ctx = rcp.Context(local)
    if args.omega_host:
        ctx.set_option("omega_host", 1)
    if args.fast_fp32:
        ctx.set_option("fp32_arith", 1)
    # N > 1: one decomposition sharded in slabs along the slab mode, the
    # library's own NCCL communicator (id broadcast through torch.distributed)
    shard = (world > 1 and not args.replicas and args.config in SHARDED_CONFIGS) or args.shard
    if world > 1 or args.shard:  # the sharded runs (this config or the scaling records) need the communicator
        uid = dist.broadcast_bytes(rcp.comm_unique_id() if rank == 0 else bytes(128))
        ctx.comm_init_nccl(world, rank, uid)
    X, slo, shi = make_tensor(rcp, synthetic, cfg, ctx, shard, world, rank)
    c = configs(cfg, rcp)
    dcfg = rcp.DecomposeConfig(rank=c["rank"], tol=c["tol"], max_iter=c["max_iter"], seed=c["seed"],
                               compress=rcp.CompressConfig(**c["compress"]))
    with ClockSampler(local) as clk:
        ms_step, pass_ms, pass_bytes, launches, model, trace = timed_decompositions(
            rcp, ctx, X, dcfg, args.steps, args.warmup, dist)
        profiled_ms = PROFILED.get("ms_per_step")

    # e2e through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    x_host = None
    if not args.no_e2e or (rank == 0 and world == 1 and not args.no_cpu_baseline):
        x_host = X.download()

    def e2e_step():
        if not shard:
            return rcp.decompose(x_host, dcfg, ctx=ctx)
        t = rcp.DeviceTensor.upload_slab(x_host, cfg.shape, slo, shi, ctx=ctx, mode=shard_mode(cfg))
        try:
            return rcp.decompose(t, dcfg, ctx=ctx)
        finally:
            t.free()

    if not args.no_e2e:
        ctx.host_register(x_host)
        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        ctx.synchronize()
        dist.barrier()
        ctx.event_record(2)
        for _ in range(args.steps):
            m2, t2 = e2e_step()
        ctx.event_record(3)
        e2e_ms = dist.max(ctx.event_elapsed_ms(2, 3) / args.steps)
        ctx.host_unregister(x_host)
        d2h = (cfg.rank + sum(cfg.shape) * cfg.rank) * np.dtype(cfg.dtype).itemsize + 2 * 8 * t2.iterations
        h2d = int(x_host.nbytes) * (world if shard else 1)  # every rank uploads its slab
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(d2h)}
    X.free()

    if rank == 0:
        sm_ms, achieved, peak, peak_kind = pass_roofline(pass_ms, pass_bytes, args.steps)
        passes = {n: {"ms_per_step": pass_ms[n] / args.steps,
                      "gbs": (pass_bytes[n] / 1e9) / (pass_ms[n] / 1e3) if pass_ms[n] > 0 and pass_bytes[n] > 0
                      else None} for n in pass_ms}
        line = {
            "metric": "rCP time-to-solution", "value": ms_step, "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
            "scaling": "strong" if shard else "weak", "vs_baseline": None,
            "dtype": "f64" if cfg.dtype == np.float64 else "f32",
            "data": "synthetic (device-generated Kruskal model + add_noise, BASELINE.json shape/distribution)",
            "config": {"workload": workload_str(cfg),
                       "parallelism": (shard_desc(cfg, world) if shard
                                       else ("replicas" if world > 1 else "single GPU")),
                       "l2": "tensor larger than L2 (no flush needed)" if cfg.nbytes() > 126e6 else "L2-resident",
                       "omega": "host-evaluated, uploaded" if args.omega_host else "device",
                       "fp32_arith": ("fast 3xTF32" if args.fast_fp32 else "faithful (fp64 products and sums)")
                       if cfg.dtype == np.float32 else "fp64",
                       "pass_events": "off in the timed region (library default); `passes`, `roofline` and "
                                      "`lu_roofline` from the same number of further steps with the per-pass CUDA "
                                      "events on (profiled_ms_per_step)"},
            "profiled_ms_per_step": profiled_ms,
            "gpu_launches": int(launches),
            "roofline": binding_roofline(cfg, pass_ms, pass_bytes, args.steps,
                                         fast_fp32=ctx.get_option("fp32_arith") == 1,
                                         traffic=profile_traffic(cfg.name)),
            "clocks": clk.summary(),
            "relerr": trace.final_relative_error, "iterations": trace.iterations, "converged": trace.converged,
            "passes": passes,
        }
        lu_ms = pass_ms.get("stab_w", 0.0) / args.steps
        if lu_ms > 0:
            lb = lu_sweep_bytes(cfg)
            line["lu_roofline"] = {"bound": "hbm", "achieved": lb / 1e9 / (lu_ms / 1e3), "peak": peak, "unit": "GB/s",
                                   "frac": lb / 1e9 / (lu_ms / 1e3) / peak, "bytes_per_step": lb, "ms_per_step": lu_ms,
                                   "kernel": "complete-pivoting LU of the W panels (stab_w; one trailing-panel "
                                             "read per pivot)"}
        if e2e:
            line["e2e"] = e2e
        if world == 1 and not args.no_cpu_baseline:
            rec, ref = cpu_baseline(cfg, x_host, c)
            rec["single_thread"] = cpu_baseline_single(cfg, x_host, c)
            line["cpu_baseline"] = rec
            line["parity"] = parity_record(cfg, model, trace, ref)
            if not line["parity"]["pass"]:
                print(f"bench.py: PARITY FAILURE vs the oracle: {json.dumps(line['parity'])}", file=sys.stderr)
    else:
        line = None

    # the sharded scaling records come last, each guarded: an exception is recorded in the
    # sub-record, and a watchdog prints the main line without them if they hang (a collective
    # that never completes must not cost the whole bench line)
    if not args.no_scaling_config:
        import threading

        def watchdog():
            if line is not None:
                line.setdefault("scaling_config", {"error": f"timeout after {limit:.0f} s"})
                print(json.dumps(line), flush=True)
            print(f"bench.py: scaling records exceeded {limit:.0f} s, exiting", file=sys.stderr, flush=True)
            os._exit(0)

        limit = float(os.environ.get("RCPG_BENCH_SCALING_TIMEOUT", "480"))
        timer = threading.Timer(limit, watchdog)
        timer.daemon = True
        timer.start()
        sh = world > 1 or args.shard
        for key, name in (("scaling_config", "C3"), ("scaling_config_C5", "C5")):
            if args.config == name:
                continue
            try:
                rec = scaling_record(args, dist, rcp, synthetic, ctx, world, rank, sh, name)
            except Exception as exc:  # recorded, not fatal
                print(f"bench.py: {key} failed: {exc!r}", file=sys.stderr, flush=True)
                rec = {"workload": name, "error": repr(exc)[:300]}
            if line is not None:
                line[key] = rec
        timer.cancel()
    if line is not None:
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
