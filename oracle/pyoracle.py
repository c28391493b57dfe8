"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/liboracle.so, the C++ restatement of the reference's
rCP hot path (/root/reference/proj/include/rcp/*.hpp; see rcp_oracle.hpp for
the per-function file:line map). Only tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py may import this module, and only as the checker
or the CPU baseline; the product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")

i64p = C.POINTER(C.c_int64)
ip = C.POINTER(C.c_int)
dp = C.POINTER(C.c_double)
fp = C.POINTER(C.c_float)


class RoCompressCfg(C.Structure):
    _fields_ = [
        ("target_rank", C.c_int64),
        ("oversampling", C.c_int64),
        ("power_iterations", C.c_int32),
        ("distribution", C.c_int32),
        ("stabilizer", C.c_int32),
        ("modes_present", C.c_int32),
        ("n_modes", C.c_int64),
        ("modes", i64p),
        ("seed", C.c_uint64),
    ]


class RoDecomposeCfg(C.Structure):
    _fields_ = [
        ("rank", C.c_int64),
        ("method", C.c_int32),
        ("randomized", C.c_int32),
        ("compress", RoCompressCfg),
        ("tol", C.c_double),
        ("max_iter", C.c_int32),
        ("init", C.c_int32),
        ("seed", C.c_uint64),
    ]


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        _lib.ro_last_error.restype = C.c_char_p
        for name in ("ro_mix64", "ro_derive_seed", "ro_stream_id"):
            getattr(_lib, name).restype = C.c_uint64
        _lib.ro_mix64.argtypes = [C.c_uint64]
        _lib.ro_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        _lib.ro_stream_id.argtypes = [C.c_uint64, C.c_uint64]
        _lib.ro_stream_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int64, dp,
                                         C.POINTER(C.c_uint64)]
        _lib.ro_sketch_matrix_d.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int, dp]
        _lib.ro_sketch_matrix_f.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int, fp]
        I, L, U, D, V = C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
        sig = {
            "ro_unfold_d": [I, V, V, L, V],
            "ro_fold_d": [I, V, V, L, L, L, V],
            "ro_khatri_rao_d": [L, L, V, L, L, V, V],
            "ro_plu_basis_d": [L, L, V, V, V], "ro_plu_basis_f": [L, L, V, V, V],
            "ro_thin_qr_d": [L, L, V, V, V], "ro_thin_qr_f": [L, L, V, V, V],
            "ro_pinv_psd_d": [L, L, V, V, V], "ro_pinv_psd_f": [L, L, V, V, V],
            "ro_sym_eig": [I, V, V, V],
            "ro_compress_d": [I, V, V, V, V, V, V, V, V, V],
            "ro_compress_f": [I, V, V, V, V, V, V, V, V, V],
            "ro_decompose_d": [I, V, V, V, V, V, V, V, V, V, V, V],
            "ro_decompose_f": [I, V, V, V, V, V, V, V, V, V, V, V],
            "ro_projection_residual_d": [I, V, V, V, V],
            "ro_validate_bound_d": [I, V, V, L, L, I, U, V, V, V],
            "ro_init_factors_d": [I, V, V, L, U, I, V],
            "ro_normalize_d": [I, V, L, V, V, V, V],
            "ro_reconstruct_d": [I, V, L, V, V, V],
            "ro_relative_error_d": [I, V, V, L, V, V, V],
            "ro_relative_error_f": [I, V, V, L, V, V, V],
            "ro_fit_d": [I, V, V, L, V, V, V],
            "ro_random_lowrank_d": [I, V, L, U, D, U, V, V, V],
            "ro_add_noise_d": [I, V, V, D, U, V],
            "ro_synth_d": [I, I, V, L, U, D, V, V, V],
            "ro_synth_f": [I, I, V, L, U, D, V, V, V],
        }
        for name, at in sig.items():
            fn = getattr(_lib, name)
            fn.argtypes = at
            fn.restype = C.c_int
        _lib.ro_sym_eig.restype = None
    return _lib


class OracleInvalidArgument(ValueError):
    pass


class OracleSolverError(RuntimeError):
    def __init__(self, msg, iteration):
        super().__init__(msg)
        self.iteration = iteration


def _check(code: int) -> None:
    if code == 0:
        return
    msg = lib().ro_last_error().decode()
    if code == 1:
        raise OracleInvalidArgument(msg)
    if code == 2:
        raise OracleSolverError(msg, lib().ro_last_error_iteration())
    raise RuntimeError(msg)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _shape(shape: Sequence[int]):
    s = np.ascontiguousarray(np.asarray(shape, dtype=np.int64))
    return s, _p(s, i64p)


# --------------------------------------------------------------------- RNG
STREAM_COMPRESS, STREAM_INIT, STREAM_FACTORS, STREAM_NOISE = 1, 2, 3, 4


def mix64(z: int) -> int:
    return lib().ro_mix64(z)


def derive_seed(seed: int, salt: int) -> int:
    return lib().ro_derive_seed(seed, salt)


def stream_id(domain: int, k: int = 0) -> int:
    return lib().ro_stream_id(domain, k)


def stream_draws(seed: int, sid: int, kind: str, n: int) -> np.ndarray:
    kinds = {"normal": 0, "uniform01": 1, "uniform_sym": 2, "bits": 3}
    out = np.zeros(n, dtype=np.float64)
    bits = np.zeros(n, dtype=np.uint64)
    lib().ro_stream_draws(seed, sid, kinds[kind], n, _p(out, dp), _p(bits, C.POINTER(C.c_uint64)))
    return bits if kind == "bits" else out


def sketch_matrix(seed: int, mode: int, rows: int, cols: int, dist: int = 0,
                  dtype=np.float64) -> np.ndarray:
    """Omega_n (rows x cols), compress.hpp:118-124; returned column-major (F order)."""
    out = np.zeros(rows * cols, dtype=dtype)
    if dtype == np.float64:
        lib().ro_sketch_matrix_d(seed, mode, rows, cols, dist, _p(out, dp))
    else:
        lib().ro_sketch_matrix_f(seed, mode, rows, cols, dist, _p(out, fp))
    return out.reshape((rows, cols), order="F")


# ----------------------------------------------------------------- tensors
def unfold(x: np.ndarray, mode: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, sp = _shape(x.shape)
    out = np.zeros(x.size, dtype=np.float64)
    _check(lib().ro_unfold_d(x.ndim, sp, _p(x, dp), mode, _p(out, dp)))
    rows = x.shape[mode]
    return out.reshape((rows, x.size // rows), order="F")


def fold(m: np.ndarray, mode: int, shape: Sequence[int]) -> np.ndarray:
    m = np.asfortranarray(m, dtype=np.float64)
    s, sp = _shape(shape)
    out = np.zeros(int(np.prod(shape)), dtype=np.float64)
    _check(lib().ro_fold_d(len(shape), sp, _p(m, dp), m.shape[0], m.shape[1], mode, _p(out, dp)))
    return out.reshape(tuple(shape))


def khatri_rao(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.asfortranarray(a, dtype=np.float64)
    b = np.asfortranarray(b, dtype=np.float64)
    out = np.zeros(a.shape[0] * b.shape[0] * a.shape[1], dtype=np.float64)
    _check(lib().ro_khatri_rao_d(a.shape[0], a.shape[1], _p(a, dp), b.shape[0], b.shape[1],
                                 _p(b, dp), _p(out, dp)))
    return out.reshape((a.shape[0] * b.shape[0], a.shape[1]), order="F")


def _matfn(name: str, m: np.ndarray, out_cols: Optional[int] = None):
    dt = m.dtype if m.dtype in (np.float32, np.float64) else np.float64
    m = np.asfortranarray(m, dtype=dt)
    r, c = m.shape
    oc = out_cols if out_cols is not None else min(r, c)
    out = np.zeros(r * oc, dtype=dt)
    rw = C.c_int(0)
    f = getattr(lib(), name + ("_d" if dt == np.float64 else "_f"))
    pt = dp if dt == np.float64 else fp
    _check(f(C.c_int64(r), C.c_int64(c), _p(m, pt), _p(out, pt), C.byref(rw)))
    return out.reshape((r, oc), order="F"), bool(rw.value)


def plu_basis(m: np.ndarray) -> np.ndarray:
    return _matfn("ro_plu_basis", m)[0]


def thin_qr(m: np.ndarray):
    """Returns (Q, rank_warning)."""
    return _matfn("ro_thin_qr", m)


def pinv_psd(v: np.ndarray) -> np.ndarray:
    return _matfn("ro_pinv_psd", v, out_cols=v.shape[0])[0]


# ----------------------------------------------------------------- configs
@dataclass
class CompressConfig:
    """Mirrors rcp::CompressConfig (compress.hpp:23-33)."""
    target_rank: int = 0
    oversampling: int = 10
    power_iterations: int = 2
    modes: Optional[List[int]] = None
    distribution: int = 0  # 0 gaussian, 1 uniform
    stabilizer: int = 0    # 0 lu, 1 qr
    seed: int = 0

    def to_c(self):
        c = RoCompressCfg()
        c.target_rank = self.target_rank
        c.oversampling = self.oversampling
        c.power_iterations = self.power_iterations
        c.distribution = self.distribution
        c.stabilizer = self.stabilizer
        c.seed = self.seed
        keep = None
        if self.modes is not None:
            keep = np.ascontiguousarray(np.asarray(self.modes, dtype=np.int64).reshape(-1))
            c.modes_present = 1
            c.n_modes = keep.size
            c.modes = _p(keep, i64p) if keep.size else None
        return c, keep


@dataclass
class DecomposeConfig:
    """Mirrors rcp::DecomposeConfig (solve.hpp:22-31)."""
    rank: int = 1
    method: int = 0
    randomized: bool = True
    compress: CompressConfig = field(default_factory=CompressConfig)
    tol: float = 1e-5
    max_iter: int = 500
    seed: int = 0
    init: int = 0

    def to_c(self):
        c = RoDecomposeCfg()
        c.rank = self.rank
        c.method = self.method
        c.randomized = 1 if self.randomized else 0
        cc, keep = self.compress.to_c()
        c.compress = cc
        c.tol = self.tol
        c.max_iter = self.max_iter
        c.init = self.init
        c.seed = self.seed
        return c, keep


@dataclass
class Compressed:
    compressed: np.ndarray
    q: List[Optional[np.ndarray]]
    identity: List[bool]
    rank_warning: List[bool]


@dataclass
class Result:
    weights: np.ndarray
    factors: List[np.ndarray]
    trace_fit: np.ndarray
    trace_seconds: np.ndarray
    iterations: int
    converged: bool
    final_relative_error: float


def _dt(x):
    return (dp, "_d") if x.dtype == np.float64 else (fp, "_f")


def compress(x: np.ndarray, cfg: CompressConfig) -> Compressed:
    pt, suf = _dt(x)
    x = np.ascontiguousarray(x)
    s, sp = _shape(x.shape)
    c, keep = cfg.to_c()
    oshape = np.zeros(x.ndim, dtype=np.int64)
    oc = np.zeros(x.size, dtype=x.dtype)
    oq = np.zeros(int(sum(e * e for e in x.shape)), dtype=x.dtype)
    oi = np.zeros(x.ndim, dtype=np.int32)
    orw = np.zeros(x.ndim, dtype=np.int32)
    oqc = np.zeros(x.ndim, dtype=np.int64)
    f = getattr(lib(), "ro_compress" + suf)
    _check(f(x.ndim, sp, _p(x, pt), C.byref(c), _p(oshape, i64p), _p(oc, pt), _p(oq, pt),
             _p(oi, ip), _p(orw, ip), _p(oqc, i64p)))
    n = int(np.prod(oshape))
    qs, off = [], 0
    for m in range(x.ndim):
        if oi[m]:
            qs.append(None)
        else:
            cnt = x.shape[m] * int(oqc[m])
            qs.append(oq[off:off + cnt].reshape((x.shape[m], int(oqc[m])), order="F").copy())
            off += cnt
    return Compressed(oc[:n].reshape(tuple(oshape)).copy(), qs, [bool(v) for v in oi],
                      [bool(v) for v in orw])


def projection_residual(x: np.ndarray, cfg: CompressConfig) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, sp = _shape(x.shape)
    c, keep = cfg.to_c()
    out = C.c_double(0)
    _check(lib().ro_projection_residual_d(x.ndim, sp, _p(x, dp), C.byref(c), C.byref(out)))
    return out.value


def theorem_bound(x: np.ndarray, k: int, p: int, trials: int = 0, seed: int = 0):
    """theorem_bound (diagnostics.hpp:36-62) -> (tail_energies, bound); with trials > 0 also the
    validate_bound (diagnostics.hpp:68-86) mean projection residual on this tensor."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, sp = _shape(x.shape)
    tails = np.zeros(x.ndim)
    b, m = C.c_double(0), C.c_double(0)
    _check(lib().ro_validate_bound_d(x.ndim, sp, _p(x, dp), C.c_int64(k), C.c_int64(p), int(trials),
                                     C.c_uint64(seed), _p(tails, dp), C.byref(b), C.byref(m)))
    return (tails, b.value) if trials <= 0 else (tails, b.value, m.value)


def decompose(x: np.ndarray, cfg: DecomposeConfig) -> Result:
    pt, suf = _dt(x)
    x = np.ascontiguousarray(x)
    s, sp = _shape(x.shape)
    c, keep = cfg.to_c()
    R = cfg.rank
    w = np.zeros(R, dtype=x.dtype)
    f = np.zeros(sum(x.shape) * R, dtype=x.dtype)
    cap = max(cfg.max_iter, 1)
    ti = np.zeros(cap, dtype=np.int32)
    tf = np.zeros(cap, dtype=np.float64)
    ts = np.zeros(cap, dtype=np.float64)
    it, conv, re = C.c_int(0), C.c_int(0), C.c_double(0)
    fn = getattr(lib(), "ro_decompose" + suf)
    _check(fn(x.ndim, sp, _p(x, pt), C.byref(c), _p(w, pt), _p(f, pt), _p(ti, ip), _p(tf, dp),
              _p(ts, dp), C.byref(it), C.byref(conv), C.byref(re)))
    facs, off = [], 0
    for e in x.shape:
        facs.append(f[off:off + e * R].reshape((e, R), order="F").copy())
        off += e * R
    n = it.value
    return Result(w, facs, tf[:n].copy(), ts[:n].copy(), n, bool(conv.value), re.value)


def _model_buffers(weights, factors):
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    f = np.concatenate([np.asarray(a, dtype=np.float64).reshape(-1, order="F") for a in factors])
    shape = [a.shape[0] for a in factors]
    return w, f, shape


def init_factors(x: np.ndarray, rank: int, seed: int, method: int = 0) -> List[np.ndarray]:
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, sp = _shape(x.shape)
    out = np.zeros(sum(x.shape) * rank, dtype=np.float64)
    _check(lib().ro_init_factors_d(x.ndim, sp, _p(x, dp), C.c_int64(rank), C.c_uint64(seed), method,
                                   _p(out, dp)))
    res, off = [], 0
    for e in x.shape:
        res.append(out[off:off + e * rank].reshape((e, rank), order="F").copy())
        off += e * rank
    return res


def normalize(weights, factors):
    w, f, shape = _model_buffers(weights, factors)
    s, sp = _shape(shape)
    ow, of = np.zeros_like(w), np.zeros_like(f)
    _check(lib().ro_normalize_d(len(shape), sp, C.c_int64(w.size), _p(w, dp), _p(f, dp), _p(ow, dp),
                                _p(of, dp)))
    R = w.size
    res, off = [], 0
    for e in shape:
        res.append(of[off:off + e * R].reshape((e, R), order="F").copy())
        off += e * R
    return ow, res


def reconstruct(weights, factors) -> np.ndarray:
    w, f, shape = _model_buffers(weights, factors)
    s, sp = _shape(shape)
    out = np.zeros(int(np.prod(shape)), dtype=np.float64)
    _check(lib().ro_reconstruct_d(len(shape), sp, C.c_int64(w.size), _p(w, dp), _p(f, dp), _p(out, dp)))
    return out.reshape(tuple(shape))


def relative_error(x: np.ndarray, weights, factors) -> float:
    out = C.c_double(0)
    s, sp = _shape(x.shape)
    if x.dtype == np.float32:
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float32))
        f = np.concatenate([np.asarray(a, dtype=np.float32).reshape(-1, order="F") for a in factors])
        x = np.ascontiguousarray(x)
        _check(lib().ro_relative_error_f(x.ndim, sp, _p(x, fp), C.c_int64(w.size), _p(w, fp), _p(f, fp),
                                         C.byref(out)))
    else:
        w, f, _ = _model_buffers(weights, factors)
        x = np.ascontiguousarray(x, dtype=np.float64)
        _check(lib().ro_relative_error_d(x.ndim, sp, _p(x, dp), C.c_int64(w.size), _p(w, dp), _p(f, dp),
                                         C.byref(out)))
    return out.value


def fit(x: np.ndarray, weights, factors) -> float:
    w, f, _ = _model_buffers(weights, factors)
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, sp = _shape(x.shape)
    out = C.c_double(0)
    _check(lib().ro_fit_d(x.ndim, sp, _p(x, dp), C.c_int64(w.size), _p(w, dp), _p(f, dp), C.byref(out)))
    return out.value


def random_lowrank(shape: Sequence[int], rank: int, seed: int, snr: float = 0.0,
                   noise_seed: int = 0):
    """random_lowrank (synthetic.hpp:21-38) [+ add_noise (42-58) when snr > 0]."""
    s, sp = _shape(shape)
    out = np.zeros(int(np.prod(shape)), dtype=np.float64)
    w = np.zeros(rank, dtype=np.float64)
    f = np.zeros(sum(shape) * rank, dtype=np.float64)
    _check(lib().ro_random_lowrank_d(len(shape), sp, C.c_int64(rank), C.c_uint64(seed), C.c_double(snr),
                                     C.c_uint64(noise_seed), _p(out, dp), _p(w, dp), _p(f, dp)))
    facs, off = [], 0
    for e in shape:
        facs.append(f[off:off + e * rank].reshape((e, rank), order="F").copy())
        off += e * rank
    return out.reshape(tuple(shape)), (w, facs)


def add_noise(x: np.ndarray, snr: float, seed: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, sp = _shape(x.shape)
    out = np.zeros_like(x)
    _check(lib().ro_add_noise_d(x.ndim, sp, _p(x, dp), C.c_double(snr), C.c_uint64(seed), _p(out, dp)))
    return out


def synth(kind: int, shape: Sequence[int], rank: int, seed: int, snr: float, dtype=np.float64):
    """Ground truth + noise for BASELINE configs C2..C5 (kind 2..5)."""
    s, sp = _shape(shape)
    out = np.zeros(int(np.prod(shape)), dtype=dtype)
    w = np.zeros(rank, dtype=dtype)
    f = np.zeros(sum(shape) * rank, dtype=dtype)
    pt, suf = (dp, "_d") if dtype == np.float64 else (fp, "_f")
    fn = getattr(lib(), "ro_synth" + suf)
    _check(fn(kind, len(shape), sp, C.c_int64(rank), C.c_uint64(seed), C.c_double(snr), _p(out, pt),
              _p(w, pt), _p(f, pt)))
    facs, off = [], 0
    for e in shape:
        facs.append(f[off:off + e * rank].reshape((e, rank), order="F").copy())
        off += e * rank
    return out.reshape(tuple(shape)), (w, facs)
