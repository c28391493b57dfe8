"""Host-side mirror of the reference's rCP C++ API over the CUDA C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/rcp/{compress,solve,kruskal}.hpp:

    rcp::CompressConfig   -> CompressConfig      (compress.hpp:23-33)
    rcp::DecomposeConfig  -> DecomposeConfig     (solve.hpp:22-31)
    rcp::Kruskal          -> Kruskal             (kruskal.hpp:16-30)
    rcp::FitTrace         -> FitTrace            (solve.hpp:35-45)
    rcp::SolverError      -> SolverError         (solve.hpp:48-57)
    std::invalid_argument -> ValueError          (types.hpp:30-32)
    rcp::compress         -> compress()          (compress.hpp:86-146)
    rcp::decompose        -> decompose()         (solve.hpp:381-398)
    rcp::relative_error   -> relative_error()    (kruskal.hpp:187-194)

Tensors are numpy arrays in C (row-major) order, exactly the reference's
storage; matrices (factors, bases) are returned as Fortran-ordered arrays of
shape (rows, cols), like the reference's column-major Eigen matrices. All
computation runs in librcpg.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as _L

GAUSSIAN, UNIFORM = 0, 1          # rcp::RandomDistribution
LU, QR = 0, 1                      # rcp::PowerStabilizer
ALS, BCD = 0, 1                    # rcp::SolveMethod
EIGENVECTORS, RANDOM = 0, 1        # rcp::InitMethod
COMPRESS, INIT, FACTORS, NOISE, PHASES, TRIAL = 1, 2, 3, 4, 5, 6  # rcp::StreamDomain (random.hpp:39-46)


class SolverError(RuntimeError):
    """rcp::SolverError (solve.hpp:48-57): numeric failure with its iteration."""

    def __init__(self, message: str, iteration: int):
        super().__init__(message)
        self._iteration = iteration

    def iteration(self) -> int:
        return self._iteration


class CudaError(RuntimeError):
    pass


@dataclass
class CompressConfig:
    target_rank: int = 0
    oversampling: int = 10
    power_iterations: int = 2
    modes: Optional[List[int]] = None  # None = all modes, [] = none
    distribution: int = GAUSSIAN
    stabilizer: int = LU
    seed: int = 0

    def _c(self):
        c = _L.CompressConfigC()
        c.target_rank = int(self.target_rank)
        c.oversampling = int(self.oversampling)
        c.power_iterations = int(self.power_iterations)
        c.distribution = int(self.distribution)
        c.stabilizer = int(self.stabilizer)
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        keep = None
        if self.modes is not None:
            keep = np.ascontiguousarray(np.asarray(list(self.modes), dtype=np.int64))
            c.modes_present = 1
            c.n_modes = keep.size
            c.modes = keep.ctypes.data_as(C.POINTER(C.c_int64)) if keep.size else None
        return c, keep


@dataclass
class DecomposeConfig:
    rank: int = 1
    method: int = ALS
    randomized: bool = True
    compress: CompressConfig = field(default_factory=CompressConfig)
    tol: float = 1e-5
    max_iter: int = 500
    seed: int = 0
    init: int = EIGENVECTORS

    def _c(self):
        c = _L.DecomposeConfigC()
        c.rank = int(self.rank)
        c.method = int(self.method)
        c.randomized = 1 if self.randomized else 0
        cc, keep = self.compress._c()
        c.compress = cc
        c.tol = float(self.tol)
        c.max_iter = int(self.max_iter)
        c.init = int(self.init)
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        return c, keep


@dataclass
class Kruskal:
    weights: np.ndarray
    factors: List[np.ndarray]

    def rank(self) -> int:
        return int(self.weights.size)

    def order(self) -> int:
        return len(self.factors)

    def shape(self) -> Tuple[int, ...]:
        return tuple(f.shape[0] for f in self.factors)


@dataclass
class FitTrace:
    @dataclass
    class Entry:
        iteration: int
        fit: float
        seconds: float

    entries: List["FitTrace.Entry"] = field(default_factory=list)
    final_relative_error: float = float("nan")
    iterations: int = 0
    converged: bool = False


@dataclass
class ModeBasis:
    q: Optional[np.ndarray]
    identity: bool
    dim: int
    rank_warning: bool

    def rows(self) -> int:
        return self.dim if self.identity else self.q.shape[0]

    def cols(self) -> int:
        return self.dim if self.identity else self.q.shape[1]


@dataclass
class CompressionResult:
    compressed: np.ndarray
    bases: List[ModeBasis]


# ------------------------------------------------------------------ context
class Context:
    """One rcpg_context (device stream + workspace); one per host thread."""

    def __init__(self, device: int = 0):
        self.lib = _L.lib()
        h = C.c_void_p()
        st = self.lib.rcpg_create(device, C.byref(h))
        if st != _L.RCPG_OK:
            raise CudaError(f"rcpg_create(device={device}) failed with status {st}: no usable CUDA device")
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.rcpg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----- sharding: one context per rank / GPU
    def comm_init_nccl(self, nranks: int, rank: int, unique_id: bytes) -> None:
        """Join an NCCL communicator (unique_id from comm_unique_id() on rank 0, broadcast by the caller)."""
        assert len(unique_id) == 128
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self.check(self.lib.rcpg_comm_init_nccl(self.h, int(nranks), int(rank), buf))

    def comm_rank(self) -> Tuple[int, int]:
        r, n = C.c_int32(), C.c_int32()
        self.lib.rcpg_comm_rank(self.h, C.byref(r), C.byref(n))
        return r.value, n.value

    def check(self, status: int) -> None:
        if status == _L.RCPG_OK:
            return
        msg = (self.lib.rcpg_last_error(self.h) or b"").decode()
        if status == _L.RCPG_INVALID_ARGUMENT:
            raise ValueError(msg)
        if status == _L.RCPG_SOLVER_ERROR:
            raise SolverError(msg, int(self.lib.rcpg_last_error_iteration(self.h)))
        if status == _L.RCPG_OOM:
            raise MemoryError(msg)
        raise CudaError(msg)

    # options (include/rcpg.h rcpg_set_option) ---------------------------
    def set_option(self, name: str, value: int) -> None:
        """"fp32_arith": 0 faithful fp64 arithmetic (default) / 1 fast 3xTF32;
        "omega_host": 0 device Omega (default) / 1 host-evaluated, uploaded (bit-identical);
        "pass_timing": 0 no per-pass events (default) / 1 events on, read with pass_timings()."""
        self.check(self.lib.rcpg_set_option(self.h, name.encode(), int(value)))

    def get_option(self, name: str) -> int:
        v = C.c_int64()
        self.check(self.lib.rcpg_get_option(self.h, name.encode(), C.byref(v)))
        return int(v.value)

    # diagnostics -------------------------------------------------------
    def pass_timings(self):
        cap = 4096
        names = C.create_string_buffer(cap * 32)
        ms = np.zeros(cap, dtype=np.float64)
        by = np.zeros(cap, dtype=np.float64)
        n = self.lib.rcpg_pass_timings(self.h, names, cap * 32, ms.ctypes.data, by.ctypes.data, cap)
        raw = names.raw.split(b"\0")
        return [(raw[i].decode(), float(ms[i]), float(by[i])) for i in range(n)]

    def pass_offsets(self):
        st = np.zeros(4096, dtype=np.float64)
        n = self.lib.rcpg_pass_offsets(self.h, st.ctypes.data, 4096)
        return [float(x) for x in st[:n]]

    def kernel_launches(self) -> int:
        return int(self.lib.rcpg_kernel_launches(self.h))

    def synchronize(self):
        self.check(self.lib.rcpg_synchronize(self.h))

    def event_record(self, slot: int):
        self.check(self.lib.rcpg_event_record(self.h, slot))

    def event_elapsed_ms(self, a: int, b: int) -> float:
        out = C.c_double()
        self.check(self.lib.rcpg_event_elapsed(self.h, a, b, C.byref(out)))
        return out.value

    def host_register(self, arr: np.ndarray):
        self.check(self.lib.rcpg_host_register(self.h, arr.ctypes.data, arr.nbytes))

    def host_unregister(self, arr: np.ndarray):
        self.check(self.lib.rcpg_host_unregister(self.h, arr.ctypes.data))


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(0)
        _tls.ctx = ctx
    return ctx


def _dtype_code(dt) -> int:
    dt = np.dtype(dt)
    if dt == np.float64:
        return _L.RCPG_F64
    if dt == np.float32:
        return _L.RCPG_F32
    raise ValueError("Tensor: unsupported dtype (float32 / float64 only)")


class DeviceTensor:
    """A tensor resident in HBM (rcpg_tensor)."""

    def __init__(self, ctx: Context, handle, shape, dtype, global_shape=None, slab=None, slab_mode=None):
        self.ctx = ctx
        self.h = handle
        self.shape = tuple(int(e) for e in shape)  # local shape (a slab's extent is hi - lo)
        self.dtype = np.dtype(dtype)
        self.global_shape = tuple(int(e) for e in (global_shape if global_shape is not None else shape))
        self.slab_range = slab  # (lo, hi) along slab_mode, or None
        self.slab_mode = slab_mode

    def slab(self, lo: int, hi: int, ctx: Optional[Context] = None, mode: Optional[int] = None) -> "DeviceTensor":
        """Slab [lo, hi) of mode `mode` (default: the last; the first is also supported) as a
        device copy, for a sharded decomposition."""
        ctx = ctx or self.ctx
        mode = len(self.shape) - 1 if mode is None else int(mode)
        h = C.c_void_p()
        ctx.check(ctx.lib.rcpg_tensor_slab_mode(ctx.h, self.h, mode, int(lo), int(hi), C.byref(h)))
        shape = list(self.shape)
        shape[mode] = int(hi) - int(lo)
        return DeviceTensor(ctx, h, shape, self.dtype, self.shape, (int(lo), int(hi)), mode)

    @classmethod
    def upload_slab(cls, x_slab: np.ndarray, global_shape: Sequence[int], lo: int, hi: int,
                    ctx: Optional[Context] = None, mode: Optional[int] = None) -> "DeviceTensor":
        """Upload this rank's slab (row-major, extent hi - lo along `mode`, default the last) of a
        tensor of `global_shape`."""
        ctx = ctx or default_context()
        x = np.ascontiguousarray(x_slab)
        gs = np.asarray(global_shape, dtype=np.int64)
        mode = len(gs) - 1 if mode is None else int(mode)
        h = C.c_void_p()
        ctx.check(ctx.lib.rcpg_tensor_upload_slab_mode(ctx.h, _dtype_code(x.dtype), len(gs), gs.ctypes.data, mode,
                                                       int(lo), int(hi), x.ctypes.data, C.byref(h)))
        return cls(ctx, h, x.shape, x.dtype, tuple(global_shape), (int(lo), int(hi)), mode)

    @classmethod
    def upload(cls, x: np.ndarray, ctx: Optional[Context] = None) -> "DeviceTensor":
        ctx = ctx or default_context()
        x = np.ascontiguousarray(x)
        code = _dtype_code(x.dtype)
        shape = np.asarray(x.shape, dtype=np.int64)
        h = C.c_void_p()
        ctx.check(ctx.lib.rcpg_tensor_upload(ctx.h, code, x.ndim, shape.ctypes.data, x.ctypes.data, C.byref(h)))
        return cls(ctx, h, x.shape, x.dtype)

    @classmethod
    def synth(cls, shape: Sequence[int], weights: np.ndarray, factors: Sequence[np.ndarray], snr: float,
              noise_seed: int, dtype=np.float64, ctx: Optional[Context] = None) -> "DeviceTensor":
        """Dense model + add_noise generated on the device (synthetic inputs)."""
        ctx = ctx or default_context()
        sh = np.asarray(shape, dtype=np.int64)
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        f = np.concatenate([np.asarray(a, dtype=np.float64).reshape(-1, order="F") for a in factors])
        h = C.c_void_p()
        ctx.check(ctx.lib.rcpg_synth(ctx.h, _dtype_code(dtype), len(shape), sh.ctypes.data, w.size,
                                     w.ctypes.data, f.ctypes.data, float(snr), int(noise_seed), C.byref(h)))
        return cls(ctx, h, shape, dtype)

    def download(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=self.dtype)
        self.ctx.check(self.ctx.lib.rcpg_tensor_download(self.ctx.h, self.h, out.ctypes.data))
        return out

    def free(self):
        if self.h:
            self.ctx.lib.rcpg_tensor_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    """128-byte NCCL unique id (create on rank 0, broadcast, then Context.comm_init_nccl on every rank)."""
    lib = _L.lib()
    buf = C.create_string_buffer(128)
    st = lib.rcpg_comm_unique_id(buf)
    if st != _L.RCPG_OK:
        raise CudaError(f"rcpg_comm_unique_id failed with status {st}")
    return buf.raw


def comm_init_loopback(contexts: Sequence[Context]) -> None:
    """Virtual ranks in one process (contexts[r] is rank r, one host thread each, any GPU)."""
    arr = (C.c_void_p * len(contexts))(*[c.h.value if isinstance(c.h, C.c_void_p) else c.h for c in contexts])
    contexts[0].check(contexts[0].lib.rcpg_comm_init_loopback(arr, len(contexts)))


def slab_range(extent: int, nranks: int, rank: int) -> Tuple[int, int]:
    """The balanced split [lo, hi) of [0, extent) that rank `rank` holds (host only)."""
    lo, hi = C.c_int64(), C.c_int64()
    _L.lib().rcpg_slab_range(int(extent), int(nranks), int(rank), C.byref(lo), C.byref(hi))
    return lo.value, hi.value


class _HostTensor:
    """A host array handed to rcpg_decompose_host (shape / dtype views like DeviceTensor's)."""

    def __init__(self, x: np.ndarray):
        self.x = x
        self.dtype = x.dtype
        self.global_shape = tuple(int(e) for e in x.shape)


def _as_device(x, ctx):
    if isinstance(x, DeviceTensor):
        return x, False
    return DeviceTensor.upload(np.asarray(x), ctx), True


# ---------------------------------------------------------------- operators
def compress(t, cfg: CompressConfig, ctx: Optional[Context] = None) -> CompressionResult:
    """rcp::compress (compress.hpp:86-146) on the GPU."""
    ctx = ctx or default_context()
    dt, tmp = _as_device(t, ctx)
    try:
        c, keep = cfg._c()
        h = C.c_void_p()
        ctx.check(ctx.lib.rcpg_compress(ctx.h, dt.h, C.byref(c), C.byref(h)))
        try:
            order = ctx.lib.rcpg_compressed_order(h)
            shape = np.zeros(order, dtype=np.int64)
            ctx.lib.rcpg_compressed_shape(h, shape.ctypes.data)
            out = np.empty(tuple(int(e) for e in shape), dtype=dt.dtype)
            ctx.check(ctx.lib.rcpg_compressed_download(ctx.h, h, out.ctypes.data))
            bases = []
            for m in range(order):
                ident, dim, cols, rw = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32()
                ctx.lib.rcpg_compressed_basis_info(h, m, C.byref(ident), C.byref(dim), C.byref(cols), C.byref(rw))
                q = None
                if not ident.value:
                    q = np.empty((dim.value, cols.value), dtype=dt.dtype, order="F")
                    ctx.check(ctx.lib.rcpg_compressed_basis_download(ctx.h, h, m, q.ctypes.data))
                bases.append(ModeBasis(q, bool(ident.value), int(dim.value), bool(rw.value)))
        finally:
            ctx.lib.rcpg_compressed_free(h)
        return CompressionResult(out, bases)
    finally:
        if tmp:
            dt.free()


def projection_residual(t, cfg: CompressConfig, ctx: Optional[Context] = None) -> float:
    """projection_residual(t, compress(t, cfg)) (compress.hpp:148-164) on the GPU."""
    ctx = ctx or default_context()
    dt, tmp = _as_device(t, ctx)
    try:
        c, keep = cfg._c()
        h = C.c_void_p()
        ctx.check(ctx.lib.rcpg_compress(ctx.h, dt.h, C.byref(c), C.byref(h)))
        try:
            out = C.c_double()
            ctx.check(ctx.lib.rcpg_projection_residual(ctx.h, dt.h, h, C.byref(out)))
            return out.value
        finally:
            ctx.lib.rcpg_compressed_free(h)
    finally:
        if tmp:
            dt.free()


@dataclass
class BoundReport:
    """rcp::BoundReport (diagnostics.hpp:23-31)."""
    tail_energies: List[float]
    bound: float
    empirical_mean: float = float("nan")
    trials: int = 0
    k: int = 0
    p: int = 0


def theorem_bound(t, k: int, p: int, ctx: Optional[Context] = None) -> BoundReport:
    """theorem_bound (diagnostics.hpp:36-62) on the GPU: per-mode tail energies of every
    unfolding (Gram eigenvalues, fp64) and sqrt(1 + k/(p-1)) sqrt(sum of tails)."""
    ctx = ctx or default_context()
    dt, tmp = _as_device(t, ctx)
    try:
        tails = np.zeros(len(dt.shape))
        b = C.c_double()
        ctx.check(ctx.lib.rcpg_theorem_bound(ctx.h, dt.h, int(k), int(p), tails.ctypes.data, C.byref(b)))
        return BoundReport([float(x) for x in tails], b.value, k=int(k), p=int(p))
    finally:
        if tmp:
            dt.free()


def validate_bound(t, k: int, p: int, trials: int, seed: int, ctx: Optional[Context] = None) -> BoundReport:
    """validate_bound (diagnostics.hpp:68-86) on a given tensor (the reference draws it with
    random_lowrank<double>(shape, rank, seed)): the theorem bound and the mean projection
    residual of `trials` single-pass compressions (q = 0) with seeds
    derive_seed(seed, stream_id(trial, t))."""
    if trials < 1:
        raise ValueError("validate_bound: need at least one trial")
    ctx = ctx or default_context()
    dt, tmp = _as_device(t, ctx)
    try:
        rep = theorem_bound(dt, k, p, ctx=ctx)
        total = 0.0
        for trial in range(trials):
            cfg = CompressConfig(target_rank=k, oversampling=p, power_iterations=0,
                                 seed=derive_seed(seed, stream_id(TRIAL, trial)))
            total += projection_residual(dt, cfg, ctx=ctx)
        rep.trials = trials
        rep.empirical_mean = total / trials
        return rep
    finally:
        if tmp:
            dt.free()


def decompose(t, cfg: DecomposeConfig, ctx: Optional[Context] = None) -> Tuple[Kruskal, FitTrace]:
    """rcp::decompose (solve.hpp:381-398) on the GPU. `t` is a numpy array
    (copied to HBM inside the call) or a DeviceTensor already in HBM."""
    ctx = ctx or default_context()
    if not isinstance(t, DeviceTensor):
        # host tensor: rcpg_decompose_host (the upload is enqueued in front of the decomposition,
        # one synchronization at the end of the call)
        x = np.ascontiguousarray(np.asarray(t))
        dt, tmp = _HostTensor(x), False
    else:
        dt, tmp = t, False
    try:
        c, keep = cfg._c()
        R = max(int(cfg.rank), 1)
        cap = max(int(cfg.max_iter), 1)
        w = np.empty(R, dtype=dt.dtype)  # (every entry read below is written by the call)
        f = np.empty(sum(dt.global_shape) * R, dtype=dt.dtype)
        ti = np.empty(cap, dtype=np.int32)
        tf = np.empty(cap, dtype=np.float64)
        ts = np.empty(cap, dtype=np.float64)
        res = _L.ResultC()
        res.weights = w.ctypes.data
        res.factors = f.ctypes.data
        res.trace_iteration = ti.ctypes.data_as(C.POINTER(C.c_int32))
        res.trace_fit = tf.ctypes.data_as(C.POINTER(C.c_double))
        res.trace_seconds = ts.ctypes.data_as(C.POINTER(C.c_double))
        res.trace_capacity = cap
        if isinstance(dt, _HostTensor):
            shape = np.asarray(dt.x.shape, dtype=np.int64)
            ctx.check(ctx.lib.rcpg_decompose_host(ctx.h, _dtype_code(dt.dtype), dt.x.ndim, shape.ctypes.data,
                                                  dt.x.ctypes.data, C.byref(c), C.byref(res)))
        else:
            ctx.check(ctx.lib.rcpg_decompose(ctx.h, dt.h, C.byref(c), C.byref(res)))
        facs, off = [], 0
        for e in dt.global_shape:
            facs.append(f[off:off + e * R].reshape((e, R), order="F").copy(order="F"))
            off += e * R
        n = int(res.iterations)
        trace = FitTrace(
            entries=[FitTrace.Entry(int(ti[i]), float(tf[i]), float(ts[i])) for i in range(min(n, cap))],
            final_relative_error=float(res.final_relative_error),
            iterations=n,
            converged=bool(res.converged),
        )
        return Kruskal(w, facs), trace
    finally:
        if tmp:
            dt.free()


def als_solve(t, cfg: DecomposeConfig, ctx: Optional[Context] = None) -> Tuple[Kruskal, FitTrace]:
    """rcp::als_solve (solve.hpp:183-262): CP-ALS on the tensor itself, no compression
    (cfg.method and cfg.randomized are ignored), on the GPU."""
    import copy
    d = copy.copy(cfg)
    d.randomized = False
    d.method = ALS
    ctx = ctx or default_context()
    dt, tmp = _as_device(t, ctx)
    try:
        c, keep = d._c()
        R = max(int(d.rank), 1)
        cap = max(int(d.max_iter), 1)
        w = np.zeros(R, dtype=dt.dtype)
        f = np.zeros(sum(dt.global_shape) * R, dtype=dt.dtype)
        ti = np.zeros(cap, dtype=np.int32)
        tf = np.zeros(cap, dtype=np.float64)
        ts = np.zeros(cap, dtype=np.float64)
        res = _L.ResultC()
        res.weights = w.ctypes.data
        res.factors = f.ctypes.data
        res.trace_iteration = ti.ctypes.data_as(C.POINTER(C.c_int32))
        res.trace_fit = tf.ctypes.data_as(C.POINTER(C.c_double))
        res.trace_seconds = ts.ctypes.data_as(C.POINTER(C.c_double))
        res.trace_capacity = cap
        ctx.check(ctx.lib.rcpg_als_solve(ctx.h, dt.h, C.byref(c), C.byref(res)))
        facs, off = [], 0
        for e in dt.global_shape:
            facs.append(f[off:off + e * R].reshape((e, R), order="F").copy(order="F"))
            off += e * R
        n = int(res.iterations)
        trace = FitTrace(
            entries=[FitTrace.Entry(int(ti[i]), float(tf[i]), float(ts[i])) for i in range(min(n, cap))],
            final_relative_error=float(res.final_relative_error),
            iterations=n,
            converged=bool(res.converged),
        )
        return Kruskal(w, facs), trace
    finally:
        if tmp:
            dt.free()


def recover(model: Kruskal, bases, ctx: Optional[Context] = None) -> Kruskal:
    """rcp::recover (kruskal.hpp:198-220) on the GPU: A_n = Q_n A~_n for every
    non-identity basis (identity modes copied), then normalize (kruskal.hpp:117-176).
    `bases` is a list of ModeBasis (CompressionResult.bases)."""
    ctx = ctx or default_context()
    w = np.ascontiguousarray(model.weights)
    dtype = w.dtype
    if dtype not in (np.float32, np.float64):
        raise TypeError("recover: float32 or float64 models")
    R = int(w.size)
    order = len(model.factors)
    if len(bases) != order:
        raise ValueError("recover: need exactly one basis per mode")
    sext = np.array([f.shape[0] for f in model.factors], dtype=np.int64)
    f = np.concatenate([np.asarray(x, dtype=dtype).reshape(-1, order="F") for x in model.factors])
    ident = np.array([1 if b.identity else 0 for b in bases], dtype=np.int32)
    dims = np.array([int(b.dim) for b in bases], dtype=np.int64)
    cols = np.array([0 if b.identity else int(np.asarray(b.q).shape[1]) for b in bases], dtype=np.int64)
    qs = [np.asarray(b.q, dtype=dtype).reshape(-1, order="F") for b in bases if not b.identity]
    q = np.concatenate(qs) if qs else np.zeros(1, dtype=dtype)
    ow = np.zeros(R, dtype=dtype)
    of = np.zeros(int(dims.sum()) * R, dtype=dtype)
    ctx.check(ctx.lib.rcpg_recover(ctx.h, _dtype_code(dtype), order, R, sext.ctypes.data, w.ctypes.data,
                                   f.ctypes.data, ident.ctypes.data, dims.ctypes.data, cols.ctypes.data,
                                   q.ctypes.data, ow.ctypes.data, of.ctypes.data))
    facs, off = [], 0
    for e in dims:
        facs.append(of[off:off + e * R].reshape((e, R), order="F").copy(order="F"))
        off += int(e) * R
    return Kruskal(ow, facs)


def relative_error(t, model: Kruskal, ctx: Optional[Context] = None) -> float:
    """rcp::relative_error (kruskal.hpp:187-194) on the GPU (double accumulation)."""
    ctx = ctx or default_context()
    dt, tmp = _as_device(t, ctx)
    try:
        w = np.ascontiguousarray(np.asarray(model.weights, dtype=dt.dtype))
        f = np.concatenate([np.asarray(a, dtype=dt.dtype).reshape(-1, order="F") for a in model.factors])
        out = C.c_double()
        ctx.check(ctx.lib.rcpg_relative_error(ctx.h, dt.h, w.size, w.ctypes.data, f.ctypes.data, C.byref(out)))
        return out.value
    finally:
        if tmp:
            dt.free()


def sketch_matrix(seed: int, mode: int, rows: int, cols: int, distribution: int = GAUSSIAN, dtype=np.float64,
                  ctx: Optional[Context] = None) -> np.ndarray:
    """Omega_n exactly as compress.hpp:118-124 draws it, generated on the GPU."""
    ctx = ctx or default_context()
    out = np.empty((rows, cols), dtype=dtype, order="F")
    ctx.check(ctx.lib.rcpg_sketch_matrix(ctx.h, _dtype_code(dtype), int(seed), mode, rows, cols, distribution,
                                         out.ctypes.data))
    return out


def stream_pass(kind: str, x: np.ndarray, p: np.ndarray, cols: int, ctx: Optional[Context] = None) -> np.ndarray:
    """One streamed mode-n pass on the GPU (compress.hpp:118-145 products).

    ``x`` is a mode view of shape (L, I, R) (row-major). ``kind="sketch"``: ``p`` has
    shape (L, cols, R), returns Y (I, cols) = sum_{a,b} x[a,:,b] p[a,:,b]^T.
    ``kind="project"``: ``p`` is Q (I, cols), returns O (L, cols, R) = Q^T x[a].
    """
    ctx = ctx or default_context()
    x = np.ascontiguousarray(x)
    L, I, R = x.shape
    if kind == "sketch":
        p = np.ascontiguousarray(p, dtype=x.dtype)
        assert p.shape == (L, cols, R)
        out = np.empty((cols, I), dtype=x.dtype)
        k = 0
    elif kind == "project":
        p = np.asfortranarray(p, dtype=x.dtype)
        assert p.shape == (I, cols)
        out = np.empty((L, cols, R), dtype=x.dtype)
        k = 1
    else:
        raise ValueError(kind)
    ctx.check(ctx.lib.rcpg_stream_pass(ctx.h, _dtype_code(x.dtype), k, L, I, R, cols, x.ctypes.data,
                                       p.ctypes.data, out.ctypes.data))
    return out.T if k == 0 else out


def plu_basis(m: np.ndarray, ctx: Optional[Context] = None) -> np.ndarray:
    """detail::plu_basis (compress.hpp:47-58) on the GPU."""
    ctx = ctx or default_context()
    m = np.asfortranarray(m)
    r = min(m.shape)
    out = np.empty((m.shape[0], r), dtype=m.dtype, order="F")
    ctx.check(ctx.lib.rcpg_plu_basis(ctx.h, _dtype_code(m.dtype), m.shape[0], m.shape[1], m.ctypes.data,
                                     out.ctypes.data))
    return out


def thin_qr(m: np.ndarray, ctx: Optional[Context] = None):
    """detail::thin_qr (compress.hpp:60-73) on the GPU: (Q, rank_warning)."""
    ctx = ctx or default_context()
    m = np.asfortranarray(m)
    r = min(m.shape)
    out = np.empty((m.shape[0], r), dtype=m.dtype, order="F")
    rw = C.c_int32()
    ctx.check(ctx.lib.rcpg_thin_qr(ctx.h, _dtype_code(m.dtype), m.shape[0], m.shape[1], m.ctypes.data,
                                   out.ctypes.data, C.byref(rw)))
    return out, bool(rw.value)


def derive_seed(seed: int, salt: int) -> int:
    """random.hpp:54-56 (pure integer arithmetic)."""
    M = 0xFFFFFFFFFFFFFFFF
    z = (seed + 0x9E3779B97F4A7C15 * (salt + 1)) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def stream_id(domain: int, k: int = 0) -> int:
    return (domain << 32) | k
