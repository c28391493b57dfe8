"""Streamed-pass kernels (compress.hpp:118-145 products) against an fp64 numpy product.

fp64 views with R > 1 run on the DMMA kernels (passes_dmma.cu). fp32 views run in one of
two arithmetics (rcpg_set_option "fp32_arith"):
  faithful (default): fp32 X, fp64 products and sums on the DMMA kernels (SIMT for R = 1 or
    unaligned views), one rounding to float -- the oracle's double-accumulated GEMM, so the
    result is the correctly rounded fp64 sum: equal to round(fp64 numpy) except where the
    exact sum sits within fp64 summation-order noise of a float rounding boundary;
  fast: the tcgen05 3xTF32 kernels (passes_tc.cu, R % 4 == 0; SIMT tiles otherwise). The
    fp32 bound (normwise relative error 1e-5) is met by 3xTF32 (~1e-7) and missed by plain
    TF32 (~5e-4).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# (L, I, R, cols): ragged M/N/K edges, several UMMA N widths, multi-n-tile (cols > 128),
# R % 4 != 0 and I % 4 != 0 (SIMT fallbacks), the last-mode view (R = 1).
VIEWS = [
    (1, 200, 1000, 70),
    (3, 130, 68, 17),
    (2, 64, 4, 48),
    (1, 1024, 4096, 80),
    (5, 37, 12, 150),
    (4, 96, 256, 128),
    (2, 50, 30, 20),
    (3, 42, 40, 33),
    (700, 20, 1, 30),
    (1, 8, 100000, 64),
]

TOL = {np.float32: 1e-5, np.float64: 1e-12}
ARITHS = [(np.float32, "faithful"), (np.float32, "fast"), (np.float64, "fp64")]


@pytest.fixture(scope="module")
def fast_ctx(rcp):
    c = rcp.Context(0)
    c.set_option("fp32_arith", 1)
    return c


def _ctx(rcp, arith, fast_ctx):
    return fast_ctx if arith == "fast" else rcp.default_context()


def _check_faithful(out, ref):
    """fp32 result of fp64 arithmetic: round(ref) almost everywhere, never more than 1 ulp off."""
    want = ref.astype(np.float32)
    frac = np.mean(out == want)
    assert frac >= 0.999, f"only {frac:.6f} of the entries equal the rounded fp64 product"
    ulp = np.abs(out.astype(np.float64) - want.astype(np.float64)) / np.spacing(np.abs(want)).astype(np.float64)
    assert ulp.max() <= 1.0, ulp.max()


def _inputs(L, I, R, cols, dtype, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((L, I, R)).astype(dtype)
    p = rng.standard_normal((L, cols, R)).astype(dtype)
    q = rng.standard_normal((I, cols)).astype(dtype)
    return x, p, q


def _check(out, ref, ref_abs, dtype):
    err = np.linalg.norm(out.astype(np.float64) - ref) / max(np.linalg.norm(ref), 1e-300)
    assert err < TOL[dtype], f"normwise relative error {err:.3e}"
    elem = np.max(np.abs(out.astype(np.float64) - ref) / np.maximum(ref_abs, 1e-300))
    assert elem < 50 * TOL[dtype], f"elementwise error / (|x||p|) {elem:.3e}"


@pytest.mark.parametrize("dtype,arith", ARITHS)
@pytest.mark.parametrize("view", VIEWS)
def test_sketch_pass(rcp, fast_ctx, view, dtype, arith):
    L, I, R, cols = view
    x, p, _ = _inputs(L, I, R, cols, dtype, 11)
    out = rcp.stream_pass("sketch", x, p, cols, ctx=_ctx(rcp, arith, fast_ctx))
    assert out.shape == (I, cols)
    xd, pd = x.astype(np.float64), p.astype(np.float64)
    ref = np.einsum("aib,acb->ic", xd, pd)
    ref_abs = np.einsum("aib,acb->ic", np.abs(xd), np.abs(pd))
    _check(out, ref, ref_abs, dtype)
    if arith == "faithful":
        _check_faithful(out, ref)


@pytest.mark.parametrize("dtype,arith", ARITHS)
@pytest.mark.parametrize("view", VIEWS)
def test_project_pass(rcp, fast_ctx, view, dtype, arith):
    L, I, R, cols = view
    x, _, q = _inputs(L, I, R, cols, dtype, 12)
    out = rcp.stream_pass("project", x, q, cols, ctx=_ctx(rcp, arith, fast_ctx))
    assert out.shape == (L, cols, R)
    xd, qd = x.astype(np.float64), q.astype(np.float64)
    ref = np.einsum("aib,ic->acb", xd, qd)
    ref_abs = np.einsum("aib,ic->acb", np.abs(xd), np.abs(qd))
    _check(out, ref, ref_abs, dtype)
    if arith == "faithful":
        _check_faithful(out, ref)


@pytest.mark.parametrize("arith", ["faithful", "fast"])
def test_pass_scaled_inputs(rcp, fast_ctx, arith):
    """Wide dynamic range: the lo plane must keep its own exponent (no flush)."""
    L, I, R, cols = 1, 256, 512, 64
    x, p, q = _inputs(L, I, R, cols, np.float32, 13)
    x *= np.float32(1e-20)
    p *= np.float32(1e15)
    q *= np.float32(1e15)
    ctx = _ctx(rcp, arith, fast_ctx)
    out = rcp.stream_pass("sketch", x, p, cols, ctx=ctx)
    ref = np.einsum("aib,acb->ic", x.astype(np.float64), p.astype(np.float64))
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-5
    out = rcp.stream_pass("project", x, q, cols, ctx=ctx)
    ref = np.einsum("aib,ic->acb", x.astype(np.float64), q.astype(np.float64))
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("arith", ["faithful", "fast"])
def test_pass_deterministic(rcp, fast_ctx, arith):
    x, p, q = _inputs(2, 300, 2000, 70, np.float32, 14)
    ctx = _ctx(rcp, arith, fast_ctx)
    a = rcp.stream_pass("sketch", x, p, 70, ctx=ctx)
    b = rcp.stream_pass("sketch", x, p, 70, ctx=ctx)
    assert np.array_equal(a, b)
    a = rcp.stream_pass("project", x, q, 70, ctx=ctx)
    b = rcp.stream_pass("project", x, q, 70, ctx=ctx)
    assert np.array_equal(a, b)


# ------------------------------------------------------- relative error
# kruskal.hpp:187-194: ||X - Xhat|| / ||X||, accumulated in fp64, for a visible residual and
# for a near-exact model (where a Gram-form evaluation would cancel).
@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-10), (np.float32, 1e-4)])
@pytest.mark.parametrize("shape,rank", [((40, 30, 20), 5), ((64, 48, 32), 12), ((9, 130, 17), 3)])
def test_relative_error_gram_and_exact(rcp, dtype, tol, shape, rank):
    rng = np.random.default_rng(sum(shape))
    fac = [rng.standard_normal((n, rank)).astype(dtype).astype(np.float64) for n in shape]
    w = np.linspace(1.0, 2.0, rank).astype(dtype).astype(np.float64)
    xh = np.einsum("r,ir,jr,kr->ijk", w, *fac)
    for noise in (0.3, 1e-7):
        x = (xh + noise * np.linalg.norm(xh) / np.sqrt(xh.size) * rng.standard_normal(shape)).astype(dtype)
        want = np.linalg.norm(x.astype(np.float64) - xh) / np.linalg.norm(x.astype(np.float64))
        k = rcp.Kruskal(weights=w.astype(dtype), factors=[f.astype(dtype) for f in fac])
        got = rcp.relative_error(x, k)
        if noise > 1e-3:
            assert abs(got - want) <= tol * want, (got, want)
        else:
            assert abs(got - want) <= (1e-12 if dtype == np.float64 else 2e-6), (got, want)


# Views big enough (L*I*R >= 2^26, I >= 8 cols) for the fp32 sketch to stream a K-tile-
# blocked copy of the panel (passes_tc.cu panel_block_kernel): R % 32 != 0 (zero-padded
# last block), cols not a multiple of the UMMA N (zero-padded columns), several slabs.
@pytest.mark.parametrize("view", [(1, 600, 131076, 70), (2, 300, 131076, 33)])
def test_sketch_pass_blocked_panel(rcp, fast_ctx, view):
    L, I, R, cols = view
    x, p, _ = _inputs(L, I, R, cols, np.float32, 13)
    out = rcp.stream_pass("sketch", x, p, cols, ctx=fast_ctx)
    ref = np.zeros((I, cols))
    ref_abs = np.zeros((I, cols))
    for a in range(L):
        xd, pd = x[a].astype(np.float64), p[a].astype(np.float64)
        ref += xd @ pd.T
        ref_abs += np.abs(xd) @ np.abs(pd).T
    _check(out, ref, ref_abs, np.float32)
