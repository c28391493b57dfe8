"""Sharded decomposition on one GPU through in-process virtual ranks.

Every rank holds a slab of the last mode (C3/C4) or of the first mode (C5) and runs the
same decompose call; the loopback
communicator stands in for NCCL (same collectives, sums in rank order). Sharding changes
only summation order, so results match the unsharded decomposition to rounding (fp64 bar
1e-8 on factors and relerr, equal iteration counts) and agree bitwise across ranks.
"""
import threading

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


def _cfg(rcp, rank, p, q, seed, tol=1e-8, max_iter=200):
    return rcp.DecomposeConfig(rank=rank, tol=tol, max_iter=max_iter, seed=seed,
                               compress=rcp.CompressConfig(target_rank=rank, oversampling=p, power_iterations=q,
                                                           seed=rcp.derive_seed(seed, rcp.stream_id(rcp.COMPRESS))))


def _run_ranks(rcp, x, n, fn, mode=-1, fast=False):
    ctxs = [rcp.Context(0) for _ in range(n)]
    rcp.comm_init_loopback(ctxs)
    mode = mode % x.ndim
    slabs = []
    for r, c in enumerate(ctxs):
        if fast:
            c.set_option("fp32_arith", 1)
        lo, hi = rcp.slab_range(x.shape[mode], n, r)
        sl = [slice(None)] * x.ndim
        sl[mode] = slice(lo, hi)
        slabs.append(rcp.DeviceTensor.upload_slab(np.ascontiguousarray(x[tuple(sl)]), x.shape, lo, hi, ctx=c,
                                                  mode=mode))
    out, errs = [None] * n, []

    def work(r):
        try:
            out[r] = fn(slabs[r], ctxs[r])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def _check_vs_single(got, want, tol):
    (m, tr), (mw, tw) = got, want
    assert tr.iterations == tw.iterations
    assert abs(tr.final_relative_error - tw.final_relative_error) <= tol * tw.final_relative_error
    for a, b in zip(m.factors, mw.factors):
        assert np.linalg.norm(a - b) <= tol * np.linalg.norm(b)
    assert np.allclose(m.weights, mw.weights, rtol=tol)


@pytest.mark.parametrize("shape,nranks,mode", [((40, 30, 20), 2, -1), ((40, 30, 21), 3, -1), ((12, 10, 14, 9), 2, -1),
                                               ((30, 24, 50), 4, -1), ((40, 30, 20), 2, 0), ((41, 30, 22), 3, 0),
                                               ((14, 10, 12, 9), 2, 0), ((64, 20, 18), 4, 0),
                                               ((40, 30, 24), 8, -1), ((64, 20, 18), 8, 0)])
def test_sharded_decompose_matches_single(rcp, oracle, shape, nranks, mode):
    x, _ = oracle.random_lowrank(list(shape), 4, 11, snr=3.0, noise_seed=11)
    cfg = _cfg(rcp, 4, 5, 2, 7)
    want = rcp.decompose(x, cfg)
    got = _run_ranks(rcp, x, nranks, lambda t, c: rcp.decompose(t, cfg, ctx=c), mode=mode)
    for g in got:
        _check_vs_single(g, want, 1e-8)
    for g in got[1:]:  # replicated results: identical on every rank
        assert g[1].final_relative_error == got[0][1].final_relative_error
        for a, b in zip(g[0].factors, got[0][0].factors):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("mode", [-1, 0])
def test_sharded_compress_matches_single(rcp, oracle, mode):
    x, _ = oracle.random_lowrank([36, 28, 22], 4, 3, snr=4.0, noise_seed=3)
    g = rcp.CompressConfig(target_rank=4, oversampling=4, power_iterations=2, seed=99)
    want = rcp.compress(x, g)
    got = _run_ranks(rcp, x, 2, lambda t, c: rcp.compress(t, g, ctx=c), mode=mode)
    for res in got:
        assert res.compressed.shape == want.compressed.shape
        assert np.max(np.abs(res.compressed - want.compressed)) <= 1e-10 * np.max(np.abs(want.compressed))
        for a, b in zip(res.bases, want.bases):
            assert a.identity == b.identity
            if not a.identity:
                assert np.max(np.abs(a.q - b.q)) <= 1e-10


@pytest.mark.parametrize("mode,modes,shape", [(-1, [0, 1], (7, 7, 9)), (0, [1, 2], (24, 7, 7))])
def test_sharded_mode_left_uncompressed(rcp, oracle, mode, modes, shape):
    """Slab mode outside the selected modes: the slabs are reassembled, the rest runs replicated."""
    x, _ = oracle.random_lowrank([24, 20, 9] if mode == -1 else [24, 20, 19], 3, 5, snr=3.0, noise_seed=5)
    g = rcp.CompressConfig(target_rank=3, oversampling=4, power_iterations=1, seed=5, modes=modes)
    want = rcp.compress(x, g)
    got = _run_ranks(rcp, x, 2, lambda t, c: rcp.compress(t, g, ctx=c), mode=mode)
    for res in got:
        assert res.compressed.shape == want.compressed.shape == shape
        assert np.max(np.abs(res.compressed - want.compressed)) <= 1e-10 * np.max(np.abs(want.compressed))


@pytest.mark.parametrize("mode,fast", [(-1, False), (0, False), (-1, True), (0, True)])
def test_sharded_fp32(rcp, oracle, mode, fast):
    """fp32: the faithful arithmetic (default) all-reduces fp64 partials and rounds once, so the
    sharded result equals the unsharded one up to fp64 summation order (same iterations, fit to
    1e-6); the fast 3xTF32 path (fp32_arith = 1) meets the fp32 bar (fit 1e-4)."""
    x, _ = oracle.random_lowrank([64, 48, 40], 5, 13, snr=4.0, noise_seed=13)
    x = x.astype(np.float32)
    cfg = _cfg(rcp, 5, 5, 2, 3, tol=1e-5, max_iter=300)
    ctx = rcp.Context(0)
    if fast:
        ctx.set_option("fp32_arith", 1)
    want = rcp.decompose(x, cfg, ctx=ctx)
    got = _run_ranks(rcp, x, 2, lambda t, c: rcp.decompose(t, cfg, ctx=c), mode=mode, fast=fast)
    for m, tr in got:
        fit_g, fit_w = 1 - tr.final_relative_error ** 2, 1 - want[1].final_relative_error ** 2
        assert abs(fit_g - fit_w) <= (1e-4 if fast else 1e-6) * abs(fit_w)
        if not fast:
            assert tr.iterations == want[1].iterations


@pytest.mark.parametrize("shape,nranks,mode", [((40, 30, 20), 2, -1), ((40, 30, 21), 3, -1), ((12, 10, 14, 9), 2, -1),
                                               ((40, 30, 20), 2, 0), ((30, 24, 50), 4, -1)])
def test_sharded_qr_stabilizer(rcp, oracle, shape, nranks, mode):
    """stabilizer = QR (compress.hpp:60-70): the row-sharded W of the modes before a last-mode slab is
    all-gathered, factored replicated and re-split; everything else factors replicated panels."""
    x, _ = oracle.random_lowrank(list(shape), 4, 21, snr=3.0, noise_seed=21)
    cfg = _cfg(rcp, 4, 5, 2, 9)
    cfg.compress.stabilizer = rcp.QR
    want = rcp.decompose(x, cfg)
    got = _run_ranks(rcp, x, nranks, lambda t, c: rcp.decompose(t, cfg, ctx=c), mode=mode)
    for g in got:
        _check_vs_single(g, want, 1e-8)
    for g in got[1:]:
        for a, b in zip(g[0].factors, got[0][0].factors):
            assert np.array_equal(a, b)


def test_sharded_qr_stabilizer_fp32(rcp, oracle):
    x, _ = oracle.random_lowrank([64, 48, 40], 5, 13, snr=4.0, noise_seed=13)
    x = x.astype(np.float32)
    cfg = _cfg(rcp, 5, 5, 2, 3, tol=1e-5, max_iter=300)
    cfg.compress.stabilizer = rcp.QR
    want = rcp.decompose(x, cfg)
    got = _run_ranks(rcp, x, 2, lambda t, c: rcp.decompose(t, cfg, ctx=c), mode=-1)
    for m, tr in got:
        fit_g, fit_w = 1 - tr.final_relative_error ** 2, 1 - want[1].final_relative_error ** 2
        assert abs(fit_g - fit_w) <= 1e-6 * abs(fit_w)
        assert tr.iterations == want[1].iterations


def test_sharded_rejects_unsupported(rcp, oracle):
    x, _ = oracle.random_lowrank([20, 18, 16], 3, 1, snr=3.0, noise_seed=1)
    det = rcp.DecomposeConfig(rank=3, randomized=False, tol=1e-8, max_iter=50)
    with pytest.raises(ValueError, match="randomized"):
        _run_ranks(rcp, x, 1, lambda t, c: rcp.decompose(t, det, ctx=c))


def test_sharded_through_nccl_single_rank(rcp, oracle):
    """The NCCL communicator (loaded at run time) on one rank: same result as unsharded."""
    x, _ = oracle.random_lowrank([30, 26, 22], 3, 17, snr=3.0, noise_seed=17)
    cfg = _cfg(rcp, 3, 4, 2, 17)
    want = rcp.decompose(x, cfg)
    ctx = rcp.Context(0)
    ctx.comm_init_nccl(1, 0, rcp.comm_unique_id())
    assert ctx.comm_rank() == (0, 1)
    t = rcp.DeviceTensor.upload_slab(x, x.shape, 0, x.shape[-1], ctx=ctx)
    _check_vs_single(rcp.decompose(t, cfg, ctx=ctx), want, 1e-8)
