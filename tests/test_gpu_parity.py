"""GPU parity: the sm_100a library (through its C ABI) against the oracle.

Bars (BASELINE.json north_star): fp64 factors within 1e-8 relative (after
the reference's canonical normalize, which fixes sign/order), relative error
within 1e-8 relative and equal iteration counts; fp32 fit within 1e-4
relative and factor match score >= 0.99.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-8


def cfgs(rcp, oracle, rank, p, q, seed, tol=1e-8, max_iter=200, stab=0, dist=0, modes=None, randomized=True,
         init=0):
    cs = oracle.derive_seed(seed, oracle.stream_id(1))
    g = rcp.DecomposeConfig(rank=rank, tol=tol, max_iter=max_iter, seed=seed, randomized=randomized, init=init,
                            compress=rcp.CompressConfig(target_rank=rank, oversampling=p, power_iterations=q,
                                                        seed=cs, stabilizer=stab, distribution=dist, modes=modes))
    o = oracle.DecomposeConfig(rank=rank, tol=tol, max_iter=max_iter, seed=seed, randomized=randomized, init=init,
                               compress=oracle.CompressConfig(target_rank=rank, oversampling=p, power_iterations=q,
                                                              seed=cs, stabilizer=stab, distribution=dist,
                                                              modes=modes))
    return g, o


def fms(w1, f1, w2, f2):
    """Factor match score with greedy |congruence| matching."""
    R = len(w1)
    score = np.ones((R, R))
    for a, b in zip(f1, f2):
        an = a / np.linalg.norm(a, axis=0)
        bn = b / np.linalg.norm(b, axis=0)
        score *= np.abs(an.T @ bn)
    used, tot = set(), 0.0
    for i in range(R):
        order = np.argsort(-score[i])
        j = next(j for j in order if j not in used)
        used.add(j)
        lam = 1 - abs(w1[i] - w2[j]) / max(abs(w1[i]), abs(w2[j]), 1e-300)
        tot += lam * score[i, j]
    return tot / R


# ----------------------------------------------------------------- RNG
def test_sketch_matrix_matches_reference_stream(rcp, oracle):
    seed = oracle.derive_seed(7, oracle.stream_id(1))
    for mode, rows, cols in [(0, 1001, 7), (2, 64, 33)]:
        got = rcp.sketch_matrix(seed, mode, rows, cols)
        want = oracle.sketch_matrix(seed, mode, rows, cols)
        ulp = np.abs(got - want) / np.spacing(np.abs(want))
        assert ulp.max() <= 8, ulp.max()
        assert np.mean(got == want) > 0.5  # CUDA libm vs glibc: ulp-level only
        gu = rcp.sketch_matrix(seed, mode, rows, cols, distribution=rcp.UNIFORM)
        wu = oracle.sketch_matrix(seed, mode, rows, cols, dist=1)
        assert np.array_equal(gu, wu)  # pure integer/affine arithmetic: bit-exact
    gf = rcp.sketch_matrix(seed, 1, 300, 9, dtype=np.float32)
    wf = oracle.sketch_matrix(seed, 1, 300, 9, dtype=np.float32)
    assert np.max(np.abs(gf - wf)) <= 1e-6


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("dist", [0, 1])
def test_omega_host_upload_bit_identical(rcp, oracle, dtype, dist):
    """north_star: Omega "bit-identical to the reference's RNG, or uploaded from host". With
    omega_host = 1 the library evaluates RandomStream::normal() (random.hpp:75-87) with the
    host's libm and uploads it: array_equal with the oracle's fill_gaussian / fill_uniform over
    10^7 draws (the device generator differs from glibc in the last ulp for ~0.1% of draws)."""
    ctx = rcp.Context(0)
    ctx.set_option("omega_host", 1)
    assert ctx.get_option("omega_host") == 1
    seed = oracle.derive_seed(12345, oracle.stream_id(1))
    for mode, rows, cols in [(0, 1_000_000, 10), (2, 999, 37)]:
        got = rcp.sketch_matrix(seed, mode, rows, cols, distribution=dist, dtype=dtype, ctx=ctx)
        want = oracle.sketch_matrix(seed, mode, rows, cols, dist=dist, dtype=dtype)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("rows,cols", [(200, 20), (1000, 30), (5000, 70), (160000, 30)])
def test_plu_basis_bitwise_random(rcp, oracle, rows, cols, dtype):
    """FullPivLU (compress.hpp:47-58) on random panels: the same pivots and the same two-rounding
    update x - m*u (no FMA contraction) as the oracle's -ffp-contract=off build: identical bits."""
    rng = np.random.default_rng(rows + 7 * cols)
    m = np.asfortranarray(rng.standard_normal((rows, cols)).astype(dtype))
    assert np.array_equal(rcp.plu_basis(m), oracle.plu_basis(m))


def test_plu_basis_bitwise_large_fp32(rcp, oracle):
    """A 10^6 x 70 fp32 panel (C3's W size) through the grid LU: identical bits."""
    rng = np.random.default_rng(70)
    m = np.asfortranarray(rng.standard_normal((1_000_000, 70)).astype(np.float32))
    assert np.array_equal(rcp.plu_basis(m), oracle.plu_basis(m))


@pytest.mark.parametrize("rows,cols", [(100, 20), (1024, 70), (10000, 80), (48, 48)])
def test_thin_qr_fp32_bitwise(rcp, oracle, rows, cols):
    """fp32 thin_qr (compress.hpp:60-73): the Householder QR in the reference's float operation
    order (fp64 dot products rounded once, separately rounded updates): identical bits."""
    rng = np.random.default_rng(rows * cols)
    m = np.asfortranarray(rng.standard_normal((rows, cols)).astype(np.float32))
    q, rw = rcp.thin_qr(m)
    qo, rwo = oracle.thin_qr(m)
    assert rw == rwo
    assert np.array_equal(q, qo)


# --------------------------------------------------------- factorizations
@pytest.mark.parametrize("rows,cols", [(200, 20), (1000, 30), (5000, 70)])
def test_plu_basis_matches_fullpivlu(rcp, oracle, rows, cols):
    rng = np.random.default_rng(rows + cols)
    m = np.asfortranarray(rng.standard_normal((rows, cols)))
    got = rcp.plu_basis(m)
    want = oracle.plu_basis(m)
    assert got.shape == want.shape
    assert np.max(np.abs(got - want)) <= 1e-12


def test_plu_basis_rank_deficient_and_ties(rcp, oracle):
    # exact zero corner -> FullPivLU early stop; integer ties -> column-major first max
    m = np.zeros((12, 5))
    m[3, 1] = 2.0
    m[7, 3] = -2.0
    m[1, 0] = 1.0
    got = rcp.plu_basis(m)
    want = oracle.plu_basis(m)
    assert np.array_equal(got, want)
    t = np.asfortranarray(np.array([[1, 2, 2], [2, 1, 2], [2, 2, 1], [1, 1, 1]], dtype=np.float64))
    assert np.array_equal(rcp.plu_basis(t), oracle.plu_basis(t))


@pytest.mark.parametrize("rows,cols,dt", [(200, 20, np.float64), (400, 30, np.float64), (900, 30, np.float64),
                                         (37, 5, np.float64), (64, 64, np.float64), (3000, 8, np.float64),
                                         (1024, 48, np.float32), (128, 48, np.float32), (12000, 30, np.float64),
                                         (20000, 70, np.float32), (160000, 30, np.float64), (50000, 48, np.float32),
                                         (416, 32, np.float64), (33, 32, np.float64), (410, 31, np.float32),
                                         (20, 30, np.float64), (10000, 80, np.float32), (4900, 70, np.float32),
                                         (1000, 80, np.float32), (3072, 48, np.float32), (7000, 17, np.float64)])
def test_plu_basis_paths_agree_bitwise(rcp, oracle, rows, cols, dt, monkeypatch):
    """Every LU path -- rows in registers (one CTA or a cluster, the default for panels it holds),
    one CTA (rows owned by threads in smem, swaps bookkept), one cluster with the
    panel resident and swaps bookkept (DSMEM exchange), one cluster with Eigen's physical swaps,
    panel resident in the SMs (smem + register columns, one grid barrier per pivot), grid over
    HBM (delayed write-back) -- makes the same pivots with the same arithmetic in the same
    order: identical bits, on random panels and on integer panels full of exact ties."""
    rng = np.random.default_rng(rows * cols)
    m = np.asfortranarray(rng.standard_normal((rows, cols)).astype(dt))
    t = np.asfortranarray(rng.integers(-2, 3, (rows, cols)).astype(dt))

    def run(x, path):
        if path:
            monkeypatch.setenv("RCPG_LU_PATH", path)
        else:
            monkeypatch.delenv("RCPG_LU_PATH", raising=False)
        return rcp.plu_basis(x)

    got, tie = run(m, ""), run(t, "")
    paths = ["resident", "coop"] + (["reg", "onchip", "cluster", "rcluster"] if rows * cols * m.itemsize <= 3_000_000
                                    else [])
    for path in paths:
        assert np.array_equal(run(m, path), got), path
        assert np.array_equal(run(t, path), tie), path
    monkeypatch.delenv("RCPG_LU_PATH", raising=False)
    if rows * cols <= 600_000:
        want = oracle.plu_basis(m.astype(np.float64))
        assert np.max(np.abs(got - want)) <= (1e-12 if dt == np.float64 else 1e-3)


@pytest.mark.parametrize("rows,cols", [(100, 20), (1024, 70)])
def test_thin_qr_matches_householder(rcp, oracle, rows, cols):
    rng = np.random.default_rng(rows)
    m = np.asfortranarray(rng.standard_normal((rows, cols)))
    q, rw = rcp.thin_qr(m)
    qo, rwo = oracle.thin_qr(m)
    assert rw == rwo
    assert np.max(np.abs(q - qo)) <= 1e-12
    assert np.max(np.abs(q.T @ q - np.eye(cols))) <= 1e-12


def test_thin_qr_rank_warning(rcp, oracle):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((50, 3))
    m = np.asfortranarray(np.hstack([a, a[:, :1] * 2.0]))
    q, rw = rcp.thin_qr(m)
    qo, rwo = oracle.thin_qr(m)
    assert rw and rwo


# ---------------------------------------------------------------- compress
def _compress_pair(rcp, oracle, x, k, p, q, seed, **kw):
    g = rcp.CompressConfig(target_rank=k, oversampling=p, power_iterations=q, seed=seed, **kw)
    o = oracle.CompressConfig(target_rank=k, oversampling=p, power_iterations=q, seed=seed, **kw)
    return rcp.compress(x, g), oracle.compress(x, o)


@pytest.mark.parametrize("shape,k,p,q", [([40, 30, 20], 4, 6, 2), ([12, 10, 14, 9], 3, 3, 1), ([60, 50, 40], 5, 5, 0)])
def test_compress_matches_oracle_fp64(rcp, oracle, shape, k, p, q):
    x, _ = oracle.random_lowrank(shape, k, 5, snr=3.0, noise_seed=5)
    got, want = _compress_pair(rcp, oracle, x, k, p, q, 99)
    assert got.compressed.shape == want.compressed.shape
    for gb, ident, wq, rw in zip(got.bases, want.identity, want.q, want.rank_warning):
        assert gb.identity == ident
        if not ident:
            assert np.max(np.abs(gb.q - wq)) <= 1e-10
            assert gb.rank_warning == rw
    scale = np.max(np.abs(want.compressed))
    assert np.max(np.abs(got.compressed - want.compressed)) <= 1e-10 * scale


def test_compress_qr_stabilizer_and_uniform(rcp, oracle):
    x, _ = oracle.random_lowrank([30, 25, 20], 3, 8, snr=2.0, noise_seed=8)
    for kw in [dict(stabilizer=1), dict(distribution=1)]:
        got, want = _compress_pair(rcp, oracle, x, 3, 4, 2, 4, **kw)
        scale = np.max(np.abs(want.compressed))
        assert np.max(np.abs(got.compressed - want.compressed)) <= 1e-10 * scale


def test_compress_mode_selection_and_clamping(rcp, oracle):
    x = np.random.default_rng(1).standard_normal((4, 30, 5))
    got, want = _compress_pair(rcp, oracle, x, 3, 10, 2, 0)
    assert [b.identity for b in got.bases] == [True, False, True]
    assert got.compressed.shape == (4, 13, 5)
    assert np.max(np.abs(got.compressed - want.compressed)) <= 1e-10 * np.max(np.abs(want.compressed))
    x = np.random.default_rng(2).standard_normal((20, 20, 20))
    got, want = _compress_pair(rcp, oracle, x, 3, 2, 2, 0, modes=[1])
    assert got.compressed.shape == (20, 5, 20)
    assert np.max(np.abs(got.compressed - want.compressed)) <= 1e-10 * np.max(np.abs(want.compressed))
    got, _ = _compress_pair(rcp, oracle, x, 2, 2, 2, 0, modes=[])
    assert np.array_equal(got.compressed, x) and all(b.identity for b in got.bases)


def test_compress_rejects_invalid(rcp):
    x = np.random.default_rng(0).standard_normal((5, 5, 5))
    with pytest.raises(ValueError):
        rcp.compress(x, rcp.CompressConfig(target_rank=0))
    with pytest.raises(ValueError):
        rcp.compress(x, rcp.CompressConfig(target_rank=2, oversampling=-1))
    with pytest.raises(ValueError):
        rcp.compress(x, rcp.CompressConfig(target_rank=2, modes=[3]))
    y = x.copy()
    y[0, 0, 0] = np.nan
    with pytest.raises(ValueError, match="finite"):
        rcp.compress(y, rcp.CompressConfig(target_rank=2))


def test_compress_bit_identical_reruns(rcp):
    x = np.random.default_rng(4).standard_normal((30, 28, 26))
    cfg = rcp.CompressConfig(target_rank=3, oversampling=4, seed=99)
    a = rcp.compress(x, cfg)
    b = rcp.compress(x, cfg)
    assert np.array_equal(a.compressed, b.compressed)
    for ba, bb in zip(a.bases, b.bases):
        assert np.array_equal(ba.q, bb.q)


# --------------------------------------------------------------- decompose
def _check_fp64(model, trace, ref, tol=FP64_TOL):
    assert trace.iterations == ref.iterations
    assert trace.converged == ref.converged
    assert abs(trace.final_relative_error - ref.final_relative_error) <= tol * ref.final_relative_error
    assert np.max(np.abs(model.weights - ref.weights) / np.abs(ref.weights)) <= tol
    for a, b in zip(model.factors, ref.factors):
        assert np.linalg.norm(a - b) <= tol * np.linalg.norm(b)
    np.testing.assert_allclose([e.fit for e in trace.entries], ref.trace_fit, rtol=0, atol=1e-10)


def test_decompose_c1_parity(rcp, oracle):
    """BASELINE config C1: 100^3 fp64, R=10, p=10, q=2, SNR 20 dB, tol 1e-8."""
    seed = 1
    x, _ = oracle.random_lowrank([100, 100, 100], 10, seed, snr=10.0, noise_seed=seed)
    g, o = cfgs(rcp, oracle, 10, 10, 2, seed)
    model, trace = rcp.decompose(x, g)
    ref = oracle.decompose(x, o)
    _check_fp64(model, trace, ref)


@pytest.mark.parametrize("split", ["0", "1"])
def test_decompose_als_pinv_placement(rcp, oracle, split, monkeypatch):
    """pinv(V) on CTA 0 after the MTTKRP (RCPG_ALS_SPLIT=0) or on its own CTA during it
    (default): both meet the fp64 bar against the oracle (C1 and a 4-way tensor)."""
    monkeypatch.setenv("RCPG_ALS_SPLIT", split)
    x, _ = oracle.random_lowrank([100, 100, 100], 10, 1, snr=10.0, noise_seed=1)
    g, o = cfgs(rcp, oracle, 10, 10, 2, 1)
    model, trace = rcp.decompose(x, g)
    _check_fp64(model, trace, oracle.decompose(x, o))
    x, _ = oracle.random_lowrank([16, 14, 12, 10], 3, 3, snr=5.0, noise_seed=3)
    g, o = cfgs(rcp, oracle, 3, 4, 2, 3)
    model, trace = rcp.decompose(x, g)
    _check_fp64(model, trace, oracle.decompose(x, o))


def test_decompose_four_way_and_options(rcp, oracle):
    x, _ = oracle.random_lowrank([16, 14, 12, 10], 3, 3, snr=5.0, noise_seed=3)
    for kw in [dict(), dict(stab=1), dict(dist=1), dict(modes=[0, 2])]:
        g, o = cfgs(rcp, oracle, 3, 4, 2, 3, **kw)
        model, trace = rcp.decompose(x, g)
        _check_fp64(model, trace, oracle.decompose(x, o))


def test_decompose_deterministic_path(rcp, oracle):
    x, _ = oracle.random_lowrank([20, 18, 16], 3, 9, snr=4.0, noise_seed=9)
    g, o = cfgs(rcp, oracle, 3, 4, 2, 9, randomized=False)
    model, trace = rcp.decompose(x, g)
    _check_fp64(model, trace, oracle.decompose(x, o))


def test_decompose_fp32_small(rcp, oracle):
    x, (tw, tf) = oracle.synth(3, [60, 50, 40], 5, 4, 10 ** (15 / 20), dtype=np.float32)
    g, o = cfgs(rcp, oracle, 5, 5, 2, 4, tol=1e-5, max_iter=500)
    model, trace = rcp.decompose(x, g)
    ref = oracle.decompose(x, o)
    fit_g = 1 - trace.final_relative_error ** 2
    fit_o = 1 - ref.final_relative_error ** 2
    assert abs(fit_g - fit_o) <= 1e-4 * abs(fit_o)
    assert fms(model.weights, model.factors, ref.weights, ref.factors) >= 0.99


def test_decompose_errors(rcp):
    x = np.random.default_rng(0).standard_normal((6, 6, 6))
    with pytest.raises(ValueError, match="target rank must equal"):
        rcp.decompose(x, rcp.DecomposeConfig(rank=2, compress=rcp.CompressConfig(target_rank=3)))
    with pytest.raises(ValueError, match="tolerance"):
        rcp.decompose(x, rcp.DecomposeConfig(rank=2, tol=0.0, randomized=False))
    y = x.copy()
    y[1, 2, 3] = np.inf
    with pytest.raises(rcp.SolverError) as e:
        rcp.decompose(y, rcp.DecomposeConfig(rank=2, randomized=False))
    assert e.value.iteration() == 0


def test_decompose_error_order_matches_reference(rcp, oracle):
    """Device-side checks are raised after the work is enqueued; the error
    reported must still be the one the sequential reference raises first."""
    x = np.random.default_rng(1).standard_normal((8, 7, 6))
    bad = x.copy()
    bad[2, 3, 1] = np.nan
    g, o = cfgs(rcp, oracle, 2, 2, 1, 3)
    with pytest.raises(ValueError, match="compress: input values must be finite"):
        rcp.decompose(bad, g)
    with pytest.raises(oracle.OracleInvalidArgument, match="compress: input values must be finite"):
        oracle.decompose(bad, o)
    # finite check precedes the mode-range check (compress.hpp:93 vs :98)
    g2, _ = cfgs(rcp, oracle, 2, 2, 1, 3, modes=[5])
    with pytest.raises(ValueError, match="finite"):
        rcp.decompose(bad, g2)
    g3, _ = cfgs(rcp, oracle, 2, 2, 1, 3, modes=[5])
    with pytest.raises(ValueError, match="mode index out of range"):
        rcp.decompose(x, g3)
    z = np.zeros((5, 4, 3))
    g4, o4 = cfgs(rcp, oracle, 2, 2, 1, 3, randomized=False)
    with pytest.raises(ValueError, match="tensor norm must be positive"):
        rcp.decompose(z, g4)
    with pytest.raises(oracle.OracleInvalidArgument, match="tensor norm must be positive"):
        oracle.decompose(z, o4)
    # the context stays usable after errors
    model, trace = rcp.decompose(x, cfgs(rcp, oracle, 2, 2, 1, 3)[0])
    assert np.isfinite(trace.final_relative_error)


def test_decompose_end_to_end_determinism(rcp, oracle):
    x, _ = oracle.random_lowrank([24, 22, 20], 3, 51, snr=2.0, noise_seed=4)
    g, _ = cfgs(rcp, oracle, 3, 10, 2, 77)
    a, ta = rcp.decompose(x, g)
    b, tb = rcp.decompose(x, g)
    assert np.array_equal(a.weights, b.weights)
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)
    assert ta.final_relative_error == tb.final_relative_error


@pytest.mark.slow
def test_decompose_c2_parity(rcp, oracle):
    """BASELINE config C2: 400^3 fp64, rank-20 Kruskal (N(0,1) factors,
    weights U[1,10]), SNR 10 dB, R=20, p=10, q=2, tol 1e-8."""
    seed = 2
    x, _ = oracle.synth(2, [400, 400, 400], 20, seed, 10 ** (10 / 20))
    g, o = cfgs(rcp, oracle, 20, 10, 2, seed)
    model, trace = rcp.decompose(x, g)
    ref = oracle.decompose(x, o)
    _check_fp64(model, trace, ref)


def test_decompose_fp32_odd_panels(rcp, oracle):
    """fp32 with odd panel sizes (mode-2 W is 81 x 9 = 729 floats): the on-chip LU keeps its
    8-byte row-base scratch aligned behind an odd-length float panel."""
    x, _ = oracle.random_lowrank([40, 32, 24], 4, 13, snr=4.0, noise_seed=13)
    x = x.astype(np.float32)
    g, o = cfgs(rcp, oracle, 4, 5, 2, 3, tol=1e-6, max_iter=300)
    model, trace = rcp.decompose(x, g)
    ref = oracle.decompose(x, o)
    assert trace.iterations == ref.iterations
    fit_g, fit_o = 1 - trace.final_relative_error ** 2, 1 - ref.final_relative_error ** 2
    assert abs(fit_g - fit_o) <= 1e-6 * abs(fit_o)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_decompose_graph_replay_identical(rcp, oracle, dtype):
    """Repeated identical calls: the second is captured as a CUDA graph and later ones replay it.
    Every call returns the same bits and counts the same kernel launches; a changed
    configuration falls back to stream launches and still matches the oracle."""
    x, _ = oracle.random_lowrank([40, 36, 30], 4, 7, snr=3.0, noise_seed=7)
    x = x.astype(dtype)
    ctx = rcp.Context(0)
    ctx.set_option("pass_timing", 1)  # the per-pass events ride in the graph as record nodes
    X = rcp.DeviceTensor.upload(x, ctx=ctx)
    g, o = cfgs(rcp, oracle, 4, 5, 2, 5, tol=1e-8 if dtype == np.float64 else 1e-6)
    outs, launches = [], []
    for _ in range(4):
        l0 = ctx.kernel_launches()
        outs.append(rcp.decompose(X, g, ctx=ctx))
        launches.append(ctx.kernel_launches() - l0)
    m0, t0 = outs[0]
    for m, t in outs[1:]:
        assert t.iterations == t0.iterations and t.final_relative_error == t0.final_relative_error
        assert np.array_equal(m.weights, m0.weights)
        for a, b in zip(m.factors, m0.factors):
            assert np.array_equal(a, b)
    assert len(set(launches)) == 1 and launches[0] > 10, launches
    timings = ctx.pass_timings()
    assert any(n == "sketch" and ms > 0 for n, ms, _ in timings)
    ref = oracle.decompose(x, o)
    assert t0.iterations == ref.iterations
    g2, o2 = cfgs(rcp, oracle, 4, 5, 1, 5, tol=1e-8 if dtype == np.float64 else 1e-6)
    m2, t2 = rcp.decompose(X, g2, ctx=ctx)
    assert t2.iterations == oracle.decompose(x, o2).iterations
    X.free()
