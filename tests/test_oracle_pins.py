"""Pins the CPU oracle (oracle/rcp_oracle.hpp) to the reference's own tests.

Each test restates a known-answer or property test from
/root/reference/proj/tests/unit/*.cpp (file:line cited) and runs it against
the oracle, so the oracle that checks the GPU path is itself checked against
everything the reference's test suite pins for this path. No GPU needed.
"""
import itertools

import numpy as np
import pytest

# ------------------------------------------------------------- helpers
RNG = np.random.default_rng(0x5EED)  # test-local randomness (oracles.hpp:101-105)


def naive_unfold(t, mode):
    """oracles.hpp:44-53: explicit fiber enumeration."""
    shape = t.shape
    m = np.zeros((shape[mode], t.size // shape[mode]))
    for idx in itertools.product(*[range(e) for e in shape]):
        col, stride = 0, 1
        for k, e in enumerate(shape):
            if k == mode:
                continue
            col += idx[k] * stride
            stride *= e
        m[idx[mode], col] = t[idx]
    return m


def naive_reconstruct(w, fs):
    """oracles.hpp:75-90."""
    shape = [f.shape[0] for f in fs]
    out = np.zeros(shape)
    for idx in itertools.product(*[range(e) for e in shape]):
        out[idx] = sum(w[r] * np.prod([f[i, r] for f, i in zip(fs, idx)]) for r in range(len(w)))
    return out


def mode_product(oracle, t, u, mode):
    shape = list(t.shape)
    shape[mode] = u.shape[0]
    return oracle.fold(u @ oracle.unfold(t, mode), mode, shape)


def random_shape(lo, hi, emax):
    return [int(e) for e in RNG.integers(1, emax + 1, size=int(RNG.integers(lo, hi + 1)))]


def det_cfg(oracle, rank, tol=1e-13, **kw):
    return oracle.DecomposeConfig(rank=rank, randomized=False, tol=tol, **kw)


# ------------------------------------------------------ test_random.cpp
def test_identical_seed_and_stream_reproduce_bits(oracle):  # test_random.cpp:11-15
    sid = oracle.stream_id(1, 1)
    assert np.array_equal(oracle.stream_draws(42, sid, "bits", 1000), oracle.stream_draws(42, sid, "bits", 1000))


def test_streams_and_salts_separate(oracle):  # test_random.cpp:17-36
    a = oracle.stream_draws(42, oracle.stream_id(1, 0), "bits", 64)
    b = oracle.stream_draws(42, oracle.stream_id(1, 1), "bits", 64)
    c = oracle.stream_draws(42, oracle.stream_id(2, 0), "bits", 64)
    assert not np.any(a == b) and not np.any(a == c)
    assert len({oracle.derive_seed(7, s) for s in range(256)}) == 256


def test_uniform_and_normal_moments(oracle):  # test_random.cpp:38-77
    u = oracle.stream_draws(3, oracle.stream_id(4), "uniform01", 100000)
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01
    x = oracle.stream_draws(11, oracle.stream_id(4), "normal", 200000)
    assert abs(x.mean()) < 0.01 and abs(x.var() - 1.0) < 0.02
    s = oracle.stream_draws(5, oracle.stream_id(1), "uniform_sym", 100000)
    assert s.min() >= -1.0 and s.max() <= 1.0 and abs((s < 0).sum() - 50000) < 2000


def test_fill_gaussian_is_column_major_sequential(oracle):  # test_random.cpp:79-88
    m = oracle.sketch_matrix(9, 2, 4, 3)  # stream (9, compress<<32|2), column-major fill
    flat = oracle.stream_draws(9, oracle.stream_id(1, 2), "normal", 12)
    assert np.array_equal(m.reshape(-1, order="F"), flat)


def test_splitmix_counter_form(oracle):
    """draw k of RandomStream(seed, id) = mix64(s0 + (k+1) gamma): the identity
    the device generator relies on (random.hpp:16-29, 54-56)."""
    seed, sid = 1234, oracle.stream_id(1, 5)
    s0 = oracle.derive_seed(seed, sid)
    bits = oracle.stream_draws(seed, sid, "bits", 50)
    G = 0x9E3779B97F4A7C15
    for k in range(50):
        assert int(bits[k]) == oracle.mix64((s0 + (k + 1) * G) & 0xFFFFFFFFFFFFFFFF)


# ------------------------------------------------------ test_tensor.cpp
def test_counting_tensor_unfoldings(oracle):  # test_tensor.cpp:39-60 (frozen)
    t = np.arange(1, 9, dtype=np.float64).reshape(2, 2, 2)
    exp = [np.array([[1, 3, 2, 4], [5, 7, 6, 8]]), np.array([[1, 5, 2, 6], [3, 7, 4, 8]]),
           np.array([[1, 5, 3, 7], [2, 6, 4, 8]])]
    for mode in range(3):
        assert np.array_equal(oracle.unfold(t, mode), exp[mode])
        assert np.array_equal(naive_unfold(t, mode), exp[mode])
    with pytest.raises(ValueError):
        oracle.unfold(t, 3)


def test_unfold_matches_fiber_oracle_random_shapes(oracle):  # test_tensor.cpp:62-69
    for _ in range(25):
        s = random_shape(1, 4, 5)
        t = RNG.standard_normal(s)
        for mode in range(len(s)):
            assert np.array_equal(oracle.unfold(t, mode), naive_unfold(t, mode))


def test_fold_inverts_unfold_and_preserves_norm(oracle):  # test_tensor.cpp:79-95
    for _ in range(20):
        t = RNG.standard_normal(random_shape(2, 4, 6))
        for mode in range(t.ndim):
            u = oracle.unfold(t, mode)
            assert np.array_equal(oracle.fold(u, mode, t.shape), t)
            assert abs(np.linalg.norm(u) - np.linalg.norm(t)) <= 1e-12 * np.linalg.norm(t)
    with pytest.raises(ValueError):
        oracle.fold(np.zeros((2, 3)), 0, [2, 2, 2])


def test_mode_products(oracle):  # test_tensor.cpp:97-125
    t = RNG.standard_normal((3, 4, 5))
    u = RNG.standard_normal((2, 4))
    got = mode_product(oracle, t, u, 1)
    want = np.einsum("jb,abc->ajc", u, t)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    v = RNG.standard_normal((6, 5))
    ab = mode_product(oracle, mode_product(oracle, t, u, 1), v, 2)
    ba = mode_product(oracle, mode_product(oracle, t, v, 2), u, 1)
    assert np.linalg.norm(ab - ba) <= 1e-12 * np.linalg.norm(ab)


def test_khatri_rao_hand_example(oracle):  # test_tensor.cpp:127-133
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.array_equal(oracle.khatri_rao(a, b), np.array([[0, 2], [1, 0], [0, 4], [3, 0]], dtype=float))


# ---------------------------------------------------- test_compress.cpp
def ccfg(oracle, k, seed=0, **kw):
    return oracle.CompressConfig(target_rank=k, seed=seed, **kw)


def test_exact_rank_capture(oracle):  # test_compress.cpp:32-39
    t, _ = oracle.random_lowrank([12, 10, 14], 3, 21)
    cfg = ccfg(oracle, 3, oversampling=3)
    assert oracle.projection_residual(t, cfg) <= 1e-10 * np.linalg.norm(t)
    assert oracle.compress(t, cfg).compressed.shape == (6, 6, 6)


def test_empty_modes_and_determinism(oracle):  # test_compress.cpp:41-75
    t = RNG.standard_normal((5, 6, 4))
    r = oracle.compress(t, ccfg(oracle, 2, modes=[]))
    assert np.array_equal(r.compressed, t) and all(r.identity)
    t = RNG.standard_normal((8, 9, 7))
    a = oracle.compress(t, ccfg(oracle, 3, 99, oversampling=2))
    b = oracle.compress(t, ccfg(oracle, 3, 99, oversampling=2))
    assert np.array_equal(a.compressed, b.compressed)
    c = oracle.compress(t, ccfg(oracle, 3, 2, oversampling=2))
    assert not np.array_equal(a.compressed, c.compressed)


@pytest.mark.parametrize("stab", [0, 1])
def test_bases_orthonormal(oracle, stab):  # test_compress.cpp:76-89
    t = RNG.standard_normal((15, 12, 18))
    r = oracle.compress(t, ccfg(oracle, 4, stabilizer=stab))
    for q, ident in zip(r.q, r.identity):
        if not ident:
            assert np.max(np.abs(q.T @ q - np.eye(q.shape[1]))) <= 1e-10


def test_compressed_equals_joint_projection(oracle):  # test_compress.cpp:91-101
    t = RNG.standard_normal((9, 11, 8))
    r = oracle.compress(t, ccfg(oracle, 3, oversampling=2))
    p = t
    for m, (q, ident) in enumerate(zip(r.q, r.identity)):
        if not ident:
            p = mode_product(oracle, p, q.T, m)
    assert np.linalg.norm(p - r.compressed) <= 1e-12 * (np.linalg.norm(p) + 1.0)


def test_clamping_and_mode_subset(oracle):  # test_compress.cpp:103-126
    r = oracle.compress(RNG.standard_normal((4, 30, 5)), ccfg(oracle, 3, oversampling=10))
    assert r.identity == [True, False, True] and r.compressed.shape == (4, 13, 5)
    r = oracle.compress(RNG.standard_normal((20, 20, 20)), ccfg(oracle, 3, oversampling=2, modes=[1]))
    assert r.identity == [True, False, True] and r.compressed.shape == (20, 5, 20)


def test_uniform_sketch_exact_rank(oracle):  # test_compress.cpp:128-133
    t, _ = oracle.random_lowrank([12, 12, 12], 3, 5)
    assert oracle.projection_residual(t, ccfg(oracle, 3, distribution=1)) <= 1e-10 * np.linalg.norm(t)


def _mean_residual(oracle, t, seeds, **kw):
    return np.mean([oracle.projection_residual(t, ccfg(oracle, 4, 1000 + s, **kw)) for s in range(seeds)])


def test_power_iterations_and_oversampling_help(oracle):  # test_compress.cpp:135-155
    clean, _ = oracle.random_lowrank([18, 18, 18], 4, 77)
    noisy = oracle.add_noise(clean, 2.0, 7)
    assert _mean_residual(oracle, noisy, 20, oversampling=2, power_iterations=2) <= \
        _mean_residual(oracle, noisy, 20, oversampling=2, power_iterations=0)
    clean, _ = oracle.random_lowrank([18, 18, 18], 4, 78)
    noisy = oracle.add_noise(clean, 2.0, 8)
    assert _mean_residual(oracle, noisy, 20, oversampling=10, power_iterations=1) <= \
        _mean_residual(oracle, noisy, 20, oversampling=0, power_iterations=1)


def test_per_mode_residual_bound(oracle):  # test_compress.cpp:157-173
    t = RNG.standard_normal((7, 6, 8))
    assert oracle.projection_residual(t, ccfg(oracle, 2, modes=[])) == 0.0
    cfg = ccfg(oracle, 2, 3)
    r = oracle.compress(t, cfg)
    s = 0.0
    for m, (q, ident) in enumerate(zip(r.q, r.identity)):
        if not ident:
            s += np.linalg.norm(mode_product(oracle, t, np.eye(q.shape[0]) - q @ q.T, m))
    assert oracle.projection_residual(t, cfg) <= s + 1e-12


def test_invalid_compress_configs(oracle):  # test_compress.cpp:175-191
    t = RNG.standard_normal((5, 5, 5))
    for cfg in [ccfg(oracle, 0), ccfg(oracle, 2, oversampling=-1), ccfg(oracle, 2, modes=[3])]:
        with pytest.raises(oracle.OracleInvalidArgument):
            oracle.compress(t, cfg)
    bad = t.copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.compress(bad, ccfg(oracle, 2))


# ----------------------------------------------------- test_kruskal.cpp
def random_model(shape, rank):
    return RNG.standard_normal(rank), [RNG.standard_normal((e, rank)) for e in shape]


def test_reconstruct_matches_naive(oracle):  # test_kruskal.cpp:40-58
    for shape in ([4, 5, 6], [3, 2, 4, 3]):
        w, fs = random_model(shape, 3)
        got = oracle.reconstruct(w, fs)
        want = naive_reconstruct(w, fs)
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_normalize_canonical_idempotent_preserving(oracle):  # test_kruskal.cpp:60-116
    w, fs = random_model([5, 4, 3], 4)
    w = np.array([0.3, -2.0, 1.4, 0.9])
    fs[0][:, 1] *= -3.0
    nw, nf = oracle.normalize(w, fs)
    for r in range(4):
        for f in nf:
            assert abs(np.linalg.norm(f[:, r]) - 1.0) <= 1e-12
        assert nw[r] >= 0 and (r == 0 or nw[r] <= nw[r - 1])
        c = nf[0][:, r]
        assert c[np.argmax(np.abs(c))] >= 0
    for _ in range(10):
        w, fs = random_model(random_shape(2, 4, 6), 3)
        w = RNG.uniform(-3, 3, 3)
        nw, nf = oracle.normalize(w, fs)
        before, after = oracle.reconstruct(w, fs), oracle.reconstruct(nw, nf)
        assert np.linalg.norm(before - after) <= 1e-12 * (np.linalg.norm(before) + 1.0)
        nw2, nf2 = oracle.normalize(nw, nf)
        assert np.array_equal(nw, nw2) and all(np.array_equal(a, b) for a, b in zip(nf, nf2))


def test_normalize_zero_column(oracle):  # test_kruskal.cpp:101-116
    w, fs = random_model([3, 3, 3], 2)
    fs[2][:, 0] = 0.0
    nw, nf = oracle.normalize(w, fs)
    assert nw[-1] == 0.0
    assert any(np.array_equal(f[:, -1], np.eye(f.shape[0])[:, 0]) for f in nf)


def test_fit_and_relative_error(oracle):  # test_kruskal.cpp:118-187
    w, fs = random_model([4, 5, 3], 2)
    nw, nf = oracle.normalize(w, fs)
    x = oracle.reconstruct(nw, nf)
    assert abs(oracle.fit(x, nw, nf) - 1.0) <= 1e-12
    assert oracle.relative_error(x, nw, nf) <= 1e-12
    assert abs(oracle.relative_error(x, np.zeros_like(nw), nf) - 1.0) <= 1e-12
    for _ in range(10):
        shape = random_shape(3, 3, 6)
        w, fs = random_model(shape, 2)
        x = RNG.standard_normal(shape)
        e = oracle.relative_error(x, w, fs)
        assert abs(oracle.fit(x, w, fs) - (1 - e * e)) <= 1e-10 * max(1.0, abs(1 - e * e))
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.relative_error(np.zeros((2, 2, 2)), *random_model([2, 2, 2], 1))


# ------------------------------------------------------- test_solve.cpp
def test_init_factors_known_answer(oracle):  # test_solve.cpp:45-62 (frozen)
    m = np.zeros((3, 8))
    m[0, 2], m[1, 0], m[2, 7] = 2.0, 5.0, 3.0
    t = oracle.fold(m, 1, [2, 3, 4])
    f = oracle.init_factors(t, 3, 0)
    assert np.all(f[0] == 0)
    e = np.eye(3)
    for j, unit in enumerate([1, 2, 0]):
        assert np.max(np.abs(f[1][:, j] - e[:, unit])) <= 1e-12


def test_init_factors_orthonormal(oracle):  # test_solve.cpp:64-71
    f = oracle.init_factors(RNG.standard_normal((6, 7, 5)), 4, 9)
    for a in f[1:]:
        assert np.max(np.abs(a.T @ a - np.eye(4))) <= 1e-10


def test_init_factors_padding_and_random(oracle):  # test_solve.cpp:73-95
    t = RNG.standard_normal((3, 3, 3))
    a, b, c = oracle.init_factors(t, 5, 31), oracle.init_factors(t, 5, 31), oracle.init_factors(t, 5, 32)
    for m in (1, 2):
        assert np.array_equal(a[m], b[m])
        assert np.allclose(np.linalg.norm(a[m], axis=0), 1.0, atol=1e-12)
    assert not np.array_equal(a[1], c[1])
    t = RNG.standard_normal((5, 5, 5))
    eig, rnd = oracle.init_factors(t, 3, 4, 0), oracle.init_factors(t, 3, 4, 1)
    assert not np.array_equal(eig[1], rnd[1])
    assert np.allclose(np.linalg.norm(rnd[1], axis=0), 1.0, atol=1e-12)


def test_pinv_psd(oracle):  # test_solve.cpp:107-118
    a = RNG.standard_normal((6, 6))
    v = a @ a.T + 0.5 * np.eye(6)
    assert np.max(np.abs(v @ oracle.pinv_psd(v) - np.eye(6))) <= 1e-10
    b = RNG.standard_normal((6, 2))
    s = b @ b.T
    ps = oracle.pinv_psd(s)
    assert np.max(np.abs(s @ ps @ s - s)) <= 1e-8 * np.max(np.abs(s))


def test_khatri_rao_gram_identity(oracle):  # test_solve.cpp:97-105
    for _ in range(10):
        a, b = RNG.standard_normal((7, 4)), RNG.standard_normal((5, 4))
        kr = oracle.khatri_rao(a, b)
        rhs = (a.T @ a) * (b.T @ b)
        assert np.max(np.abs(kr.T @ kr - rhs)) <= 1e-12 * np.max(np.abs(rhs))


def test_als_exact_recovery_and_monotone_fit(oracle):  # test_solve.cpp:120-144
    t, _ = oracle.random_lowrank([20, 20, 20], 3, 17)
    res = oracle.decompose(t, det_cfg(oracle, 3))
    assert res.converged and res.final_relative_error <= 1e-6
    for seed in range(3):
        t, _ = oracle.random_lowrank([10, 11, 9], 3, 40 + seed)
        res = oracle.decompose(t, det_cfg(oracle, 3, tol=1e-9, seed=seed))
        assert np.all(np.diff(res.trace_fit) >= -1e-12)


def test_als_max_iter_and_trace(oracle):  # test_solve.cpp:146-159
    t, _ = oracle.random_lowrank([10, 10, 10], 2, 6)
    res = oracle.decompose(t, det_cfg(oracle, 2, tol=1e-300, max_iter=7))
    assert not res.converged and res.iterations == 7
    assert np.all(np.diff(res.trace_seconds) >= 0)


def test_solver_rejects_invalid(oracle):  # test_solve.cpp:161-186
    t, _ = oracle.random_lowrank([5, 5, 5], 2, 1)
    for cfg in [det_cfg(oracle, 0), det_cfg(oracle, 2, tol=0.0), det_cfg(oracle, 2, max_iter=0)]:
        with pytest.raises(oracle.OracleInvalidArgument):
            oracle.decompose(t, cfg)
    bad = RNG.standard_normal((4, 4, 4))
    bad.reshape(-1)[5] = np.inf
    with pytest.raises(oracle.OracleSolverError) as e:
        oracle.decompose(bad, det_cfg(oracle, 2))
    assert e.value.iteration == 0


def test_randomized_decompose(oracle):  # test_solve.cpp:231-289
    t, _ = oracle.random_lowrank([20, 20, 20], 3, 23)
    cfg = det_cfg(oracle, 3)
    cfg.randomized = True
    cfg.compress.seed = 5
    assert oracle.decompose(t, cfg).final_relative_error <= 1e-6
    t, _ = oracle.random_lowrank([15, 15, 15], 4, 29)
    det = oracle.decompose(t, det_cfg(oracle, 4))
    rnd = det_cfg(oracle, 4)
    rnd.randomized = True
    rnd.compress.seed = 11
    assert abs(oracle.decompose(t, rnd).final_relative_error - det.final_relative_error) <= 1e-4
    # empty mode list == deterministic path, bit for bit (test_solve.cpp:252-265)
    t, _ = oracle.random_lowrank([9, 8, 7], 2, 44)
    d = oracle.decompose(t, det_cfg(oracle, 2, seed=13))
    e = det_cfg(oracle, 2, seed=13)
    e.randomized = True
    e.compress.modes = []
    r = oracle.decompose(t, e)
    assert np.array_equal(d.weights, r.weights) and all(np.array_equal(a, b) for a, b in zip(d.factors, r.factors))
    assert d.final_relative_error == r.final_relative_error
    # compression rank must equal the CP rank (test_solve.cpp:267-273)
    bad = det_cfg(oracle, 2)
    bad.randomized = True
    bad.compress.target_rank = 3
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.decompose(t, bad)


def test_decompose_end_to_end_determinism(oracle):  # test_solve.cpp:275-289
    clean, _ = oracle.random_lowrank([12, 12, 12], 3, 51)
    t = oracle.add_noise(clean, 2.0, 4)
    cfg = oracle.DecomposeConfig(rank=3, seed=77, compress=oracle.CompressConfig(seed=78))
    a, b = oracle.decompose(t, cfg), oracle.decompose(t, cfg)
    assert np.array_equal(a.weights, b.weights) and a.final_relative_error == b.final_relative_error


def test_acceptance_exact_recovery_randomized(oracle):  # acceptance/main.cpp:64-81 (ALS rows)
    t, _ = oracle.random_lowrank([40, 40, 40], 5, 1)
    for randomized in (False, True):
        cfg = oracle.DecomposeConfig(rank=5, randomized=randomized, tol=1e-12, seed=2,
                                     compress=oracle.CompressConfig(target_rank=5, oversampling=10,
                                                                    power_iterations=2,
                                                                    seed=oracle.derive_seed(2, oracle.stream_id(1))))
        assert oracle.decompose(t, cfg).final_relative_error <= 1e-5


def test_probe_c1_known_values(oracle):
    """Cross-check against SURVEY.md's independent numpy probe (Appendix):
    C1 geometry relerr 0.0992737 after 6 ALS iterations."""
    x, _ = oracle.random_lowrank([100, 100, 100], 10, 1, snr=10.0, noise_seed=1)
    cfg = oracle.DecomposeConfig(rank=10, tol=1e-8, max_iter=200, seed=1,
                                 compress=oracle.CompressConfig(target_rank=10, oversampling=10, power_iterations=2,
                                                                seed=oracle.derive_seed(1, oracle.stream_id(1))))
    res = oracle.decompose(x, cfg)
    assert res.iterations == 6 and abs(res.final_relative_error - 0.0992737) < 5e-8


# ------------------------------------------------------ BCD (solve.hpp:264-376)
def check_factors_match(got_f, want_f, tol):  # test_solve.cpp:26-41
    R = got_f[0].shape[1]
    for r in range(R):
        sign_product = 1.0
        for g, w in zip(got_f, want_f):
            s = 1.0 if g[:, r] @ w[:, r] >= 0 else -1.0
            sign_product *= s
            assert np.max(np.abs(g[:, r] - s * w[:, r])) <= tol
        assert sign_product == 1.0


def test_bcd_rank1_recovery(oracle):  # test_solve.cpp:188-195
    t, (w, fs) = oracle.random_lowrank([12, 9, 11], 1, 3)
    res = oracle.decompose(t, det_cfg(oracle, 1, method=1))
    assert abs(res.weights[0] - w[0]) <= 1e-8 * abs(w[0])
    check_factors_match(res.factors, fs, 1e-6)


def test_bcd_orthogonal_rank2_in_weight_order(oracle):  # test_solve.cpp:197-217
    rng = np.random.default_rng(5)
    fs = [oracle.thin_qr(rng.standard_normal((e, 2)))[0] for e in (10, 12, 9)]
    w, fs = oracle.normalize(np.array([3.0, 1.5]), fs)
    t = oracle.reconstruct(w, fs)
    res = oracle.decompose(t, det_cfg(oracle, 2, tol=1e-12, method=1))
    assert res.final_relative_error <= 1e-6
    assert np.allclose(res.weights, w, rtol=1e-5)
    check_factors_match(res.factors, fs, 1e-5)


def test_bcd_reports_nonconvergence(oracle):  # test_solve.cpp:219-229
    clean, _ = oracle.random_lowrank([8, 8, 8], 3, 12)
    t = oracle.add_noise(clean, 2.0, 1)
    res = oracle.decompose(t, det_cfg(oracle, 3, tol=1e-300, method=1, max_iter=5))
    assert not res.converged and res.iterations <= 5


def test_bcd_rejects_invalid(oracle):  # test_solve.cpp:161-166
    t, _ = oracle.random_lowrank([5, 5, 5], 2, 1)
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.decompose(t, det_cfg(oracle, 0, method=1))


# ------------------------------------------------ diagnostics.hpp (bound)
def test_theorem_bound_tails_are_svd_tails(oracle):  # diagnostics.hpp:36-62
    x, _ = oracle.random_lowrank([12, 10, 9], 4, 2, snr=3.0, noise_seed=2)
    tails, bound = oracle.theorem_bound(x, 3, 4)
    for m in range(3):
        sv = np.linalg.svd(oracle.unfold(x, m), compute_uv=False)
        assert abs(tails[m] - np.sum(sv[3:] ** 2)) <= 1e-12 * np.sum(sv ** 2)
    assert abs(bound - np.sqrt(1 + 3 / 3) * np.sqrt(tails.sum())) <= 1e-14 * bound
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.theorem_bound(x, 1, 4)
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.theorem_bound(x, 9, 4)


def test_validate_bound_holds_below_rank(oracle):  # diagnostics.hpp:68-86 (acceptance criterion 4 shape)
    x, _ = oracle.random_lowrank([15, 15, 15], 6, 8)
    tails, bound, mean = oracle.theorem_bound(x, 3, 4, trials=10, seed=5)
    assert 0 < mean <= bound
