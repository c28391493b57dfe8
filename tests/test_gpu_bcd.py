"""BCD solver (bcd_solve, solve.hpp:264-376) on the GPU: the reference's own BCD tests
(test_solve.cpp:188-229) and parity with the oracle's restatement, deterministic and
randomized (decompose(method = bcd) on the compressed tensor, solve.hpp:381-398).
"""
import numpy as np
import pytest

from test_oracle_pins import check_factors_match

pytestmark = pytest.mark.gpu


def _pair(rcp, oracle, rank, tol=1e-10, max_iter=500, randomized=False, seed=0, p=5, q=2, cseed=9):
    kw = dict(rank=rank, method=1, randomized=randomized, tol=tol, max_iter=max_iter, seed=seed)
    g = rcp.DecomposeConfig(**kw, compress=rcp.CompressConfig(target_rank=rank, oversampling=p, power_iterations=q,
                                                               seed=cseed))
    o = oracle.DecomposeConfig(**kw, compress=oracle.CompressConfig(target_rank=rank, oversampling=p,
                                                                     power_iterations=q, seed=cseed))
    return g, o


def test_bcd_rank1_recovery(rcp, oracle):  # test_solve.cpp:188-195
    t, (w, fs) = oracle.random_lowrank([12, 9, 11], 1, 3)
    g, _ = _pair(rcp, oracle, 1, tol=1e-13)
    model, trace = rcp.decompose(t, g)
    assert abs(model.weights[0] - w[0]) <= 1e-8 * abs(w[0])
    check_factors_match(model.factors, fs, 1e-6)


def test_bcd_orthogonal_rank2_in_weight_order(rcp, oracle):  # test_solve.cpp:197-217
    rng = np.random.default_rng(5)
    fs = [oracle.thin_qr(rng.standard_normal((e, 2)))[0] for e in (10, 12, 9)]
    w, fs = oracle.normalize(np.array([3.0, 1.5]), fs)
    t = oracle.reconstruct(w, fs)
    g, _ = _pair(rcp, oracle, 2, tol=1e-12)
    model, trace = rcp.decompose(t, g)
    assert trace.final_relative_error <= 1e-6
    assert np.allclose(model.weights, w, rtol=1e-5)
    check_factors_match(model.factors, fs, 1e-5)


def test_bcd_reports_nonconvergence(rcp, oracle):  # test_solve.cpp:219-229
    clean, _ = oracle.random_lowrank([8, 8, 8], 3, 12)
    t = oracle.add_noise(clean, 2.0, 1)
    g, o = _pair(rcp, oracle, 3, tol=1e-300, max_iter=5)
    model, trace = rcp.decompose(t, g)
    ref = oracle.decompose(t, o)
    assert not trace.converged and trace.iterations <= 5
    assert trace.iterations == ref.iterations


def test_bcd_rejects_invalid(rcp, oracle):
    t, _ = oracle.random_lowrank([5, 5, 5], 2, 1)
    g, _ = _pair(rcp, oracle, 0)
    with pytest.raises(ValueError):
        rcp.decompose(t, g)


@pytest.mark.parametrize("randomized", [False, True])
@pytest.mark.parametrize("shape,rank", [((20, 18, 16), 3), ((40, 30, 20), 4), ((12, 10, 14, 9), 3)])
def test_bcd_matches_oracle_fp64(rcp, oracle, shape, rank, randomized):
    """fp64: the same inner-iteration count, fit trace, factors and relative error as the oracle."""
    t, _ = oracle.random_lowrank(list(shape), rank, 11, snr=3.0, noise_seed=11)
    g, o = _pair(rcp, oracle, rank, tol=1e-8, randomized=randomized, seed=7)
    model, trace = rcp.decompose(t, g)
    ref = oracle.decompose(t, o)
    assert trace.iterations == ref.iterations and trace.converged == ref.converged
    fit = np.array([e.fit for e in trace.entries])
    assert np.max(np.abs(fit - ref.trace_fit)) <= 1e-10
    assert abs(trace.final_relative_error - ref.final_relative_error) <= 1e-8 * ref.final_relative_error
    for a, b in zip(model.factors, ref.factors):
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)


@pytest.mark.parametrize("randomized", [False, True])
def test_bcd_matches_oracle_fp32(rcp, oracle, randomized):
    """fp32 (faithful arithmetic): same iterations, fit within 1e-6."""
    t, _ = oracle.random_lowrank([40, 32, 24], 4, 13, snr=4.0, noise_seed=13)
    t = t.astype(np.float32)
    g, o = _pair(rcp, oracle, 4, tol=1e-6, randomized=randomized, seed=3)
    model, trace = rcp.decompose(t, g)
    ref = oracle.decompose(t, o)
    assert trace.iterations == ref.iterations
    fit_g, fit_o = 1 - trace.final_relative_error ** 2, 1 - ref.final_relative_error ** 2
    assert abs(fit_g - fit_o) <= 1e-6 * abs(fit_o)


def test_bcd_deterministic_reruns(rcp, oracle):
    t, _ = oracle.random_lowrank([30, 25, 20], 3, 4, snr=3.0, noise_seed=4)
    g, _ = _pair(rcp, oracle, 3, tol=1e-8, randomized=True, seed=1)
    m1, t1 = rcp.decompose(t, g)
    m2, t2 = rcp.decompose(t, g)
    assert t1.final_relative_error == t2.final_relative_error and t1.iterations == t2.iterations
    for a, b in zip(m1.factors, m2.factors):
        assert np.array_equal(a, b)
