"""GPU: the standalone recover and als_solve entry points of the C ABI.

rcpg_recover restates kruskal.hpp:198-220 (A_n = Q_n A~_n, identity modes
copied, then normalize kruskal.hpp:117-176); checked against numpy's product
and the oracle's normalize. rcpg_als_solve is solve.hpp:183-262 (ALS on the
tensor itself) and must equal decompose(randomized=False) bit for bit.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def model_and_bases(rcp, dtype, seed, shape=(40, 33, 27), small=(6, 33, 5), R=4):
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.5, 2.0, R).astype(dtype)
    facs = [np.asfortranarray(rng.standard_normal((e, R)).astype(dtype)) for e in small]
    bases = []
    for e, k in zip(shape, small):
        if e == k:
            bases.append(rcp.ModeBasis(q=None, identity=True, dim=e, rank_warning=False))
        else:
            q, _ = np.linalg.qr(rng.standard_normal((e, k)))
            bases.append(rcp.ModeBasis(q=np.asfortranarray(q.astype(dtype)), identity=False, dim=e,
                                       rank_warning=False))
    return rcp.Kruskal(w, facs), bases


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
def test_recover_matches_product_then_normalize(rcp, oracle, dtype, tol):
    k, bases = model_and_bases(rcp, dtype, 7)
    out = rcp.recover(k, bases)
    big = [f.astype(np.float64) if b.identity else b.q.astype(np.float64) @ f.astype(np.float64)
           for f, b in zip(k.factors, bases)]
    ew, ef = oracle.normalize(k.weights.astype(np.float64), big)
    assert out.weights.dtype == dtype
    np.testing.assert_allclose(out.weights, ew, rtol=tol, atol=0)
    for a, e in zip(out.factors, ef):
        assert a.shape == e.shape
        np.testing.assert_allclose(a, e, rtol=0, atol=tol * 10)


def test_recover_rejects_mismatched_bases(rcp):
    k, bases = model_and_bases(rcp, np.float64, 3)
    with pytest.raises(Exception, match="one basis per mode"):
        rcp.recover(k, bases[:2])
    bad = list(bases)
    bad[0] = rcp.ModeBasis(q=np.zeros((40, 7)), identity=False, dim=40, rank_warning=False)
    with pytest.raises(Exception, match="basis columns"):
        rcp.recover(k, bad)


def test_recover_of_compress_bases(rcp):
    """recover(decompose of the compressed tensor, compress bases) is what
    the randomized decompose does internally (solve.hpp:392-396)."""
    rng = np.random.default_rng(11)
    A = [rng.standard_normal((e, 3)) for e in (30, 28, 26)]
    x = np.einsum("ir,jr,kr->ijk", *A)
    comp = rcp.compress(x, rcp.CompressConfig(target_rank=3, oversampling=2, power_iterations=1, seed=5))
    cm, _ = rcp.decompose(comp.compressed, rcp.DecomposeConfig(rank=3, randomized=False, tol=1e-12,
                                                               max_iter=200, seed=9))
    full = rcp.recover(cm, comp.bases)
    assert [f.shape[0] for f in full.factors] == [30, 28, 26]
    assert rcp.relative_error(x, full) < 1e-6


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_als_solve_is_plain_decompose(rcp, dtype):
    rng = np.random.default_rng(5)
    A = [rng.standard_normal((e, 3)) for e in (20, 18, 16)]
    x = (np.einsum("ir,jr,kr->ijk", *A) + 0.01 * rng.standard_normal((20, 18, 16))).astype(dtype)
    cfg = rcp.DecomposeConfig(rank=3, tol=1e-8, max_iter=50, seed=3, randomized=True,
                              compress=rcp.CompressConfig(target_rank=3, oversampling=2, power_iterations=1, seed=4))
    m1, t1 = rcp.als_solve(x, cfg)
    assert cfg.randomized  # the caller's config is not modified
    cfg.randomized = False
    m2, t2 = rcp.decompose(x, cfg)
    assert t1.iterations == t2.iterations
    assert t1.final_relative_error == t2.final_relative_error
    np.testing.assert_array_equal(m1.weights, m2.weights)
    for a, b in zip(m1.factors, m2.factors):
        np.testing.assert_array_equal(a, b)
