"""fp64 tensor-core products (DMMA, kernels_dmma.cu) and the recursive Cholesky + inverse
(pipeline.cu chol_inv) against numpy fp64 — the arithmetic behind the fp64 configs' sketch
and residual (c1/c2) and behind every orthonormal basis of the path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    from paper_1703_06065_b200 import bcur
    return bcur


def rel_fro(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.mark.parametrize("m,n,N", [(500, 2000, 15), (64, 20000, 10), (1, 7, 3), (129, 65, 1), (300, 301, 130),
                                   (2048, 512, 256), (777, 333, 16), (1000, 64, 9), (70, 5000, 17)])
def test_dmma_products(B, m, n, N):
    gen = np.random.default_rng(m * 7 + n + N)
    a = np.asfortranarray(gen.standard_normal((m, n)))
    x = np.asfortranarray(gen.standard_normal((n, N)))
    assert rel_fro(B.sketch_product(a, x), a @ x) < 1e-14
    q = np.asfortranarray(gen.standard_normal((m, N)))
    ref = a.T @ q
    assert rel_fro(B.sketch_product(a, q, transpose=True), ref) < 1e-14
    rows = B.sketch_product(a, q, transpose=True, row_sumsq=True)
    np.testing.assert_allclose(rows, np.sum(ref * ref, axis=1), rtol=1e-13)


@pytest.mark.parametrize("m,n", [(500, 200), (96, 1000), (300, 129)])
def test_dmma_structured(B, m, n):
    gen = np.random.default_rng(m + n)
    a = np.asfortranarray(gen.standard_normal((m, n)))
    g = B.structured_product(a, gram=True)
    ref = a.T @ a
    iu = np.triu_indices(n)
    assert np.max(np.abs(g[iu] - ref[iu])) <= 1e-13 * np.max(np.abs(ref))
    xu = np.asfortranarray(np.triu(gen.standard_normal((n, n))))
    np.testing.assert_allclose(B.structured_product(a, xu, x_upper=True), a @ xu, rtol=1e-12, atol=1e-12)


def spd(gen, w, cond_pow=2.0):
    x = gen.standard_normal((w + 40, w)) * (np.arange(1, w + 1) ** (-cond_pow / 2.0 / max(w, 1)))[None, :]
    return np.asfortranarray(x.T @ x)


@pytest.mark.parametrize("w", [1, 5, 37, 128, 129, 200, 384, 1000, 1536, 2113])
def test_cholesky_inverse(B, w):
    gen = np.random.default_rng(w)
    g = spd(gen, w)
    r, ri, info, mn = B.cholesky(g)
    assert info == 0
    ref = np.linalg.cholesky(g).T
    assert np.allclose(np.tril(r, -1), 0.0) and np.allclose(np.tril(ri, -1), 0.0)
    assert rel_fro(r, ref) < 1e-12
    assert np.max(np.abs(ri @ r - np.eye(w))) < 1e-11
    assert mn == pytest.approx(float(np.min(np.diag(ref))), rel=1e-12)
    # only the upper triangle of G is read
    g2 = g.copy()
    g2[np.tril_indices(w, -1)] = np.nan
    r2, _, info2, _ = B.cholesky(g2)
    assert info2 == 0 and np.array_equal(r2, r)


def test_cholesky_hybrid_tensor_core_products(B, monkeypatch):
    """The factorization path of the fp32 pipelines' basis Grams at w >= 3072: one recursion level
    around two persistent launches, the off-diagonal quarter on tcgen05 3xFP16 products (an
    fp32-class result by design: the Gram it factors is one).  R, R^-1 and min diag are checked,
    with R requested (the pipelines skip it)."""
    w = 3072
    gen = np.random.default_rng(11)
    x = gen.standard_normal((w + 256, w)) / np.sqrt(w + 256.0)
    g = np.asfortranarray(x.T @ x + 0.5 * np.eye(w))  # kappa ~ 10
    monkeypatch.setenv("BCUR_CHOL_TC", "1")
    r, ri, info, mn = B.cholesky(g)
    monkeypatch.delenv("BCUR_CHOL_TC")
    assert info == 0
    ref = np.linalg.cholesky(g).T
    assert np.allclose(np.tril(r, -1), 0.0) and np.allclose(np.tril(ri, -1), 0.0)
    assert rel_fro(r, ref) < 1e-5
    assert np.max(np.abs(ri @ ref - np.eye(w))) < 1e-4
    assert mn == pytest.approx(float(np.min(np.diag(ref))), rel=1e-4)
    r64, ri64, _, _ = B.cholesky(g)  # the fp64 path on the same input
    assert rel_fro(r64, ref) < 1e-12


@pytest.mark.parametrize("w,bad", [(50, 17), (200, 150), (700, 300), (700, 650)])
def test_cholesky_reports_failed_pivot(B, w, bad):
    gen = np.random.default_rng(bad)
    x = gen.standard_normal((w + 10, w))
    x[:, bad] = x[:, :bad] @ gen.standard_normal(bad)  # column `bad` in the span of the earlier ones
    g = np.asfortranarray(x.T @ x)
    g[bad, bad] -= 1e-3 * abs(g[bad, bad])             # … and pushed below: pivot `bad` is negative
    _, _, info, _ = B.cholesky(g)
    assert info == bad + 1
