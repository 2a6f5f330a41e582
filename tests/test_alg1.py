"""The reference's default Algorithm 1 (blockcur.cpp:54-109): uniform rows → R,
approximate block leverage of R (leverage.cpp:155-164), g blocks → C, W, U = W⁺
(matcore.cpp:85-91), ‖A − CUR‖_F for U and U_k (matcore.cpp:81-83) — GPU against the
oracle's restatement; the host row draws (sampler.cpp:54-95) against the oracle on CPU."""
import numpy as np
import pytest

from oracle import bcur_oracle as O


@pytest.fixture(scope="module")
def B():
    from paper_1703_06065_b200 import bcur
    return bcur


@pytest.mark.parametrize("m,r,seed", [(100, 10, 0), (7, 30, 3), (1000, 1, 9)])
def test_row_draws_match_reference_semantics(B, m, r, seed):
    got = B.draw_rows(m, r, B.Rng(seed))
    ref = O.draw_rows(m, r, O.Rng(seed))
    assert [(x.row, x.probability, x.scale) for x in got] == [(x.row, x.probability, x.scale) for x in ref]
    if r <= m:
        got = B.draw_rows_distinct(m, r, B.Rng(seed))
        ref = O.draw_rows_distinct(m, r, O.Rng(seed))
        assert [x.row for x in got] == [x.row for x in ref]
        assert len(set(x.row for x in got)) == r


def lowrank(m, n, rank, seed, noise, dt):
    g = np.random.default_rng(seed)
    a = g.standard_normal((m, rank)) @ (g.standard_normal((rank, n)) * np.logspace(0, -2, rank)[:, None])
    return np.asfortranarray((a + noise * g.standard_normal((m, n))).astype(dt))


@pytest.mark.gpu
@pytest.mark.parametrize("dt,m,n,s,k,r,g,mode,distinct,seed", [
    (np.float64, 300, 1200, 20, 8, 40, 6, O.WITH_REPLACEMENT, False, 5),
    (np.float64, 300, 1200, 30, 8, 25, 5, O.WITHOUT_REPLACEMENT, True, 6),
    (np.float32, 256, 1024, 32, 6, 48, 8, O.WITHOUT_REPLACEMENT, False, 7),
    (np.float64, 64, 3000, 100, 5, 64, 4, O.WITH_REPLACEMENT, True, 8),
])
def test_alg1_matches_oracle(B, dt, m, n, s, k, r, g, mode, distinct, seed):
    a = lowrank(m, n, 12, seed, 1e-3, dt)
    pg, po = B.BlockPartition.equal_blocks(n, s), O.BlockPartition.equal_blocks(n, s)
    got = B.block_cur_reference(a, pg, k, r, g, B.Rng(seed), block_mode=mode, distinct_rows=distinct)
    ref = O.block_cur_alg1(a, po, k, r, g, O.Rng(seed), block_mode=mode, distinct_rows=distinct)
    assert [x.row for x in got.rows] == [x.row for x in ref.rows]
    assert got.scores.normalizer == ref.scores.normalizer
    tol = 1e-9 if dt == np.float64 else 1e-4
    np.testing.assert_allclose(got.scores.scores, ref.scores.scores, rtol=tol, atol=tol * 1e-3)
    assert got.block_plan.blocks() == ref.plan.blocks()
    assert got.a_norm == pytest.approx(ref.a_norm, rel=1e-12)
    assert got.abs_err_u == pytest.approx(ref.abs_err_u, rel=1e-6, abs=1e-9 * ref.a_norm)
    assert got.abs_err_uk == pytest.approx(ref.abs_err_uk, rel=1e-6, abs=1e-9 * ref.a_norm)
    assert got.u.shape == ref.u.shape
    assert np.max(np.abs(got.u - ref.u)) <= 1e-6 * np.max(np.abs(ref.u))


@pytest.mark.gpu
def test_alg1_degenerate_r(B):
    part = B.BlockPartition.equal_blocks(40, 10)
    with pytest.raises(B.DegenerateR):
        B.block_cur_reference(np.zeros((10, 40)), part, 2, 3, 2, B.Rng(0))


@pytest.mark.gpu
def test_alg1_boosted_matches_oracle(B):
    a = lowrank(200, 900, 10, 11, 1e-3, np.float64)
    pg, po = B.BlockPartition.equal_blocks(900, 30), O.BlockPartition.equal_blocks(900, 30)
    got, ge = B.block_cur_reference_boosted(a, pg, 6, 30, 4, 3, B.Rng(12))
    ref, re_ = O.block_cur_alg1_boosted(a, po, 6, 30, 4, 3, O.Rng(12))
    np.testing.assert_allclose(ge, re_, rtol=1e-6, atol=1e-9 * ref.a_norm)
    assert got.block_plan.blocks() == ref.plan.blocks()


# ---- score diagnostics (leverage.cpp:123-153): block stable rank and incoherence
@pytest.mark.gpu
@pytest.mark.parametrize("n,k,s", [(600, 10, 20), (2000, 50, 128), (777, 64, 100)])
def test_block_diagnostics(B, n, k, s):
    gen = np.random.default_rng(n + k)
    v, _ = np.linalg.qr(gen.standard_normal((n, k)) * np.logspace(0, -1, k))
    u, _ = np.linalg.qr(gen.standard_normal((3 * k, k)))
    pg, po = B.BlockPartition.equal_blocks(n, s), O.BlockPartition.equal_blocks(n, s)
    sr, alpha, mu = B.block_diagnostics(np.asfortranarray(v), np.asfortranarray(u), pg)
    np.testing.assert_allclose(sr, O.column_block_stable_ranks(v.T, po), rtol=1e-10)
    assert alpha == pytest.approx(O.block_stable_rank(v, po), rel=1e-10)
    assert mu == pytest.approx(O.incoherence(u), rel=1e-12)


@pytest.mark.gpu
def test_block_diagnostics_zero_block(B):
    v = np.zeros((40, 3))
    v[:30, :] = np.linalg.qr(np.random.default_rng(0).standard_normal((30, 3)))[0]
    with pytest.raises(B.ZeroBlock):
        B.block_diagnostics(v, None, B.BlockPartition.equal_blocks(40, 10))
