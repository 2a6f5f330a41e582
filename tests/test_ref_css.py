"""Ports of the reference's factor/residual tests (test_sketch.cpp:243-268,
test_blockcur.cpp:139-173) plus the oracle's agreement with the reference's
literal exact-SVD + pinv semantics (sketch.cpp:68-82)."""
import numpy as np
import pytest

from helpers import random_matrix, random_rank_k
from oracle import bcur_oracle as O


def test_css_exact_span(impl):  # test_sketch.cpp:245-250
    rng = impl.Rng(22)
    a = random_rank_k(O.Rng(22), 8, 12, 2)
    part = impl.BlockPartition.equal_blocks(12, 3)
    _, err, _ = impl.block_css(a, part, 2, 2, rng)
    assert err <= 1e-8 * np.linalg.norm(a)


def test_css_whole_block(impl):  # test_sketch.cpp:252-255
    noisy = random_matrix(O.Rng(23), 6, 9)
    _, err, _ = impl.block_css(noisy, impl.BlockPartition.equal_blocks(9, 9), 3, 1, impl.Rng(23))
    assert err <= 1e-8 * np.linalg.norm(noisy)


def test_css_monotone_in_g(impl):  # test_sketch.cpp:257-267 (paired draws)
    g0 = O.Rng(24)
    hard = random_rank_k(g0, 10, 16, 4) + 0.05 * random_matrix(g0, 10, 16)
    part = impl.BlockPartition.equal_blocks(16, 2)
    for seed in range(1, 11 if impl.name == "oracle" else 4):
        prev = np.inf
        for g in (1, 2, 4, 8):
            _, err, _ = impl.block_css(hard, part, 4, g, impl.Rng(seed))
            assert err <= prev + 1e-9
            prev = err


def test_css_scale_equivariance(impl):  # test_blockcur.cpp:75-88 analogue
    g0 = O.Rng(103)
    a = random_rank_k(g0, 16, 24, 3) + 0.05 * random_matrix(g0, 16, 24)
    part = impl.BlockPartition.equal_blocks(24, 4)
    b1, e1, _ = impl.block_css(a, part, 3, 3, impl.Rng(77))
    b2, e2, _ = impl.block_css(37.5 * a, part, 3, 3, impl.Rng(77))
    assert b1 == b2
    assert e2 == pytest.approx(37.5 * e1, rel=1e-10)


def test_error_report_edge_cases(impl):  # test_blockcur.cpp:139-161
    a = random_matrix(O.Rng(107), 6, 8)
    ae, rel = impl.error_report(a, a, np.eye(8), np.eye(8))
    assert ae <= 1e-12 and rel <= 1e-12
    ae, _ = impl.error_report(a, a, np.zeros((8, 8)), np.eye(8))
    assert ae == pytest.approx(np.linalg.norm(a), rel=1e-12)
    with pytest.raises(impl.DimensionMismatch):
        impl.error_report(a, a, np.eye(7, 8), np.eye(8))


def test_oracle_range_finder_css_equals_reference_semantics():
    """With a generous sketch (q=3) the oracle selects the same blocks and reaches the
    same projection error as the literal reference (exact SVD + SVD pinv)."""
    gen = np.random.default_rng(11)
    for trial in range(12):
        m, n, s = int(gen.integers(20, 60)), int(gen.integers(40, 120)), int(gen.integers(2, 9))
        rank = int(gen.integers(2, 8))
        a = np.asfortranarray(gen.standard_normal((m, rank)) @ gen.standard_normal((rank, n))
                              + 1e-3 * gen.standard_normal((m, n)))
        part = O.BlockPartition.equal_blocks(n, s)
        k = rank
        g = min(part.num_blocks(), int(gen.integers(1, 6)))
        ours = O.block_css(a, part, k, g, O.Rng(trial), p=6, q=3, mode=O.WITHOUT_REPLACEMENT)
        ref = O.reference_block_css(a, part, k, g, O.Rng(trial), mode=O.WITHOUT_REPLACEMENT)
        np.testing.assert_allclose(ours.scores.scores, ref.scores.scores, rtol=1e-6, atol=1e-12)
        if min(ours.plan.margins) > 1e-6:
            assert ours.plan.blocks() == ref.plan.blocks()
            assert ours.abs_err == pytest.approx(ref.abs_err, rel=1e-8, abs=1e-12 * ref.a_norm)


def test_oracle_c1_matches_reference_semantics():
    """Config 1 (the reference's CPU-runnable case): oracle range-finder pipeline vs
    the literal reference pipeline on the same input and seed."""
    c = O.CONFIGS["c1"]
    a = O.gen_lowrank(c["m"], c["n"], O.spectrum(c["spectrum"], c["rank"]), c["noise"], c["seed"])
    part = O.BlockPartition.equal_blocks(c["n"], c["s"])
    ours = O.block_css(a, part, c["k"], c["g"], O.Rng(c["seed"]), p=c["p"], q=c["q"], mode=c["mode"])
    ref = O.reference_block_css(a, part, c["k"], c["g"], O.Rng(c["seed"]), mode=c["mode"])
    assert ours.plan.blocks() == ref.plan.blocks()
    assert ours.abs_err == pytest.approx(ref.abs_err, rel=1e-9)
    # randomized (p=5, q=0) vs exact scores differ at the sketch's accuracy (2.2e-3)
    assert np.max(np.abs(ours.scores.scores - ref.scores.scores) / ref.scores.scores) < 1e-2


def test_oracle_cur_u_matches_pinv_definition():
    gen = np.random.default_rng(3)
    m, n = 48, 64
    a = np.asfortranarray(gen.standard_normal((m, 6)) @ gen.standard_normal((6, n)) + 1e-2 * gen.standard_normal((m, n)))
    cp = O.BlockPartition.equal_blocks(n, 8)
    rp = O.BlockPartition.equal_blocks(m, 8)
    r = O.block_cur_rows_cols(a, cp, rp, 5, 3, 3, O.Rng(5), p=5, q=1)
    c = O.materialize_columns(a, cp, r.col_plan)
    rr = O.materialize_row_blocks(a, rp, r.row_plan)
    u_ref = O.pinv(c) @ a @ O.pinv(rr)
    np.testing.assert_allclose(r.u, u_ref, rtol=1e-7, atol=1e-9 * np.abs(u_ref).max())
    abs_err, _ = O.error_report(a, c, u_ref, rr)
    assert r.abs_err == pytest.approx(abs_err, rel=1e-9)


def test_oracle_greedy_first_pick_is_heaviest_block():
    gen = np.random.default_rng(8)
    a = np.asfortranarray(gen.standard_normal((30, 60)) * np.linspace(0.1, 2.0, 60)[None, :])
    part = O.BlockPartition.equal_blocks(60, 5)
    r = O.greedy_select(a, part, 3, 4, 0)
    bn = O.block_norms2(a, part)
    assert r.steps[0].block == int(np.argmax(bn))
    # residual equals the projection residual of the selected blocks
    qc, _ = O.column_basis(a, part, r.blocks(), a.dtype, bn)
    x = a - qc @ (qc.T @ a)
    assert r.abs_err == pytest.approx(float(np.linalg.norm(x)), rel=1e-9)
    # each greedy pick maximises the residual among the remaining blocks
    assert len(set(r.blocks())) == 4
