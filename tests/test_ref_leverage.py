"""Ports of the reference's score tests (proj/tests/test_leverage.cpp, acceptance
criterion 1) — each runs against the oracle and (marker gpu) the GPU product."""
import numpy as np
import pytest

from helpers import hadamard4, max_abs_diff, random_matrix, random_orthonormal, random_partition
from oracle import bcur_oracle as O


def exact_right(a, k):
    return O.exact_subspace(a, k).v_k


def test_partition_construction(impl):  # test_leverage.cpp:42-62
    P = impl.BlockPartition
    part = P.equal_blocks(10, 4)
    assert part.num_blocks() == 3
    off = part.offsets()
    assert off[2] == 8 and off[3] == 10
    assert part.max_width() == 4
    assert part.block_of_column(0) == 0 and part.block_of_column(7) == 1 and part.block_of_column(9) == 2
    ex = P.from_boundaries(8, [3, 5])
    assert ex.num_blocks() == 3 and list(ex.offsets()) == [0, 3, 5, 8]
    with pytest.raises(ValueError):
        P.from_boundaries(8, [5, 3])
    with pytest.raises(ValueError):
        P.from_boundaries(8, [8])
    with pytest.raises(ValueError):
        P(4, [(0, 2), (3, 4)])
    with pytest.raises(ValueError):
        P(4, [(0, 2), (2, 2)])


def test_column_leverage_canonical_bases(impl):  # test_leverage.cpp:64-75
    v = np.eye(5, 2)
    s = impl.column_leverage(v)
    assert s.scores[0] == pytest.approx(1.0) and s.scores[1] == pytest.approx(1.0)
    assert np.all(s.scores[2:] == 0.0)
    assert s.normalizer == 2.0
    h = impl.column_leverage(np.asfortranarray(hadamard4()[:, :2]))
    assert max_abs_diff(h.scores, 0.5) <= 1e-12


def test_column_leverage_sums_to_k_and_rejects_skew(impl):  # test_leverage.cpp:77-89
    rng = O.Rng(41)
    for _ in range(10):
        v = exact_right(random_matrix(rng, 9, 7), 3)
        s = impl.column_leverage(v)
        assert abs(s.scores.sum() - 3.0) <= 1e-10 * 3.0
        assert abs(s.probabilities().sum() - 1.0) <= 1e-10
    skew = np.eye(4, 2)
    skew[0, 1] = 0.5
    with pytest.raises(impl.InvalidBasis):
        impl.column_leverage(skew)


def test_block_leverage_degenerate_partitions(impl):  # test_leverage.cpp:91-104
    v = random_orthonormal(O.Rng(43), 8, 3)
    cols = impl.column_leverage(v)
    singles = impl.block_leverage(v, impl.BlockPartition.equal_blocks(8, 1))
    assert max_abs_diff(cols.scores, singles.scores) < 1e-12
    whole = impl.block_leverage(v, impl.BlockPartition.equal_blocks(8, 8))
    assert whole.scores.size == 1 and abs(whole.scores[0] - 3.0) <= 1e-10 * 3.0


def test_block_leverage_matches_slab_oracle(impl):  # test_leverage.cpp:106-128
    v = exact_right(random_matrix(O.Rng(47), 12, 12), 3)
    part = impl.BlockPartition.equal_blocks(12, 3)
    s = impl.block_leverage(v, part)
    assert abs(s.scores.sum() - 3.0) <= 1e-10 * 3
    cols = impl.column_leverage(v).scores
    for g in range(4):
        e = np.zeros((12, 3))
        for j in range(3):
            e[3 * g + j, j] = 1.0
        slab = v.T @ e
        assert s.scores[g] == pytest.approx(float(np.sum(slab * slab)), rel=1e-12)
        assert s.scores[g] == pytest.approx(float(cols[3 * g:3 * g + 3].sum()), rel=1e-12)


def test_block_leverage_permutation_invariance(impl):  # test_leverage.cpp:130-141
    a = random_matrix(O.Rng(53), 10, 8)
    part = impl.BlockPartition.equal_blocks(8, 4)
    before = impl.block_leverage(exact_right(a, 3), part)
    p = a.copy()
    p[:, [1, 3]] = p[:, [3, 1]]
    p[:, [5, 6]] = p[:, [6, 5]]
    after = impl.block_leverage(exact_right(np.asfortranarray(p), 3), part)
    assert max_abs_diff(before.scores, after.scores) < 1e-9


def test_single_row_scores(impl):  # test_leverage.cpp:223-237 (approx_block_leverage of one row)
    v = np.array([1.0, 2.0, 0.0, -1.0, 3.0, 0.5])
    part = impl.BlockPartition.equal_blocks(6, 2)
    basis = (v / np.linalg.norm(v)).reshape(6, 1)
    s = impl.block_leverage(basis, part)
    total = float(v @ v)
    for g in range(3):
        seg = v[2 * g:2 * g + 2]
        assert s.scores[g] == pytest.approx(float(seg @ seg) / total, rel=1e-12)
    assert s.distribution().sum() == pytest.approx(1.0, abs=1e-15)


def test_score_identities_random_sweep(impl):  # acceptance.cpp:68-91 (criterion 1)
    gen = O.Rng(1001)
    worst_sum, worst_col = 0.0, 0.0
    trials = 100 if impl.name == "oracle" else 25
    for _ in range(trials):
        m = 2 + gen.below(63)
        n = 2 + gen.below(63)
        k = 1 + gen.below(min(m, n))
        v = exact_right(random_matrix(gen, m, n), k)
        part = random_partition(gen, n, 8)
        part = impl.BlockPartition(n, list(zip(part.offsets()[:-1], part.offsets()[1:])))
        blocks = impl.block_leverage(v, part)
        worst_sum = max(worst_sum, abs(blocks.scores.sum() - v.shape[1]))
        singles = impl.block_leverage(v, impl.BlockPartition.equal_blocks(n, 1))
        cols = impl.column_leverage(v)
        worst_col = max(worst_col, max_abs_diff(singles.scores, cols.scores))
    assert worst_sum <= 1e-10
    assert worst_col <= 1e-12


def test_dimension_and_basis_errors(impl):
    v = random_orthonormal(O.Rng(3), 8, 2)
    with pytest.raises(impl.DimensionMismatch):
        impl.block_leverage(v, impl.BlockPartition.equal_blocks(9, 3))
    with pytest.raises(impl.InvalidBasis):
        impl.block_leverage(np.ones((2, 3)), impl.BlockPartition.equal_blocks(2, 1))
