"""Ports of the reference's sampling tests (proj/tests/test_sampler.cpp) —
oracle and (marker gpu) the GPU draw/gather kernels."""
import math

import numpy as np
import pytest

from helpers import max_abs_diff, random_matrix
from oracle import bcur_oracle as O


def test_identical_seeds_identical_plans(impl):  # test_sampler.cpp:25-48
    a, b = impl.Rng(99), impl.Rng(99)
    probs = [0.2, 0.5, 0.3]
    pa = impl.draw_blocks(probs, 7, impl.WITH, a)
    pb = impl.draw_blocks(probs, 7, impl.WITH, b)
    assert [d.block for d in pa.draws] == [d.block for d in pb.draws]
    assert [d.scale for d in pa.draws] == [d.scale for d in pb.draws]


def test_degenerate_distributions(impl):  # test_sampler.cpp:76-97
    rng = impl.Rng(4)
    plan = impl.draw_blocks([1.0], 9, impl.WITH, rng)
    for d in plan.draws:
        assert d.block == 0 and d.scale == pytest.approx(1.0 / math.sqrt(9.0))
    only0 = impl.draw_blocks([1.0, 0.0, 0.0], 50, impl.WITH, rng)
    assert all(d.block == 0 for d in only0.draws)
    with pytest.raises(impl.DistributionInvalid):
        impl.draw_blocks([0.5, 0.4], 3, impl.WITH, rng)
    with pytest.raises(ValueError):
        impl.draw_blocks([1.0], 0, impl.WITH, rng)
    with pytest.raises(impl.DistributionInvalid):
        impl.draw_blocks([0.5, -0.1, 0.6], 1, impl.WITH, rng)


def test_block_frequencies_concentrate(impl):  # test_sampler.cpp:99-111
    plan = impl.draw_blocks([0.25] * 4, 40000, impl.WITH, impl.Rng(77))
    counts = np.bincount([d.block for d in plan.draws], minlength=4)
    sigma = math.sqrt(40000 * 0.25 * 0.75)
    assert np.all(np.abs(counts - 10000.0) <= 3.0 * sigma)


def test_without_replacement(impl):  # test_sampler.cpp:113-129
    probs = [0.4, 0.3, 0.1, 0.1, 0.1]
    plan = impl.draw_blocks(probs, 5, impl.WITHOUT, impl.Rng(6))
    seen = set()
    for d in plan.draws:
        seen.add(d.block)
        assert d.probability == pytest.approx(probs[d.block])
        assert d.scale == pytest.approx(1.0 / math.sqrt(5.0 * probs[d.block]))
    assert seen == {0, 1, 2, 3, 4}
    with pytest.raises(impl.NotEnoughBlocks):
        impl.draw_blocks([0.6, 0.4, 0.0, 0.0], 3, impl.WITHOUT, impl.Rng(6))


def test_materialize_hand_checkable(impl):  # test_sampler.cpp:131-149
    a = random_matrix(O.Rng(7), 5, 6)
    whole = impl.BlockPartition.equal_blocks(6, 6)
    assert max_abs_diff(impl.materialize_columns(a, whole, [(0, 1.0, 1.0)]), a) < 1e-15
    eye = np.eye(4)
    halves = impl.BlockPartition.equal_blocks(4, 2)
    c = impl.materialize_columns(eye, halves, [(1, 0.5, 1.0 / math.sqrt(0.5))])
    assert c.shape == (4, 2)
    assert c[2, 0] == pytest.approx(math.sqrt(2.0)) and c[3, 1] == pytest.approx(math.sqrt(2.0))
    assert np.all(c[:2] == 0.0)
    with pytest.raises(impl.DimensionMismatch):
        impl.materialize_columns(eye, halves, [(5, 0.5, 1.0)])


def test_identity_plan_exact(impl):  # test_sampler.cpp:151-157
    a = random_matrix(O.Rng(8), 4, 9)
    part = impl.BlockPartition.equal_blocks(9, 3)
    assert np.array_equal(impl.materialize_columns(a, part, impl.identity_plan(part)), a)


def test_sampled_mass_unbiased(impl):  # test_sampler.cpp:159-185
    rng = impl.Rng(2025)
    q = random_matrix(O.Rng(2025), 5, 8)
    part = impl.BlockPartition.equal_blocks(8, 3)
    probs = [0.5, 0.2, 0.3]
    trials = 4000 if impl.name == "oracle" else 800
    norms2 = np.array([float(q[:, part.offsets()[b]:part.offsets()[b + 1]].__pow__(2).sum()) for b in range(3)])
    samples = []
    for _ in range(trials):
        plan = impl.draw_blocks(probs, 4, impl.WITH, rng)
        samples.append(sum(norms2[d.block] * d.scale ** 2 for d in plan.draws))
    samples = np.array(samples)
    sigma_mean = samples.std(ddof=1) / math.sqrt(trials)
    assert abs(samples.mean() - float(np.sum(q * q))) <= 3.0 * sigma_mean


@pytest.mark.gpu
def test_gpu_draws_match_oracle_draws():
    """Same distribution + same Rng stream ⇒ same blocks (ties excepted, D14)."""
    from paper_1703_06065_b200 import bcur
    gen = np.random.default_rng(5)
    for trial in range(30):
        G = int(gen.integers(1, 3000))
        s = gen.random(G) ** 3
        s[gen.random(G) < 0.1] = 0.0
        if s.sum() == 0:
            s[0] = 1.0
        p = s / s.sum()
        positive = int(np.sum(p > 0))
        for mode in (O.WITH_REPLACEMENT, O.WITHOUT_REPLACEMENT):
            g = int(gen.integers(1, max(2, min(64, positive))))
            ref = O.draw_blocks(p, g, mode, O.Rng(trial))
            got = bcur.draw_blocks(p, g, mode, bcur.Rng(trial))
            for t, (dr, dg) in enumerate(zip(ref.draws, got.draws)):
                if ref.margins[t] > 1e-12:
                    assert dr.block == dg.block, (trial, mode, t)
                    assert dr.scale == pytest.approx(dg.scale, rel=1e-15)
                else:
                    break  # after a near-tie the streams may legitimately diverge
