"""GPU-vs-oracle parity of the whole hot path (BASELINE.json north star bars):
identical block selections for the same seed (when the selection has no near-tie),
block leverage within 1e-9 relative (fp64) / 1e-4 (fp32), CUR/CSS residual within
1e-6 relative of the oracle's.  All calls go through the C ABI."""
import threading

import numpy as np
import pytest

from oracle import bcur_oracle as O

pytestmark = pytest.mark.gpu

SCORE_TOL = {np.dtype(np.float64): 1e-9, np.dtype(np.float32): 1e-4}
ERR_TOL = 1e-6


@pytest.fixture(scope="module")
def B():
    from paper_1703_06065_b200 import bcur
    return bcur


def lowrank(m, n, r, spec, noise, seed, dt):
    return O.gen_lowrank(m, n, O.spectrum(spec, r), noise, seed, dtype=dt)


def check_scores(got, ref, dt):
    ref = np.asarray(ref)
    rel = np.abs(np.asarray(got) - ref) / np.maximum(np.abs(ref), 1e-300)
    assert float(np.max(rel)) <= SCORE_TOL[np.dtype(dt)], float(np.max(rel))


def check_err(got, ref, a_norm, dt):
    floor = (1e-12 if np.dtype(dt) == np.float64 else 1e-6) * a_norm
    assert abs(got - ref) <= ERR_TOL * abs(ref) + floor, (got, ref)


def check_plan(got_blocks, ref_plan):
    for t, (bg, dr) in enumerate(zip(got_blocks, ref_plan.draws)):
        if ref_plan.margins[t] < 1e-9:
            return  # near-tie (D14): later draws may legitimately differ
        assert bg == dr.block, (t, got_blocks, ref_plan.blocks())


def run_css(B, a, s, k, p, q, g, mode, seed):
    n = a.shape[1]
    pg = B.BlockPartition.equal_blocks(n, s)
    po = O.BlockPartition.equal_blocks(n, s)
    got = B.block_css(a, pg, k, g, B.Rng(seed), p=p, q=q, mode=mode, return_c=False)
    ref = O.block_css(a, po, k, g, O.Rng(seed), p=p, q=q, mode=mode)
    check_scores(got.scores.scores, ref.scores.scores, a.dtype)
    assert got.scores.normalizer == ref.scores.normalizer
    check_plan(got.plan.blocks(), ref.plan)
    if got.plan.blocks() == ref.plan.blocks():
        check_err(got.projection_error, ref.abs_err, ref.a_norm, a.dtype)
        assert got.rank_c == ref.rank_c
    assert got.a_norm == pytest.approx(ref.a_norm, rel=1e-12 if a.dtype == np.float64 else 1e-10)
    return got, ref


def test_generator_lowrank_matches_oracle(B):
    for dt in (np.float64, np.float32):
        m, n, r = 300, 700, 7
        sig = O.spectrum("geom:10:0.8", r)
        dm = B.DeviceMatrix.generate("lowrank", dt, m, n, seed=5, sigma=sig, noise=1e-3)
        got = dm.to_host()
        ref = O.gen_lowrank(m, n, sig, 1e-3, 5, dtype=dt)
        tol = 1e-12 if dt == np.float64 else 2.0 ** -22
        assert np.max(np.abs(got.astype(np.float64) - ref.astype(np.float64))) <= tol * np.max(np.abs(ref))
        # a column shard generates exactly the same columns
        sh = B.DeviceMatrix.generate("lowrank", dt, m, 200, seed=5, sigma=sig, noise=1e-3, col0=300, n_global=n)
        assert np.array_equal(sh.to_host(), got[:, 300:500])


def test_generator_biometric_matches_oracle(B):
    m, n = 16, 3000
    got = B.DeviceMatrix.generate("biometric", np.float64, m, n, seed=3).to_host()
    ref = O.gen_biometric(m, n, 3)
    assert np.max(np.abs(got - ref)) <= 1e-10 * np.max(np.abs(ref))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_range_finder_matches_oracle(B, dt):
    a = lowrank(600, 1500, 12, "geom:10:0.8", 1e-3, 9, dt)
    key = O.omega_key_from_seed(4)
    for q in (0, 2):
        got = B.range_finder(a, 10, 5, q, key)
        ref = O.range_finder(a, 10, 5, q, key)
        assert got.k_eff == ref.k_eff
        np.testing.assert_allclose(got.sigma, ref.sigma[:got.k_eff], rtol=1e-9 if dt == np.float64 else 1e-5)
        part = O.BlockPartition.equal_blocks(1500, 30)
        check_scores(O.block_sums(np.sum(got.v_k ** 2, axis=1), part),
                     O.block_sums(np.sum(ref.v_k ** 2, axis=1), part), dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_range_finder_wide_sketch_one_sided_jacobi(B, dt):
    # ℓ = k + p = 130: the ℓ×ℓ eigenproblem no longer fits shared memory and runs on the
    # one-sided (column-coalesced) Jacobi — same subspace, same σ as the oracle
    a = lowrank(700, 2400, 150, "pow:1", 1e-4, 5, dt)
    key = O.omega_key_from_seed(6)
    got = B.range_finder(a, 120, 10, 1, key)
    ref = O.range_finder(a, 120, 10, 1, key)
    assert got.k_eff == ref.k_eff
    np.testing.assert_allclose(got.sigma, ref.sigma[:got.k_eff], rtol=1e-9 if dt == np.float64 else 1e-5)
    part = O.BlockPartition.equal_blocks(2400, 40)
    check_scores(O.block_sums(np.sum(got.v_k ** 2, axis=1), part),
                 O.block_sums(np.sum(ref.v_k ** 2, axis=1), part), dt)


def test_config1_full(B):
    c = O.CONFIGS["c1"]
    a = lowrank(c["m"], c["n"], c["rank"], c["spectrum"], c["noise"], c["seed"], np.float64)
    got, ref = run_css(B, a, c["s"], c["k"], c["p"], c["q"], c["g"], c["mode"], c["seed"])
    assert got.plan.blocks() == ref.plan.blocks()


@pytest.mark.parametrize("m,n,s,dt", [(333, 420, 7, np.float64), (333, 420, 7, np.float32), (250, 600, 12, np.float64)])
def test_block_gather_odd_shapes(B, m, n, s, dt):
    """The one-launch block gather (k_copy_segments) on blocks whose byte size or offset is not a
    multiple of 16 (odd m: the 4-byte path) and on 16-byte aligned ones, against the oracle."""
    a = lowrank(m, n, 9, "pow:1", 1e-3, 5, dt)
    run_css(B, a, s, 6, 4, 1, 5, O.WITHOUT_REPLACEMENT, 2)


def test_config2_full_greedy(B):
    c = O.CONFIGS["c2"]
    a = O.gen_biometric(c["m"], c["n"], c["seed"])
    pg = B.BlockPartition.equal_blocks(c["n"], c["s"])
    po = O.BlockPartition.equal_blocks(c["n"], c["s"])
    got = B.greedy_select(a, pg, c["k"], c["g"], seed=c["seed"], p=c["p"], q=c["q"])
    ref = O.greedy_select(a, po, c["k"], c["g"], O.omega_key_from_seed(c["seed"]), p=c["p"], q=c["q"])
    assert got.blocks() == ref.blocks()
    assert [s.saturated for s in got.steps] == [s.saturated for s in ref.steps]
    assert [s.rank_added for s in got.steps] == [s.rank_added for s in ref.steps]
    check_err(got.abs_err, ref.abs_err, ref.a_norm, np.float64)


def test_config3_scaled(B):
    # config-3 structure (fp32, power-law rank 50, q=2, 128-wide blocks) at 2048 × 8192
    a = lowrank(2048, 8192, 50, "pow:1.5", 1e-4, 0, np.float32)
    run_css(B, a, 128, 50, 10, 2, 8, O.WITHOUT_REPLACEMENT, 0)


def test_config5_scaled_leverage_and_greedy(B):
    a = lowrank(1024, 16384, 60, "pow:1", 1e-4, 1, np.float32)
    run_css(B, a, 128, 40, 10, 0, 8, O.WITHOUT_REPLACEMENT, 3)
    pg = B.BlockPartition.equal_blocks(16384, 128)
    po = O.BlockPartition.equal_blocks(16384, 128)
    got = B.greedy_select(a, pg, 40, 6, seed=3, p=10)
    ref = O.greedy_select(a, po, 40, 6, O.omega_key_from_seed(3), p=10)
    for t, (sg, sr) in enumerate(zip(got.steps, ref.steps)):
        assert sg.block == sr.block, t
        if sr.margin < 1e-6 * ref.a_norm ** 2:
            break
    check_err(got.abs_err, ref.abs_err, ref.a_norm, np.float32)


def test_config4_scaled_cur(B):
    a = lowrank(1536, 2048, 40, "geom:1:0.97", 1e-3, 2, np.float32)
    cg, rg = B.BlockPartition.equal_blocks(2048, 128), B.BlockPartition.equal_blocks(1536, 128)
    co, ro = O.BlockPartition.equal_blocks(2048, 128), O.BlockPartition.equal_blocks(1536, 128)
    got = B.block_cur(a, cg, rg, 30, 4, 3, B.Rng(11), p=10)
    ref = O.block_cur_rows_cols(a, co, ro, 30, 4, 3, O.Rng(11), p=10)
    check_scores(got.col_scores.scores, ref.col_scores.scores, np.float32)
    check_scores(got.row_scores.scores, ref.row_scores.scores, np.float32)
    assert got.col_plan.blocks() == ref.col_plan.blocks()
    assert got.row_plan.blocks() == ref.row_plan.blocks()
    check_err(got.abs_err, ref.abs_err, ref.a_norm, np.float32)
    assert got.u.shape == ref.u.shape
    assert np.max(np.abs(got.u - ref.u)) <= 1e-4 * np.max(np.abs(ref.u))


@pytest.mark.parametrize("case", ["ragged", "single_block", "singleton_blocks", "with_replacement_dups",
                                  "all_blocks"])
def test_edge_partitions(B, case):
    gen = np.random.default_rng(17)
    m, n = 80, 203
    a = np.asfortranarray(gen.standard_normal((m, 9)) @ gen.standard_normal((9, n)) + 1e-2 * gen.standard_normal((m, n)))
    if case == "ragged":
        run_css(B, a, 20, 6, 4, 1, 5, O.WITHOUT_REPLACEMENT, 1)
    elif case == "single_block":
        got, ref = run_css(B, a, n, 6, 4, 0, 1, O.WITH_REPLACEMENT, 2)
        assert got.projection_error <= 1e-8 * got.a_norm
    elif case == "singleton_blocks":
        run_css(B, a[:, :60].copy(order="F"), 1, 5, 4, 1, 12, O.WITHOUT_REPLACEMENT, 3)
    elif case == "with_replacement_dups":
        run_css(B, a, 50, 6, 4, 1, 12, O.WITH_REPLACEMENT, 4)
    else:
        got, ref = run_css(B, a, 29, 6, 4, 0, 7, O.WITHOUT_REPLACEMENT, 5)
        assert got.projection_error <= 1e-8 * got.a_norm


def test_errors(B):
    part = B.BlockPartition.equal_blocks(40, 10)
    with pytest.raises(B.ZeroMatrix):
        B.block_css(np.zeros((10, 40)), part, 2, 2, B.Rng(0))
    sparse = np.zeros((10, 40))
    sparse[:, :10] = np.random.default_rng(0).standard_normal((10, 10))
    with pytest.raises(B.NotEnoughBlocks):
        B.block_css(sparse, part, 1, 3, B.Rng(0), mode=B.SamplingMode.without_replacement)
    with pytest.raises(B.DimensionMismatch):
        B.block_css(np.ones((10, 41)), part, 2, 2, B.Rng(0))
    # require_finite (matcore.cpp:26-33): NaN / Inf inputs are rejected, not propagated
    for bad in (np.nan, np.inf):
        a = np.random.default_rng(1).standard_normal((10, 40))
        a[3, 17] = bad
        with pytest.raises(ValueError):
            B.block_css(a, part, 2, 2, B.Rng(0))
        with pytest.raises(ValueError):
            B.greedy_select(a, part, 2, 2, seed=0)
        # block_css reads its finiteness verdict after the range finder has run (one host round
        # trip for both): every kernel before that read must survive NaN / Inf data — the packed
        # Jacobi's eigenvalue ranking did not (profiles/r02al) — also on the tcgen05 fp32 path
        big = np.random.default_rng(2).standard_normal((512, 4096)).astype(np.float32)
        big[7, 300] = bad
        with pytest.raises(ValueError):
            B.block_css(big, B.BlockPartition.equal_blocks(4096, 128), 20, 6, B.Rng(0), p=10, q=1)
    # the context is still usable afterwards
    ok = B.block_css(np.random.default_rng(3).standard_normal((10, 40)), part, 2, 2, B.Rng(0))
    assert np.isfinite(ok.projection_error)


def test_bitwise_rerun_determinism(B):
    a = lowrank(512, 4096, 30, "pow:1", 1e-4, 6, np.float32)
    part = B.BlockPartition.equal_blocks(4096, 128)
    r1 = B.block_css(a, part, 20, 6, B.Rng(8), p=10, q=1, mode=B.SamplingMode.without_replacement)
    r2 = B.block_css(a, part, 20, 6, B.Rng(8), p=10, q=1, mode=B.SamplingMode.without_replacement)
    assert r1.plan.blocks() == r2.plan.blocks()
    assert np.array_equal(r1.scores.scores, r2.scores.scores)
    assert r1.projection_error == r2.projection_error
    assert np.array_equal(r1.c, r2.c)


def test_result_downloads_pageable_and_pinned(B):
    """Device → host result copies: a pageable destination above 1 MB goes through the two-buffer
    pinned staging pipeline (ragged last chunk, pitched destination), a pinned one takes one copy;
    block_cur's U arrives the same in a caller-owned pinned buffer (out_u) as in a fresh array."""
    gen = np.random.default_rng(3)
    a = np.asfortranarray(gen.standard_normal((3001, 1237)))  # 29.7 MB: four 8 MB chunks, ragged
    dm = B.DeviceMatrix.from_host(a)
    assert np.array_equal(dm.to_host(), a)
    pin = B.pinned_empty((3001, 1237))
    assert pin.flags.f_contiguous and pin.dtype == np.float64
    B._check(B.L.lib.bcur_dmat_download(dm.ctx.handle, dm.handle, pin.ctypes.data_as(B.C.c_void_p), 3001))
    assert np.array_equal(pin, a)
    s = 32
    m = lowrank(256, 512, 12, "pow:1", 1e-3, 4, np.float64)
    cpart, rpart = B.BlockPartition.equal_blocks(512, s), B.BlockPartition.equal_blocks(256, s)
    r0 = B.block_cur(m, cpart, rpart, 8, 3, 3, B.Rng(2), p=4, q=1)
    buf = B.pinned_empty((3 * s, 3 * s))
    r1 = B.block_cur(m, cpart, rpart, 8, 3, 3, B.Rng(2), p=4, q=1, out_u=buf)
    assert np.shares_memory(r1.u, buf)
    assert np.array_equal(r0.u, r1.u) and r0.abs_err == r1.abs_err
    with pytest.raises(ValueError):
        B.block_cur(m, cpart, rpart, 8, 3, 3, B.Rng(2), p=4, q=1, out_u=np.zeros((4, 4), order="F"))


def test_wide_sketch_eigensolve_repeatable(B):
    """The packed Jacobi at sketch widths that need 1024-thread launches (l = k + p >= 84; c4 runs
    l = 110).  A missing barrier before its per-sweep flag reset let a late warp leave the sweep
    loop alone — an illegal access in about half of c4's 20-step runs (profiles/r02at) — so the
    same decomposition is repeated and must reproduce bit for bit."""
    a = np.asfortranarray(lowrank(384, 4096, 100, "geom:1:0.97", 1e-3, 12, np.float64))
    dm = B.DeviceMatrix.from_host(a)
    part = B.BlockPartition.equal_blocks(4096, 128)
    first = None
    for _ in range(25):
        r = B.block_css(dm, part, 100, 2, B.Rng(5), p=10, q=0)
        key = (r.plan.blocks(), r.projection_error, r.scores.scores.tobytes())
        if first is None:
            first = key
        assert key == first


def run_ranks(B, a, s, world, call):
    """Run `call(dm, ctx)` on `world` contexts of one GPU, each holding a contiguous column
    shard of `a` (blocks of width s).  The collectives are a host rendezvous after each rank
    synchronises its own stream (no device-side waiting between kernels): allreduce (fp64 sum)
    and broadcast (bytes from the root)."""
    import ctypes

    n = a.shape[1]
    G = n // s
    barrier = threading.Barrier(world)
    bufs = [None] * world
    results = [None] * world
    errors = []
    traffic = [0]

    def worker(rank):
        try:
            ctx = B.Context(0)
            lib = B.L.lib

            def allreduce(ptr, count, stream):
                h = B.DeviceMatrix.wrap(ptr, np.float64, count, 1, count, ctx)
                ctx.synchronize()
                bufs[rank] = h.to_host()[:, 0].copy()
                barrier.wait()
                total = sum(bufs)
                barrier.wait()
                lib.bcur_dmat_upload(ctx.handle, h.handle, total.ctypes.data_as(ctypes.c_void_p), count)
                h.close()

            def broadcast(ptr, nbytes, root, stream):
                h = B.DeviceMatrix.wrap(ptr, np.float32, nbytes // 4, 1, nbytes // 4, ctx)
                ctx.synchronize()
                if rank == root:
                    bufs[root] = h.to_host()[:, 0].copy()
                    traffic[0] += nbytes
                barrier.wait()
                data = bufs[root]
                barrier.wait()
                if rank != root:
                    lib.bcur_dmat_upload(ctx.handle, h.handle, data.ctypes.data_as(ctypes.c_void_p), nbytes // 4)
                ctx.synchronize()
                h.close()

            ctx.set_comm(rank, world, allreduce, broadcast)
            g0, g1 = rank * G // world, (rank + 1) * G // world
            dm = B.DeviceMatrix.from_host(np.asfortranarray(a[:, g0 * s:g1 * s]), ctx)
            dm.set_shard(g0 * s, n)
            results[rank] = call(dm, ctx)
            ctx.synchronize()
        except Exception as e:  # pragma: no cover
            errors.append(e)
            barrier.abort()

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    return results, traffic[0]


def test_two_rank_column_sharding_matches_single_rank(B):
    a = lowrank(384, 4096, 20, "pow:1", 1e-4, 12, np.float32)
    part = B.BlockPartition.equal_blocks(4096, 128)
    kw = dict(p=8, q=1, mode=B.SamplingMode.without_replacement, return_c=False)
    single = B.block_css(a, part, 16, 6, B.Rng(21), **kw)
    res, _ = run_ranks(B, a, 128, 2, lambda dm, ctx: B.block_css(dm, part, 16, 6, B.Rng(21), ctx=ctx, **kw))
    for r in res:
        assert r.plan.blocks() == single.plan.blocks()
        np.testing.assert_allclose(r.scores.scores, single.scores.scores, rtol=1e-6)
        assert r.projection_error == pytest.approx(single.projection_error, rel=1e-6)


def test_two_rank_pythagoras_css_ships_blocks_in_split_form(B):
    # C narrower than m: the residual takes the Pythagoras path and C's 3×FP16 split is
    # broadcast by each selected block's owner — 4 bytes per element, no fp64 panels
    a = lowrank(2048, 8192, 30, "pow:1", 1e-3, 5, np.float32)
    part = B.BlockPartition.equal_blocks(8192, 128)
    kw = dict(p=10, q=1, mode=B.SamplingMode.without_replacement, return_c=False)
    single = B.block_css(a, part, 20, 8, B.Rng(4), **kw)
    assert single.residual_path == "pythagoras"
    res, traffic = run_ranks(B, a, 128, 2, lambda dm, ctx: B.block_css(dm, part, 20, 8, B.Rng(4), ctx=ctx, **kw))
    for r in res:
        assert r.plan.blocks() == single.plan.blocks()
        np.testing.assert_allclose(r.scores.scores, single.scores.scores, rtol=1e-6)
        assert r.projection_error == pytest.approx(single.projection_error, rel=1e-6)
    assert traffic <= 2048 * 8 * 128 * 4 + 8 * 128 * 4  # m·c·4 bytes + the exponents


def test_two_rank_greedy_matches_single_rank(B):
    a = lowrank(1024, 4096, 30, "pow:1", 1e-4, 3, np.float32)
    part = B.BlockPartition.equal_blocks(4096, 128)
    single = B.greedy_select(a, part, 16, 5, seed=2, p=10)
    res, _ = run_ranks(B, a, 128, 2, lambda dm, ctx: B.greedy_select(dm, part, 16, 5, seed=2, p=10, ctx=ctx))
    for r in res:
        assert r.blocks() == single.blocks()
        assert r.abs_err == pytest.approx(single.abs_err, rel=1e-6)


def test_two_rank_block_cur_matches_single_rank(B):
    a = lowrank(1536, 2048, 40, "geom:1:0.97", 1e-3, 2, np.float32)
    cg, rg = B.BlockPartition.equal_blocks(2048, 128), B.BlockPartition.equal_blocks(1536, 128)
    single = B.block_cur(a, cg, rg, 30, 4, 3, B.Rng(11), p=10)
    res, _ = run_ranks(B, a, 128, 2, lambda dm, ctx: B.block_cur(dm, cg, rg, 30, 4, 3, B.Rng(11), p=10, ctx=ctx))
    for r in res:
        assert r.col_plan.blocks() == single.col_plan.blocks()
        assert r.row_plan.blocks() == single.row_plan.blocks()
        assert r.abs_err == pytest.approx(single.abs_err, rel=1e-6)
        np.testing.assert_allclose(r.u, single.u, rtol=1e-5, atol=1e-6 * np.max(np.abs(single.u)))


# Blocked fp64 Cholesky (w > 144: 128-wide diagonal blocks, the block-row solve split between
# the chain and a side stream, trailing DSYRK on a third stream, R⁻¹ assembled on a fourth)
# inside the whole-C CholQR2: ragged last block (fp64, w = 700) and a 12-step chain (fp32,
# w = 1536, 3×FP16 products) against the oracle's CUR error.
@pytest.mark.parametrize("dt,m,n,s,g", [(np.float64, 1024, 4096, 100, 7), (np.float32, 2048, 8192, 128, 12)])
def test_blocked_factorization_widths(B, dt, m, n, s, g):
    a = lowrank(m, n, 40, "pow:1", 1e-3, 9, dt)
    got, ref = run_css(B, a, s, 30, 10, 1, g, O.WITHOUT_REPLACEMENT, 9)
    assert got.plan.blocks() == ref.plan.blocks()
    assert got.rank_c == g * s


# fp32 shapes off the 64-row grid of the fp16 copy (TF32 fallbacks) and a whole-C basis whose
# width is not a multiple of 64 with a ragged block (3×FP16 partial tiles)
@pytest.mark.parametrize("m,n,s,g", [(1000, 3000, 100, 6), (2048, 1050, 100, 11)])
def test_fp32_off_grid_shapes(B, m, n, s, g):
    a = lowrank(m, n, 30, "pow:1", 1e-4, 13, np.float32)
    got, ref = run_css(B, a, s, 20, 10, 1, g, O.WITHOUT_REPLACEMENT, 13)
    assert got.plan.blocks() == ref.plan.blocks()


def run_css_forced(B, a, s, k, p, q, g, mode, seed, residual):
    """run_css with the ABI's residual mode forced on both sides."""
    n = a.shape[1]
    pg, po = B.BlockPartition.equal_blocks(n, s), O.BlockPartition.equal_blocks(n, s)
    code = {"explicit": B.L.RESID_EXPLICIT, "pythagoras": B.L.RESID_PYTHAGORAS}[residual]
    got = B.block_css(a, pg, k, g, B.Rng(seed), p=p, q=q, mode=mode, return_c=False, residual=code)
    ref = O.block_css(a, po, k, g, O.Rng(seed), p=p, q=q, mode=mode, residual=residual)
    check_scores(got.scores.scores, ref.scores.scores, a.dtype)
    assert got.plan.blocks() == ref.plan.blocks()
    assert got.residual_path == ref.residual_path == residual
    check_err(got.projection_error, ref.abs_err, ref.a_norm, a.dtype)
    return got, ref


def test_config3_shape_pythagoras_path(B):
    # the c3 structure at 2048 × 8192 with the noise raised so that rel_err² > θ_explicit = 0.1:
    # the residual takes the same Pythagoras path as full-size c3 (‖A‖² − the fp16 row-Σ² pass)
    a = lowrank(2048, 8192, 50, "pow:1.5", 3e-4, 0, np.float32)
    got, ref = run_css(B, a, 128, 50, 10, 2, 8, O.WITHOUT_REPLACEMENT, 0)
    assert ref.residual_path == "pythagoras" and got.residual_path == "pythagoras"
    assert got.plan.blocks() == ref.plan.blocks()


def planted(m, n, s, heavy, r, seed, noise, dt):
    """Low rank with coherent right factors: the rows of V in the `heavy` column blocks are
    scaled up before orthonormalization, so block leverage is far from uniform and a wrong
    score would change the selection (the Philox generator's V is nearly incoherent)."""
    gen = np.random.default_rng(seed)
    u, _ = np.linalg.qr(gen.standard_normal((m, r)))
    v0 = gen.standard_normal((n, r))
    for i, b in enumerate(heavy):
        v0[b * s:(b + 1) * s] *= 4.0 + i
    v, _ = np.linalg.qr(v0)
    sig = 10.0 * 0.85 ** np.arange(r)
    a = (u * sig) @ v.T + noise * gen.standard_normal((m, n))
    return np.asfortranarray(a.astype(dt))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_planted_heavy_blocks_coherent_leverage(B, dt):
    s, heavy = 64, [3, 17, 40, 41, 58]
    a = planted(768, 64 * s, s, heavy, 24, 31, 1e-3, dt)
    got, ref = run_css(B, a, s, 20, 8, 1, 6, O.WITHOUT_REPLACEMENT, 5)
    sc = np.asarray(ref.scores.scores)
    assert sc[heavy].min() > 5.0 * np.median(sc)  # the planted blocks dominate
    assert got.plan.blocks() == ref.plan.blocks()
    assert len(set(ref.plan.blocks()) & set(heavy)) >= 2


def test_row_scaled_fp32_dynamic_range(B):
    # rows spanning 2^±24 inside every column (e.g. users in different units): the per-column
    # fp16 scaling of the 3×FP16 split cannot hold the small rows' significands
    gen = np.random.default_rng(3)
    a = lowrank(1024, 4096, 30, "pow:1", 1e-3, 4, np.float64)
    a *= (2.0 ** gen.uniform(-24, 24, size=1024))[:, None]
    a = np.asfortranarray(a.astype(np.float32))
    got, ref = run_css(B, a, 128, 20, 10, 1, 6, O.WITHOUT_REPLACEMENT, 2)
    assert got.plan.blocks() == ref.plan.blocks()
    cg, rg = B.BlockPartition.equal_blocks(4096, 128), B.BlockPartition.equal_blocks(1024, 128)
    co, ro = O.BlockPartition.equal_blocks(4096, 128), O.BlockPartition.equal_blocks(1024, 128)
    gc = B.block_cur(a, cg, rg, 20, 4, 3, B.Rng(7), p=10)
    rc = O.block_cur_rows_cols(a, co, ro, 20, 4, 3, O.Rng(7), p=10)
    check_scores(gc.col_scores.scores, rc.col_scores.scores, np.float32)
    check_scores(gc.row_scores.scores, rc.row_scores.scores, np.float32)
    check_err(gc.abs_err, rc.abs_err, rc.a_norm, np.float32)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_steep_spectrum_keeps_k_like_the_reference(B, dt):
    # σ_i = 0.8^i: σ_40/σ_1 ≈ 1.3e-4 — the reference's rank cut (1e-12·max(m,n)·σ₁,
    # matcore.cpp:35-49) keeps all k = 40; the working-precision floor is opt-in only
    a = lowrank(1024, 4096, 60, "geom:1:0.8", 0.0, 8, dt)
    part = B.BlockPartition.equal_blocks(4096, 128)
    ex = O.exact_subspace(a, 40)
    got = B.block_css(a, part, 40, 4, B.Rng(1), p=10, q=2, mode=B.SamplingMode.without_replacement,
                      return_c=False)
    assert got.scores.normalizer == ex.k_eff == 40
    floor = B.block_css(a, part, 40, 4, B.Rng(1), p=10, q=2, mode=B.SamplingMode.without_replacement,
                        return_c=False, rank_floor=True)
    ref_floor = O.block_css(a, O.BlockPartition.equal_blocks(4096, 128), 40, 4, O.Rng(1), p=10, q=2,
                            mode=O.WITHOUT_REPLACEMENT, rank_floor=True)
    assert floor.scores.normalizer == ref_floor.scores.normalizer


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_forced_residual_paths(B, dt):
    # the explicit streamed residual Σ(A − Q_C X)² (and Pythagoras) forced through the ABI's
    # residual mode, on a low-noise input (rel_err ≈ 1e-3) with n ≥ 256
    a = lowrank(1024, 4096, 20, "geom:1:0.7", 1e-5, 21, dt)
    for mode in ("explicit", "pythagoras"):
        if dt == np.float32 and mode == "pythagoras":
            continue  # ‖A‖² − ‖QᵀA‖² cancels to noise in fp32 at rel_err 1e-3 (why AUTO goes explicit)
        run_css_forced(B, a, 128, 15, 10, 1, 6, O.WITHOUT_REPLACEMENT, 4, mode)


def test_config3_shape_low_noise_explicit_residual(B):
    # c3 structure with little noise (rel_err ≈ 1e-2 < √θ_explicit): AUTO takes the explicit path —
    # X = QᵀA and Σ(A − QX)² on tcgen05 3×FP16 with the subtraction fused into the epilogue
    a = lowrank(2048, 8192, 50, "pow:1.5", 1e-6, 0, np.float32)
    got, ref = run_css(B, a, 128, 50, 10, 2, 8, O.WITHOUT_REPLACEMENT, 0)
    assert ref.residual_path == "explicit" and got.residual_path == "explicit"
    assert got.plan.blocks() == ref.plan.blocks()
    forced, ref_f = run_css_forced(B, a, 128, 50, 10, 2, 8, O.WITHOUT_REPLACEMENT, 0, "explicit")
    assert forced.projection_error == pytest.approx(got.projection_error, rel=1e-9)
