"""tcgen05 3×TF32 sketch products vs exact fp64 products of the same fp32 A
(the accuracy the range finder and residual passes rely on)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    from paper_1703_06065_b200 import bcur
    return bcur


def rel_fro(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.mark.parametrize("m,n,N", [(512, 1024, 60), (1024, 768, 110), (256, 4096, 220), (2048, 512, 256),
                                   (96, 1000, 17), (64, 200, 64)])
def test_ax_and_atx(B, m, n, N):
    gen = np.random.default_rng(m + n + N)
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    a64 = a.astype(np.float64)
    x = np.asfortranarray(gen.standard_normal((n, N)))
    y = B.sketch_product(a, x)
    assert rel_fro(y, a64 @ x) < 2e-6
    q = np.asfortranarray(gen.standard_normal((m, N)))
    z = B.sketch_product(a, q, transpose=True)
    assert rel_fro(z, a64.T @ q) < 2e-6


def test_low_mantissa_bits_are_kept(B):
    """Inputs whose information sits below the TF32 mantissa: a plain TF32 product would
    lose it (rel. error ~1e-3); the 3×TF32 split must keep fp32 accuracy."""
    gen = np.random.default_rng(1)
    m, n, N = 256, 512, 64
    base = np.float32(1.0) + gen.integers(0, 1 << 13, size=(m, n)).astype(np.float32) * np.float32(2.0 ** -23)
    a = np.asfortranarray(base * np.sign(gen.standard_normal((m, n))).astype(np.float32))
    x = np.asfortranarray(gen.standard_normal((n, N)))
    ref = a.astype(np.float64) @ x
    assert rel_fro(B.sketch_product(a, x), ref) < 2e-6
    q = np.asfortranarray(gen.standard_normal((m, N)))
    assert rel_fro(B.sketch_product(a, q, transpose=True), a.astype(np.float64).T @ q) < 2e-6


@pytest.mark.parametrize("N", [40, 128, 300, 1024])
def test_fused_row_sumsq(B, N):
    gen = np.random.default_rng(N)
    m, n = 512, 1000
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    q = np.asfortranarray(gen.standard_normal((m, N)))
    ref = np.sum((a.astype(np.float64).T @ q) ** 2, axis=1)
    got = B.sketch_product(a, q, transpose=True, row_sumsq=True)
    # 1×TF32 with both operands rounded to nearest: unbiased per-element errors ~2⁻¹² that
    # average out — a row (N·K terms) is good to ~1e-4, the grand total to ~1e-7
    assert np.max(np.abs(got - ref) / ref) < 5e-4
    # the total's random part shrinks like 1/sqrt(#dot products); systematic part ≲ 2e-6
    assert abs(got.sum() - ref.sum()) / ref.sum() < 3e-6 + 4 * 2.5e-4 / np.sqrt(n * N)


# CTA-pair 3×TF32 path (k_umma2_x3): NT = 2 products with ≥ 74 pair tiles; odd tile counts
# leave the last pair's second CTA on zero-filled A rows
@pytest.mark.parametrize("m,n,N", [(8288, 256, 600), (8192, 96, 1000)])
def test_pair_ax(B, m, n, N):
    gen = np.random.default_rng(m + N)
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    x = np.asfortranarray(gen.standard_normal((n, N)))
    assert rel_fro(B.sketch_product(a, x), a.astype(np.float64) @ x) < 2e-6


@pytest.mark.parametrize("m,n,N", [(512, 8288, 600), (224, 8192, 1000)])
def test_pair_atx(B, m, n, N):
    gen = np.random.default_rng(m + n + N)
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    q = np.asfortranarray(gen.standard_normal((m, N)))
    assert rel_fro(B.sketch_product(a, q, transpose=True), a.astype(np.float64).T @ q) < 2e-6


@pytest.mark.parametrize("m,n", [(1024, 4224), (480, 2176)])
def test_gram_upper(B, m, n):
    gen = np.random.default_rng(m + n)
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    a64 = a.astype(np.float64)
    g = B.structured_product(a, gram=True)
    ref = a64.T @ a64
    iu = np.triu_indices(n)
    assert rel_fro(g[iu], ref[iu]) < 2e-6


@pytest.mark.parametrize("m,n", [(8192, 640), (4096, 200)])
def test_x_upper(B, m, n):
    gen = np.random.default_rng(m + n + 1)
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    x = np.asfortranarray(np.triu(gen.standard_normal((n, n))))
    assert rel_fro(B.structured_product(a, x, x_upper=True), a.astype(np.float64) @ x) < 2e-6


# fp16 row-Σ² path (kind::f16 on block_sumsq's per-column-scaled copy): single-CTA NT = 1/2/4
# and the CTA-pair kernel; columns spanning many binades exercise the per-column scales
@pytest.mark.parametrize("m,n,N", [(512, 1000, 40), (512, 1000, 128), (1024, 768, 300), (2048, 1024, 1024)])
def test_rowsq_f16(B, m, n, N):
    gen = np.random.default_rng(m + n + N)
    a = gen.standard_normal((m, n)) * np.exp2(gen.integers(-40, 40, size=n))[None, :]
    a = np.asfortranarray(a.astype(np.float32))
    q = np.asfortranarray(gen.standard_normal((m, N)) * 1e-3)
    ref = np.sum((a.astype(np.float64).T @ q) ** 2, axis=1)
    got = B.structured_product(a, q, rowsq_f16=True)
    # same rounding model as the 1×TF32 pass (11-bit significands, round to nearest)
    rel = (got - ref) / ref
    assert np.max(np.abs(rel)) < 5e-4
    # unbiased: the per-row errors average out (column scales span 2^±40, so the plain
    # total would be one column's error)
    assert abs(rel.mean()) < 3e-6 + 4 * rel.std() / np.sqrt(n)


# ---- 3×FP16 (fp16 hi + lo split with exact power-of-two column scales) --------------
@pytest.mark.parametrize("m,n,N", [(512, 1024, 60), (1024, 768, 110), (256, 4096, 220), (2048, 512, 256),
                                   (128, 1000, 17), (64, 200, 64), (4096, 2048, 60)])
def test_h3_ax_and_atx(B, m, n, N):
    gen = np.random.default_rng(7 * m + n + N)
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    a64 = a.astype(np.float64)
    x = np.asfortranarray(gen.standard_normal((n, N)))
    assert rel_fro(B.structured_product(a, x, h3=True), a64 @ x) < 2e-6
    q = np.asfortranarray(gen.standard_normal((m, N)))
    assert rel_fro(B.structured_product(a, q, transpose=True, h3=True), a64.T @ q) < 2e-6


def test_h3_scales_and_low_bits(B):
    """Columns of A spanning 2^±20 and rows of X spanning 2^±12 (the exact per-column
    scales must keep every column's own precision), with information below the fp16
    significand (1 + k·2⁻²³)."""
    gen = np.random.default_rng(3)
    m, n, N = 256, 640, 64
    base = np.float32(1.0) + gen.integers(0, 1 << 13, size=(m, n)).astype(np.float32) * np.float32(2.0 ** -23)
    a = base * np.sign(gen.standard_normal((m, n))).astype(np.float32)
    a = np.asfortranarray(a * np.float32(2.0) ** gen.integers(-20, 21, size=n).astype(np.float32))
    a64 = a.astype(np.float64)
    x = np.asfortranarray(gen.standard_normal((n, N)) * 2.0 ** gen.integers(-12, 13, size=(n, 1)))
    ref = a64 @ x
    got = B.structured_product(a, x, h3=True)
    # every output column is dominated by its largest terms: compare per element against
    # the exact sum of |terms| (the conditioning-free bound)
    bound = np.abs(a64) @ np.abs(x)
    assert np.max(np.abs(got - ref) / bound) < 1e-6
    q = np.asfortranarray(gen.standard_normal((m, N)))
    got_t = B.structured_product(a, q, transpose=True, h3=True)
    bound_t = np.abs(a64).T @ np.abs(q)
    assert np.max(np.abs(got_t - a64.T @ q) / bound_t) < 1e-6


@pytest.mark.parametrize("m,n", [(1024, 384), (512, 200)])
def test_h3_gram_and_triangular(B, m, n):
    gen = np.random.default_rng(m + n)
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    a64 = a.astype(np.float64)
    g = B.structured_product(a, gram=True, h3=True)
    iu = np.triu_indices(n)
    ref = a64.T @ a64
    assert rel_fro(g[iu], ref[iu]) < 2e-6
    r = np.triu(gen.standard_normal((n, n)))
    got = B.structured_product(a, r, x_upper=True, h3=True)
    assert rel_fro(got, a64 @ r) < 2e-6


@pytest.mark.parametrize("m,n,N,upper", [(8192, 512, 1100, False), (8192, 640, 1100, True)])
def test_h3_fast_acc(B, m, n, N, upper):
    """GEMM_FAST_ACC (k_umma2_h3m): the three fp16 MMAs of a k-step into one fp32 accumulator —
    fp32-grade (the tensor core's round-toward-zero over 24 accumulations per chunk, ~1e-6)
    instead of the split accumulators' ~2⁻²².  Shapes large enough for the CTA-pair path."""
    gen = np.random.default_rng(m + n + N)
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    x = gen.standard_normal((n, N))
    if upper:
        x = np.triu(x)
    x = np.asfortranarray(x)
    ref = a.astype(np.float64) @ x
    fast = B.structured_product(a, x, x_upper=upper, h3=True, fast_acc=True)
    exact = B.structured_product(a, x, x_upper=upper, h3=True)
    assert rel_fro(exact, ref) < 2e-6
    assert rel_fro(fast, ref) < 5e-6
    # the bias is systematic (toward zero) but bounded by the accumulation count per chunk
    assert abs(np.sum(fast * ref) / np.sum(ref * ref) - 1.0) < 3e-6


@pytest.mark.parametrize("m,n,N", [(8192, 640, 1100)])
def test_h3_hi_only_correction(B, m, n, N):
    """GEMM_HI_ONLY (k_umma2_h3m, one MMA: a_hi·x_hi): the CholQR2 second pass's correction
    Q1·(−F) with ‖F‖ ~ 1e-4.  The product alone is 2⁻¹¹-relative; added to Q1 (the basis
    epilogue), its error is ≲ 1e-7 of the result."""
    gen = np.random.default_rng(m + n + N + 1)
    a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    x = np.asfortranarray(np.triu(gen.standard_normal((n, N))))
    ref = a.astype(np.float64) @ x
    hi = B.structured_product(a, x, x_upper=True, h3=True, fast_acc=True, hi_only=True)
    err = rel_fro(hi, ref)
    assert 1e-5 < err < 1e-3  # one fp16 MMA: well above the 3×FP16 error, below 2⁻¹⁰
