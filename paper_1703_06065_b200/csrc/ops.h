// ops.h — host-side launchers for every device kernel of the hot path.
// Everything takes the context (stream, workspace pool) and raw device pointers.
#pragma once

#include "common.cuh"

namespace bcur_b200 {
namespace ops {

enum Op { OP_N = 0, OP_T = 1 };

// ---- reductions (kernels_reduce.cu) --------------------------------------
// out[g] = Σ_{j∈block g} Σ_i a(i,j)²  (fp64; offsets are device, relative to a's first column)
// shadow (nullable, fp32 A only): also write the TF32-rounded copy of A (ld lds)
// Optional copies written in the same pass (fp32 A): `shadow` = TF32-rounded fp32, or
// `sh16` = fp16 scaled per column by 2^colexp[j] (exact; see gemm_rowsumsq_f16), and with
// it optionally `sl16` = hi and the fp16 remainder lo interleaved per 64-row chunk, 2m halves
// per column (m % 64 == 0): the A operand of the 3×FP16 products
void block_sumsq(Ctx* c, const void* a, int dt, int64_t m, int64_t ld, const int64_t* d_offsets, int64_t G,
                 double* d_out, float* shadow = nullptr, int64_t lds = 0, uint16_t* sh16 = nullptr,
                 int* colexp = nullptr, uint16_t* sl16 = nullptr);
// out[j] = Σ_c v(j,c)²   then segmented into blocks: out_blocks[g]
void row_sumsq_blocks(Ctx* c, const void* v, int dt, int64_t n, int64_t k, int64_t ld, const int64_t* d_offsets,
                      int64_t G, double* d_rows /*nullable*/, double* d_blocks);
// segmented sum of a fp64 vector over block offsets
void segment_sum(Ctx* c, const double* x, const int64_t* d_offsets, int64_t G, double* d_out);
// max |G - I| over the upper triangle of a symmetric w×w fp64 matrix → d_out[0]
void max_dev_identity(Ctx* c, const double* g, int64_t w, int64_t ld, double* d_out);
// per row block g of V (n × k, k ≤ 64): ‖V_g‖_F² and ‖V_g‖_2² (stable-rank diagnostics)
void block_spectral(Ctx* c, const double* v, int64_t ld, int64_t k, const int64_t* d_offsets, int64_t G, double* d_fro2,
                    double* d_spec2);
// max_i Σ_c u(i, c)² → d_out[0]
void max_row_sumsq(Ctx* c, const double* u, int64_t m, int64_t ld, int64_t k, double* d_out);
// ordered sum of x[0..n) → d_out[0]
void sum_vector(Ctx* c, const double* x, int64_t n, double* d_out);
// Σ x[i]² over x[0..n) → d_out[0] (fixed-order, deterministic)
void sumsq_vector(Ctx* c, const double* x, int64_t n, double* d_out);

// ---- dense products (kernels_gemm.cu), fp64 accumulation ------------------
// C(M×N fp64) = alpha·op(A)·op(B) + beta·C.  Structure hints (exploited by the tcgen05 path
// only; other paths compute the full product):
//   GEMM_SYM_UPPER  op(A)·op(B) is the Gram AᵀA (B == A): only C's upper triangle is needed
//   GEMM_B_UPPER    op(B) is upper triangular
//   GEMM_X1         the product is a small correction (‖op(B)‖ ≲ 1e-4): one round-to-nearest
//                   TF32 pass suffices (errors ~1e-4 × the correction)
//   GEMM_A_UPPER / GEMM_A_LOWER / GEMM_B_LOWER   op(A) upper / lower, op(B) lower triangular
//                   (the fp64 DMMA path skips the zero blocks)
//   GEMM_FAST_ACC   3×FP16 only: the three MMAs of a k-step into one fp32 accumulator (CTA pairs,
//                   N = 256 tiles; fp32-grade, ~1e-6 relative): for products whose error is
//                   corrected downstream or far inside its bar
//   GEMM_HI_ONLY    with GEMM_FAST_ACC: a_hi·x_hi alone (one of the three MMAs; the lo halves are
//                   not loaded): 2⁻¹¹-relative, for corrections ≲ 1e-4 of the result they are
//                   added to (the CholQR2 second pass), whose error is then ≲ 1e-7 of the result
enum GemmFlags { GEMM_SYM_UPPER = 1, GEMM_B_UPPER = 2, GEMM_X1 = 4, GEMM_A_UPPER = 8, GEMM_A_LOWER = 16,
                 GEMM_B_LOWER = 32, GEMM_FAST_ACC = 64, GEMM_HI_ONLY = 128 };
void gemm(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, double alpha, const void* A, int dta, int64_t lda,
          const void* B, int dtb, int64_t ldb, double beta, double* C, int64_t ldc, int flags = 0);
// rowsq[i] = Σ_j (op(A)·op(B))(i,j)²   (product never stored)
// a_rounded: A is already rounded to TF32 (block_sumsq's shadow) — the X1 pass skips its transform
void gemm_rowsumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                   const void* B, int dtb, int64_t ldb, double* rowsq, bool a_rounded = false);
// rowsq[j] = Σ_c (AᵀX)_jc² from block_sumsq's fp16 copy of A (K × M, ld lda, column j scaled
// by 2^colexp[j]).  X (K × N, fp32/fp64) is converted to fp16 scaled by a power of two
// from its max; the tensor cores run kind::f16 (same 11-bit significand as the
// round-to-nearest 1×TF32 pass, twice the MMA rate, half the bytes) and the scales are
// removed exactly in fp64.
// interleaved: A16 is the [hi 64 | lo 64]-per-chunk copy (only hi is read), else compact hi.
// x16_pre (nullable): X already in fp16 (K × N, ld K) scaled by 2^q_pre (B is then unused);
// x16_il: x16_pre is an interleaved hi/lo split (2K halves per column) whose hi part is X
// d_tiles (nullable, ntiles entries): compute only these 128-row tiles of the output (the other
// rows are zero) — needs rowsq_tiles_ok(M, N) (the CTA-pair path)
void gemm_rowsumsq_f16(Ctx* c, int64_t M, int64_t N, int64_t K, const uint16_t* A16, int64_t lda, const int* colexp,
                       const void* B, int dtb, int64_t ldb, double* rowsq, bool interleaved = true,
                       const uint16_t* x16_pre = nullptr, int q_pre = 0, bool x16_il = false,
                       const int* d_tiles = nullptr, int ntiles = 0);
bool rowsq_tiles_ok(int64_t M, int64_t N);
// orthonormal Q (fp64) → fp32 basis + its fp16 copy scaled by 2^14 (one pass)
void basis_out(Ctx* c, const double* q, int64_t K, int64_t N, int64_t ldq, float* q32, uint16_t* q16);
// out[0] = Σ_ij (D − op(A)·op(B))(i,j)²
void gemm_resid_sumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                      const void* B, int dtb, int64_t ldb, const void* D, int dtd, int64_t ldd, double* out);

// ---- fp64 tensor-core products (kernels_dmma.cu, mma.sync m8n8k4 .f64) -----
// C = alpha·op(A)·op(B) + beta·C, fp32/fp64 operands, fp64 accumulation; flags as gemm()
void dgemm(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, double alpha, const void* A, int dta, int64_t lda,
           const void* B, int dtb, int64_t ldb, double beta, double* C, int64_t ldc, int flags = 0);
void dgemm_rowsumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                    const void* B, int dtb, int64_t ldb, double* rowsq);
void dgemm_resid_sumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                       const void* B, int dtb, int64_t ldb, const void* D, int dtd, int64_t ldd, double* out);
// st = {int info, int pad, double min diag(R) = +inf, double max diag(G)} before a factorization
void chol_status_init(Ctx* c, const double* g, int64_t w, int64_t ldg, int* st);
// w > 128: R (upper, ld w) with G = RᵀR (G's upper triangle read, ldg) and X = R⁻¹ (upper, ld w)
// in one cooperative persistent launch (blocked right-looking, fp64 DMMA); st as chol_status_init
// (initialized by the caller), info = failed pivot + 1
// want_r = false: R's diagonal blocks are not written (its off-diagonal blocks always are)
void chol_persistent(Ctx* c, const double* g, int64_t w, int64_t ldg, double* r, double* x, int* st, bool want_r = true);
// *flag = 1 unless the factorization with status st passed min diag(R) > tau·sqrt(max diag(G))
void chol_flag(Ctx* c, const int* st, double tau, int* flag);
// w ≤ 128, one CTA: R (upper, lower zeroed) with G = RᵀR from G's upper triangle, and X = R⁻¹
// (upper).  Chained status: skipped when *info != 0; failure → info = info_offset + j + 1;
// diag[0] = running min diag(R).  flags: 1 = R not written (r may be null), 2 = the lower
// triangles of R and X are already zero (only the upper triangles are written)
void chol_inv_leaf(Ctx* c, const double* g, int64_t w, int64_t ldg, double* r, int64_t ldr, double* x, int64_t ldx,
                   int* info, double* diag, int64_t info_offset, int flags = 0);

// ---- tcgen05 3×TF32 A-passes (kernels_umma.cu), fp32 A only ----------------
bool umma_ok(int dta, int64_t m, int64_t lda, const void* a);
// Out(n×N) = alpha·Aᵀ X + beta·Out (fp64) or rowsq[j] = Σ_c (AᵀX)_jc²; X fp32 or fp64.
// sym: X holds the same matrix as A (a Gram) — only the upper triangle of Out is written.
void umma_atx(Ctx* c, const float* A, int64_t m, int64_t n, int64_t lda, const void* X, int dtx, int64_t N,
              int64_t ldx, double alpha, double beta, double* out, int64_t ldo, double* rowsq, bool sym = false,
              bool a_rounded = false);
// Out(m×N) = alpha·A X + beta·Out (fp64); X fp32 or fp64; x_upper_tri: X[k,j] = 0 for k > j
void umma_ax(Ctx* c, const float* A, int64_t m, int64_t n, int64_t lda, const void* X, int dtx, int64_t N,
             int64_t ldx, double alpha, double beta, double* out, int64_t ldo, bool x_upper_tri = false,
             bool x1 = false);

// ---- 3×FP16 products (kernels_umma.cu, H3) --------------------------------
// An fp16 hi + lo split of a K × N operand (ld K), column j scaled by 2^exps[j] (exact).
struct SplitF16 {
    DevBuf hi, lo, exps;
    int64_t K = 0, N = 0, ld = 0;  // ld: K rounded up to 8 (TMA strides are multiples of 16 bytes)
};
// A non-owning view of one (a SplitF16, or — lo == nullptr — an interleaved split_il buffer
// read as the K-major X operand, K % 64 == 0)
struct F16View {
    const uint16_t* hi;
    const uint16_t* lo;
    const int* exps;
    int64_t K, N;
    int64_t ld = 0;  // separate hi/lo: leading dimension in halves (0: K)
    int part = -1;   // interleaved only: 0 / 1 = read the hi / lo part alone as X (the other reads as zero)
};
inline F16View view(const SplitF16& s) {
    return {s.hi.as<uint16_t>(), s.lo.as<uint16_t>(), s.exps.as<int>(), s.K, s.N, s.ld};
}
// fold (nullable, K ints): exponents subtracted from row k first (A·X with a scaled A)
void split_f16(Ctx* c, const void* x, int dtx, int64_t K, int64_t N, int64_t ldx, const int* fold, SplitF16* out);
// A (m × n, fp32/fp64, lda) → the interleaved hi/lo A operand (2m halves per column; m % 64 == 0)
// with per-column exponents
void split_il(Ctx* c, const void* a, int dta, int64_t m, int64_t n, int64_t lda, DevBuf* il, DevBuf* exps);
void split_il_into(Ctx* c, const void* a, int dta, int64_t m, int64_t n, int64_t lda, uint16_t* il, int* exps);
// umma_h3 on operands split here (a_mn: A·X, else AᵀX; GEMM_SYM_UPPER: AᵀA with X == A)
void gemm_h3(Ctx* c, bool a_mn, const void* A, int dta, int64_t m, int64_t n, int64_t lda, const void* X, int dtx,
             int64_t N, int64_t ldx, double alpha, double beta, double* out, int64_t ldo, int flags = 0);
// A (m × n) given as block_sumsq's interleaved fp16 hi/lo copy AL (2m halves per column) with
// column exponents ea; needs m % 64 == 0.
bool h3_ok(int64_t m);
// a_mn: Out(m×N) = alpha·A·X + beta·Out (X: n × N); else Out(n×N) = alpha·AᵀX + beta·Out (X: m × N).
// flags: GEMM_SYM_UPPER (AᵀA with X the split of A itself: upper tiles only), GEMM_B_UPPER (A·X, X upper).
// Every product is hi·hi + hi·lo + lo·hi on kind::f16 tensor cores (fp32 accumulate, drained to
// compensated fp32 every 8 MMAs), scales removed exactly in the fp64 epilogue.
void umma_h3(Ctx* c, bool a_mn, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const F16View& X,
             double alpha, double beta, double* out, int64_t ldo, int flags = 0);
void umma_h3(Ctx* c, bool a_mn, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const void* X, int dtx,
             int64_t N, int64_t ldx, double alpha, double beta, double* out, int64_t ldo, int flags = 0);

// Out = alpha·A·X (a_mn form; N > 64, m % 64 == 0) written straight into the interleaved split
// layout (2m halves per column) with the fixed column exponent 14 (fill_basis_exps): for
// outputs with |entries| < 2 (orthonormal-basis candidates, e.g. Q1 = C·R⁻¹)
void umma_h3_to_split(Ctx* c, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const void* X, int dtx,
                      int64_t N, int64_t ldx, double alpha, uint16_t* out_il, int flags = 0);
// Q = alpha·A·X (+ addend_il read back from its fixed-exponent split, nullable) written as the
// fp32 basis q32 (m × N, ld m) and its fp16 copy q16: the interleaved split of Q·2^14 (2m halves
// per column; hi = the row-Σ² passes' operand, lo = hi's rounding error)
void umma_h3_basis(Ctx* c, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const void* X, int dtx, int64_t N,
                   int64_t ldx, double alpha, const uint16_t* addend_il, float* q32, uint16_t* q16, int flags = 0);
// exps[0..n) = 14, the column exponents of umma_h3_to_split's output
void fill_basis_exps(Ctx* c, int* exps, int64_t n);

// Σ_ij (D − A·X)_ij² with A the interleaved split (m × n, exps ea), X fp64 (n × N, ldx), D fp32
// (m × N, ldd): the explicit residual's second product fused with the subtraction (tcgen05 3×FP16)
void umma_h3_resid(Ctx* c, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const void* X, int dtx, int64_t N,
                   int64_t ldx, const float* D, int64_t ldd, double* d_sum);

// ---- small dense factorizations (kernels_small.cu), single CTA, fp64 ------
// R upper (ld ldr, may alias g) with G = RᵀR, only g's upper triangle is read; info[0] = 0 ok / j+1 failed pivot;
// diag[0] = min diag(R), diag[1] = max diag(G) (input)
// chained: part of a blocked factorization (skip if *info != 0; failures report info_offset + j + 1;
// diag[0] accumulates the min across the chain)
void cholesky_upper(Ctx* c, const double* g, int64_t w, int64_t ldg, double* r, int64_t ldr, int* info, double* diag,
                    int64_t info_offset = 0, bool chained = false);
// X = I − F where F = strict_upper(E) + diag(E)/2, E = G − I (first-order inverse of the
// Cholesky factor of a near-identity Gram)
// minus_identity: return −F instead (the correction of Q = Q1·(I − F) = Q1 + Q1·(−F))
void near_identity_rinv(Ctx* c, const double* g, int64_t w, int64_t ldg, double* x, bool minus_identity = false);
// P ← R⁻ᵀ·P in place (R upper kb × kb, kb ≤ 128; P kb × n): the blocked Cholesky's panel solve
void trsm_upper_t(Ctx* c, const double* r, int64_t kb, int64_t ldr, double* p, int64_t ldp, int64_t n);
// X = R⁻¹ (upper triangular, w ≤ 128; only R's upper triangle is read; X's lower is zeroed)
void tri_inv_upper(Ctx* c, const double* r, int64_t w, int64_t ldr, double* x, int64_t ldx);
// symmetric eig, eigenvalues descending in lam, eigenvectors in columns of V (w×w)
void sym_eig(Ctx* c, const double* g, int64_t w, int64_t ldg, double* lam, double* v);

// ---- elementwise / layout (kernels_misc.cu) -------------------------------
void convert(Ctx* c, const void* src, int dts, int64_t m, int64_t n, int64_t lds, void* dst, int dtd, int64_t ldd);
// nsegs contiguous device → device copies in one launch (d_segs on the device; bytes % 4 == 0)
struct CopySeg {
    const void* src;
    void* dst;
    size_t bytes;
};
void copy_segments(Ctx* c, const CopySeg* d_segs, int nsegs, size_t max_bytes);
// dst[i] = fp32(src[i] as fp16) · scale
void f16_to_f32(Ctx* c, const uint16_t* src, int64_t count, float scale, float* dst);
void transpose(Ctx* c, const void* src, int dts, int64_t m, int64_t n, int64_t lds, void* dst, int dtd, int64_t ldd);
void zero_lower(Ctx* c, double* x, int64_t w, int64_t ld);
void convert_to_f64(Ctx* c, const void* src, int dt, int64_t m, int64_t n, int64_t lds, double* dst, int64_t ldd);
void fill_f64(Ctx* c, double* p, int64_t count, double v);
// *d_flag |= 1 when any of x[0..count) is NaN or Inf (the loader's require_finite)
void flag_nonfinite(Ctx* c, const double* x, int64_t count, unsigned int* d_flag);
void axpy_neg(Ctx* c, const double* x, double* y, int64_t n);  // y -= x
void scale_columns(Ctx* c, double* x, int64_t m, int64_t n, int64_t ld, const double* d_scale /*n*/);
void scale_rows(Ctx* c, double* x, int64_t m, int64_t n, int64_t ld, const double* d_scale /*m*/);
// out[j] = Σ_{i ∈ ranges} v(i, j)² for j < k (ranges: nr pairs [r0, r1) on the device)
void colsumsq_ranges(Ctx* c, const double* v, int64_t ld, int64_t k, const int64_t* d_ranges, int nr, double* d_out);
// scale[k] = σ[k]·√max(0, 1 − lev[k])
void sigma_weights(Ctx* c, const double* d_sigma, const double* d_lev, int64_t n, double* d_scale);
void copy_f64(Ctx* c, const double* src, int64_t m, int64_t n, int64_t lds, double* dst, int64_t ldd);
void transpose_to_f64(Ctx* c, const void* src, int dt, int64_t m, int64_t n, int64_t lds, double* dst, int64_t ldd);

// ---- generators (kernels_gen.cu) ------------------------------------------
void omega(Ctx* c, uint64_t key, int64_t n_rows, int64_t row0, int64_t l, double* out, int64_t ld);
void gaussian_matrix(Ctx* c, uint64_t key, uint32_t stream, int64_t m, int64_t n, double* out, int64_t ld);
void lowrank_assemble(Ctx* c, const double* us /*m×r*/, const double* v /*n_global×r*/, int64_t m, int64_t n,
                      int64_t r, int64_t col0, int64_t n_global, double noise, uint64_t seed, void* a, int dt,
                      int64_t lda);
void biometric(Ctx* c, int64_t m, int64_t n, int64_t col0, int64_t n_global, uint64_t seed, void* a, int dt,
               int64_t lda);

// ---- sampling (kernels_sample.cu) -----------------------------------------
// scores (G) → distribution → draws with the given uniforms.  status[0] = bcur_status.
void distribution_draw(Ctx* c, const double* d_scores, int64_t G, int normalize, int64_t g, int mode,
                       const double* d_uniforms, bcur_block_draw* d_draws, double* d_margins, int* d_status);
// C[:, dst cols of draw t] = scale_t · A[:, block_t]  (or rows when rows=1: gathers row blocks into R)
void gather_blocks(Ctx* c, const void* a, int dt, int64_t m, int64_t n, int64_t lda, const int64_t* d_offsets,
                   const bcur_block_draw* d_draws, const int64_t* d_dst_off, int64_t ndraws, int rows, int scaled,
                   void* out, int dto, int64_t ldo);
// argmax over unselected entries (ties → lowest index); out_vals = {top1, top2}
// count successive picks, each masking its block: out3[3t..] = {index (as double), best, second best}
void argmax_masked_seq(Ctx* c, const double* x, unsigned char* mask_selected, int64_t G, int count, double* out3);
void argmax_masked(Ctx* c, const double* x, const unsigned char* mask_selected, int64_t G, int64_t* out_idx,
                   double* out_vals);

}  // namespace ops
}  // namespace bcur_b200
