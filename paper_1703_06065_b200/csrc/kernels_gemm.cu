// kernels_gemm.cu — product dispatch: every op(A)·op(B) of the hot path goes to one of
// the hand-written tensor-core kernels.
//
//   fp32 A-passes and wide fp32 products  → tcgen05 (kernels_umma.cu: 3×FP16 on the split
//                                           copies, 3×TF32 on raw fp32 A)
//   everything else (fp64 inputs, Grams,   → DMMA fp64 (kernels_dmma.cu), fused epilogues
//   factor products, mixed fp32/fp64)        STORE / ROWSQ / RESID
#include "ops.h"

namespace bcur_b200 {

namespace ops {

void gemm(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, double alpha, const void* A, int dta, int64_t lda,
          const void* B, int dtb, int64_t ldb, double beta, double* C, int64_t ldc, int flags) {
    if (M <= 0 || N <= 0) return;
    // fp32 products wide enough to be tensor-bound (N ≥ 256, Grams) → 3×FP16 on operands split
    // here (the split is one extra pass over A: worth it only where the MMAs dominate).  This
    // includes the GEMM_X1 corrections: 3×FP16 is both faster than the 1×TF32 pass (no in-kernel
    // rounding) and exact to ~2⁻²² instead of 2⁻¹¹ of the correction.
    if (dta == BCUR_F32 && K > 0 && tb == OP_N && (N >= 256 || (flags & GEMM_SYM_UPPER)) &&
        h3_ok(ta == OP_N ? M : K) && ((uintptr_t)A % 16) == 0) {
        const bool sym = (flags & GEMM_SYM_UPPER) && A == B && dta == dtb && lda == ldb && M == N && beta == 0.0;
        if (ta == OP_N)
            gemm_h3(c, true, A, dta, M, K, lda, B, dtb, N, ldb, alpha, beta, C, ldc, flags & GEMM_B_UPPER);
        else
            gemm_h3(c, false, A, dta, K, M, lda, B, dtb, N, ldb, alpha, beta, C, ldc, sym ? GEMM_SYM_UPPER : 0);
        return;
    }
    // fp32 A-passes → tcgen05 3×TF32 kernels
    if (dta == BCUR_F32 && K > 0 && tb == OP_N) {
        if (ta == OP_N && K % 4 == 0 && umma_ok(dta, M, lda, A)) {
            umma_ax(c, (const float*)A, M, K, lda, B, dtb, N, ldb, alpha, beta, C, ldc, (flags & GEMM_B_UPPER) != 0,
                    (flags & GEMM_X1) != 0);
            return;
        }
        if (ta == OP_T && umma_ok(dta, K, lda, A)) {
            const bool sym = (flags & GEMM_SYM_UPPER) && A == B && dta == dtb && lda == ldb && M == N && beta == 0.0;
            umma_atx(c, (const float*)A, K, M, lda, B, dtb, N, ldb, alpha, beta, C, ldc, nullptr, sym);
            return;
        }
    }
    dgemm(c, ta, tb, M, N, K, alpha, A, dta, lda, B, dtb, ldb, beta, C, ldc, flags);
}

void gemm_rowsumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                   const void* B, int dtb, int64_t ldb, double* rowsq, bool a_rounded) {
    if (M <= 0) return;
    if (ta == OP_T && tb == OP_N && dta == BCUR_F32 && N > 0 && K > 0 && umma_ok(dta, K, lda, A)) {
        umma_atx(c, (const float*)A, K, M, lda, B, dtb, N, ldb, 1.0, 0.0, nullptr, 0, rowsq, false, a_rounded);
        return;
    }
    dgemm_rowsumsq(c, ta, tb, M, N, K, A, dta, lda, B, dtb, ldb, rowsq);
}

void gemm_resid_sumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                      const void* B, int dtb, int64_t ldb, const void* D, int dtd, int64_t ldd, double* out) {
    dgemm_resid_sumsq(c, ta, tb, M, N, K, A, dta, lda, B, dtb, ldb, D, dtd, ldd, out);
}

}  // namespace ops
}  // namespace bcur_b200
