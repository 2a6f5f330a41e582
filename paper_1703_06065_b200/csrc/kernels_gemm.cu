// kernels_gemm.cu — register-tiled SIMT products with fp64 accumulation.
//
// Used for every fp64-input product (configs 1–2, the Grams/CGS2 panels and
// small factor products of all configs) and as the exact-arithmetic path for
// the skinny products of the range finder.  The wide fp32 A-passes of configs
// 3–5 go through the tcgen05 3×TF32 kernels in kernels_umma.cu.
//
// Epilogues: STORE (alpha·AB + beta·C, deterministic split-K), ROWSQ (per-row
// Σ_j (AB)_ij², product never stored — the fused ‖Q_Cᵀ A_g‖² of sketch.cpp:80 /
// blockcur.cpp:46), RESID (Σ (D − AB)², the explicit residual of blockcur.cpp:46).
#include "ops.h"

namespace bcur_b200 {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;
enum { EPI_STORE = 0, EPI_ROWSQ = 1, EPI_RESID = 2 };

template <class T>
__device__ __forceinline__ double ld_as_f64(const T* p) { return (double)__ldg(p); }

template <typename TA, typename TB, int TRA, int TRB, int EPI>
__global__ void __launch_bounds__(NT) k_gemm(int64_t M, int64_t N, int64_t K, int64_t kchunk, double alpha,
                                             const TA* __restrict__ A, int64_t lda, const TB* __restrict__ B,
                                             int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
                                             double* __restrict__ partial, const void* __restrict__ D, int dtd,
                                             int64_t ldd) {
    __shared__ double As[2][BK][BM];
    __shared__ double Bs[2][BK][BN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
    const int64_t kend = min(K, kbeg + kchunk);
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    double ra[4], rb[4];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            int i, kk;
            if (TRA == 0) { i = tid & 63; kk = (tid >> 6) + 4 * r; } else { kk = tid & 15; i = (tid >> 4) + 16 * r; }
            const int64_t gi = m0 + i, gk = k0 + kk;
            double v = 0.0;
            if (gi < M && gk < kend) v = TRA == 0 ? ld_as_f64(A + gi + gk * lda) : ld_as_f64(A + gk + gi * lda);
            ra[r] = v;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            int j, kk;
            if (TRB == 0) { kk = tid & 15; j = (tid >> 4) + 16 * r; } else { j = tid & 63; kk = (tid >> 6) + 4 * r; }
            const int64_t gj = n0 + j, gk = k0 + kk;
            double v = 0.0;
            if (gj < N && gk < kend) v = TRB == 0 ? ld_as_f64(B + gk + gj * ldb) : ld_as_f64(B + gj + gk * ldb);
            rb[r] = v;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            int i, kk;
            if (TRA == 0) { i = tid & 63; kk = (tid >> 6) + 4 * r; } else { kk = tid & 15; i = (tid >> 4) + 16 * r; }
            As[buf][kk][i] = ra[r];
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            int j, kk;
            if (TRB == 0) { kk = tid & 15; j = (tid >> 4) + 16 * r; } else { j = tid & 63; kk = (tid >> 6) + 4 * r; }
            Bs[buf][kk][j] = rb[r];
        }
    };

    int buf = 0;
    if (kbeg < kend) {
        load(kbeg);
        store(0);
        __syncthreads();
        for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
            const bool more = k0 + BK < kend;
            if (more) load(k0 + BK);
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                double a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
            }
            if (more) {
                store(buf ^ 1);
                __syncthreads();
                buf ^= 1;
            }
        }
    }

    if (EPI == EPI_STORE) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t gi = m0 + ty + 16 * i;
            if (gi >= M) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t gj = n0 + tx + 16 * j;
                if (gj >= N) continue;
                if (partial) {
                    partial[(int64_t)blockIdx.z * M * N + gi + gj * M] = acc[i][j];
                } else {
                    double* cp = C + gi + gj * ldc;
                    *cp = beta == 0.0 ? alpha * acc[i][j] : fma(beta, *cp, alpha * acc[i][j]);
                }
            }
        }
    } else if (EPI == EPI_ROWSQ) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j) s = fma(acc[i][j], acc[i][j], s);  // out-of-range cols are exact zeros
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const int64_t gi = m0 + ty + 16 * i;
            if (tx == 0 && gi < M) partial[(int64_t)blockIdx.y * M + gi] = s;
        }
    } else {  // EPI_RESID
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t gi = m0 + ty + 16 * i;
            if (gi >= M) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t gj = n0 + tx + 16 * j;
                if (gj >= N) continue;
                const double d = dtd == BCUR_F32 ? (double)((const float*)D)[gi + gj * ldd]
                                                 : ((const double*)D)[gi + gj * ldd];
                const double e = d - acc[i][j];
                s = fma(e, e, s);
            }
        }
        __shared__ double red[NT / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((tid & 31) == 0) red[tid >> 5] = s;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < NT / 32; ++w) t += red[w];
            partial[(int64_t)blockIdx.x + (int64_t)blockIdx.y * gridDim.x] = t;
        }
    }
}

// C = alpha·Σ_z partial[z] + beta·C  (fixed order ⇒ deterministic)
__global__ void k_splitk_reduce(int64_t M, int64_t N, int splits, const double* __restrict__ partial, double alpha,
                                double beta, double* __restrict__ C, int64_t ldc) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= M * N) return;
    const int64_t i = idx % M, j = idx / M;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * M * N + idx];
    double* cp = C + i + j * ldc;
    *cp = beta == 0.0 ? alpha * s : fma(beta, *cp, alpha * s);
}

__global__ void k_sum_rows_partials(int64_t M, int tiles, const double* __restrict__ partial, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    double s = 0.0;
    for (int t = 0; t < tiles; ++t) s += partial[(int64_t)t * M + i];
    out[i] = s;
}

template <typename TA, typename TB, int EPI>
void launch(Ctx* c, ops::Op ta, ops::Op tb, dim3 grid, int64_t M, int64_t N, int64_t K, int64_t kchunk, double alpha,
            const void* A, int64_t lda, const void* B, int64_t ldb, double beta, double* C, int64_t ldc,
            double* partial, const void* D, int dtd, int64_t ldd) {
#define BCUR_GEMM_CASE(TRA, TRB)                                                                              \
    k_gemm<TA, TB, TRA, TRB, EPI><<<grid, NT, 0, c->stream>>>(M, N, K, kchunk, alpha, (const TA*)A, lda,     \
                                                              (const TB*)B, ldb, beta, C, ldc, partial, D, dtd, \
                                                              ldd)
    if (ta == ops::OP_N && tb == ops::OP_N) BCUR_GEMM_CASE(0, 0);
    else if (ta == ops::OP_N && tb == ops::OP_T) BCUR_GEMM_CASE(0, 1);
    else if (ta == ops::OP_T && tb == ops::OP_N) BCUR_GEMM_CASE(1, 0);
    else BCUR_GEMM_CASE(1, 1);
#undef BCUR_GEMM_CASE
    LAUNCH_CHECK(c);
}

template <int EPI>
void dispatch(Ctx* c, ops::Op ta, ops::Op tb, dim3 grid, int64_t M, int64_t N, int64_t K, int64_t kchunk,
              double alpha, const void* A, int dta, int64_t lda, const void* B, int dtb, int64_t ldb, double beta,
              double* C, int64_t ldc, double* partial, const void* D, int dtd, int64_t ldd) {
    if (dta == BCUR_F32 && dtb == BCUR_F32)
        launch<float, float, EPI>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, partial, D, dtd, ldd);
    else if (dta == BCUR_F32)
        launch<float, double, EPI>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, partial, D, dtd, ldd);
    else if (dtb == BCUR_F32)
        launch<double, float, EPI>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, partial, D, dtd, ldd);
    else
        launch<double, double, EPI>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, partial, D, dtd, ldd);
}

}  // namespace

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
    // plain fp64 GEMMs of the small factorizations (Grams, Cholesky/inverse updates, factor
    // products) → cuBLAS DGEMM (DMMA tensor cores); deterministic for a fixed device.
    if (dta == BCUR_F64 && dtb == BCUR_F64 && K > 0 && (double)M * N * K >= 32768.0) {
        ProfScope prof(c, "dgemm_cublas", 2.0 * M * N * K, 8.0 * ((double)M * K + (double)K * N + (double)M * N));
        cublas_dgemm(c, ta == OP_T, tb == OP_T, M, N, K, alpha, (const double*)A, lda, (const double*)B, ldb, beta,
                     C, ldc);
        return;
    }
    ProfScope prof(c, (dta == BCUR_F32 || dtb == BCUR_F32) ? "gemm_store_f32" : "gemm_store_f64", 2.0 * M * N * K,
                   (double)M * K * dtype_size(dta) + (double)K * N * dtype_size(dtb) + 8.0 * M * N);
    if (K <= 0) {
        // C = beta·C
        if (beta == 0.0) {
            for (int64_t j = 0; j < N; ++j) CUDA_CHECK(cudaMemsetAsync(C + j * ldc, 0, M * sizeof(double), c->stream));
            return;
        }
        K = 0;
    }
    const int64_t mt = (M + BM - 1) / BM, nt = (N + BN - 1) / BN;
    const int64_t tiles = mt * nt;
    int splits = 1;
    const int64_t target = 2LL * c->sm_count;
    if (tiles < target && K >= 4 * BK) {
        splits = (int)std::min<int64_t>((target + tiles - 1) / tiles, std::max<int64_t>(1, K / (8 * BK)));
        splits = std::min(splits, 256);
    }
    int64_t kchunk = (K + splits - 1) / splits;
    kchunk = (kchunk + BK - 1) / BK * BK;
    if (kchunk <= 0) kchunk = BK;
    splits = (int)((K + kchunk - 1) / kchunk);
    if (splits < 1) splits = 1;
    dim3 grid((unsigned)mt, (unsigned)nt, (unsigned)splits);
    if (splits == 1) {
        dispatch<EPI_STORE>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, dta, lda, B, dtb, ldb, beta, C, ldc, nullptr,
                            nullptr, 0, 0);
    } else {
        DevBuf part(c, (size_t)splits * M * N * sizeof(double));
        dispatch<EPI_STORE>(c, ta, tb, grid, M, N, K, kchunk, 1.0, A, dta, lda, B, dtb, ldb, 0.0, nullptr, 0,
                            part.as<double>(), nullptr, 0, 0);
        const int64_t total = M * N;
        k_splitk_reduce<<<(unsigned)((total + 255) / 256), 256, 0, c->stream>>>(M, N, splits, part.as<double>(), alpha,
                                                                                beta, C, ldc);
        LAUNCH_CHECK(c);
    }
}

void gemm_rowsumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                   const void* B, int dtb, int64_t ldb, double* rowsq, bool a_rounded) {
    if (M <= 0) return;
    if (ta == OP_T && tb == OP_N && dta == BCUR_F32 && N > 0 && K > 0 && umma_ok(dta, K, lda, A)) {
        umma_atx(c, (const float*)A, K, M, lda, B, dtb, N, ldb, 1.0, 0.0, nullptr, 0, rowsq, false, a_rounded);
        return;
    }
    ProfScope prof(c, (dta == BCUR_F32 || dtb == BCUR_F32) ? "gemm_rowsumsq_f32" : "gemm_rowsumsq_f64",
                   2.0 * M * N * K, (double)M * K * dtype_size(dta) + (double)K * N * dtype_size(dtb) + 8.0 * M);
    if (N <= 0) {
        CUDA_CHECK(cudaMemsetAsync(rowsq, 0, M * sizeof(double), c->stream));
        return;
    }
    const int64_t mt = (M + BM - 1) / BM, nt = (N + BN - 1) / BN;
    DevBuf part(c, (size_t)nt * M * sizeof(double));
    dim3 grid((unsigned)mt, (unsigned)nt, 1);
    dispatch<EPI_ROWSQ>(c, ta, tb, grid, M, N, K, std::max<int64_t>(K, 1), 1.0, A, dta, lda, B, dtb, ldb, 0.0,
                        nullptr, 0, part.as<double>(), nullptr, 0, 0);
    k_sum_rows_partials<<<(unsigned)((M + 255) / 256), 256, 0, c->stream>>>(M, (int)nt, part.as<double>(), rowsq);
    LAUNCH_CHECK(c);
}

void gemm_resid_sumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                      const void* B, int dtb, int64_t ldb, const void* D, int dtd, int64_t ldd, double* out) {
    ProfScope prof(c, "gemm_resid", 2.0 * M * N * K,
                   (double)M * K * dtype_size(dta) + (double)K * N * dtype_size(dtb) + (double)M * N * dtype_size(dtd));
    const int64_t mt = (M + BM - 1) / BM, nt = (N + BN - 1) / BN;
    DevBuf part(c, (size_t)mt * nt * sizeof(double));
    dim3 grid((unsigned)mt, (unsigned)nt, 1);
    dispatch<EPI_RESID>(c, ta, tb, grid, M, N, K, std::max<int64_t>(K, 1), 1.0, A, dta, lda, B, dtb, ldb, 0.0,
                        nullptr, 0, part.as<double>(), D, dtd, ldd);
    sum_vector(c, part.as<double>(), mt * nt, out);
}

}  // namespace ops
}  // namespace bcur_b200
