// kernels_dmma.cu — fp64 products on the tensor cores (DMMA, mma.sync m8n8k4 .f64) and
// the fused single-CTA Cholesky + triangular inverse that the recursive factorization
// (pipeline.cu chol_inv) uses as its leaf.
//
// k_dgemm: C = alpha·op(A)·op(B) + beta·C with fp64 accumulation, every operand converted
// to fp64 on its way into shared memory (fp32 or fp64 inputs).  It serves every product that
// is not an fp32 A-pass: the fp64 configs' sketch (Y = AΩ, B = QᵀA — the reference's
// BDCSVD/GEMMs, matcore.cpp:39-56, blockcur.cpp:46), Grams, CholQR2 panels, the recursive
// Cholesky's updates, U assembly.  Epilogues:
//   STORE  alpha·AB + beta·C (split-K partials reduced in a fixed order: deterministic)
//   ROWSQ  rowsq[i] = Σ_j (AB)_ij² without storing the product (‖Q_Cᵀ A_g‖², sketch.cpp:80)
//   RESID  Σ (D − AB)² (the explicit residual ‖A − C(UR)‖_F², blockcur.cpp:46)
// Structure flags shrink each tile's K range (triangular operands) or skip tiles (a product
// known to be symmetric, of which only the upper triangle is consumed).
//
// CTA tile 64×64×16, 4 warps as 2×2, each warp 32×32 = 4×4 DMMA tiles; a 4-stage cp.async
// pipeline (3 k-tiles in flight: the latency-bound small products of the factorizations and
// orthonormalizations wait on L2 once, not once per k-tile); conflict-free fragment pitches
// (DTile).
#include "ops.h"

namespace bcur_b200 {
namespace {

constexpr int DBM = 64, DBN = 64, DBK = 16, DNT = 128;
enum { DEPI_STORE = 0, DEPI_ROWSQ = 1, DEPI_RESID = 2 };

template <class T>
__device__ __forceinline__ double ldg64(const T* p) { return (double)__ldg(p); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Shared-memory tiles keep each operand's stored contiguous direction (so cp.async copies
// elements straight from global memory): op(A) is [k][m] when A is column-major (TRA = 0) and
// [m][k] when transposed; op(B) is [n][k] when B is K-major (TRB = 0) and [k][n] otherwise.
// Pitches make the DMMA fragment loads conflict-free: [·][k] rows hold 16 k + 4 pad (20 ≡ 4 mod
// 16 doubles / ≡ 20 mod 32 floats), [k][·] rows 64 + 4 doubles or 64 + 8 floats.
// ROWS: the tile's extent along M (64) or N (the kernel's NB: 64, or 16 for thin outputs — an
// N = 15 sketch product on a 64-wide tile spent three quarters of its DMMAs on zero columns,
// and the DMMA pipe, one m8n8k4 per 4 clocks per SM, was what bound it: profiles/r02ae)
template <typename T, bool KMAJOR, int ROWS = 64>
struct DTile {
    static constexpr int P = KMAJOR ? (DBK + 4) : (ROWS + (sizeof(T) == 8 ? 4 : 8));
    static constexpr int ELEMS = KMAJOR ? ROWS * P : DBK * P;
};
constexpr int DSTAGES = 4;

__device__ __forceinline__ void cp_async_elem(void* smem, const void* gmem, int bytes, bool valid) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    const int src = valid ? bytes : 0;  // src-size 0: the destination is zero-filled
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(gmem), "r"(src) : "memory");
}

template <typename TA, typename TB, int TRA, int TRB, int EPI, int NB = DBN>
__global__ void __launch_bounds__(DNT) k_dgemm(int64_t M, int64_t N, int64_t K, int64_t kchunk, double alpha,
                                               const TA* __restrict__ A, int64_t lda, const TB* __restrict__ B,
                                               int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
                                               double* __restrict__ partial, const void* __restrict__ D, int dtd,
                                               int64_t ldd, int flags) {
    using TLA = DTile<TA, TRA == 1>;
    using TLB = DTile<TB, TRB == 0, NB>;
    // warps: 2 × 2 of 32 × 32 (NB = 64) or 4 × 1 of 16 × 16 (NB = 16)
    constexpr int WN = NB == 64 ? 2 : 1, WM = 4 / WN, MI = DBM / WM / 8, NJ = NB / WN / 8;
    extern __shared__ __align__(16) unsigned char dsm[];
    TA* As = reinterpret_cast<TA*>(dsm);
    TB* Bs = reinterpret_cast<TB*>(dsm + (size_t)DSTAGES * TLA::ELEMS * sizeof(TA));
    __shared__ double red[2][DBM];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % WM, wn = warp / WM;
    // triangular operands: the tiles with the longest K range are scheduled first (the block
    // scheduler dispatches in blockIdx order; the last wave should hold the short tiles)
    const int64_t bx = (flags & ops::GEMM_A_LOWER) ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
    const int64_t by = (flags & ops::GEMM_B_UPPER) ? gridDim.y - 1 - blockIdx.y : blockIdx.y;
    const int64_t m0 = bx * DBM, n0 = by * NB;
    const bool split = partial != nullptr && EPI == DEPI_STORE;
    // a symmetric product of which only the upper triangle is consumed: tiles strictly
    // below the diagonal are not computed (zeros into their split-K partials)
    const bool skip = (flags & ops::GEMM_SYM_UPPER) && m0 >= n0 + NB;
    if (skip && !split) return;
    int64_t kbeg = (int64_t)blockIdx.z * kchunk, kend = min(K, kbeg + kchunk);
    if (flags & ops::GEMM_A_UPPER) kbeg = max(kbeg, m0 / DBK * DBK);   // op(A)[i,k] = 0 for k < i
    if (flags & ops::GEMM_A_LOWER) kend = min(kend, m0 + DBM);         // op(A)[i,k] = 0 for k > i
    if (flags & ops::GEMM_B_UPPER) kend = min(kend, n0 + NB);         // op(B)[k,j] = 0 for k > j
    if (flags & ops::GEMM_B_LOWER) kbeg = max(kbeg, n0 / DBK * DBK);   // op(B)[k,j] = 0 for k < j
    if (skip) kend = kbeg;

    double acc[MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // one stage: op(A) (DBM × DBK) and op(B) (DBK × DBN), 1024 elements each = 8 cp.async per
    // thread and operand, the thread map following the stored contiguous direction (coalesced)
    auto issue = [&](int st, int64_t k0) {
        TA* as = As + st * TLA::ELEMS;
        TB* bs = Bs + st * TLB::ELEMS;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int i, kk;
            if (TRA == 0) { i = tid & 63; kk = (tid >> 6) + 2 * r; } else { kk = tid & 15; i = (tid >> 4) + 8 * r; }
            const int64_t gi = m0 + i, gk = k0 + kk;
            const bool v = gi < M && gk < kend;
            const TA* src = A + (v ? (TRA == 0 ? gi + gk * lda : gk + gi * lda) : 0);
            cp_async_elem(TRA == 0 ? as + kk * TLA::P + i : as + i * TLA::P + kk, src, (int)sizeof(TA), v);
        }
#pragma unroll
        for (int r = 0; r < NB / 8; ++r) {
            int j, kk;
            if (TRB == 0) { kk = tid & 15; j = (tid >> 4) + 8 * r; } else { j = tid & (NB - 1); kk = tid / NB + (DNT / NB) * r; }
            const int64_t gj = n0 + j, gk = k0 + kk;
            const bool v = gj < N && gk < kend;
            const TB* src = B + (v ? (TRB == 0 ? gk + gj * ldb : gj + gk * ldb) : 0);
            cp_async_elem(TRB == 0 ? bs + j * TLB::P + kk : bs + kk * TLB::P + j, src, (int)sizeof(TB), v);
        }
    };

    if (kbeg < kend) {
        const int nk = (int)((kend - kbeg + DBK - 1) / DBK);
#pragma unroll
        for (int st = 0; st < DSTAGES - 1; ++st) {  // prologue: DSTAGES−1 stages in flight
            if (st < nk) issue(st, kbeg + (int64_t)st * DBK);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        const int fk = lane & 3, fm = lane >> 2;
        for (int kt = 0; kt < nk; ++kt) {
            asm volatile("cp.async.wait_group %0;" ::"n"(DSTAGES - 2) : "memory");
            __syncthreads();  // stage kt landed for every thread; stage kt−1 is free again
            if (kt + DSTAGES - 1 < nk) issue((kt + DSTAGES - 1) % DSTAGES, kbeg + (int64_t)(kt + DSTAGES - 1) * DBK);
            asm volatile("cp.async.commit_group;" ::: "memory");
            const TA* as = As + (kt % DSTAGES) * TLA::ELEMS;
            const TB* bs = Bs + (kt % DSTAGES) * TLB::ELEMS;
#pragma unroll
            for (int k4 = 0; k4 < DBK; k4 += 4) {
                double af[MI], bf[NJ];
#pragma unroll
                for (int i = 0; i < MI; ++i) {
                    const int mm = wm * (MI * 8) + i * 8 + fm;
                    af[i] = (double)(TRA == 0 ? as[(k4 + fk) * TLA::P + mm] : as[mm * TLA::P + k4 + fk]);
                }
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    const int nn = wn * (NJ * 8) + j * 8 + fm;
                    bf[j] = (double)(TRB == 0 ? bs[nn * TLB::P + k4 + fk] : bs[(k4 + fk) * TLB::P + nn]);
                }
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }

    // accumulator fragment: row = lane>>2, columns 2·(lane&3) + {0,1} of each 8×8 tile
    const int er = lane >> 2, ec = 2 * (lane & 3);
    if (EPI == DEPI_STORE) {
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            const int64_t gi = m0 + wm * (MI * 8) + i * 8 + er;
            if (gi >= M) continue;
#pragma unroll
            for (int j = 0; j < NJ; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t gj = n0 + wn * (NJ * 8) + j * 8 + ec + h;
                    if (gj >= N) continue;
                    if (split) {
                        partial[(int64_t)blockIdx.z * M * N + gi + gj * M] = acc[i][j][h];
                    } else {
                        double* cp = C + gi + gj * ldc;
                        *cp = beta == 0.0 ? alpha * acc[i][j][h] : fma(beta, *cp, alpha * acc[i][j][h]);
                    }
                }
        }
    } else if (EPI == DEPI_ROWSQ) {
        // out-of-range columns hold exact zeros (zero-filled operands)
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NJ; ++j) s = fma(acc[i][j][0], acc[i][j][0], fma(acc[i][j][1], acc[i][j][1], s));
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            if ((lane & 3) == 0) red[wn][wm * (MI * 8) + i * 8 + er] = s;
        }
        __syncthreads();
        for (int i = tid; i < DBM; i += DNT) {
            const int64_t gi = m0 + i;
            if (gi < M) partial[(int64_t)blockIdx.y * M + gi] = WN == 2 ? red[0][i] + red[1][i] : red[0][i];
        }
    } else {  // DEPI_RESID
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            const int64_t gi = m0 + wm * (MI * 8) + i * 8 + er;
            if (gi >= M) continue;
#pragma unroll
            for (int j = 0; j < NJ; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t gj = n0 + wn * (NJ * 8) + j * 8 + ec + h;
                    if (gj >= N) continue;
                    const double d = dtd == BCUR_F32 ? (double)((const float*)D)[gi + gj * ldd]
                                                     : ((const double*)D)[gi + gj * ldd];
                    const double e = d - acc[i][j][h];
                    s = fma(e, e, s);
                }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[0][warp] = s;
        __syncthreads();
        if (tid == 0)
            partial[(int64_t)blockIdx.x + (int64_t)blockIdx.y * gridDim.x] = (red[0][0] + red[0][1]) + (red[0][2] + red[0][3]);
    }
}

// C = alpha·Σ_z partial[z] + beta·C  (fixed order ⇒ deterministic)
__global__ void k_dsplitk_reduce(int64_t M, int64_t N, int splits, const double* __restrict__ partial, double alpha,
                                 double beta, double* __restrict__ C, int64_t ldc, int sym_upper) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= M * N) return;
    const int64_t i = idx % M, j = idx / M;
    if (sym_upper && i / DBM >= j / DBN + 1) return;  // tiles the product skipped
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * M * N + idx];
    double* cp = C + i + j * ldc;
    *cp = beta == 0.0 ? alpha * s : fma(beta, *cp, alpha * s);
}

// the same with many splits (thin Grams: 60 × 60 over K = 16384): one warp per element, lanes
// over the splits, a fixed shuffle tree (deterministic)
__global__ void k_dsplitk_reduce_warp(int64_t M, int64_t N, int splits, const double* __restrict__ partial,
                                      double alpha, double beta, double* __restrict__ C, int64_t ldc, int sym_upper) {
    const int64_t idx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (idx >= M * N) return;
    const int64_t i = idx % M, j = idx / M;
    if (sym_upper && i / DBM >= j / DBN + 1) return;
    double s = 0.0;
    for (int z = lane; z < splits; z += 32) s += partial[(int64_t)z * M * N + idx];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        double* cp = C + i + j * ldc;
        *cp = beta == 0.0 ? alpha * s : fma(beta, *cp, alpha * s);
    }
}

__global__ void k_dsum_rows(int64_t M, int tiles, const double* __restrict__ partial, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    double s = 0.0;
    for (int t = 0; t < tiles; ++t) s += partial[(int64_t)t * M + i];
    out[i] = s;
}

template <typename TA, typename TB, int TRA, int TRB, int NB>
size_t dgemm_smem() {
    return (size_t)DSTAGES * (DTile<TA, TRA == 1>::ELEMS * sizeof(TA) + DTile<TB, TRB == 0, NB>::ELEMS * sizeof(TB));
}

template <typename TA, typename TB, int EPI, int NB = DBN>
void dlaunch(Ctx* c, ops::Op ta, ops::Op tb, dim3 grid, int64_t M, int64_t N, int64_t K, int64_t kchunk, double alpha,
             const void* A, int64_t lda, const void* B, int64_t ldb, double beta, double* C, int64_t ldc,
             double* partial, const void* D, int dtd, int64_t ldd, int flags) {
#define BCUR_DGEMM_CASE(TRA, TRB)                                                                                  \
    do {                                                                                                           \
        static bool attr = false;                                                                                  \
        const size_t sm = dgemm_smem<TA, TB, TRA, TRB, NB>();                                                      \
        if (!attr) {                                                                                               \
            CUDA_CHECK(cudaFuncSetAttribute(k_dgemm<TA, TB, TRA, TRB, EPI, NB>,                                    \
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));                \
            attr = true;                                                                                           \
        }                                                                                                          \
        k_dgemm<TA, TB, TRA, TRB, EPI, NB><<<grid, DNT, sm, c->stream>>>(                                          \
            M, N, K, kchunk, alpha, (const TA*)A, lda, (const TB*)B, ldb, beta, C, ldc, partial, D, dtd, ldd, flags); \
    } while (0)
    if (ta == ops::OP_N && tb == ops::OP_N) BCUR_DGEMM_CASE(0, 0);
    else if (ta == ops::OP_N && tb == ops::OP_T) BCUR_DGEMM_CASE(0, 1);
    else if (ta == ops::OP_T && tb == ops::OP_N) BCUR_DGEMM_CASE(1, 0);
    else BCUR_DGEMM_CASE(1, 1);
#undef BCUR_DGEMM_CASE
    LAUNCH_CHECK(c);
}

template <int EPI, int NB = DBN>
void ddispatch(Ctx* c, ops::Op ta, ops::Op tb, dim3 grid, int64_t M, int64_t N, int64_t K, int64_t kchunk,
               double alpha, const void* A, int dta, int64_t lda, const void* B, int dtb, int64_t ldb, double beta,
               double* C, int64_t ldc, double* partial, const void* D, int dtd, int64_t ldd, int flags) {
    if (dta == BCUR_F32 && dtb == BCUR_F32)
        dlaunch<float, float, EPI, NB>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, partial, D,
                                   dtd, ldd, flags);
    else if (dta == BCUR_F32)
        dlaunch<float, double, EPI, NB>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, partial, D,
                                    dtd, ldd, flags);
    else if (dtb == BCUR_F32)
        dlaunch<double, float, EPI, NB>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, partial, D,
                                    dtd, ldd, flags);
    else
        dlaunch<double, double, EPI, NB>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, partial,
                                     D, dtd, ldd, flags);
}

// ------------------------------------------- fused Cholesky + inverse (w ≤ 128)
// G (upper triangle read) → R upper with G = RᵀR and X = R⁻¹, one CTA of 256 threads.
// Factor: right-looking 32-column panels on the lower triangle L = Rᵀ held in shared memory
// (warp 0 factors the 32×32 diagonal block in registers, one thread per row solves the panel,
// all warps apply the rank-32 update).  Inverse, in the free upper triangle of the same
// array: the diagonal 32-blocks X_bb by one warp each (lane = column, back substitution in
// registers), then the off-diagonal blocks by superdiagonal, X_ij = −X_ii·Σ_{i<l≤j} R_il·X_lj.
// Status: chained (part of a recursive factorization) — skip when *info != 0 on entry,
// failures report info_offset + j + 1, diag[0] = running min diag(R).
// Pitches ≡ 4 (mod 16) doubles: a DMMA fragment (8 rows × 4 consecutive k, or 8 columns × 4
// k) then hits 16 distinct 8-byte bank pairs per half-warp — with an odd pitch it was 4-way
// conflicted and the leaf's DMMA phases ran at the shared-memory wavefront rate
constexpr int LF_T = 256, LF_MAX = 128, LF_LD = LF_MAX + 4, LF_TP = 36;
// chol_inv_leaf flags (ops.h).  QUIET: no timing print.  SYM: g holds the full symmetric block
// (both triangles) with 16-byte aligned columns and w == 128 — it is then copied column by column
// (M's lower triangle is g's) with cp.async instead of the transposing load
enum { LEAF_NO_R = 1, LEAF_ZEROED = 2, LEAF_QUIET = 4, LEAF_SYM = 8 };
__device__ int g_leaf_timing = 0;  // BCUR_LEAF_TIMING=1: thread 0 prints the phase clocks (diagnostics)
#define LF_CLK(i) do { if (timing && threadIdx.x == 0) clk[i] = clock64(); } while (0)

__device__ __forceinline__ double lf_rsqrt(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double hx = 0.5 * x;
    r = r * fma(-hx * r, r, 1.5);
    r = r * fma(-hx * r, r, 1.5);
    return r;
}

// The leaf as a device function of 256 threads (k_chol_inv_leaf, and the FACT step of the
// persistent factorization k_chol_persistent); smlf: LF_SMEM bytes of dynamic shared memory.
// g is read through L2 (ld.global.cg): inside the persistent kernel other CTAs wrote it.
__device__ __forceinline__ void chol_leaf_dev(double* smlf, const double* __restrict__ g, int w, int64_t ldg,
                                              double* __restrict__ r, int64_t ldr, double* __restrict__ x,
                                              int64_t ldx, int* info, double* diag, int info_offset, int flags) {
    double* M = smlf;                       // M[i + k·LD]: i ≥ k → L = Rᵀ; i < k → X[i][k]
    double* Tb = smlf + LF_MAX * LF_LD;     // 3 × 32 × LF_TP temporaries of the inverse
    double* Xd = Tb + 3 * 32 * LF_TP;       // 4 × 32 × LF_TP: the diagonal blocks of X as full squares
    __shared__ double invd[LF_MAX];
    __shared__ double xch[32];
    __shared__ int stop_sh;
    __shared__ double mn_sh;
    if (*(volatile int*)info != 0) return;
    const int timing = g_leaf_timing && !(flags & LEAF_QUIET);
    long long clk[16] = {0};
    LF_CLK(0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wp = (w + 31) & ~31;
    // the (padded) square in 8-deep batches of independent loads (a loop over one column at
    // a time left each warp with ~40 dependent L2 round trips)
    // the padded wp × wp square in 8-row × 4-column lane tiles (lane → row 8·ib + lane/4, column
    // 4·kb + lane%4): the shared-memory side of both the load and the final store is then
    // conflict-free at the 4-mod-16 pitch; batches of 16 independent global loads
    const int nib = wp >> 3, total = wp * wp;
    auto tile_ik = [&](int e, int& i, int& k) {
        const int blk = e >> 5, ln = e & 31;
        i = (blk % nib) * 8 + (ln >> 2);
        k = (blk / nib) * 4 + (ln & 3);
    };
    const bool sym_load = (flags & LEAF_SYM) && w == LF_MAX && (ldg % 2) == 0 && ((uintptr_t)g % 16) == 0;
    if (sym_load) {  // 128 columns × 64 16-byte pairs, through L2 (other CTAs wrote g)
        for (int e = tid; e < LF_MAX * (LF_MAX / 2); e += LF_T) {
            const int c = e >> 6, r = 2 * (e & 63);
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(M + r + c * LF_LD);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g + r + (int64_t)c * ldg) : "memory");
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    }
    for (int q0 = 0; !sym_load && q0 * LF_T < total; q0 += 16) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {  // addresses clamped, no branches
            int i, k;
            tile_ik(min((q0 + q) * LF_T + tid, total - 1), i, k);
            v[q] = __ldcg(g + min(i, w - 1) + (int64_t)min(k, w - 1) * ldg);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int e = (q0 + q) * LF_T + tid;
            int i, k;
            tile_ik(e, i, k);
            if (e < total && i <= k) M[k + i * LF_LD] = (i < w && k < w) ? v[q] : (i == k ? 1.0 : 0.0);
        }
    }
    if (tid == 0) {
        stop_sh = 0;
        mn_sh = INFINITY;
    }
    __syncthreads();
    LF_CLK(1);
    for (int c0 = 0; c0 < wp; c0 += 32) {
        if (warp == 0) {
            double a[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) a[k] = M[(c0 + lane) + (c0 + k) * LF_LD];
            // The next pivot is formed by its own lane (a[j+1] − l²) and shuffled right away, so
            // the pivot chain is shuffle → rsqrt → multiply → FMA → shuffle, without the
            // shared-memory exchange (which only feeds the rest of the row updates).  A failed
            // pivot is recorded, not branched on: the NaNs it spreads are never stored.
            int bad = 0;
            double mn = INFINITY, dl = 1.0;
            double dcur = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const double d = dcur;
                if (bad == 0 && (!(d > 0.0) || !isfinite(d))) bad = c0 + j + 1;
                const double ri = lf_rsqrt(d), rj = d * ri;
                if (c0 + j < w) mn = fmin(mn, rj);
                if (lane == j) dl = ri;
                const double lij = a[j] * ri;
                a[j] = lane == j ? rj : lij;
                if (j + 1 < 32) dcur = __shfl_sync(0xffffffffu, fma(-lij, lij, a[j + 1]), j + 1);
                xch[lane] = lij;
                __syncwarp();
#pragma unroll
                for (int k = j + 1; k < 32; ++k) a[k] = fma(-lij, xch[k], a[k]);
                __syncwarp();
            }
            if (!bad) {
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    if (k <= lane) M[(c0 + lane) + (c0 + k) * LF_LD] = a[k];
                invd[c0 + lane] = dl;
            }
            if (lane == 0) {
                if (bad) stop_sh = bad;
                mn_sh = fmin(mn_sh, mn);
            }
        }
        __syncthreads();
        if (c0 == 0) LF_CLK(2);
        if (stop_sh) break;
        const int base = c0 + 32, nr = wp - base;
        if (nr <= 0) break;
        if (tid < nr) {  // panel solve, right-looking (2 dependent ops per column)
            const int i = base + tid;
            double xr[32];
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) xr[cc] = M[i + (c0 + cc) * LF_LD];
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
                xr[cc] *= invd[c0 + cc];
#pragma unroll
                for (int c2 = cc + 1; c2 < 32; ++c2) xr[c2] = fma(-xr[cc], M[(c0 + c2) + (c0 + cc) * LF_LD], xr[c2]);
            }
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) M[i + (c0 + cc) * LF_LD] = xr[cc];
        }
        __syncthreads();
        if (c0 == 0) LF_CLK(3);
        {   // trailing lower triangle −= P·Pᵀ (P = the solved panel, nr × 32) on DMMA: 8×8 tiles
            // on or below the diagonal, round-robin over the warps, fragments from shared memory
            const int t8 = nr >> 3, ntiles = t8 * (t8 + 1) / 2;
            const int fr = lane >> 2, fk = lane & 3;
            for (int t = warp; t < ntiles; t += LF_T / 32) {
                int ti = 0;
                while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
                const int tk = t - ti * (ti + 1) / 2;  // tk ≤ ti
                const int ra = base + ti * 8 + fr, rb = base + tk * 8 + fr;
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int k4 = 0; k4 < 32; k4 += 4) {
                    const int kc = (c0 + k4 + fk) * LF_LD;
                    dmma(d0, d1, M[ra + kc], M[rb + kc]);
                }
                const int row = base + ti * 8 + fr, col = base + tk * 8 + 2 * fk;
                if (col <= row) M[row + col * LF_LD] -= d0;
                if (col + 1 <= row) M[row + (col + 1) * LF_LD] -= d1;
            }
        }
        __syncthreads();
    }
    LF_CLK(4);
    const int stop = stop_sh;
    if (!stop) {
        const int nb = wp / 32;
        // (a) diagonal blocks: warp b solves R_bb·x = e_c for lane c (back substitution)
        if (warp < nb) {
            const int b0 = warp * 32;
            double xv[32];
#pragma unroll
            for (int t = 0; t < 32; ++t) xv[t] = t == lane ? 1.0 : 0.0;
#pragma unroll
            for (int t = 31; t >= 0; --t) {
                xv[t] *= invd[b0 + t];
#pragma unroll
                for (int i = 0; i < t; ++i) xv[i] = fma(-M[(b0 + t) + (b0 + i) * LF_LD], xv[t], xv[i]);  // R[i][t]
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (i < lane) M[(b0 + i) + (b0 + lane) * LF_LD] = xv[i];
                // full square copy (zeros below, the diagonal): the DMMA operand of (b)
                Xd[warp * 32 * LF_TP + i * LF_TP + lane] = i < lane ? xv[i] : (i == lane ? invd[b0 + lane] : 0.0);
            }
        }
        __syncthreads();
        LF_CLK(5);
        // (b) off-diagonal blocks, superdiagonal by superdiagonal, on DMMA (8×8 output tiles,
        // 16 per 32×32 block, round-robin over the warps):
        //   T_ij = Σ_{i<l≤j} R_il·X_lj   (K = 32·d),   X_ij = −X_ii·T_ij   (K = 32)
        const int fr = lane >> 2, fk = lane & 3;
        constexpr int NW8 = LF_T / 32;
        for (int d = 1; d < nb; ++d) {
            const int nblk = nb - d, ntl = nblk * 16;
            // two independent tiles per warp and pass (the K loops are equally long: 32·d)
            for (int t0 = warp; t0 < ntl; t0 += 2 * NW8) {
                const int t1 = t0 + NW8 < ntl ? t0 + NW8 : t0;
                int gr[2], gc[2], i0[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int t = u ? t1 : t0, bi = t >> 4, tr = (t >> 2) & 3, tc = t & 3;
                    i0[u] = bi * 32;
                    gr[u] = i0[u] + tr * 8 + fr;
                    gc[u] = (bi + d) * 32 + tc * 8 + fr;
                }
                double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
                for (int k4 = 32; k4 < 32 * (d + 1); k4 += 4) {
                    const bool diag_blk = k4 >= 32 * d;  // rows of X_jj (warp-uniform)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int tk = i0[u] + k4 + fk;
                        const double av = M[tk + gr[u] * LF_LD];  // R[gr][tk]
                        const int j0 = i0[u] + 32 * d;
                        const double bv = diag_blk ? Xd[(j0 >> 5) * 32 * LF_TP + (tk - j0) * LF_TP + (gc[u] - j0)]
                                                   : M[tk + gc[u] * LF_LD];  // X[tk][gc]
                        dmma(acc[u][0], acc[u][1], av, bv);
                    }
                }
#pragma unroll
                for (int u = 0; u < (t1 != t0 ? 2 : 1); ++u) {
                    const int t = u ? t1 : t0, bi = t >> 4, tr = (t >> 2) & 3, tc = t & 3;
                    double* T = Tb + bi * 32 * LF_TP;
                    T[(tr * 8 + fr) * LF_TP + tc * 8 + 2 * fk] = acc[u][0];
                    T[(tr * 8 + fr) * LF_TP + tc * 8 + 2 * fk + 1] = acc[u][1];
                }
            }
            __syncthreads();
            for (int t0 = warp; t0 < ntl; t0 += 2 * NW8) {
                const int t1 = t0 + NW8 < ntl ? t0 + NW8 : t0;
                double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                for (int k4 = 0; k4 < 32; k4 += 4) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int t = u ? t1 : t0, bi = t >> 4, tr = (t >> 2) & 3, tc = t & 3;
                        const int ii = bi * 32, r_ = tr * 8 + fr, uu = k4 + fk;
                        const double av = Xd[bi * 32 * LF_TP + r_ * LF_TP + uu];  // X_ii[r_][uu]
                        const double bv = Tb[bi * 32 * LF_TP + uu * LF_TP + tc * 8 + fr];
                        dmma(acc[u][0], acc[u][1], av, bv);
                    }
                }
#pragma unroll
                for (int u = 0; u < (t1 != t0 ? 2 : 1); ++u) {
                    const int t = u ? t1 : t0, bi = t >> 4, tr = (t >> 2) & 3, tc = t & 3;
                    const int ii = bi * 32, jj = (bi + d) * 32, r_ = tr * 8 + fr, cc = tc * 8 + 2 * fk;
                    M[(ii + r_) + (jj + cc) * LF_LD] = -acc[u][0];
                    M[(ii + r_) + (jj + cc + 1) * LF_LD] = -acc[u][1];
                }
            }
            __syncthreads();
        }
    }
    LF_CLK(6);
    // X (and R unless LEAF_NO_R): with LEAF_ZEROED the lower triangles are already zero (the
    // recursion memsets R and X), so only the upper triangles are written — X by 16-byte stores,
    // one column per warp, consecutive row pairs per lane (a 512-byte run per warp and column)
    const bool zeroed = (flags & LEAF_ZEROED) != 0, want_r = !(flags & LEAF_NO_R);
    if (zeroed && !stop && ((uintptr_t)x % 16) == 0 && (ldx % 2) == 0) {
        for (int k = warp; k < w; k += LF_T / 32) {
            for (int p = lane; 2 * p <= k; p += 32) {
                const int i = 2 * p;
                const double v0 = i < k ? M[i + k * LF_LD] : invd[k];
                const double v1 = i + 1 < k ? M[i + 1 + k * LF_LD] : (i + 1 == k ? invd[k] : 0.0);
                if (i + 1 < w) *reinterpret_cast<double2*>(x + i + (int64_t)k * ldx) = make_double2(v0, v1);
                else x[i + (int64_t)k * ldx] = v0;
            }
        }
        if (want_r) {
#pragma unroll 4
            for (int q = 0; q * LF_T < total; ++q) {
                const int e = q * LF_T + tid;
                int i, k;
                tile_ik(e, i, k);
                if (e < total && i <= k && k < w) r[i + (int64_t)k * ldr] = M[k + i * LF_LD];
            }
        }
    } else {
#pragma unroll 4
        for (int q = 0; q * LF_T < total; ++q) {
            const int e = q * LF_T + tid;
            int i, k;
            tile_ik(e, i, k);
            if (e < total && i < w && k < w && !(zeroed && i > k)) {
                x[i + (int64_t)k * ldx] = stop ? 0.0 : (i < k ? M[i + k * LF_LD] : (i == k ? invd[i] : 0.0));
                if (want_r) r[i + (int64_t)k * ldr] = i <= k && !stop ? M[k + i * LF_LD] : 0.0;
            }
        }
    }
    LF_CLK(7);
    if (tid == 0) {
        if (stop) *info = info_offset + stop;
        diag[0] = stop ? 0.0 : fmin(diag[0], mn_sh);
    }
    if (timing && tid == 0)
        printf("leaf w=%d clocks: load %lld | panel0 diag %lld | panel0 trsm %lld | panels rest %lld | inv diag %lld | "
               "inv offdiag %lld | store %lld | total %lld\n", w, clk[1] - clk[0], clk[2] - clk[1], clk[3] - clk[2],
               clk[4] - clk[3], clk[5] - clk[4], clk[6] - clk[5], clk[7] - clk[6], clk[7] - clk[0]);
}
constexpr size_t LF_SMEM = (size_t)(LF_MAX * LF_LD + 7 * 32 * LF_TP) * sizeof(double);
// the leaf as a call of its own (register allocation independent of the caller: inlined into
// the persistent kernel it shared that kernel's budget, spilled, and ran at half speed)
__device__ __noinline__ void chol_leaf_call(double* smlf, const double* g, int w, int64_t ldg, double* r, int64_t ldr,
                                            double* x, int64_t ldx, int* info, double* diag, int info_offset, int flags) {
    chol_leaf_dev(smlf, g, w, ldg, r, ldr, x, ldx, info, diag, info_offset, flags);
}

__global__ void __launch_bounds__(LF_T) k_chol_inv_leaf(const double* __restrict__ g, int w, int64_t ldg,
                                                        double* __restrict__ r, int64_t ldr, double* __restrict__ x,
                                                        int64_t ldx, int* info, double* diag, int info_offset,
                                                        int flags) {
    extern __shared__ double smlf[];
    chol_leaf_dev(smlf, g, w, ldg, r, ldr, x, ldx, info, diag, info_offset, flags);
}

// st = {info, pad, min diag(R) (running), max diag(G)}
__global__ void k_chol_status_init(const double* __restrict__ g, int64_t w, int64_t ldg, int* st) {
    __shared__ double red[32];
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i < w; i += blockDim.x) mx = fmax(mx, g[i + i * ldg]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mx = fmax(mx, red[i]);
        st[0] = 0;
        st[1] = 0;
        reinterpret_cast<double*>(st)[1] = INFINITY;
        reinterpret_cast<double*>(st)[2] = mx;
    }
}

// *flag = 1 unless the factorization behind st succeeded with min diag(R) > tau·sqrt(max diag(G))
// (the host-side chol_ok test of orth, decided on the device so no round trip is needed)
__global__ void k_chol_flag(const int* __restrict__ st, double tau, int* flag) {
    if (threadIdx.x != 0) return;
    const double mn = reinterpret_cast<const double*>(st)[1], mx = reinterpret_cast<const double*>(st)[2];
    const bool ok = st[0] == 0 && isfinite(mn) && mn > tau * sqrt(fmax(mx, 0.0));
    if (!ok) *flag = 1;
}


// ------------------------------------- persistent blocked Cholesky + inverse (w > 128)
// One cooperative launch (one 256-thread CTA per SM) runs the whole right-looking blocked
// factorization of a w × w SPD G (upper triangle read) with 128-wide blocks, R and X = R⁻¹
// together, all fp64 DMMA.  Step j (nb = ⌈w/128⌉ steps), three phases between grid barriers:
//   1  CTA 0: FACT(j) — the leaf (chol_leaf_dev) on the updated diagonal block: R_jj, X_jj.
//      The other CTAs meanwhile: the trailing update of step j−1 for block rows ≥ j+1
//      (W_ik −= R_{j−1,i}ᵀ R_{j−1,k}) and T = X[0:j,0:j]·R[0:j, j] for X's block column j.
//   2  PANEL: R_jk = X_jjᵀ W_jk for every k > j.
//   3  lookahead: block row j+1 gets step j's update (W_{j+1,k} −= R_{j,j+1}ᵀ R_jk), so FACT(j+1)
//      and PANEL(j+1) can start at once; X[0:j, j] = −T·X_jj.
// Work items are 128 × 128 blocks (phase 1) or 64 × 64 sub-tiles (phases 2, 3; tile_mm),
// dealt round-robin over CTAs 1.. — CTA 0 runs only the leaf, which keeps its long
// straight-line code warm in that SM's instruction cache (run between tile products, each
// FACT re-fetched it from a busy L2 and took ~2× the standalone leaf's time).  The
// critical path per step is FACT + one sub-tile in each of phases 2 and 3 + three barriers;
// the O(w³) updates and the inverse fill the SMs while CTA 0 factors (the launch-per-product
// recursion it replaces spent ~5 ms of a 4096-wide factorization on small dependent launches).
constexpr int PC_T = 256;
constexpr int PC_KC = 16;            // k-chunk per shared-memory stage
constexpr int PC_PK = PC_KC + 4;     // [m][k] / [n][k] pitch (≡ 4 mod 16: conflict-free fragments)
constexpr size_t PC_SMEM = LF_SMEM;       // the leaf's; the two workers' rings fit in it (static_assert below)

// Grid-wide barrier of a cooperative launch (sense by generation; bar[0] = arrivals, bar[1] = generation)
__device__ __forceinline__ void pc_grid_sync(unsigned int* bar, unsigned int& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int g = gen;
        if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
            bar[0] = 0;
            __threadfence();
            atomicExch(&bar[1], g + 1);
        } else {
            unsigned int v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1) : "memory");
            } while (v == g);
        }
    }
    gen += 1;
    __syncthreads();
}

// Tile operands are streamed by cp.async.cg (16-byte pairs, L2 only — coherent with the other
// CTAs' writes) through a PC_STAGES-deep shared-memory ring: three k-chunks in flight, no
// register staging.  Needs even leading dimensions and 16-byte aligned bases.
constexpr int PC_STAGES = 4;
__device__ __forceinline__ void cp16(double* smem, const double* gmem, int bytes) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}
// One 64 × 64 output sub-tile on a 4-warp group (two groups per CTA work independently, each
// with its own cp.async ring and named barrier, as two co-resident CTAs would: one 8-warp
// CTA stalled the whole SM's DMMA pipe at every chunk barrier — ncu put the persistent kernel's
// DMMA pipe at 26 % with barrier stalls first).  Same operand conventions as tile_mm_async.
constexpr int PG_STAGE = 2 * 64 * PC_PK;  // doubles per stage and group
static_assert((size_t)2 * PC_STAGES * PG_STAGE * 8 <= PC_SMEM, "two group rings");
template <int NW, bool TA, bool TB>
__device__ void tile_mm_grp(double* sm, int gtid, int bar_id, const double* __restrict__ A, int64_t lda,
                            const double* __restrict__ B, int64_t ldb, int mv, int nv, int k1, double alpha,
                            double* __restrict__ C, int64_t ldc, bool accumulate) {
    // NW = 4: a worker group (warp tile 32 × 32); NW = 8: the whole CTA (warp tile 16 × 32) for the
    // critical-path items, which then finish in half the time
    constexpr int TM = 64, TN = 64, PMA = TM + 4, PMB = TN + 4, NT = 32 * NW;
    constexpr int WMN = NW == 4 ? 2 : 4;             // warps along m
    constexpr int MF = TM / WMN / 8, NF = 4;          // 8 × 8 fragments per warp
    constexpr int CP = 512 / NT;                      // 16-byte pairs per thread and operand
    const int lane = gtid & 31, gw = gtid >> 5, wm = gw % WMN, wn = gw / WMN;
    double acc[MF][NF][2];
#pragma unroll
    for (int a = 0; a < MF; ++a)
#pragma unroll
        for (int b = 0; b < NF; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    double oldv[MF][NF][2];
    if (accumulate) {  // issued first: the latency hides behind the products
#pragma unroll
        for (int a = 0; a < MF; ++a)
#pragma unroll
            for (int b = 0; b < NF; ++b)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = wm * (MF * 8) + a * 8 + (lane >> 2), j = wn * 32 + b * 8 + 2 * (lane & 3) + e;
                    oldv[a][b][e] = (i < mv && j < nv) ? __ldcg(C + i + (int64_t)j * ldc) : 0.0;
                }
    }
    const int nc = k1 > 0 ? (k1 + PC_KC - 1) / PC_KC : 0;
    auto bar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(NT) : "memory"); };
    auto issue = [&](int c) {
        double* as = sm + (c % PC_STAGES) * PG_STAGE;
        double* bs = as + 64 * PC_PK;
        const int kb = c * PC_KC;
#pragma unroll
        for (int r = 0; r < CP; ++r) {  // 512 16-byte pairs of A, then of B
            const int t = gtid + r * NT;
            if (TA) {
                const int kk = 2 * (t & 7), i = t >> 3, gk = kb + kk;
                const int n = (i < mv && gk < k1) ? (gk + 1 < k1 ? 16 : 8) : 0;
                cp16(as + i * PC_PK + kk, n ? A + gk + (int64_t)i * lda : A, n);
            } else {
                const int i = 2 * (t & 31), kk = t >> 5, gk = kb + kk;
                const int n = (i < mv && gk < k1) ? (i + 1 < mv ? 16 : 8) : 0;
                cp16(as + kk * PMA + i, n ? A + i + (int64_t)gk * lda : A, n);
            }
            if (TB) {
                const int j = 2 * (t & 31), kk = t >> 5, gk = kb + kk;
                const int n = (j < nv && gk < k1) ? (j + 1 < nv ? 16 : 8) : 0;
                cp16(bs + kk * PMB + j, n ? B + j + (int64_t)gk * ldb : B, n);
            } else {
                const int kk = 2 * (t & 7), j = t >> 3, gk = kb + kk;
                const int n = (j < nv && gk < k1) ? (gk + 1 < k1 ? 16 : 8) : 0;
                cp16(bs + j * PC_PK + kk, n ? B + gk + (int64_t)j * ldb : B, n);
            }
        }
    };
#pragma unroll
    for (int c = 0; c < PC_STAGES - 1; ++c) {
        if (c < nc) issue(c);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const int fr = lane >> 2, fk = lane & 3;
    for (int c = 0; c < nc; ++c) {
        asm volatile("cp.async.wait_group %0;" ::"n"(PC_STAGES - 2) : "memory");
        bar();
        if (c + PC_STAGES - 1 < nc) issue(c + PC_STAGES - 1);
        asm volatile("cp.async.commit_group;" ::: "memory");
        const double* as = sm + (c % PC_STAGES) * PG_STAGE;
        const double* bs = as + 64 * PC_PK;
#pragma unroll
        for (int k4 = 0; k4 < PC_KC; k4 += 4) {
            double af[MF], bf[NF];
#pragma unroll
            for (int a = 0; a < MF; ++a) {
                const int i = wm * (MF * 8) + a * 8 + fr, kk = k4 + fk;
                af[a] = TA ? as[i * PC_PK + kk] : as[kk * PMA + i];
            }
#pragma unroll
            for (int b = 0; b < NF; ++b) {
                const int j = wn * 32 + b * 8 + fr, kk = k4 + fk;
                bf[b] = TB ? bs[kk * PMB + j] : bs[j * PC_PK + kk];
            }
#pragma unroll
            for (int a = 0; a < MF; ++a)
#pragma unroll
                for (int b = 0; b < NF; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int a = 0; a < MF; ++a)
#pragma unroll
        for (int b = 0; b < NF; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = wm * (MF * 8) + a * 8 + (lane >> 2), j = wn * 32 + b * 8 + 2 * (lane & 3) + e;
                if (i < mv && j < nv)
                    C[i + (int64_t)j * ldc] = accumulate ? fma(alpha, acc[a][b][e], oldv[a][b][e]) : alpha * acc[a][b][e];
            }
    bar();  // the ring is reused by the next item
}

// W (w × w working copy of G, upper blocks updated in place), R and X (zeroed, ld w),
// T (zeroed, w × w: the accumulated products X[0:j, 0:j]·R[0:j, j] of X's block columns),
// st = chol_status_init's status, bar = 2 zeroed words.  w even (16-byte cp.async pairs).
__global__ void __launch_bounds__(PC_T, 1) k_chol_persistent(double* __restrict__ W, double* __restrict__ R,
                                                            double* __restrict__ X, double* __restrict__ T, int w,
                                                            int* st, unsigned int* bar, int want_r) {
    extern __shared__ double pcs[];
    const int64_t ld = w;
    const int nb = (w + 127) / 128;
    const int cta = blockIdx.x, G = gridDim.x;
    unsigned int gen = 0;
    auto bs = [&](int b) { return min(128, w - b * 128); };
    // CTAs 1.. run two independent 4-warp groups ("workers"); CTA 0 runs only the leaf
    const int grp = threadIdx.x >> 7, gtid = threadIdx.x & 127, bar_id = 1 + grp;
    double* gsm = pcs + grp * PC_STAGES * PG_STAGE;
    // The SM that shares CTA 0's TPC stays idle: the leaf's long straight-line code is fetched
    // once per FACT, and tile products on the neighbouring SM evicted it from the shared
    // instruction cache (the leaf's first panel ran at 1.5–3× its standalone time, profiles/r02s)
    if (threadIdx.x == 0) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if (cta == 0) atomicExch(&bar[2], smid + 1);
        while (atomicAdd(&bar[2], 0u) == 0u) {}
        if (cta != 0 && (smid >> 1) == ((atomicAdd(&bar[2], 0u) - 1) >> 1)) atomicExch(&bar[3], (unsigned int)cta);
    }
    pc_grid_sync(bar, gen);
    const int quiet = (int)*(volatile unsigned int*)&bar[3];  // 0: none
    const int nq = G - 1 - (quiet ? 1 : 0);                    // CTAs with items
    const int crank = cta - 1 - (quiet && cta > quiet ? 1 : 0);
    const bool busy = cta > 0 && cta != quiet;
    const int worker = 2 * crank + grp, nwork = 2 * nq;
    // BCUR_LEAF_TIMING=1: CTA 0 sums its clocks per phase (FACT, the wait for the other CTAs'
    // phase-1 work, phases 2 and 3) and prints them at the end (diagnostics)
    const bool timing = g_leaf_timing && cta == 0 && threadIdx.x == 0;
    long long tf = 0, tw = 0, t2 = 0, t3 = 0, c0 = 0, c1 = 0;
    // W_{i,k} sub-tile (a, b) −= R_{s,i}[:, a]ᵀ · R_{s,k}[:, b]
    auto update = [&](int s, int i, int k, int a, int b, bool whole) {
        const int mv = min(64, bs(i) - a * 64), nv = min(64, bs(k) - b * 64);
        if (mv <= 0 || nv <= 0) return;  // diagonal blocks whole: they stay symmetric (LEAF_SYM loads)
        if (whole) tile_mm_grp<8, true, false>(pcs, threadIdx.x, 1, R + s * 128 + (int64_t)(i * 128 + a * 64) * ld, ld,
                                               R + s * 128 + (int64_t)(k * 128 + b * 64) * ld, ld, mv, nv, bs(s), -1.0,
                                               W + (i * 128 + a * 64) + (int64_t)(k * 128 + b * 64) * ld, ld, true);
        else tile_mm_grp<4, true, false>(gsm, gtid, bar_id, R + s * 128 + (int64_t)(i * 128 + a * 64) * ld, ld,
                                 R + s * 128 + (int64_t)(k * 128 + b * 64) * ld, ld, mv, nv, bs(s), -1.0,
                                 W + (i * 128 + a * 64) + (int64_t)(k * 128 + b * 64) * ld, ld, true);
    };
    // the diagonal blocks made symmetric (lower ← upper: the Gram kernels may write only the upper
    // triangle); every later update keeps them so, and the leaf copies them column by column
    for (int b = cta; b < nb; b += G) {
        const int wb = bs(b);
        double* D = W + b * 128 + (int64_t)(b * 128) * ld;
        for (int e = threadIdx.x; e < wb * wb; e += PC_T) {
            const int i = e % wb, k = e / wb;
            if (i > k) D[i + (int64_t)k * ld] = D[k + (int64_t)i * ld];
        }
    }
    pc_grid_sync(bar, gen);
    const int leaf_flags = LEAF_ZEROED | LEAF_SYM | (want_r ? 0 : LEAF_NO_R) | (g_leaf_timing == 2 ? 0 : LEAF_QUIET);
    for (int j = 0; j < nb; ++j) {
        const int J = j * 128;
        if (timing) c0 = clock64();
        // ---- phase 1: FACT(j) on CTA 0 | the workers: step j−1's trailing update of block rows
        //      ≥ j+1 and X's block column j−1 into the inverse accumulators
        //      (T[0:J, k] += X[0:J, j−1]·R[j−1, k], k ≥ j), as 64 × 64 sub-tiles
        if (cta == 0) {
            chol_leaf_call(pcs, W + J + (int64_t)J * ld, bs(j), ld, R + J + (int64_t)J * ld, ld, X + J + (int64_t)J * ld,
                           ld, st, reinterpret_cast<double*>(st) + 1, J, leaf_flags);
        } else if (j >= 1) {
            const int s = j - 1, S = s * 128, n = nb - j - 1;
            const int nupd = 4 * (n * (n + 1) / 2);  // blocks (i, k), j+1 ≤ i ≤ k
            const int ninv = 4 * (j * (nb - j));     // blocks (r, k), r < j, k ≥ j
            for (int t = worker; busy && t < nupd + ninv; t += nwork) {
                const int a = (t >> 1) & 1, b = t & 1, tb = t >> 2;
                if (t < nupd) {
                    int i = j + 1, u = tb;           // row i holds nb − i blocks
                    while (u >= nb - i) { u -= nb - i; ++i; }
                    update(s, i, i + u, a, b, false);
                } else {
                    const int u = tb - nupd / 4, r = u / (nb - j), k = j + u % (nb - j);
                    const int mv = min(64, bs(r) - a * 64), nv = min(64, bs(k) - b * 64);
                    if (mv > 0 && nv > 0)
                        tile_mm_grp<4, false, false>(gsm, gtid, bar_id, X + r * 128 + a * 64 + (int64_t)S * ld, ld,
                                                  R + S + (int64_t)(k * 128 + b * 64) * ld, ld, mv, nv, bs(s), 1.0,
                                                  T + r * 128 + a * 64 + (int64_t)(k * 128 + b * 64) * ld, ld, true);
                }
            }
        }
        if (timing) { c1 = clock64(); tf += c1 - c0; c0 = c1; }
        pc_grid_sync(bar, gen);
        if (timing) { c1 = clock64(); tw += c1 - c0; c0 = c1; }
        if (*(volatile int*)st != 0) return;  // a failed pivot (info) stops every CTA
        // ---- phase 2: PANEL(j): R_jk = X_jjᵀ W_jk, k > j (whole-CTA items: the critical path)
        if (cta > 0) {
            const int n2 = (nb - 1 - j) * 4;
            for (int t = crank; busy && t < n2; t += nq) {
                const int k = j + 1 + t / 4, a = (t >> 1) & 1, b = t & 1;
                const int mv = min(64, bs(j) - a * 64), nv = min(64, bs(k) - b * 64);
                if (mv <= 0 || nv <= 0) continue;
                // (X_jjᵀ)[a·64 + i, kk] = X[J + kk, J + a·64 + i], non-zero for kk ≤ a·64 + i
                tile_mm_grp<8, true, false>(pcs, threadIdx.x, 1, X + J + (int64_t)(J + a * 64) * ld, ld,
                                         W + J + (int64_t)(k * 128 + b * 64) * ld, ld, mv, nv, min(bs(j), a * 64 + 64),
                                         1.0, R + J + a * 64 + (int64_t)(k * 128 + b * 64) * ld, ld, false);
            }
        }
        pc_grid_sync(bar, gen);
        if (timing) { c1 = clock64(); t2 += c1 - c0; c0 = c1; }
        // ---- phase 3: lookahead — block row j+1 gets step j's update; X[0:J, j] = −T[0:J, j]·X_jj
        if (cta > 0) {
            const int nupd = j + 1 < nb ? 4 * (nb - 1 - j) : 0;
            const int nx = (J / 64) * 2;
            for (int t = crank; busy && t < nupd + nx; t += nq) {
                if (t < nupd) {
                    update(j, j + 1, j + 1 + t / 4, (t >> 1) & 1, t & 1, true);
                } else {
                    const int u = t - nupd, r = u >> 1, b = u & 1;
                    const int nv = min(64, bs(j) - b * 64);
                    if (nv <= 0) continue;
                    // X_jj upper: row kk of column b·64 + jj is non-zero for kk ≤ b·64 + jj
                    tile_mm_grp<8, false, false>(pcs, threadIdx.x, 1, T + r * 64 + (int64_t)J * ld, ld,
                                              X + J + (int64_t)(J + b * 64) * ld, ld, 64, nv, min(bs(j), b * 64 + 64),
                                              -1.0, X + r * 64 + (int64_t)(J + b * 64) * ld, ld, false);
                }
            }
        }
        pc_grid_sync(bar, gen);
        if (timing) { c1 = clock64(); t3 += c1 - c0; }
    }
    if (timing)
        printf("chol_persistent w=%d nb=%d grid=%d clocks: fact %lld | wait phase-1 %lld | phase 2 %lld | phase 3 %lld\n", w,
               nb, G, tf, tw, t2, t3);
}

}  // namespace

namespace ops {

// Split-K count: about two CTAs per SM.  Thin outputs (≤ 1 M elements, reduced by a warp per
// element) may split up to that many ways — the 60 × 60 Gram of a 65536-row panel ran 64
// splits of K = 1024 at one SM's DMMA rate (55 µs); wider outputs stay at ≤ 64 splits.
static int dgemm_splits(const Ctx* c, int64_t tiles, int64_t K, int64_t MN) {
    const int64_t target = 2LL * c->sm_count;
    if (tiles >= target || K < 8 * DBK) return 1;
    // (under half a wave of tiles — c1's 200 × 200 Grams over K = 500 ran 10 CTAs of 32 k-tiles, 29 µs
    // at one SM's DMMA rate each — split down to 4 k-tiles per CTA)
    int64_t s = std::min<int64_t>((target + tiles - 1) / tiles, K / ((tiles <= 64 ? 4 : 16) * DBK));
    return (int)std::max<int64_t>(1, std::min<int64_t>(s, MN <= (1 << 20) ? target : 64));
}

void dgemm(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, double alpha, const void* A, int dta, int64_t lda,
           const void* B, int dtb, int64_t ldb, double beta, double* C, int64_t ldc, int flags) {
    if (M <= 0 || N <= 0) return;
    ProfScope prof(c, "dgemm_dmma", 2.0 * M * N * std::max<int64_t>(K, 0),
                   (double)M * K * dtype_size(dta) + (double)K * N * dtype_size(dtb) + 8.0 * M * N);
    if (K <= 0) {
        if (beta == 0.0) {
            CUDA_CHECK(cudaMemset2DAsync(C, ldc * sizeof(double), 0, M * sizeof(double), N, c->stream));
            return;
        }
        K = 0;
    }
    static const bool no_thin = getenv("BCUR_DGEMM_NO_THIN") != nullptr;  // experiments
    const bool thin = N <= 16 && !no_thin;  // 64 × 16 tiles (the sketch's ℓ-wide products of c1/c2)
    const int64_t nb = thin ? 16 : DBN;
    const int64_t mt = (M + DBM - 1) / DBM, nt = (N + nb - 1) / nb;
    int64_t tiles = mt * nt;
    if (flags & GEMM_SYM_UPPER) tiles = (tiles + std::min(mt, nt)) / 2;
    int splits = dgemm_splits(c, tiles, K, M * N);
    int64_t kchunk = (std::max<int64_t>(K, 1) + splits - 1) / splits;
    kchunk = (kchunk + DBK - 1) / DBK * DBK;
    splits = (int)((std::max<int64_t>(K, 1) + kchunk - 1) / kchunk);
    dim3 grid((unsigned)mt, (unsigned)nt, (unsigned)splits);
    if (splits == 1) {
        if (thin)
            ddispatch<DEPI_STORE, 16>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, dta, lda, B, dtb, ldb, beta, C, ldc,
                                      nullptr, nullptr, 0, 0, flags);
        else
            ddispatch<DEPI_STORE>(c, ta, tb, grid, M, N, K, kchunk, alpha, A, dta, lda, B, dtb, ldb, beta, C, ldc,
                                  nullptr, nullptr, 0, 0, flags);
        return;
    }
    DevBuf part(c, (size_t)splits * M * N * sizeof(double));
    if (thin)
        ddispatch<DEPI_STORE, 16>(c, ta, tb, grid, M, N, K, kchunk, 1.0, A, dta, lda, B, dtb, ldb, 0.0, nullptr, 0,
                                  part.as<double>(), nullptr, 0, 0, flags);
    else
        ddispatch<DEPI_STORE>(c, ta, tb, grid, M, N, K, kchunk, 1.0, A, dta, lda, B, dtb, ldb, 0.0, nullptr, 0,
                              part.as<double>(), nullptr, 0, 0, flags);
    const int64_t total = M * N;
    if (splits >= 16 && total <= (1 << 20))
        k_dsplitk_reduce_warp<<<(unsigned)((total * 32 + 255) / 256), 256, 0, c->stream>>>(
            M, N, splits, part.as<double>(), alpha, beta, C, ldc, (flags & GEMM_SYM_UPPER) ? 1 : 0);
    else
        k_dsplitk_reduce<<<(unsigned)((total + 255) / 256), 256, 0, c->stream>>>(
            M, N, splits, part.as<double>(), alpha, beta, C, ldc, (flags & GEMM_SYM_UPPER) ? 1 : 0);
    LAUNCH_CHECK(c);
}

void dgemm_rowsumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                    const void* B, int dtb, int64_t ldb, double* rowsq) {
    if (M <= 0) return;
    ProfScope prof(c, "dgemm_rowsq_dmma", 2.0 * M * N * K,
                   (double)M * K * dtype_size(dta) + (double)K * N * dtype_size(dtb) + 8.0 * M);
    if (N <= 0 || K <= 0) {
        CUDA_CHECK(cudaMemsetAsync(rowsq, 0, M * sizeof(double), c->stream));
        return;
    }
    const int64_t mt = (M + DBM - 1) / DBM, nt = (N + DBN - 1) / DBN;
    DevBuf part(c, (size_t)nt * M * sizeof(double));
    dim3 grid((unsigned)mt, (unsigned)nt, 1);
    ddispatch<DEPI_ROWSQ>(c, ta, tb, grid, M, N, K, K, 1.0, A, dta, lda, B, dtb, ldb, 0.0, nullptr, 0,
                          part.as<double>(), nullptr, 0, 0, 0);
    k_dsum_rows<<<(unsigned)((M + 255) / 256), 256, 0, c->stream>>>(M, (int)nt, part.as<double>(), rowsq);
    LAUNCH_CHECK(c);
}

void dgemm_resid_sumsq(Ctx* c, Op ta, Op tb, int64_t M, int64_t N, int64_t K, const void* A, int dta, int64_t lda,
                       const void* B, int dtb, int64_t ldb, const void* D, int dtd, int64_t ldd, double* out) {
    ProfScope prof(c, "dgemm_resid_dmma", 2.0 * M * N * K,
                   (double)M * K * dtype_size(dta) + (double)K * N * dtype_size(dtb) + (double)M * N * dtype_size(dtd));
    const int64_t mt = (M + DBM - 1) / DBM, nt = (N + DBN - 1) / DBN;
    DevBuf part(c, (size_t)mt * nt * sizeof(double));
    dim3 grid((unsigned)mt, (unsigned)nt, 1);
    ddispatch<DEPI_RESID>(c, ta, tb, grid, M, N, std::max<int64_t>(K, 0), std::max<int64_t>(K, 1), 1.0, A, dta, lda, B,
                          dtb, ldb, 0.0, nullptr, 0, part.as<double>(), D, dtd, ldd, 0);
    sum_vector(c, part.as<double>(), mt * nt, out);
}

void chol_status_init(Ctx* c, const double* g, int64_t w, int64_t ldg, int* st) {
    k_chol_status_init<<<1, 256, 0, c->stream>>>(g, w, ldg, st);
    LAUNCH_CHECK(c);
}

void chol_persistent(Ctx* c, const double* g, int64_t w, int64_t ldg, double* r, double* x, int* st, bool want_r) {
    if (w < 2 || w % 2 != 0 || w > (1 << 20)) fail(BCUR_E_INVALID_ARGUMENT, "chol_persistent: needs an even width");
    ProfScope prof(c, "chol_inv", 2.0 * w * w * w / 3.0, 8.0 * 4 * w * w);
    static int grid = 0;
    if (!grid) {
        CUDA_CHECK(cudaFuncSetAttribute(k_chol_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PC_SMEM));
        int per_sm = 0;
        CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chol_persistent, PC_T, PC_SMEM));
        grid = std::max(1, per_sm) * c->sm_count;
        const char* t = getenv("BCUR_LEAF_TIMING");  // 1: phase clocks; 2: also each leaf's own
        const int on = t ? atoi(t) : 0;
        if (on) CUDA_CHECK(cudaMemcpyToSymbol(g_leaf_timing, &on, sizeof on));
    }
    if (grid < 2) fail(BCUR_E_CUDA, "chol_persistent: needs two co-resident CTAs");
    DevBuf W(c, (size_t)w * w * sizeof(double)), T(c, (size_t)w * w * sizeof(double)), bar(c, 64);
    CUDA_CHECK(cudaMemcpy2DAsync(W.ptr, w * sizeof(double), g, ldg * sizeof(double), w * sizeof(double), w,
                                 cudaMemcpyDeviceToDevice, c->stream));
    CUDA_CHECK(cudaMemsetAsync(r, 0, (size_t)w * w * sizeof(double), c->stream));
    CUDA_CHECK(cudaMemsetAsync(x, 0, (size_t)w * w * sizeof(double), c->stream));
    CUDA_CHECK(cudaMemsetAsync(T.ptr, 0, T.bytes, c->stream));
    CUDA_CHECK(cudaMemsetAsync(bar.ptr, 0, 64, c->stream));
    double* wp = W.as<double>();
    double* tp = T.as<double>();
    unsigned int* bp = bar.as<unsigned int>();
    int wi = (int)w, wr = want_r ? 1 : 0;
    void* args[] = {&wp, &r, &x, &tp, &wi, &st, &bp, &wr};
    CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_chol_persistent, dim3(grid), dim3(PC_T), args, PC_SMEM,
                                           c->stream));
    LAUNCH_CHECK(c);
}

void chol_flag(Ctx* c, const int* st, double tau, int* flag) {
    k_chol_flag<<<1, 32, 0, c->stream>>>(st, tau, flag);
    LAUNCH_CHECK(c);
}

void chol_inv_leaf(Ctx* c, const double* g, int64_t w, int64_t ldg, double* r, int64_t ldr, double* x, int64_t ldx,
                   int* info, double* diag, int64_t info_offset, int flags) {
    if (w > LF_MAX || w < 1) fail(BCUR_E_INVALID_ARGUMENT, "chol_inv_leaf: 1 <= w <= 128");
    ProfScope prof(c, "chol_inv_leaf", 2.0 * w * w * w / 3.0, 8.0 * 3 * w * w);
    constexpr size_t smem = (size_t)(LF_MAX * LF_LD + 7 * 32 * LF_TP) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_chol_inv_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const char* t = getenv("BCUR_LEAF_TIMING");
        const int on = (t && t[0] == '1') ? 1 : 0;
        if (on) CUDA_CHECK(cudaMemcpyToSymbol(g_leaf_timing, &on, sizeof on));
        attr = true;
    }
    k_chol_inv_leaf<<<1, LF_T, smem, c->stream>>>(g, (int)w, ldg, r, ldr, x, ldx, info, diag, (int)info_offset, flags);
    LAUNCH_CHECK(c);
}

}  // namespace ops
}  // namespace bcur_b200
