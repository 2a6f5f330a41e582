// kernels_small.cu — single-CTA fp64 factorizations of the small (≤ a few
// hundred) matrices of the hot path: Cholesky (CholQR2 of the sketch / C panels,
// diagonal blocks of the blocked factorization), triangular inverse, and a
// parallel-ordered cyclic Jacobi eigensolver (SVQB rank revealing and the ℓ×ℓ
// eigenproblem of B·Bᵀ that replaces the reference's BDCSVD, matcore.cpp:39-56).
// Working matrices sit in shared memory when they fit and in an L2-resident global
// scratch otherwise; all index math is 32-bit and loops are warp-strided so that
// global accesses coalesce.
#include "ops.h"

namespace bcur_b200 {
namespace {

constexpr int ST = 1024;

// 1/x to full double precision from the hardware approximation + two Newton steps (the
// IEEE-exact division is a long software sequence that sat on the factorizations'
// serial critical paths).
// 1/√x to full double precision: hardware approximation + two Newton steps (4 DFMA deep)
__device__ __forceinline__ double fast_rsqrt(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double hx = 0.5 * x;
    r = r * fma(-hx * r, r, 1.5);
    r = r * fma(-hx * r, r, 1.5);
    return r;
}
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    r = fma(r, fma(-x, r, 1.0), r);
    return r;
}
constexpr int NW = ST / 32;
constexpr int SMEM_MAX_W = 144;

// --------------------------------------------------------------- Cholesky
// Right-looking with delayed scaling on the LOWER triangle L of the working copy
// (M[i,k], i ≥ k, holds Gᵀ's entries): step j subtracts M[i,j]·M[k,j]/M[j,j] from every
// trailing M[i,k] (j < k ≤ i) — column j is read contiguously, one barrier per column —
// and R[j,k] = M[k,j]/√M[j,j] is formed once at the end.  Input: the upper triangle of g.
// Chained use (blocked factorization): a nonzero *info on entry means an earlier block
// failed — return untouched; on failure write info = info_offset + j + 1.  diag[0]
// accumulates min diag(R) across the chain (caller initialises it), diag[1] = max diag(G).
__global__ void __launch_bounds__(ST) k_cholesky(const double* g, int w, int64_t ldg, double* r, int64_t ldr,
                                                 double* __restrict__ work, int* info, double* diag,
                                                 int info_offset, int chained) {
    extern __shared__ double sm[];
    if (chained && *info != 0) return;
    double* M = work ? work : sm;
    const int ldm = w | 1;  // odd stride: row-wise walks of the final transpose hit distinct banks
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = warp; k < w; k += NW)
        for (int i = lane; i <= k; i += 32) M[k + i * ldm] = g[i + k * ldg];  // upper of g → lower of M
    __syncthreads();
    if (warp == 0) {
        double mx = 0.0;
        for (int j = lane; j < w; j += 32) mx = fmax(mx, M[j + j * ldm]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && !chained) diag[1] = mx;
    }
    int stop = 0;
    double mn = INFINITY;
    for (int j = 0; j < w; ++j) {
        const double d = M[j + j * ldm];  // final after step j-1's barrier; identical in all threads
        if (!(d > 0.0) || !isfinite(d)) {
            stop = j + 1;
            break;
        }
        mn = fmin(mn, d);
        const double inv = fast_rcp(d);
        const double* colj = M + j * ldm;
        for (int k = j + 1 + warp; k < w; k += NW) {
            const double a = colj[k] * inv;
            double* colk = M + k * ldm;
            for (int i = k + lane; i < w; i += 32) colk[i] = fma(-a, colj[i], colk[i]);
        }
        __syncthreads();
    }
    for (int k = warp; k < w; k += NW)
        for (int i = lane; i < w; i += 32)
            r[i + k * ldr] = i <= k && !stop ? M[k + i * ldm] / sqrt(M[i + i * ldm]) : 0.0;
    if (threadIdx.x == 0) {
        mn = sqrt(mn);
        if (chained) {
            if (stop) *info = info_offset + stop;
            diag[0] = stop ? 0.0 : fmin(diag[0], mn);
        } else {
            *info = stop;
            diag[0] = stop ? 0.0 : mn;
        }
    }
}

// ------------------------------------------------- panel Cholesky (w ≤ 128)
// Same contract as k_cholesky, for the diagonal blocks of the blocked factorization.
// 32-column panels: (1) one warp factors the 32×32 diagonal block in registers (lane i
// holds row i; pivots and multipliers move by shuffles — no barriers), (2) one thread per
// remaining row forward-substitutes its 32 panel entries (TRSM), (3) all 8 warps apply the
// rank-32 SYRK update to the trailing lower triangle with 6×6 register tiles.  Three
// barriers per panel instead of one per column; ~5× fewer instructions than k_cholesky.
constexpr int CP_T = 256, CP_MAX = 128, CP_LD = CP_MAX + 1;
__global__ void __launch_bounds__(CP_T) k_chol_panel(const double* g, int w, int64_t ldg, double* r, int64_t ldr,
                                                     int* info, double* diag, int info_offset, int chained) {
    extern __shared__ double smc[];
    double* M = smc;                    // lower triangle, M[i + k·LD] (i ≥ k), padded with identity
    __shared__ double invd[CP_MAX];
    __shared__ double xch[32];
    __shared__ int stop_sh;
    __shared__ double mn_sh;
    if (chained && *info != 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wp = (w + 31) & ~31;
    for (int k = warp; k < wp; k += CP_T / 32)
        for (int i = lane; i <= k; i += 32)
            M[k + i * CP_LD] = (i < w && k < w) ? g[i + (int64_t)k * ldg] : (i == k ? 1.0 : 0.0);
    if (tid == 0) {
        stop_sh = 0;
        mn_sh = INFINITY;
    }
    __syncthreads();
    if (warp == 0) {
        double mx = 0.0;
        for (int j = lane; j < w; j += 32) mx = fmax(mx, M[j + j * CP_LD]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && !chained) diag[1] = mx;
    }
    for (int c0 = 0; c0 < wp; c0 += 32) {
        // (1) 32×32 diagonal block, warp 0, registers
        if (warp == 0) {
            double a[32];
#pragma unroll
            // row `lane` of the block; entries k > lane are upper-triangle garbage that is
            // updated harmlessly and never stored or read for a lower entry (no per-lane
            // predicates in the step: they cost more than the arithmetic)
            for (int k = 0; k < 32; ++k) a[k] = M[(c0 + lane) + (c0 + k) * CP_LD];
            int bad = 0;
            double mn = INFINITY, dl = 1.0;  // dl: this lane's 1/r_ii
#pragma unroll
            for (int j = 0; j < 32; ++j) {  // fully unrolled: a[] stays in registers (no break)
                const double d = __shfl_sync(0xffffffffu, a[j], j);
                if (!bad && (!(d > 0.0) || !isfinite(d))) bad = c0 + j + 1;
                if (bad) continue;
                const double ri = fast_rsqrt(d), rj = d * ri;
                if (c0 + j < w) mn = fmin(mn, rj);  // padding pivots are 1
                if (lane == j) dl = ri;
                const double lij = a[j] * ri;  // l(lane, j) for lane > j (garbage above)
                a[j] = lane == j ? rj : lij;
                // multipliers exchanged through shared memory (broadcast loads pipeline;
                // 31 dependent-issue double shuffles per step dominated the step time)
                xch[lane] = lij;
                __syncwarp();
#pragma unroll
                for (int k = j + 1; k < 32; ++k) a[k] = fma(-lij, xch[k], a[k]);
                __syncwarp();
            }
            if (!bad) {
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    if (k <= lane) M[(c0 + lane) + (c0 + k) * CP_LD] = a[k];
                invd[c0 + lane] = dl;
            }
            if (lane == 0) {
                if (bad) stop_sh = bad;
                mn_sh = fmin(mn_sh, mn);
            }
        }
        __syncthreads();
        if (stop_sh) break;
        const int base = c0 + 32, nr = wp - base;
        if (nr <= 0) break;
        // (2) TRSM: row i of the panel below the diagonal block, x = m · L_ppᵀ⁻¹
        if (tid < nr) {
            // right-looking: each solved x_c immediately updates every later entry, so the
            // dependent chain is 2 ops per column (a dot-product form is a 528-deep chain)
            const int i = base + tid;
            double x[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] = M[i + (c0 + c) * CP_LD];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                x[c] *= invd[c0 + c];
#pragma unroll
                for (int cc = c + 1; cc < 32; ++cc) x[cc] = fma(-x[c], M[(c0 + cc) + (c0 + c) * CP_LD], x[cc]);
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) M[i + (c0 + c) * CP_LD] = x[c];
        }
        __syncthreads();
        // (3) SYRK: M[i,k] -= Σ_c L[i,c]·L[k,c] over the trailing lower triangle
        {
            const int ty = tid >> 4, tx = tid & 15;
            double acc[6][6];
#pragma unroll
            for (int u = 0; u < 6; ++u)
#pragma unroll
                for (int v = 0; v < 6; ++v) acc[u][v] = 0.0;
#pragma unroll 4
            for (int c = 0; c < 32; ++c) {
                const double* col = M + (c0 + c) * CP_LD + base;
                double li[6], lk[6];
#pragma unroll
                for (int u = 0; u < 6; ++u) {
                    li[u] = (ty + 16 * u) < nr ? col[ty + 16 * u] : 0.0;
                    lk[u] = (tx + 16 * u) < nr ? col[tx + 16 * u] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 6; ++u)
#pragma unroll
                    for (int v = 0; v < 6; ++v) acc[u][v] = fma(li[u], lk[v], acc[u][v]);
            }
#pragma unroll
            for (int u = 0; u < 6; ++u)
#pragma unroll
                for (int v = 0; v < 6; ++v) {
                    const int i = ty + 16 * u, k = tx + 16 * v;
                    if (i < nr && k <= i) M[(base + i) + (base + k) * CP_LD] -= acc[u][v];
                }
        }
        __syncthreads();
    }
    const int stop = stop_sh;
    for (int k = warp; k < w; k += CP_T / 32)
        for (int i = lane; i < w; i += 32) r[i + (int64_t)k * ldr] = i <= k && !stop ? M[k + i * CP_LD] : 0.0;
    if (tid == 0) {
        if (chained) {
            if (stop) *info = info_offset + stop;
            diag[0] = stop ? 0.0 : fmin(diag[0], mn_sh);
        } else {
            *info = stop;
            diag[0] = stop ? 0.0 : mn_sh;
        }
    }
}

// ------------------------------------------------- panel solve (kb ≤ 128)
// P ← R⁻ᵀ·P in place for an upper-triangular R (kb × kb, ld ldr) and P (kb × N, ld ldp): the
// block-row solve of the blocked Cholesky.  One CTA per 32 columns of P; Lᵀ = R staged in
// shared memory; four 32-row blocks: each column's 32×32 triangle solved by its own thread in
// registers (right-looking: 2 dependent ops per row), then the 32-row block's contribution
// subtracted from the rows below by all 8 warps.
constexpr int TS_T = 256, TS_C = 32, TS_LD = 129;
__global__ void __launch_bounds__(TS_T) k_trsm128(const double* __restrict__ R, int kb, int64_t ldr, double* P,
                                                  int64_t ldp, int N) {
    extern __shared__ double sm_ts[];
    double* L = sm_ts;                 // L[i + k·TS_LD] = R[k][i] (lower), i ≥ k
    double* X = L + 128 * TS_LD;       // X[r + c·TS_LD], 128 × 32 slab
    __shared__ double dinv[128];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c0 = blockIdx.x * TS_C, nc = min(TS_C, N - c0);
    const int kp = (kb + 31) & ~31;
    for (int i = warp; i < kp; i += TS_T / 32)  // column i of R (contiguous) → row i of L
        for (int k = lane; k <= i; k += 32)
            L[i + k * TS_LD] = (i < kb) ? R[k + (int64_t)i * ldr] : (i == k ? 1.0 : 0.0);
    for (int c = warp; c < TS_C; c += TS_T / 32)
        for (int r = lane; r < kp; r += 32)
            X[r + c * TS_LD] = (c < nc && r < kb) ? P[r + (int64_t)(c0 + c) * ldp] : 0.0;
    __syncthreads();
    for (int i = tid; i < kp; i += TS_T) dinv[i] = 1.0 / L[i + i * TS_LD];
    __syncthreads();
    for (int b0 = 0; b0 < kp; b0 += 32) {
        if (warp == 0) {  // lane = column
            double x[32];
#pragma unroll
            for (int r = 0; r < 32; ++r) x[r] = X[(b0 + r) + lane * TS_LD];
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                x[r] *= dinv[b0 + r];
#pragma unroll
                for (int j = r + 1; j < 32; ++j) x[j] = fma(-L[(b0 + j) + (b0 + r) * TS_LD], x[r], x[j]);
            }
#pragma unroll
            for (int r = 0; r < 32; ++r) X[(b0 + r) + lane * TS_LD] = x[r];
        }
        __syncthreads();
        // rows below the block: X[i, c] −= Σ_r L[i, b0 + r]·X[b0 + r, c]
        for (int i = b0 + 32 + warp; i < kp; i += TS_T / 32) {
            double acc = X[i + lane * TS_LD];
#pragma unroll 8
            for (int r = 0; r < 32; ++r) acc = fma(-L[i + (b0 + r) * TS_LD], X[(b0 + r) + lane * TS_LD], acc);
            X[i + lane * TS_LD] = acc;
        }
        __syncthreads();
    }
    for (int c = warp; c < nc; c += TS_T / 32)
        for (int r = lane; r < kb; r += 32) P[r + (int64_t)(c0 + c) * ldp] = X[r + c * TS_LD];
}

// ------------------------------------------------------ triangular inverse
// X = R⁻¹ for upper-triangular R, w ≤ TRI_MAX_W, one CTA, 16-wide blocks (the matrix is
// padded with identity to a multiple of 16).  Storage: one padded square S holds R's
// upper triangle in place and Xᵀ's strictly-lower part (X[i,c] at S[c + i·ld], c > i), X's
// diagonal in xd.  Phase A inverts all diagonal blocks at once (thread per column, a
// ≤16-deep back substitution); phase B sweeps block columns j = 1.. : T = X[0:j,0:j]·R[0:j,j],
// then X[0:j,j] = −T·X_jj.  ~8 barriers instead of a w-deep serial chain.
constexpr int TRI_MAX_W = 128;
constexpr int TRI_B = 16;
constexpr int TRI_LD = TRI_MAX_W + 1;
__global__ void __launch_bounds__(ST) k_tri_inv_upper(const double* __restrict__ r, int w, int64_t ldr,
                                                      double* __restrict__ x, int64_t ldx) {
    extern __shared__ double sm_tri[];
    double* S = sm_tri;                      // TRI_LD × TRI_LD
    double* T = S + TRI_LD * TRI_LD;         // (TRI_MAX_W − TRI_B) × TRI_B, row r at T[r·TRI_B + c]
    __shared__ double xd[TRI_MAX_W];
    const int wp = (w + TRI_B - 1) / TRI_B * TRI_B;
    const int nb = wp / TRI_B;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = warp; k < wp; k += NW)
        for (int i = lane; i <= k; i += 32)
            S[i + k * TRI_LD] = (i < w && k < w) ? r[i + k * ldr] : (i == k ? 1.0 : 0.0);
    __syncthreads();
    for (int c = threadIdx.x; c < wp; c += ST) xd[c] = fast_rcp(S[c + c * TRI_LD]);
    __syncthreads();
    // phase A: column c of the inverse of its diagonal block
    for (int c = threadIdx.x; c < wp; c += ST) {
        const int b0 = c / TRI_B * TRI_B;
        const double xcc = xd[c];
        for (int i = c - 1; i >= b0; --i) {
            double s = S[i + c * TRI_LD] * xcc;
            for (int t = i + 1; t < c; ++t) s = fma(S[i + t * TRI_LD], S[c + t * TRI_LD], s);
            S[c + i * TRI_LD] = -s * xd[i];
        }
    }
    __syncthreads();
    // phase B
    for (int jb = 1; jb < nb; ++jb) {
        const int j0 = jb * TRI_B;
        for (int e = threadIdx.x; e < j0 * TRI_B; e += ST) {
            const int cc = e % TRI_B, rr = e / TRI_B, c = j0 + cc;
            double s = xd[rr] * S[rr + c * TRI_LD];
            for (int t = rr + 1; t < j0; ++t) s = fma(S[t + rr * TRI_LD], S[t + c * TRI_LD], s);
            T[rr * TRI_B + cc] = s;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < j0 * TRI_B; e += ST) {
            const int cc = e % TRI_B, rr = e / TRI_B, c = j0 + cc;
            double s = T[rr * TRI_B + cc] * xd[c];
            for (int u = j0; u < c; ++u) s = fma(T[rr * TRI_B + (u - j0)], S[c + u * TRI_LD], s);
            S[c + rr * TRI_LD] = -s;
        }
        __syncthreads();
    }
    for (int k = warp; k < w; k += NW)
        for (int i = lane; i < w; i += 32) x[i + k * ldx] = i < k ? S[k + i * TRI_LD] : (i == k ? xd[i] : 0.0);
}

// ---------------------------------------------------------------- Jacobi
// Parallel (round-robin) cyclic Jacobi; A (w×w, column-major) in `A`, V (w×w) in `V`.
__global__ void __launch_bounds__(ST) k_jacobi(const double* __restrict__ g, int w, int64_t ldg,
                                               double* __restrict__ Aglob, double* V,
                                               double* __restrict__ lam, double* __restrict__ vout, int max_sweeps) {
    extern __shared__ double sm[];
    const int la = w | 1;  // odd leading dimension: row rotations (stride la) hit distinct banks
    double* A = Aglob ? Aglob : sm;
    if (!V) V = sm + w * la;  // V in shared memory after A (sym_eig sizes the allocation)
    __shared__ int pos[512];
    __shared__ double cs[256], sn[256], np_[256], nq_[256];
    __shared__ int pp[256], qq[256];
    __shared__ int rotated;
    __shared__ double floor_abs;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NWB = blockDim.x >> 5, NTB = blockDim.x;  // (256 threads measured slower for w = 64)
    const int wp = (w + 1) & ~1;  // even number of players (w..wp-1 is a bye)
    const int half = wp / 2;
    for (int j = warp; j < w; j += NWB)
        for (int i = lane; i < w; i += 32) {
            A[i + j * la] = g[i + j * ldg];
            V[i + j * la] = i == j ? 1.0 : 0.0;
        }
    for (int i = threadIdx.x; i < wp; i += NTB) pos[i] = i;
    // absolute floor: off-diagonal rounding noise of the input (≈ eps·‖G‖) is not rotated away
    if (threadIdx.x == 0) {
        double f = 0.0;
        for (int j = 0; j < w; ++j) f = fmax(f, fabs(g[j + j * ldg]));
        floor_abs = 1e-16 * f * (double)w;
    }
    __syncthreads();
    const int msw = max_sweeps < 0 ? -max_sweeps : max_sweeps;
    for (int sweep = 0; sweep < msw; ++sweep) {
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int round = 0; round < wp - 1; ++round) {
            for (int i = threadIdx.x; i < half; i += NTB) {
                // circle method: player wp-1 fixed, the others rotate (all pairs in wp-1 rounds)
                const int mrot = wp - 1;
                int p = i == 0 ? round : (round + i) % mrot;
                int q = i == 0 ? wp - 1 : (round - i + mrot) % mrot;
                if (p > q) { const int t = p; p = q; q = t; }
                double c = 1.0, s = 0.0;
                if (q < w) {
                    const double apq = A[p + q * la];
                    const double app = A[p + p * la], aqq = A[q + q * la];
                    if (fabs(apq) > floor_abs && apq * apq > 1e-30 * fabs(app * aqq)) {  // |apq| > 1e-15·√|app·aqq|
                        // rotation from rsqrt/rcp approximations refined to ~1 ulp (the
                        // IEEE sqrt/div sequences made each round a long serial chain)
                        const double tau = (aqq - app) * fast_rcp(2.0 * apq);
                        const double q2 = fma(tau, tau, 1.0);
                        const double root = q2 * rsqrt(q2);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) * fast_rcp(fabs(tau) + root);
                        c = rsqrt(fma(t, t, 1.0));
                        s = t * c;
                        np_[i] = app - t * apq;  // exact post-rotation diagonal (Golub–Van Loan 8.4)
                        nq_[i] = aqq + t * apq;
                        rotated = 1;
                    }
                }
                pp[i] = p;
                qq[i] = q;
                cs[i] = c;
                sn[i] = s;
            }
            __syncthreads();
            // rows: A ← Jᵀ A   (warp per pair, lanes over columns)
            for (int i = warp; i < half; i += NWB) {
                const int p = pp[i], q = qq[i];
                if (q >= w || sn[i] == 0.0) continue;
                const double c = cs[i], s = sn[i];
                for (int k = lane; k < w; k += 32) {
                    const double ap = A[p + k * la], aq = A[q + k * la];
                    A[p + k * la] = c * ap - s * aq;
                    A[q + k * la] = s * ap + c * aq;
                }
            }
            __syncthreads();
            // columns: A ← A J, V ← V J   (coalesced along the column)
            for (int i = warp; i < half; i += NWB) {
                const int p = pp[i], q = qq[i];
                if (q >= w || sn[i] == 0.0) continue;
                const double c = cs[i], s = sn[i];
                for (int k = lane; k < w; k += 32) {
                    const double ap = A[k + p * la], aq = A[k + q * la];
                    A[k + p * la] = c * ap - s * aq;
                    A[k + q * la] = s * ap + c * aq;
                    const double vp = V[k + p * la], vq = V[k + q * la];
                    V[k + p * la] = c * vp - s * vq;
                    V[k + q * la] = s * vp + c * vq;
                }
                // the rotated pair is annihilated exactly (rounding noise would retrigger
                // rotations); columns p and q belong to this warp alone in this phase
                __syncwarp();
                if (lane == 0) {
                    A[p + q * la] = 0.0;
                    A[q + p * la] = 0.0;
                    A[p + p * la] = np_[i];
                    A[q + q * la] = nq_[i];
                }
            }
            __syncthreads();
        }
        if (!rotated) {
            if (threadIdx.x == 0 && max_sweeps < 0) printf("jacobi w=%d sweeps=%d\n", w, sweep + 1);
            break;
        }
        __syncthreads();
    }
    // sort eigenvalues descending (stable selection on indices), permute V
    __shared__ int order[512];
    if (threadIdx.x == 0) {
        for (int i = 0; i < w; ++i) order[i] = i;
        for (int i = 0; i < w; ++i) {
            int best = i;
            for (int j = i + 1; j < w; ++j)
                if (A[order[j] + order[j] * la] > A[order[best] + order[best] * la]) best = j;
            const int t = order[i]; order[i] = order[best]; order[best] = t;
        }
    }
    __syncthreads();
    for (int j = warp; j < w; j += NWB)
        for (int i = lane; i < w; i += 32) vout[i + j * w] = V[i + order[j] * la];
    for (int j = threadIdx.x; j < w; j += NTB) lam[j] = A[order[j] + order[j] * la];
}

// ---------------------------------------- packed two-sided Jacobi (any w ≤ 220)
// The same rotations as k_jacobi (circle-method rounds, the same angle formula and stopping
// rule), restructured so that a round is ONE pass over the matrix: under a round's pairing
// the 2×2 blocks (pair P rows × pair Q columns) partition A, and each is updated from both
// sides at once, A[P,Q] ← J_Pᵀ A[P,Q] J_Q, by one thread (blocks are disjoint: no barrier
// between the row and the column rotation).  Only the lower triangle is stored (packed),
// so w = 220 fits in shared memory (194 KB).  V is not accumulated here: every round's
// rotations are logged (p, q, c, s) and k_jacobi_replay applies them to the rows of V on
// many SMs afterwards.
constexpr int JP_T = 1024;
__device__ int g_jac_timing = 0;  // BCUR_JACOBI_TIMING=1: thread 0 prints the phase clocks (diagnostics)
struct JRot {
    double c, s;
    int p, q;
};
__device__ __forceinline__ int tri_at(int i, int j) { return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i; }
__global__ void __launch_bounds__(JP_T) k_jacobi_packed(const double* __restrict__ g, int w, int64_t ldg,
                                                        JRot* __restrict__ log, int* __restrict__ nrounds_out,
                                                        double* __restrict__ lam, int* __restrict__ order_out,
                                                        int max_sweeps) {
    extern __shared__ double Ap[];  // packed lower triangle
    auto at = [&](int i, int j) { return tri_at(i, j); };
    __shared__ double cs[256], sn[256], np_[256], nq_[256];
    __shared__ int pp[256], qq[256];
    __shared__ int rotated;
    __shared__ double floor_abs;
    const int wp = (w + 1) & ~1, half = wp / 2, mrot = wp - 1;
    const int NT = blockDim.x;
    for (int i = threadIdx.x; i < w; i += NT)
        for (int j = 0; j <= i; ++j) Ap[at(i, j)] = g[i + (int64_t)j * ldg];  // lower of a symmetric G
    if (threadIdx.x == 0) {
        double f = 0.0;
        for (int j = 0; j < w; ++j) f = fmax(f, fabs(g[j + j * ldg]));
        floor_abs = 1e-16 * f * (double)w;
    }
    __syncthreads();
    const int nblk = half * (half + 1) / 2;
    int P0 = (int)((sqrtf(8.0f * (float)threadIdx.x + 1.0f) - 1.0f) * 0.5f);  // block threadIdx.x → (P0, Q0), P0 ≥ Q0
    if (P0 * (P0 + 1) / 2 > (int)threadIdx.x) --P0;
    if ((P0 + 1) * (P0 + 2) / 2 <= (int)threadIdx.x) ++P0;
    const int Q0 = (int)threadIdx.x - P0 * (P0 + 1) / 2;
    int rounds = 0;
    const bool timing = g_jac_timing && threadIdx.x == 0;
    long long ta = 0, tb = 0, c0 = 0, c1 = 0;
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int round = 0; round < mrot; ++round, ++rounds) {
            if (timing) c0 = clock64();
            for (int i = threadIdx.x; i < half; i += NT) {
                // (round ± i) mod mrot without the integer divisions (0 ≤ round, i < mrot)
                int p = round + i, q = round - i;
                if (p >= mrot) p -= mrot;
                if (q < 0) q += mrot;
                if (i == 0) q = wp - 1;
                if (p > q) { const int t = p; p = q; q = t; }
                double c = 1.0, sv = 0.0;
                if (q < w) {
                    const double apq = Ap[at(q, p)];
                    const double app = Ap[at(p, p)], aqq = Ap[at(q, q)];
                    if (fabs(apq) > floor_abs && apq * apq > 1e-30 * fabs(app * aqq)) {
                        // The small-angle rotation with tan 2θ = 2a_pq/(a_qq − a_pp), from the double
                        // angle: cos 2θ = |d|/√h, h = d² + (2a_pq)²; cos²θ = (1 + cos 2θ)/2;
                        // |sin θ| = |2a_pq|/(2√h·cos θ); sign θ = sign(d·a_pq).  Two rsqrt chains
                        // instead of rcp → rsqrt → rcp → rsqrt: the rotation is this phase's whole
                        // latency (a ~33-deep dependent fp64 chain cut to ~21; profiles/r02aq →
                        // r02as jacobi_clocks).  h outside the normal range: the tangent form.
                        const double d = aqq - app, b2 = 2.0 * apq;
                        const double h = fma(d, d, b2 * b2);
                        double t;
                        if (h > 1e-280 && h < 1e280) {
                            const double r = fast_rsqrt(h);
                            const double c2 = fma(0.5 * fabs(d), r, 0.5);
                            const double rc = fast_rsqrt(c2);
                            c = c2 * rc;
                            sv = (d * b2 >= 0.0 ? 0.5 : -0.5) * fabs(b2) * r * rc;
                            t = sv * rc;
                        } else {
                            const double tau = d * fast_rcp(b2);
                            const double q2 = fma(tau, tau, 1.0);
                            const double root = q2 * fast_rsqrt(q2);
                            t = (tau >= 0.0 ? 1.0 : -1.0) * fast_rcp(fabs(tau) + root);
                            c = fast_rsqrt(fma(t, t, 1.0));
                            sv = t * c;
                        }
                        np_[i] = app - t * apq;
                        nq_[i] = aqq + t * apq;
                        rotated = 1;
                    }
                }
                pp[i] = p;
                qq[i] = q;
                cs[i] = c;
                sn[i] = sv;
                log[(int64_t)rounds * half + i] = JRot{c, sv, p, q};
            }
            __syncthreads();
            if (timing) { c1 = clock64(); ta += c1 - c0; c0 = c1; }
            // block (P, Q), P ≥ Q, enumerated over the packed block triangle
            for (int b = threadIdx.x; b < nblk; b += NT) {
                int P = P0, Q = Q0;  // the thread's first block, decoded once before the sweeps
                if (b != (int)threadIdx.x) {
                    P = (int)((sqrtf(8.0f * (float)b + 1.0f) - 1.0f) * 0.5f);
                    if (P * (P + 1) / 2 > b) --P;
                    if ((P + 1) * (P + 2) / 2 <= b) ++P;
                    Q = b - P * (P + 1) / 2;
                }
                const int p1 = pp[P], q1 = qq[P], p2 = pp[Q], q2 = qq[Q];
                const double s1 = sn[P], s2 = sn[Q];
                if (s1 == 0.0 && s2 == 0.0) continue;
                if (P == Q) {  // diagonal block: exact annihilation
                    if (q1 >= w) continue;
                    Ap[at(q1, p1)] = 0.0;
                    Ap[at(p1, p1)] = np_[P];
                    Ap[at(q1, q1)] = nq_[P];
                    continue;
                }
                const double c1 = cs[P], c2 = cs[Q];
                const bool r2 = q1 < w, c2v = q2 < w;  // byes: a padding index has no row/column
                const int i_pp = at(p1, p2), i_pq = c2v ? at(p1, q2) : 0;
                const int i_qp = r2 ? at(q1, p2) : 0, i_qq = (r2 && c2v) ? at(q1, q2) : 0;
                const double a_pp = Ap[i_pp], a_pq = c2v ? Ap[i_pq] : 0.0;
                const double a_qp = r2 ? Ap[i_qp] : 0.0, a_qq = (r2 && c2v) ? Ap[i_qq] : 0.0;
                // rows: [p1; q1] ← [c1 −s1; s1 c1]·[.]   (Jᵀ A with J = [c s; −s c] convention of k_jacobi)
                const double b_pp = c1 * a_pp - s1 * a_qp, b_pq = c1 * a_pq - s1 * a_qq;
                const double b_qp = s1 * a_pp + c1 * a_qp, b_qq = s1 * a_pq + c1 * a_qq;
                // columns: [p2, q2] ← [.]·J
                const double o_pp = c2 * b_pp - s2 * b_pq, o_pq = s2 * b_pp + c2 * b_pq;
                const double o_qp = c2 * b_qp - s2 * b_qq, o_qq = s2 * b_qp + c2 * b_qq;
                Ap[i_pp] = o_pp;
                if (c2v) Ap[i_pq] = o_pq;
                if (r2) Ap[i_qp] = o_qp;
                if (r2 && c2v) Ap[i_qq] = o_qq;
            }
            __syncthreads();
            if (timing) tb += clock64() - c0;
        }
        if (!rotated) break;
        // would the next sweep rotate at all?  (The same test as the rounds' on every off-diagonal
        // pair: none passing it means that sweep would change nothing — skipping it is exact.)
        __syncthreads();  // every thread has read the sweep's flag before thread 0 clears it: without
                          // this barrier a late warp could read the cleared flag and leave the loop alone
                          // (c4's 1024-thread launches faulted in about half of 20-step runs, profiles/r02at)
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int e = threadIdx.x; e < w * (w - 1) / 2; e += NT) {
            int i = (int)((sqrtf(8.0f * (float)e + 1.0f) + 1.0f) * 0.5f);  // strict lower (i > j): e = i(i−1)/2 + j
            if (i * (i - 1) / 2 > e) --i;
            if ((i + 1) * i / 2 <= e) ++i;
            const int j = e - i * (i - 1) / 2;
            const double apq = Ap[at(i, j)];
            if (fabs(apq) > floor_abs && apq * apq > 1e-30 * fabs(Ap[at(i, i)] * Ap[at(j, j)])) rotated = 1;
        }
        __syncthreads();
        if (!rotated) break;
        __syncthreads();
    }
    // eigenvalues descending: rank by counting (ties keep index order), one thread per entry
    __shared__ int order[512];
    // (a total order even for NaN input — NaNs rank last, among themselves by index — so `order`
    // is always a permutation: the caller's finiteness verdict arrives after this kernel ran)
    for (int j = threadIdx.x; j < w; j += NT) {
        const double lj = Ap[at(j, j)];
        const bool nj = lj != lj;
        int rank = 0;
        for (int i = 0; i < w; ++i) {
            const double li = Ap[at(i, i)];
            const bool ni = li != li;
            const bool before = ni ? (nj && i < j) : (nj || li > lj || (li == lj && i < j));
            rank += before ? 1 : 0;
        }
        order[rank] = j;
    }
    if (threadIdx.x == 0) {
        *nrounds_out = rounds;
        if (timing) printf("jacobi_packed w=%d threads=%d rounds=%d clocks/round: rotations %lld | updates %lld\n", w, NT,
                           rounds, ta / (rounds ? rounds : 1), tb / (rounds ? rounds : 1));
    }
    __syncthreads();
    for (int j = threadIdx.x; j < w; j += NT) {
        lam[j] = Ap[at(order[j], order[j])];
        order_out[j] = order[j];
    }
}

// V = the product of the logged rotations (V ← V·J per round), rows of V spread over warps:
// every row goes through all rounds independently and within a round the pairs are disjoint, so
// a warp owns JR_RW rows outright (lanes over the round's pairs) and separates rounds with
// __syncwarp only; the CTA shares the staged log.  vout[:, j] = V[:, order[j]].
constexpr int JR_T = 256, JR_RW = 2, JR_ROWS = JR_RW * (JR_T / 32), JR_CHUNK = 4096;  // log entries per chunk (96 KB)
constexpr size_t JR_SMEM = JR_CHUNK * sizeof(JRot) + (size_t)JR_ROWS * 512 * sizeof(double);
__global__ void __launch_bounds__(JR_T) k_jacobi_replay(const JRot* __restrict__ log, const int* __restrict__ nrounds,
                                                        const int* __restrict__ order, int w, double* __restrict__ vout) {
    extern __shared__ uint8_t jr_smem[];
    JRot* stage = reinterpret_cast<JRot*>(jr_smem);                        // a chunk of whole rounds
    double* V = reinterpret_cast<double*>(jr_smem + JR_CHUNK * sizeof(JRot));  // [JR_ROWS][512]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r0 = blockIdx.x * JR_ROWS;
    const int wp = (w + 1) & ~1, half = wp / 2;
    for (int e = threadIdx.x; e < JR_ROWS * wp; e += JR_T) {
        const int rr = e / wp, j = e % wp;
        V[rr * 512 + j] = (r0 + rr < w && j == r0 + rr) ? 1.0 : 0.0;
    }
    double* v0 = V + (warp * JR_RW) * 512;
    double* v1 = v0 + 512;
    const int n = *nrounds, per = JR_CHUNK / half;
    for (int t0 = 0; t0 < n; t0 += per) {
        const int nr = min(per, n - t0);
        __syncthreads();
        for (int e = threadIdx.x; e < nr * half; e += JR_T) stage[e] = log[(int64_t)t0 * half + e];
        __syncthreads();
        for (int t = 0; t < nr; ++t) {
            const JRot* lr = stage + t * half;
            for (int i = lane; i < half; i += 32) {
                const JRot r = lr[i];
                if (r.s == 0.0) continue;
                const double a0 = v0[r.p], b0 = v0[r.q], a1 = v1[r.p], b1 = v1[r.q];
                v0[r.p] = r.c * a0 - r.s * b0;
                v0[r.q] = r.s * a0 + r.c * b0;
                v1[r.p] = r.c * a1 - r.s * b1;
                v1[r.q] = r.s * a1 + r.c * b1;
            }
            __syncwarp();
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < JR_ROWS * w; e += JR_T) {
        const int rr = e / w, j = e % w;
        if (r0 + rr < w) vout[(r0 + rr) + (int64_t)j * w] = V[rr * 512 + order[j]];
    }
}

// ------------------------------------------------ one-sided Jacobi (large w)
// Hestenes one-sided Jacobi on a symmetric PSD G (its singular values are its
// eigenvalues): column pairs of W = G·V are orthogonalised in the same circle-method
// rounds; only column operations (coalesced, in an L2-resident global scratch), one
// barrier per round.  λ_i = ‖W e_i‖, eigenvectors = V e_i.  Used when G does not fit in
// shared memory (the two-sided rotations' row updates would be uncoalesced there).
__global__ void __launch_bounds__(ST) k_jacobi1s(const double* __restrict__ g, int w, int64_t ldg,
                                                 double* __restrict__ W, double* __restrict__ V,
                                                 double* __restrict__ lam, double* __restrict__ vout, int max_sweeps) {
    __shared__ int rotated;
    __shared__ int order[512];
    __shared__ double nrm[512];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wp = (w + 1) & ~1, half = wp / 2, mrot = wp - 1;
    for (int j = warp; j < w; j += NW)
        for (int i = lane; i < w; i += 32) {
            W[i + (int64_t)j * w] = g[i + (int64_t)j * ldg];
            V[i + (int64_t)j * w] = i == j ? 1.0 : 0.0;
        }
    __syncthreads();
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int round = 0; round < mrot; ++round) {
            for (int i = warp; i < half; i += NW) {
                int p = i == 0 ? round : (round + i) % mrot;
                int q = i == 0 ? mrot : (round - i + mrot) % mrot;
                if (p > q) { const int t = p; p = q; q = t; }
                if (q >= w) continue;
                double* wp_ = W + (int64_t)p * w;
                double* wq_ = W + (int64_t)q * w;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int k = lane; k < w; k += 32) {
                    const double x = wp_[k], y = wq_[k];
                    al = fma(x, x, al);
                    be = fma(y, y, be);
                    ga = fma(x, y, ga);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (!(ga * ga > 1e-30 * al * be) || ga == 0.0) continue;  // |γ| ≤ 1e-15·√(αβ): orthogonal
                const double zeta = (be - al) * fast_rcp(2.0 * ga);
                const double q2 = fma(zeta, zeta, 1.0);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) * fast_rcp(fabs(zeta) + q2 * rsqrt(q2));
                const double c = rsqrt(fma(t, t, 1.0)), s = t * c;
                double* vp = V + (int64_t)p * w;
                double* vq = V + (int64_t)q * w;
                for (int k = lane; k < w; k += 32) {
                    const double x = wp_[k], y = wq_[k];
                    wp_[k] = c * x - s * y;
                    wq_[k] = s * x + c * y;
                    const double a = vp[k], b = vq[k];
                    vp[k] = c * a - s * b;
                    vq[k] = s * a + c * b;
                }
                if (lane == 0) rotated = 1;
            }
            __syncthreads();
        }
        if (!rotated) break;
        __syncthreads();
    }
    for (int j = warp; j < w; j += NW) {
        double s = 0.0;
        for (int k = lane; k < w; k += 32) {
            const double x = W[k + (int64_t)j * w];
            s = fma(x, x, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) nrm[j] = sqrt(s);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < w; ++i) order[i] = i;
        for (int i = 0; i < w; ++i) {
            int best = i;
            for (int j = i + 1; j < w; ++j)
                if (nrm[order[j]] > nrm[order[best]]) best = j;
            const int t = order[i]; order[i] = order[best]; order[best] = t;
        }
    }
    __syncthreads();
    for (int j = warp; j < w; j += NW)
        for (int i = lane; i < w; i += 32) vout[i + (int64_t)j * w] = V[i + (int64_t)order[j] * w];
    for (int j = threadIdx.x; j < w; j += ST) lam[j] = nrm[order[j]];
}

void ensure_attrs() {
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_cholesky, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_CHECK(cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
}

}  // namespace

namespace ops {

void cholesky_upper(Ctx* c, const double* g, int64_t w, int64_t ldg, double* r, int64_t ldr, int* info, double* diag,
                    int64_t info_offset, bool chained) {
    if (w > 4096) fail(BCUR_E_INVALID_ARGUMENT, "cholesky_upper: single-CTA path limited to w <= 4096");
    ensure_attrs();
    ProfScope prof(c, "cholesky", w * w * w / 3.0, 8.0 * w * w);
    if (w <= CP_MAX) {
        static bool attr_p = false;
        constexpr size_t smem_p = (size_t)CP_MAX * CP_LD * sizeof(double);
        if (!attr_p) {
            CUDA_CHECK(cudaFuncSetAttribute(k_chol_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p));
            attr_p = true;
        }
        k_chol_panel<<<1, CP_T, smem_p, c->stream>>>(g, (int)w, ldg, r, ldr, info, diag, (int)info_offset,
                                                     chained ? 1 : 0);
        LAUNCH_CHECK(c);
        return;
    }
    DevBuf work;
    size_t smem = 0;
    const size_t bytes = (size_t)w * (size_t)(w | 1) * sizeof(double);
    if (w <= SMEM_MAX_W) smem = bytes;
    else work = DevBuf(c, bytes);
    k_cholesky<<<1, ST, smem, c->stream>>>(g, (int)w, ldg, r, ldr, work.as<double>(), info, diag, (int)info_offset,
                                           chained ? 1 : 0);
    LAUNCH_CHECK(c);
}

void trsm_upper_t(Ctx* c, const double* r, int64_t kb, int64_t ldr, double* p, int64_t ldp, int64_t n) {
    if (kb > 128) fail(BCUR_E_INVALID_ARGUMENT, "trsm_upper_t: kb <= 128");
    if (kb <= 0 || n <= 0) return;
    ProfScope prof(c, "trsm", 1.0 * kb * kb * n, 8.0 * (kb * kb / 2.0 + 2.0 * kb * n));
    constexpr size_t smem = (size_t)(128 + TS_C) * TS_LD * sizeof(double);
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_trsm128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    k_trsm128<<<(unsigned)((n + TS_C - 1) / TS_C), TS_T, smem, c->stream>>>(r, (int)kb, ldr, p, ldp, (int)n);
    LAUNCH_CHECK(c);
}

void tri_inv_upper(Ctx* c, const double* r, int64_t w, int64_t ldr, double* x, int64_t ldx) {
    if (w > TRI_MAX_W) fail(BCUR_E_INVALID_ARGUMENT, "tri_inv_upper: single-CTA path limited to w <= 128");
    if (w == 0) return;
    ProfScope prof(c, "tri_inv", w * w * w / 3.0, 8.0 * w * w);
    static bool attr = false;
    constexpr size_t smem = (size_t)(TRI_LD * TRI_LD + (TRI_MAX_W - TRI_B) * TRI_B) * sizeof(double);
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_tri_inv_upper, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    k_tri_inv_upper<<<1, ST, smem, c->stream>>>(r, (int)w, ldr, x, ldx);
    LAUNCH_CHECK(c);
}

void sym_eig(Ctx* c, const double* g, int64_t w, int64_t ldg, double* lam, double* v) {
    if (w > 512) fail(BCUR_E_INVALID_ARGUMENT, "sym_eig: w > 512 not supported");
    if (w <= 0) return;
    ensure_attrs();
    ProfScope prof(c, "sym_eig", 0.0, 8.0 * w * w);
    const size_t packed = (size_t)w * (w + 1) / 2 * sizeof(double);
    static const char* legacy = getenv("BCUR_JACOBI_LEGACY");
    if (packed <= 200 * 1024 && !(legacy && legacy[0] == '1')) {
        // packed two-sided rounds + logged rotations replayed onto V across SMs
        static bool attr = false;
        if (!attr) {
            CUDA_CHECK(cudaFuncSetAttribute(k_jacobi_packed, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            attr = true;
        }
        static bool timing_set = false;
        if (!timing_set) {
            const char* t = getenv("BCUR_JACOBI_TIMING");
            const int on = (t && t[0] == '1') ? 1 : 0;
            if (on) CUDA_CHECK(cudaMemcpyToSymbol(g_jac_timing, &on, sizeof on));
            timing_set = true;
        }
        constexpr int max_sweeps = 40;
        const int64_t half = (w + 1) / 2, rounds_max = (int64_t)max_sweeps * (2 * half - 1);
        DevBuf log(c, (size_t)rounds_max * half * sizeof(JRot)), meta(c, (size_t)(w + 16) * sizeof(int));
        int* nrounds = meta.as<int>();
        int* order = nrounds + 16;
        // threads: one per 2×2 block of a round (fewer warps per barrier for small w).  A full-square
        // variant whose warps read contiguous runs (the circle method's r ± i pairs) measured slower:
        // 1616 vs 1066 update cycles per round at ℓ = 60 (twice the blocks, profiles/r02y)
        const int64_t nblk = half * (half + 1) / 2;
        const int nt = (int)std::min<int64_t>(JP_T, std::max<int64_t>(128, (nblk + 127) / 128 * 128));
        k_jacobi_packed<<<1, nt, packed, c->stream>>>(g, (int)w, ldg, log.as<JRot>(), nrounds, lam, order,
                                                      max_sweeps);
        LAUNCH_CHECK(c);
        static bool attr_r = false;
        if (!attr_r) {
            CUDA_CHECK(cudaFuncSetAttribute(k_jacobi_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)JR_SMEM));
            attr_r = true;
        }
        k_jacobi_replay<<<(unsigned)((w + JR_ROWS - 1) / JR_ROWS), JR_T, JR_SMEM, c->stream>>>(
            log.as<JRot>(), nrounds, order, (int)w, v);
        if (getenv("BCUR_JACOBI_DEBUG")) {
            int hr = 0;
            CUDA_CHECK(cudaMemcpyAsync(&hr, nrounds, sizeof hr, cudaMemcpyDeviceToHost, c->stream));
            CUDA_CHECK(cudaStreamSynchronize(c->stream));
            fprintf(stderr, "sym_eig w=%d rounds=%d sweeps=%.1f\n", (int)w, hr, hr / (double)(2 * half - 1));
        }
        LAUNCH_CHECK(c);
        return;
    }
    // A and V both in shared memory when they fit (every rotation updates two rows and
    // two columns of each; a global V made a 64×64 solve take 3.4 ms)
    const size_t mat = (size_t)w * (size_t)(w | 1) * sizeof(double);
    DevBuf work, vtmp;
    size_t smem = 0;
    if (2 * mat > 200 * 1024) {  // too big for shared memory: one-sided, column-coalesced
        work = DevBuf(c, (size_t)w * w * sizeof(double));
        vtmp = DevBuf(c, (size_t)w * w * sizeof(double));
        k_jacobi1s<<<1, ST, 0, c->stream>>>(g, (int)w, ldg, work.as<double>(), vtmp.as<double>(), lam, v, 40);
        LAUNCH_CHECK(c);
        return;
    }
    smem = 2 * mat;
    static const int dbg = getenv("BCUR_JACOBI_DEBUG") ? -1 : 1;
    k_jacobi<<<1, ST, smem, c->stream>>>(g, (int)w, ldg, work.as<double>(), vtmp.as<double>(), lam, v, 40 * dbg);
    LAUNCH_CHECK(c);
}

}  // namespace ops
}  // namespace bcur_b200
