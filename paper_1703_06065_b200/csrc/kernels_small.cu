// kernels_small.cu — single-CTA fp64 factorizations of the small (≤ a few
// hundred) matrices of the hot path: Cholesky (CholQR2 of the sketch / C panels),
// triangular inverse, and a parallel-ordered cyclic Jacobi eigensolver (SVQB
// rank revealing and the ℓ×ℓ eigenproblem of B·Bᵀ that replaces the reference's
// BDCSVD, matcore.cpp:39-56).  The working matrix sits in shared memory when it
// fits (w ≤ 144) and in an L2-resident global scratch otherwise.
#include "ops.h"

namespace bcur_b200 {
namespace {

constexpr int ST = 1024;
constexpr int64_t SMEM_MAX_W = 144;

// --------------------------------------------------------------- Cholesky
__global__ void __launch_bounds__(ST) k_cholesky(const double* __restrict__ g, int64_t w, int64_t ldg,
                                                 double* __restrict__ r, double* __restrict__ work, int* info,
                                                 double* mindiag) {
    extern __shared__ double sm[];
    double* M = work ? work : sm;  // column-major w×w
    __shared__ int stop;
    __shared__ double rdiag;
    for (int64_t e = threadIdx.x; e < w * w; e += ST) M[e] = g[(e % w) + (e / w) * ldg];
    if (threadIdx.x == 0) {
        stop = 0;
        double mx = 0.0;
        for (int64_t j = 0; j < w; ++j) mx = fmax(mx, g[j + j * ldg]);
        mindiag[1] = mx;
    }
    __syncthreads();
    double mn = INFINITY;
    for (int64_t j = 0; j < w; ++j) {
        if (threadIdx.x == 0) {
            const double d = M[j + j * w];
            if (!(d > 0.0) || !isfinite(d)) {
                stop = (int)j + 1;
            } else {
                rdiag = sqrt(d);
                M[j + j * w] = rdiag;
            }
        }
        __syncthreads();
        if (stop) break;
        const double rj = rdiag;
        if (threadIdx.x == 0) mn = fmin(mn, rj);
        for (int64_t k = j + 1 + threadIdx.x; k < w; k += ST) M[j + k * w] /= rj;
        __syncthreads();
        const int64_t t = w - j - 1;
        for (int64_t e = threadIdx.x; e < t * t; e += ST) {
            const int64_t i = j + 1 + e % t, k = j + 1 + e / t;
            if (i <= k) M[i + k * w] = fma(-M[j + i * w], M[j + k * w], M[i + k * w]);
        }
        __syncthreads();
    }
    for (int64_t e = threadIdx.x; e < w * w; e += ST) {
        const int64_t i = e % w, k = e / w;
        r[e] = i <= k ? M[e] : 0.0;
    }
    if (threadIdx.x == 0) {
        *info = stop;
        *mindiag = stop ? 0.0 : mn;
    }
}

// ------------------------------------------------------ triangular inverse
__global__ void __launch_bounds__(ST) k_tri_inv_upper(const double* __restrict__ r, int64_t w, double* __restrict__ x,
                                                      bool use_smem) {
    extern __shared__ double sm[];
    const double* R = r;
    if (use_smem) {
        for (int64_t e = threadIdx.x; e < w * w; e += ST) sm[e] = r[e];
        __syncthreads();
        R = sm;
    }
    for (int64_t c = threadIdx.x; c < w; c += ST) {
        for (int64_t i = c + 1; i < w; ++i) x[i + c * w] = 0.0;
        x[c + c * w] = 1.0 / R[c + c * w];
        for (int64_t i = c - 1; i >= 0; --i) {
            double s = 0.0;
            for (int64_t t = i + 1; t <= c; ++t) s = fma(R[i + t * w], x[t + c * w], s);
            x[i + c * w] = -s / R[i + i * w];
        }
    }
}

// ---------------------------------------------------------------- Jacobi
// Parallel (round-robin) cyclic Jacobi; A (w×w, column-major) in `A`, V (w×w) in `V`.
__global__ void __launch_bounds__(ST) k_jacobi(const double* __restrict__ g, int64_t w, int64_t ldg,
                                               double* __restrict__ Aglob, double* __restrict__ V,
                                               double* __restrict__ lam, double* __restrict__ vout, int max_sweeps) {
    extern __shared__ double sm[];
    double* A = Aglob ? Aglob : sm;
    __shared__ int pos[512];
    __shared__ double cs[256], sn[256];
    __shared__ int pp[256], qq[256];
    __shared__ int rotated;
    const int64_t wp = (w + 1) & ~1LL;  // even number of players (w..wp-1 is a bye)
    const int half = (int)(wp / 2);
    for (int64_t e = threadIdx.x; e < w * w; e += ST) {
        const int64_t i = e % w, j = e / w;
        A[e] = g[i + j * ldg];
        V[e] = i == j ? 1.0 : 0.0;
    }
    for (int i = threadIdx.x; i < wp; i += ST) pos[i] = i;
    // absolute floor: off-diagonal rounding noise of the input (≈ eps·‖G‖_F) is not rotated away
    __shared__ double floor_abs;
    if (threadIdx.x == 0) {
        double f = 0.0;
        for (int64_t j = 0; j < w; ++j) f = fmax(f, fabs(g[j + j * ldg]));
        floor_abs = 1e-17 * f * (double)w;
    }
    __syncthreads();
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int round = 0; round < wp - 1; ++round) {
            // pair i: pos[i] vs pos[wp-1-i]
            for (int i = threadIdx.x; i < half; i += ST) {
                int p = pos[i], q = pos[wp - 1 - i];
                if (p > q) { const int t = p; p = q; q = t; }
                double c = 1.0, s = 0.0;
                if (q < w) {
                    const double apq = A[p + q * w];
                    const double app = A[p + p * w], aqq = A[q + q * w];
                    if (fabs(apq) > floor_abs && fabs(apq) > 1e-16 * sqrt(fabs(app * aqq))) {
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                        rotated = 1;
                    }
                }
                pp[i] = p;
                qq[i] = q;
                cs[i] = c;
                sn[i] = s;
            }
            __syncthreads();
            // rows: A ← Jᵀ A
            for (int64_t e = threadIdx.x; e < (int64_t)half * w; e += ST) {
                const int i = (int)(e % half);
                const int64_t k = e / half;
                const int p = pp[i], q = qq[i];
                if (q >= w || sn[i] == 0.0) continue;
                const double c = cs[i], s = sn[i];
                const double ap = A[p + k * w], aq = A[q + k * w];
                A[p + k * w] = c * ap - s * aq;
                A[q + k * w] = s * ap + c * aq;
            }
            __syncthreads();
            // columns: A ← A J, V ← V J
            for (int64_t e = threadIdx.x; e < (int64_t)half * w; e += ST) {
                const int i = (int)(e % half);
                const int64_t k = e / half;
                const int p = pp[i], q = qq[i];
                if (q >= w || sn[i] == 0.0) continue;
                const double c = cs[i], s = sn[i];
                const double ap = A[k + p * w], aq = A[k + q * w];
                A[k + p * w] = c * ap - s * aq;
                A[k + q * w] = s * ap + c * aq;
                const double vp = V[k + p * w], vq = V[k + q * w];
                V[k + p * w] = c * vp - s * vq;
                V[k + q * w] = s * vp + c * vq;
            }
            __syncthreads();
            // rotate positions 1..wp-1
            if (threadIdx.x == 0) {
                const int last = pos[wp - 1];
                for (int i = (int)wp - 1; i > 1; --i) pos[i] = pos[i - 1];
                pos[1] = last;
            }
            __syncthreads();
        }
        if (!rotated) break;
        __syncthreads();
    }
    // sort eigenvalues descending (stable selection on indices), permute V
    __shared__ int order[512];
    if (threadIdx.x == 0) {
        for (int i = 0; i < w; ++i) order[i] = i;
        for (int i = 0; i < w; ++i) {
            int best = i;
            for (int j = i + 1; j < w; ++j)
                if (A[order[j] + order[j] * w] > A[order[best] + order[best] * w]) best = j;
            const int t = order[i]; order[i] = order[best]; order[best] = t;
        }
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < w * w; e += ST) {
        const int64_t i = e % w, j = e / w;
        vout[i + j * w] = V[i + (int64_t)order[j] * w];
    }
    for (int64_t j = threadIdx.x; j < w; j += ST) lam[j] = A[order[j] + (int64_t)order[j] * w];
}

void ensure_attrs() {
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_cholesky, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_CHECK(cudaFuncSetAttribute(k_tri_inv_upper, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_CHECK(cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
}

}  // namespace

namespace ops {

void cholesky_upper(Ctx* c, const double* g, int64_t w, int64_t ldg, double* r, int* info, double* mindiag) {
    DevBuf work;
    size_t smem = 0;
    if (w <= SMEM_MAX_W) {
        smem = (size_t)w * w * sizeof(double);
    } else {
        work = DevBuf(c, (size_t)w * w * sizeof(double));
    }
    ensure_attrs();
    ProfScope prof(c, "cholesky", w * w * w / 3.0, 8.0 * w * w);
    k_cholesky<<<1, ST, smem, c->stream>>>(g, w, ldg, r, work.as<double>(), info, mindiag);
    LAUNCH_CHECK(c);
}

void tri_inv_upper(Ctx* c, const double* r, int64_t w, double* x) {
    ensure_attrs();
    ProfScope prof(c, "tri_inv", w * w * w / 3.0, 8.0 * w * w);
    const bool use = w <= SMEM_MAX_W;
    k_tri_inv_upper<<<1, ST, use ? (size_t)w * w * sizeof(double) : 0, c->stream>>>(r, w, x, use);
    LAUNCH_CHECK(c);
}

void sym_eig(Ctx* c, const double* g, int64_t w, int64_t ldg, double* lam, double* v) {
    if (w > 512) fail(BCUR_E_INVALID_ARGUMENT, "sym_eig: w > 512 not supported");
    ensure_attrs();
    ProfScope prof(c, "sym_eig", 0.0, 8.0 * w * w);
    DevBuf work, vtmp(c, (size_t)w * w * sizeof(double));
    size_t smem = 0;
    if (w <= SMEM_MAX_W) smem = (size_t)w * w * sizeof(double);
    else work = DevBuf(c, (size_t)w * w * sizeof(double));
    k_jacobi<<<1, ST, smem, c->stream>>>(g, w, ldg, work.as<double>(), vtmp.as<double>(), lam, v, 40);
    LAUNCH_CHECK(c);
}

}  // namespace ops
}  // namespace bcur_b200
