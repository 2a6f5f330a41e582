// Times the single-CTA factorization kernels in isolation (includes kernels_small.cu).
#include "../paper_1703_06065_b200/csrc/kernels_small.cu"

#include <cstdio>
#include <vector>
namespace bcur_b200 { namespace {

__global__ void __launch_bounds__(CP_T) k_chol_panel_t(const double* g, int w, int64_t ldg, double* r, int64_t ldr,
                                                     int* info, double* diag, int info_offset, int chained, long long* tt) {
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
    long long t0 = clock64(), t1 = 0, t2 = 0, t3 = 0;
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
        t1 += clock64() - t0; t0 = clock64();
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
        t2 += clock64() - t0; t0 = clock64();
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
        t3 += clock64() - t0; t0 = clock64();
    }
    if (threadIdx.x == 0) { tt[0] = t1; tt[1] = t2; tt[2] = t3; }
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

} }
using namespace bcur_b200;
int main() {
    for (int w : {20, 60, 128}) {
        std::vector<double> h(w * w);
        for (int j = 0; j < w; ++j)
            for (int i = 0; i < w; ++i) h[i + j * w] = (i == j ? w + 1.0 : 0.0) + 1.0 / (1 + i + j);
        double *g, *r, *diag; int* info;
        cudaMalloc(&g, w * w * 8); cudaMalloc(&r, w * w * 8); cudaMalloc(&diag, 64); cudaMalloc(&info, 64);
        cudaMemcpy(g, h.data(), w * w * 8, cudaMemcpyHostToDevice);
        constexpr size_t smem_p = (size_t)CP_MAX * CP_LD * sizeof(double);
        cudaFuncSetAttribute(k_chol_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
        cudaFuncSetAttribute(k_cholesky, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            for (int it = 0; it < 20; ++it) k_chol_panel<<<1, CP_T, smem_p>>>(g, w, w, r, w, info, diag, 0, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            cudaEventRecord(e0);
            for (int it = 0; it < 20; ++it)
                k_cholesky<<<1, ST, (size_t)w * (w | 1) * 8>>>(g, w, w, r, w, nullptr, info, diag, 0, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms2; cudaEventElapsedTime(&ms2, e0, e1);
            long long* tt; cudaMalloc(&tt, 64);
            cudaFuncSetAttribute(k_chol_panel_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
            k_chol_panel_t<<<1, CP_T, smem_p>>>(g, w, w, r, w, info, diag, 0, 0, tt);
            long long ht[3]; cudaMemcpy(ht, tt, 24, cudaMemcpyDeviceToHost);
            if (rep == 2) printf("  phase cycles: diag %lld trsm %lld syrk %lld\n", ht[0], ht[1], ht[2]);
            if (rep == 2) printf("w=%d  chol_panel %.1f us  cholesky %.1f us  (%s)\n", w, ms * 1000 / 20, ms2 * 1000 / 20,
                                 cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
