// kernels_gen.cu — counter-based generators (Philox4x32-10): the Rademacher
// sketch Ω of the range finder and the synthetic inputs of the five configs
// (K14).  Every value is a pure function of (key, stream, element index), so a
// column shard generates exactly the columns the full matrix would have, and the
// numpy oracle (oracle/bcur_oracle.py: philox4x32, omega, gaussian) reproduces
// Ω bit-for-bit.
#include "ops.h"

namespace bcur_b200 {

__device__ __forceinline__ void philox4x32_10(uint64_t key, uint32_t c[4]) {
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__device__ __forceinline__ double gauss_at(uint64_t key, uint32_t stream, uint64_t e) {
    uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), 0u, stream};
    philox4x32_10(key, c);
    const uint64_t a = ((((uint64_t)c[0]) << 32) | c[1]) >> 11;
    const uint64_t b = ((((uint64_t)c[2]) << 32) | c[3]) >> 11;
    const double u1 = 1.0 - (double)a * 0x1.0p-53;
    const double u2 = (double)b * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

__device__ __forceinline__ double uniform_at(uint64_t key, uint32_t stream, uint64_t e) {
    uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), 0u, stream};
    philox4x32_10(key, c);
    const uint64_t a = ((((uint64_t)c[0]) << 32) | c[1]) >> 11;
    return (double)a * 0x1.0p-53;
}

namespace {

constexpr uint32_t STREAM_OMEGA = 0x4F4D4547u, STREAM_E = 3, STREAM_WALK = 4, STREAM_LOAD = 5, STREAM_PHASE = 6;

// one thread per (row, group of 128 sketch columns)
__global__ void k_omega(uint64_t key, int64_t n_rows, int64_t row0, int64_t l, double* __restrict__ out, int64_t ld) {
    const int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int grp = blockIdx.y;
    if (jj >= n_rows) return;
    const uint64_t j = (uint64_t)(row0 + jj);
    uint32_t c[4] = {(uint32_t)j, (uint32_t)(j >> 32), (uint32_t)grp, STREAM_OMEGA};
    philox4x32_10(key, c);
    const int cmax = (int)imin64(128, l - (int64_t)grp * 128);
    for (int b = 0; b < cmax; ++b) {
        const uint32_t bit = (c[b >> 5] >> (b & 31)) & 1u;
        out[jj + ((int64_t)grp * 128 + b) * ld] = bit ? -1.0 : 1.0;
    }
}

__global__ void k_gauss(uint64_t key, uint32_t stream, int64_t m, int64_t n, double* __restrict__ out, int64_t ld) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m * n) return;
    const int64_t i = e % m, j = e / m;
    out[i + j * ld] = gauss_at(key, stream, (uint64_t)e);
}

// A(:, jj) for global column j = col0 + jj:  Σ_t us(i,t)·v(j,t) (ordered, unfused) + ν·E(i,j)
template <class T>
__global__ void __launch_bounds__(256) k_lowrank(const double* __restrict__ us, const double* __restrict__ v,
                                                 int64_t m, int64_t n, int64_t r, int64_t col0, int64_t n_global,
                                                 double noise, uint64_t key, T* __restrict__ a, int64_t lda) {
    __shared__ double su[16][64];
    __shared__ double sv[16][64];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t i0 = (int64_t)blockIdx.x * 64, j0 = (int64_t)blockIdx.y * 64;
    double acc[4][4] = {};
    for (int64_t t0 = 0; t0 < r; t0 += 16) {
        for (int e = tid; e < 16 * 64; e += 256) {
            const int ii = e & 63, tt = e >> 6;
            const int64_t gi = i0 + ii, gj = col0 + j0 + ii, gt = t0 + tt;
            su[tt][ii] = (gi < m && gt < r) ? us[gi + gt * m] : 0.0;
            sv[tt][ii] = (j0 + ii < n && gt < r) ? v[gj + gt * n_global] : 0.0;
        }
        __syncthreads();
        const int tmax = (int)imin64(16, r - t0);
        for (int tt = 0; tt < tmax; ++tt) {
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y)
                    acc[x][y] = __dadd_rn(acc[x][y], __dmul_rn(su[tt][ty + 16 * x], sv[tt][tx + 16 * y]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
        const int64_t gi = i0 + ty + 16 * x;
        if (gi >= m) continue;
#pragma unroll
        for (int y = 0; y < 4; ++y) {
            const int64_t jj = j0 + tx + 16 * y;
            if (jj >= n) continue;
            double val = acc[x][y];
            if (noise > 0.0) {
                const uint64_t e = (uint64_t)gi + (uint64_t)(col0 + jj) * (uint64_t)m;
                val = __dadd_rn(val, __dmul_rn(noise, gauss_at(key, STREAM_E, e)));
            }
            a[gi + jj * lda] = (T)val;
        }
    }
}

// Config-2 surrogate: per row, trailing moving average of a Gaussian random walk
// plus 5 cosine trends with Gaussian loadings (oracle: gen_biometric).
template <class T>
__global__ void k_biometric(int64_t m, int64_t n, int64_t col0, int64_t n_global, uint64_t key, T* __restrict__ a,
                            int64_t lda) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    constexpr int W = 50, NT = 5;
    double load[NT], phase[NT];
    for (int t = 0; t < NT; ++t) {
        load[t] = gauss_at(key, STREAM_LOAD, (uint64_t)(i + t * m));
        phase[t] = 2.0 * 3.141592653589793 * uniform_at(key, STREAM_PHASE, (uint64_t)t);
    }
    // cs[j+1] = Σ_{t≤j} walk[t]; keep a ring of the last W+1 prefix sums
    double ring[W + 1];
    ring[0] = 0.0;
    double walk = 0.0, cs = 0.0;
    for (int64_t j = 0; j < col0 + n; ++j) {
        walk += 0.05 * gauss_at(key, STREAM_WALK, (uint64_t)(i + j * m));
        cs += walk;
        ring[(j + 1) % (W + 1)] = cs;
        if (j < col0) continue;
        const int64_t lo = j + 1 - W > 0 ? j + 1 - W : 0;
        const double ma = (cs - ring[lo % (W + 1)]) / (double)(j + 1 - lo);
        double tr = 0.0;
        for (int t = 0; t < NT; ++t) tr += load[t] * cos(2.0 * 3.141592653589793 * (t + 1) * (double)j / (double)n_global + phase[t]);
        a[i + (j - col0) * lda] = (T)(ma + tr);
    }
}

inline unsigned nblk(int64_t count) { return (unsigned)((count + 255) / 256); }

}  // namespace

namespace ops {

void omega(Ctx* c, uint64_t key, int64_t n_rows, int64_t row0, int64_t l, double* out, int64_t ld) {
    if (n_rows <= 0 || l <= 0) return;
    dim3 grid(nblk(n_rows), (unsigned)((l + 127) / 128));
    k_omega<<<grid, 256, 0, c->stream>>>(key, n_rows, row0, l, out, ld);
    LAUNCH_CHECK(c);
}

void gaussian_matrix(Ctx* c, uint64_t key, uint32_t stream, int64_t m, int64_t n, double* out, int64_t ld) {
    if (m * n == 0) return;
    k_gauss<<<nblk(m * n), 256, 0, c->stream>>>(key, stream, m, n, out, ld);
    LAUNCH_CHECK(c);
}

void lowrank_assemble(Ctx* c, const double* us, const double* v, int64_t m, int64_t n, int64_t r, int64_t col0,
                      int64_t n_global, double noise, uint64_t seed, void* a, int dt, int64_t lda) {
    dim3 grid((unsigned)((m + 63) / 64), (unsigned)((n + 63) / 64));
    if (dt == BCUR_F32)
        k_lowrank<float><<<grid, 256, 0, c->stream>>>(us, v, m, n, r, col0, n_global, noise, seed, (float*)a, lda);
    else
        k_lowrank<double><<<grid, 256, 0, c->stream>>>(us, v, m, n, r, col0, n_global, noise, seed, (double*)a, lda);
    LAUNCH_CHECK(c);
}

void biometric(Ctx* c, int64_t m, int64_t n, int64_t col0, int64_t n_global, uint64_t seed, void* a, int dt,
               int64_t lda) {
    if (dt == BCUR_F32)
        k_biometric<float><<<(unsigned)((m + 63) / 64), 64, 0, c->stream>>>(m, n, col0, n_global, seed, (float*)a, lda);
    else
        k_biometric<double><<<(unsigned)((m + 63) / 64), 64, 0, c->stream>>>(m, n, col0, n_global, seed, (double*)a, lda);
    LAUNCH_CHECK(c);
}

}  // namespace ops
}  // namespace bcur_b200
