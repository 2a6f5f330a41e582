// kernels_misc.cu — layout/elementwise helpers (dtype conversion, transposes, scaling, copies).
#include "ops.h"
#include <cuda_fp16.h>

namespace bcur_b200 {
namespace {

template <class TS, class TD>
__global__ void k_convert(const TS* __restrict__ src, int64_t m, int64_t n, int64_t lds, TD* __restrict__ dst,
                          int64_t ldd) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m * n) return;
    const int64_t i = e % m, j = e / m;
    dst[i + j * ldd] = (TD)src[i + j * lds];
}

template <class TS, class TD>
__global__ void k_transpose(const TS* __restrict__ src, int64_t m, int64_t n, int64_t lds, TD* __restrict__ dst,
                            int64_t ldd) {
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + threadIdx.x, j = j0 + r;
        if (i < m && j < n) tile[r][threadIdx.x] = (double)src[i + j * lds];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + threadIdx.x, i = i0 + r;  // dst(j, i) = src(i, j)
        if (i < m && j < n) dst[j + i * ldd] = (TD)tile[threadIdx.x][r];
    }
}

// Several contiguous device → device copies in one launch (the selected blocks of a column
// basis: c3 gathered its 32 blocks and their exponents with 64 dependent cudaMemcpyAsync calls,
// 0.4 ms of a 21 ms step — profiles/r02an/step_c3.txt).  Every segment is a multiple of 4 bytes;
// 16-byte aligned ones move as uint4.  grid = (chunks, segments).
__global__ void __launch_bounds__(256) k_copy_segments(const ops::CopySeg* __restrict__ segs) {
    const ops::CopySeg sg = segs[blockIdx.y];
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
    const bool a16 = ((((uintptr_t)sg.src) | ((uintptr_t)sg.dst) | (uintptr_t)sg.bytes) & 15) == 0;
    if (a16) {
        const uint4* s = reinterpret_cast<const uint4*>(sg.src);
        uint4* d = reinterpret_cast<uint4*>(sg.dst);
        const size_t n = sg.bytes / 16;
        size_t i = tid;
        for (; i + 3 * nth < n; i += 4 * nth) {  // four independent loads in flight per thread
            const uint4 v0 = s[i], v1 = s[i + nth], v2 = s[i + 2 * nth], v3 = s[i + 3 * nth];
            d[i] = v0; d[i + nth] = v1; d[i + 2 * nth] = v2; d[i + 3 * nth] = v3;
        }
        for (; i < n; i += nth) d[i] = s[i];
    } else {
        const uint32_t* s = reinterpret_cast<const uint32_t*>(sg.src);
        uint32_t* d = reinterpret_cast<uint32_t*>(sg.dst);
        const size_t n = sg.bytes / 4;
        for (size_t i = tid; i < n; i += nth) d[i] = s[i];
    }
}

__global__ void k_count_nonfinite(const double* __restrict__ x, int64_t count, unsigned int* __restrict__ flag) {
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[e]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

__global__ void k_fill(double* p, int64_t count, double v) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < count) p[e] = v;
}

__global__ void k_scale_columns(double* x, int64_t m, int64_t n, int64_t ld, const double* __restrict__ s) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m * n) return;
    const int64_t i = e % m, j = e / m;
    x[i + j * ld] *= s[j];
}

// out[k] = Σ over the row ranges [r0, r1) (pairs) of v(i, k)², one block per column k
__global__ void k_colsumsq_ranges(const double* __restrict__ v, int64_t ld, const int64_t* __restrict__ ranges, int nr,
                                  double* __restrict__ out) {
    const double* col = v + (int64_t)blockIdx.x * ld;
    double s = 0.0;
    for (int r = 0; r < nr; ++r)
        for (int64_t i = ranges[2 * r] + threadIdx.x; i < ranges[2 * r + 1]; i += blockDim.x) s = fma(col[i], col[i], s);
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        out[blockIdx.x] = t;
    }
}

// s[k] = σ[k]·sqrt(max(0, 1 − lev[k]))
__global__ void k_sigma_weights(const double* __restrict__ sigma, const double* __restrict__ lev, int n,
                                double* __restrict__ s) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) s[k] = sigma[k] * sqrt(fmax(0.0, 1.0 - lev[k]));
}

__global__ void k_scale_rows(double* x, int64_t m, int64_t n, int64_t ld, const double* __restrict__ s) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m * n) return;
    const int64_t i = e % m, j = e / m;
    x[i + j * ld] *= s[i];
}

__global__ void k_axpy_neg(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) y[e] -= x[e];
}

__global__ void k_zero_lower(double* x, int64_t w, int64_t ld) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= w * w) return;
    const int64_t i = e % w, j = e / w;
    if (i > j) x[i + j * ld] = 0.0;
}

__global__ void k_near_identity_rinv(const double* __restrict__ g, int64_t w, int64_t ldg, double* __restrict__ x,
                                     double one) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= w * w) return;
    const int64_t i = e % w, j = e / w;
    double v = 0.0;
    if (i == j) v = one - 0.5 * (g[i + j * ldg] - 1.0);
    else if (i < j) v = -g[i + j * ldg];
    x[i + j * w] = v;
}

inline unsigned nblk(int64_t count) { return (unsigned)((count + 255) / 256); }

}  // namespace

__global__ void k_f16_to_f32(const uint16_t* __restrict__ src, int64_t count, float scale, float* __restrict__ dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) dst[i] = __half2float(__ushort_as_half(src[i])) * scale;
}

namespace ops {

void f16_to_f32(Ctx* c, const uint16_t* src, int64_t count, float scale, float* dst) {
    if (count <= 0) return;
    k_f16_to_f32<<<nblk(count), 256, 0, c->stream>>>(src, count, scale, dst);
    LAUNCH_CHECK(c);
}

void convert(Ctx* c, const void* src, int dts, int64_t m, int64_t n, int64_t lds, void* dst, int dtd, int64_t ldd) {
    if (m * n == 0) return;
    const unsigned g = nblk(m * n);
    if (dts == BCUR_F32 && dtd == BCUR_F32)
        k_convert<float, float><<<g, 256, 0, c->stream>>>((const float*)src, m, n, lds, (float*)dst, ldd);
    else if (dts == BCUR_F32)
        k_convert<float, double><<<g, 256, 0, c->stream>>>((const float*)src, m, n, lds, (double*)dst, ldd);
    else if (dtd == BCUR_F32)
        k_convert<double, float><<<g, 256, 0, c->stream>>>((const double*)src, m, n, lds, (float*)dst, ldd);
    else
        k_convert<double, double><<<g, 256, 0, c->stream>>>((const double*)src, m, n, lds, (double*)dst, ldd);
    LAUNCH_CHECK(c);
}

void copy_segments(Ctx* c, const CopySeg* d_segs, int nsegs, size_t max_bytes) {
    if (nsegs <= 0 || max_bytes == 0) return;
    // ~4 CTAs per SM in total, each thread moving at least a few 16-byte words
    const size_t per = std::max<size_t>(1, (size_t)(4 * c->sm_count + nsegs - 1) / nsegs);
    const size_t want = (max_bytes / 16 + 256 * 4 - 1) / (256 * 4);
    const unsigned chunks = (unsigned)std::max<size_t>(1, std::min(per, want));
    k_copy_segments<<<dim3(chunks, (unsigned)nsegs), 256, 0, c->stream>>>(d_segs);
    LAUNCH_CHECK(c);
}

void convert_to_f64(Ctx* c, const void* src, int dt, int64_t m, int64_t n, int64_t lds, double* dst, int64_t ldd) {
    convert(c, src, dt, m, n, lds, dst, BCUR_F64, ldd);
}

void transpose(Ctx* c, const void* src, int dts, int64_t m, int64_t n, int64_t lds, void* dst, int dtd, int64_t ldd) {
    if (m * n == 0) return;
    dim3 grid((unsigned)((m + 31) / 32), (unsigned)((n + 31) / 32));
    dim3 block(32, 8);
    if (dts == BCUR_F32 && dtd == BCUR_F32)
        k_transpose<float, float><<<grid, block, 0, c->stream>>>((const float*)src, m, n, lds, (float*)dst, ldd);
    else if (dts == BCUR_F32)
        k_transpose<float, double><<<grid, block, 0, c->stream>>>((const float*)src, m, n, lds, (double*)dst, ldd);
    else if (dtd == BCUR_F32)
        k_transpose<double, float><<<grid, block, 0, c->stream>>>((const double*)src, m, n, lds, (float*)dst, ldd);
    else
        k_transpose<double, double><<<grid, block, 0, c->stream>>>((const double*)src, m, n, lds, (double*)dst, ldd);
    LAUNCH_CHECK(c);
}

void transpose_to_f64(Ctx* c, const void* src, int dt, int64_t m, int64_t n, int64_t lds, double* dst, int64_t ldd) {
    transpose(c, src, dt, m, n, lds, dst, BCUR_F64, ldd);
}

void flag_nonfinite(Ctx* c, const double* x, int64_t count, unsigned int* d_flag) {
    if (count <= 0) return;
    const unsigned g = (unsigned)std::min<int64_t>((count + 255) / 256, 4LL * c->sm_count);
    k_count_nonfinite<<<g, 256, 0, c->stream>>>(x, count, d_flag);
    LAUNCH_CHECK(c);
}

void fill_f64(Ctx* c, double* p, int64_t count, double v) {
    if (count <= 0) return;
    k_fill<<<nblk(count), 256, 0, c->stream>>>(p, count, v);
    LAUNCH_CHECK(c);
}

void axpy_neg(Ctx* c, const double* x, double* y, int64_t n) {
    if (n <= 0) return;
    k_axpy_neg<<<nblk(n), 256, 0, c->stream>>>(x, y, n);
    LAUNCH_CHECK(c);
}

void scale_columns(Ctx* c, double* x, int64_t m, int64_t n, int64_t ld, const double* d_scale) {
    if (m * n == 0) return;
    k_scale_columns<<<nblk(m * n), 256, 0, c->stream>>>(x, m, n, ld, d_scale);
    LAUNCH_CHECK(c);
}

void colsumsq_ranges(Ctx* c, const double* v, int64_t ld, int64_t k, const int64_t* d_ranges, int nr, double* d_out) {
    if (k <= 0) return;
    k_colsumsq_ranges<<<(unsigned)k, 256, 0, c->stream>>>(v, ld, d_ranges, nr, d_out);
    LAUNCH_CHECK(c);
}

void sigma_weights(Ctx* c, const double* d_sigma, const double* d_lev, int64_t n, double* d_scale) {
    if (n <= 0) return;
    k_sigma_weights<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(d_sigma, d_lev, (int)n, d_scale);
    LAUNCH_CHECK(c);
}

void scale_rows(Ctx* c, double* x, int64_t m, int64_t n, int64_t ld, const double* d_scale) {
    if (m <= 0 || n <= 0) return;
    k_scale_rows<<<nblk(m * n), 256, 0, c->stream>>>(x, m, n, ld, d_scale);
    LAUNCH_CHECK(c);
}

void copy_f64(Ctx* c, const double* src, int64_t m, int64_t n, int64_t lds, double* dst, int64_t ldd) {
    convert(c, src, BCUR_F64, m, n, lds, dst, BCUR_F64, ldd);
}

void near_identity_rinv(Ctx* c, const double* g, int64_t w, int64_t ldg, double* x, bool minus_identity) {
    if (w <= 0) return;
    k_near_identity_rinv<<<nblk(w * w), 256, 0, c->stream>>>(g, w, ldg, x, minus_identity ? 0.0 : 1.0);
    LAUNCH_CHECK(c);
}

void zero_lower(Ctx* c, double* x, int64_t w, int64_t ld) {
    if (w <= 0) return;
    k_zero_lower<<<nblk(w * w), 256, 0, c->stream>>>(x, w, ld);
    LAUNCH_CHECK(c);
}

}  // namespace ops
}  // namespace bcur_b200
