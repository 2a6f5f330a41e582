// kernels_reduce.cu — HBM-streaming reductions with fp64 accumulation.
//
//  * block_sumsq      ‖A_g‖_F² per column block (sketch.cpp:21-26), whose sum is
//                     ‖A‖_F² (matcore.cpp:93-95).  Pure streaming pass over A.
//  * row_sumsq_blocks block leverage ℓ_g = Σ_{j∈g} ‖V_k[j,:]‖² (leverage.cpp:108-121),
//                     coalesced along the rows of column-major V_k.
// All sums are deterministic (fixed-order partials, no floating atomics), so a
// rerun with the same inputs reproduces results bit-for-bit.
#include "ops.h"
#include <cuda_fp16.h>

namespace bcur_b200 {
namespace {

constexpr int RT = 256;

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// Fixed-order block reduction of one value per thread (RT threads).
__device__ double block_sum(double s) {
    __shared__ double red[32];
    s = warp_sum(s);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = s;
    __syncthreads();
    double t = 0.0;
    if (w == 0) {
        t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
        t = warp_sum(t);
    }
    return t;  // valid in thread 0
}

// Block-wide max of one non-negative value per thread, broadcast to every thread.
__device__ float block_max_all(float v) {
    __shared__ float red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    float t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, o));
    return t;
}

// Power-of-two scale exponent p for a column with max |value| mx: mx·2^p < 2^15, so the
// scaled column fits fp16 (max 65504) with 29 binades of normal range below its largest
// entry.  Scaling by 2^p is exact; fp16 round-to-nearest then keeps the same 11-bit
// significand as a TF32 round-to-nearest of the unscaled value.
__device__ __forceinline__ int f16_scale_exp(float mx) {
    if (!(mx > 0.0f) || !isfinite(mx)) return 0;
    int e;
    frexpf(mx, &e);  // mx = f·2^e, f ∈ [0.5, 1)
    return 15 - e;
}

// Σ col[i]²; fp32 columns optionally also write their TF32-rounded copy to `shadow`
// (one read of A serves the norms and the pre-rounded operand of the X1 passes).
template <class T>
__device__ __forceinline__ double sq_col(const T* __restrict__ col, int64_t m, bool vec, float* __restrict__ shadow) {
    double s0 = 0.0, s1 = 0.0;
    if (vec && sizeof(T) == 4) {
        const float4* c4 = reinterpret_cast<const float4*>(col);
        float4* sh4 = reinterpret_cast<float4*>(shadow);
        const int64_t m4 = m >> 2;
        for (int64_t i = threadIdx.x; i < m4; i += RT) {
            const float4 v = __ldcs(c4 + i);
            s0 = fma((double)v.x, (double)v.x, s0);
            s1 = fma((double)v.y, (double)v.y, s1);
            s0 = fma((double)v.z, (double)v.z, s0);
            s1 = fma((double)v.w, (double)v.w, s1);
            if (shadow)
                __stcs(sh4 + i, make_float4(rn_tf32_dev(v.x), rn_tf32_dev(v.y), rn_tf32_dev(v.z), rn_tf32_dev(v.w)));
        }
        for (int64_t i = (m4 << 2) + threadIdx.x; i < m; i += RT) {
            const double v = (double)col[i];
            s0 = fma(v, v, s0);
            if (shadow) shadow[i] = rn_tf32_dev((float)v);
        }
    } else if (vec) {
        const double2* c2 = reinterpret_cast<const double2*>(col);
        const int64_t m2 = m >> 1;
        for (int64_t i = threadIdx.x; i < m2; i += RT) {
            const double2 v = __ldcs(c2 + i);
            s0 = fma(v.x, v.x, s0);
            s1 = fma(v.y, v.y, s1);
        }
        for (int64_t i = (m2 << 1) + threadIdx.x; i < m; i += RT) {
            const double v = (double)col[i];
            s0 = fma(v, v, s0);
        }
    } else {
        for (int64_t i = threadIdx.x; i < m; i += RT) {
            const double v = (double)col[i];
            s0 = fma(v, v, s0);
            if (shadow) shadow[i] = rn_tf32_dev((float)v);
        }
    }
    return s0 + s1;
}

// Σ col[i]² of an fp32 column (m % 4 == 0, 16-byte aligned) that also writes its fp16 copy
// scaled by 2^p (p = f16_scale_exp(max |col|), stored in colexp[j]): the max pass reads the
// column from HBM; the scaling pass re-reads it from L2.
// il16 (nullable, m % 64 == 0): also the 3×FP16 operand of the column (kernels_umma.cu, H3) —
// hi and the fp16 remainder lo = rn(col·2^p − hi), interleaved per 64-row chunk
// [hi 64 | lo 64] (2m halves per column), so a tile's hi and lo rows are one 256-byte run.
// hi + lo carry 22 significant bits.
__device__ double sq_col_f16(const float* __restrict__ col, int64_t m, uint16_t* __restrict__ sh16,
                             uint16_t* __restrict__ sl16, int* colexp_j) {
    double s0 = 0.0, s1 = 0.0;
    float mx = 0.0f;
    const float4* c4 = reinterpret_cast<const float4*>(col);
    const int64_t m4 = m >> 2;
    for (int64_t i = threadIdx.x; i < m4; i += RT) {
        const float4 v = c4[i];
        s0 = fma((double)v.x, (double)v.x, s0);
        s1 = fma((double)v.y, (double)v.y, s1);
        s0 = fma((double)v.z, (double)v.z, s0);
        s1 = fma((double)v.w, (double)v.w, s1);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    const int p = f16_scale_exp(block_max_all(mx));
    if (threadIdx.x == 0) *colexp_j = p;
    uint2* o4 = reinterpret_cast<uint2*>(sh16);
    uint2* l4 = reinterpret_cast<uint2*>(sl16);
    for (int64_t i = threadIdx.x; i < m4; i += RT) {
        const float4 v = __ldcs(c4 + i);
        const float x0 = ldexpf(v.x, p), x1 = ldexpf(v.y, p), x2 = ldexpf(v.z, p), x3 = ldexpf(v.w, p);
        const __half2 h01 = __floats2half2_rn(x0, x1);
        const __half2 h23 = __floats2half2_rn(x2, x3);
        if (sh16)
            __stcs(o4 + i, make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23)));
        if (sl16) {  // exact fp32 remainders (x and hi share the binade), rounded to fp16
            const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
            const __half2 l01 = __floats2half2_rn(x0 - f01.x, x1 - f01.y);
            const __half2 l23 = __floats2half2_rn(x2 - f23.x, x3 - f23.y);
            const int64_t r = i << 2, at = ((r >> 6) << 5) + ((r & 63) >> 2);  // uint2 units: chunk = 32
            __stcs(l4 + at, make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23)));
            __stcs(l4 + at + 16, make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23)));
        }
    }
    return s0 + s1;
}

// The interleaved-copy form only (m % 64 == 0): 8 rows per thread and step, so the max pass
// keeps two 16-byte loads in flight per thread and the write pass stores 16-byte hi and lo
// runs (the uint2 form stored 8 bytes per instruction and ran the norms pass at 4.4 TB/s).
__device__ double sq_col_il(const float* __restrict__ col, int64_t m, uint16_t* __restrict__ il, int* colexp_j) {
    double s0 = 0.0, s1 = 0.0;
    float mx = 0.0f;
    const float4* c4 = reinterpret_cast<const float4*>(col);
    const int64_t m8 = m >> 3;
    for (int64_t i = threadIdx.x; i < m8; i += RT) {
        const float4 v = c4[2 * i], u = c4[2 * i + 1];
        s0 = fma((double)v.x, (double)v.x, s0);
        s1 = fma((double)v.y, (double)v.y, s1);
        s0 = fma((double)v.z, (double)v.z, s0);
        s1 = fma((double)v.w, (double)v.w, s1);
        s0 = fma((double)u.x, (double)u.x, s0);
        s1 = fma((double)u.y, (double)u.y, s1);
        s0 = fma((double)u.z, (double)u.z, s0);
        s1 = fma((double)u.w, (double)u.w, s1);
        mx = fmaxf(mx, fmaxf(fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))),
                             fmaxf(fmaxf(fabsf(u.x), fabsf(u.y)), fmaxf(fabsf(u.z), fabsf(u.w)))));
    }
    const int p = f16_scale_exp(block_max_all(mx));
    if (threadIdx.x == 0) *colexp_j = p;
    uint4* o = reinterpret_cast<uint4*>(il);  // 16-byte units: a 64-row chunk = 8 hi + 8 lo units
    for (int64_t i = threadIdx.x; i < m8; i += RT) {
        const float4 v = __ldcs(c4 + 2 * i), u = __ldcs(c4 + 2 * i + 1);
        const float x[8] = {ldexpf(v.x, p), ldexpf(v.y, p), ldexpf(v.z, p), ldexpf(v.w, p),
                            ldexpf(u.x, p), ldexpf(u.y, p), ldexpf(u.z, p), ldexpf(u.w, p)};
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const __half2 h = __floats2half2_rn(x[2 * t], x[2 * t + 1]);
            const float2 f = __half22float2(h);
            const __half2 l = __floats2half2_rn(x[2 * t] - f.x, x[2 * t + 1] - f.y);
            hw[t] = *reinterpret_cast<const uint32_t*>(&h);
            lw[t] = *reinterpret_cast<const uint32_t*>(&l);
        }
        const int64_t at = (i >> 3) * 16 + (i & 7);  // row 8i: chunk i/8, 16-byte unit i%8
        __stcs(o + at, make_uint4(hw[0], hw[1], hw[2], hw[3]));
        __stcs(o + at + 8, make_uint4(lw[0], lw[1], lw[2], lw[3]));
    }
    return s0 + s1;
}

// grid (G, Z): CTA (g, z) sums columns off[g]+z, off[g]+z+Z, ...  Optional copies of the
// column: the TF32-rounded fp32 `shadow`, or the scaled fp16 `sh16` (+ per-column exponents).
template <class T>
__global__ void __launch_bounds__(RT) k_block_sumsq(const T* __restrict__ a, int64_t m, int64_t ld,
                                                    const int64_t* __restrict__ off, int Z, bool vec,
                                                    double* __restrict__ partial, float* __restrict__ shadow,
                                                    int64_t lds, uint16_t* __restrict__ sh16,
                                                    uint16_t* __restrict__ sl16, int* __restrict__ colexp) {
    const int64_t g = blockIdx.x;
    const int z = blockIdx.y;
    double s = 0.0;
    for (int64_t j = off[g] + z; j < off[g + 1]; j += Z) {
        if (sizeof(T) == 4 && sl16 && !sh16 && (m & 63) == 0)
            s += sq_col_il(reinterpret_cast<const float*>(a + j * ld), m, sl16 + 2 * j * m, colexp + j);
        else if (sizeof(T) == 4 && (sh16 || sl16))
            s += sq_col_f16(reinterpret_cast<const float*>(a + j * ld), m, sh16 ? sh16 + j * lds : nullptr,
                            sl16 ? sl16 + 2 * j * m : nullptr, colexp + j);
        else
            s += sq_col(a + j * ld, m, vec, shadow ? shadow + j * lds : nullptr);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partial[g * Z + z] = s;
}

__global__ void k_segment_rows(const double* __restrict__ partial, int Z, int64_t G, double* __restrict__ out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    double s = 0.0;
    for (int z = 0; z < Z; ++z) s += partial[g * Z + z];
    out[g] = s;
}

template <class T>
__global__ void k_row_sumsq(const T* __restrict__ v, int64_t n, int64_t k, int64_t ld, double* __restrict__ rows) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int64_t c = 0; c < k; ++c) {
        const double x = (double)v[j + c * ld];
        s = fma(x, x, s);
    }
    rows[j] = s;
}

// one warp per segment
__global__ void k_segment_sum(const double* __restrict__ x, const int64_t* __restrict__ off, int64_t G,
                              double* __restrict__ out) {
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= G) return;
    double s = 0.0;
    for (int64_t j = off[g] + lane; j < off[g + 1]; j += 32) s += x[j];
    s = warp_sum(s);
    if (lane == 0) out[g] = s;
}

__global__ void k_sum_vector(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
    s = block_sum(s);
    if (threadIdx.x == 0) out[0] = s;
}

// Σ x[i]² over a contiguous vector: a fixed grid of block partials (deterministic order)
__global__ void k_sumsq_part(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s = fma(x[i], x[i], s);
    s = block_sum(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// max |G − I| over a w×w matrix: warp per column (lanes over rows, coalesced), block max,
// then an integer atomicMax on the bit pattern (non-negative doubles order like their bits;
// a NaN's pattern exceeds +inf, so NaN propagates).  *out must be zeroed first.
__global__ void k_max_dev_identity(const double* __restrict__ g, int w, int64_t ld,
                                   unsigned long long* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double mx = 0.0;
    for (int j = blockIdx.x * nw + warp; j < w; j += gridDim.x * nw) {
        const double* col = g + (int64_t)j * ld;
        for (int i = lane; i <= j; i += 32) {  // upper triangle (G is symmetric; Grams may hold only it)
            const double d = fabs(col[i] - (i == j ? 1.0 : 0.0));
            mx = d > mx || d != d ? d : mx;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = v > mx || v != v ? v : mx;
    }
    if (lane == 0) atomicMax(out, (unsigned long long)__double_as_longlong(mx));
}

// Per column block g of M (rows × n, ld): ‖M_g‖_F² and ‖M_g‖_2² (leverage.cpp:123-139
// column_block_stable_ranks on V_kᵀ, i.e. M = V_k with blocks of rows — here M's rows are V_k's
// rows, each block a w × k slab).  One CTA per block: the k × k Gram of the slab in shared
// memory, then power iteration with a Rayleigh quotient (exact to rounding even when the top
// eigenvalues cluster: the quotient error is the residual weight times the top gap).
constexpr int BS_T = 256, BS_KMAX = 64;
__global__ void __launch_bounds__(BS_T) k_block_spectral(const double* __restrict__ v, int64_t ld, int k,
                                                          const int64_t* __restrict__ off, double* __restrict__ fro2,
                                                          double* __restrict__ spec2) {
    __shared__ double Gm[BS_KMAX * BS_KMAX];
    __shared__ double x[BS_KMAX], y[BS_KMAX], red[BS_T / 32];
    const int64_t g = blockIdx.x, j0 = off[g], w = off[g + 1] - off[g];
    double f = 0.0;
    for (int e = threadIdx.x; e < k * k; e += BS_T) {
        const int a = e % k, b = e / k;
        double sacc = 0.0;
        for (int64_t i = 0; i < w; ++i) sacc = fma(v[j0 + i + a * ld], v[j0 + i + b * ld], sacc);
        Gm[e] = sacc;
        if (a == b) f += sacc;
    }
    f = block_sum(f);
    __syncthreads();
    if (threadIdx.x == 0) fro2[g] = f;
    for (int a = threadIdx.x; a < k; a += BS_T) x[a] = 1.0 / sqrt((double)k) * (1.0 + 0.01 * a);  // generic start
    __syncthreads();
    double lam = 0.0;
    for (int it = 0; it < 2000; ++it) {
        for (int a = threadIdx.x; a < k; a += BS_T) {
            double sacc = 0.0;
            for (int b = 0; b < k; ++b) sacc = fma(Gm[a + b * k], x[b], sacc);
            y[a] = sacc;
        }
        __syncthreads();
        double num = 0.0, den = 0.0;  // Rayleigh quotient xᵀGx / xᵀx and ‖y‖
        for (int a = 0; a < k; ++a) {
            num = fma(x[a], y[a], num);
            den = fma(y[a], y[a], den);
        }
        double xx = 0.0;
        for (int a = 0; a < k; ++a) xx = fma(x[a], x[a], xx);
        const double rq = xx > 0.0 ? num / xx : 0.0;
        const double ny = sqrt(den);
        __syncthreads();
        for (int a = threadIdx.x; a < k; a += BS_T) x[a] = ny > 0.0 ? y[a] / ny : 0.0;
        __syncthreads();
        const bool done = it > 8 && fabs(rq - lam) <= 1e-16 * fabs(rq);
        lam = rq;
        if (done || !(ny > 0.0)) break;
    }
    if (threadIdx.x == 0) spec2[g] = lam;
}

// max over rows of Σ_c u(i, c)² (incoherence of U_k)
__global__ void k_max_row_sumsq(const double* __restrict__ u, int64_t m, int64_t ld, int k,
                                unsigned long long* __restrict__ out) {
    double mx = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double sacc = 0.0;
        for (int c = 0; c < k; ++c) sacc = fma(u[i + c * ld], u[i + c * ld], sacc);
        mx = fmax(mx, sacc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(mx));
}

}  // namespace

namespace ops {

void block_sumsq(Ctx* c, const void* a, int dt, int64_t m, int64_t ld, const int64_t* d_offsets, int64_t G,
                 double* d_out, float* shadow, int64_t lds, uint16_t* sh16, int* colexp, uint16_t* sl16) {
    if (G <= 0) return;
    ProfScope prof(c, "block_sumsq", 0.0, 0.0);
    // enough CTAs to fill the machine several times over
    int Z = (int)std::max<int64_t>(1, std::min<int64_t>(64, (8LL * c->sm_count + G - 1) / G));
    const size_t es = dtype_size(dt);
    const bool vec = ((ld * es) % 16 == 0) && (((uintptr_t)a) % 16 == 0);
    DevBuf part(c, (size_t)G * Z * sizeof(double));
    dim3 grid((unsigned)G, (unsigned)Z);
    if (dt == BCUR_F32)
    {
        if ((sh16 || sl16) && !(vec && m % 4 == 0 && lds % 4 == 0))
            fail(BCUR_E_INVALID_ARGUMENT, "block_sumsq: the fp16 copy needs aligned columns with m % 4 == 0");
        if (sl16 && m % 64 != 0) fail(BCUR_E_INVALID_ARGUMENT, "block_sumsq: the 3×FP16 copy needs m % 64 == 0");
        k_block_sumsq<float><<<grid, RT, 0, c->stream>>>((const float*)a, m, ld, d_offsets, Z,
                                                         vec && (shadow == nullptr || (lds % 4 == 0)),
                                                         part.as<double>(), shadow, lds, sh16, sl16, colexp);
    } else
        k_block_sumsq<double><<<grid, RT, 0, c->stream>>>((const double*)a, m, ld, d_offsets, Z, vec, part.as<double>(),
                                                          nullptr, 0, nullptr, nullptr, nullptr);
    LAUNCH_CHECK(c);
    k_segment_rows<<<(unsigned)((G + 255) / 256), 256, 0, c->stream>>>(part.as<double>(), Z, G, d_out);
    LAUNCH_CHECK(c);
}

void row_sumsq_blocks(Ctx* c, const void* v, int dt, int64_t n, int64_t k, int64_t ld, const int64_t* d_offsets,
                      int64_t G, double* d_rows, double* d_blocks) {
    ProfScope prof(c, "block_scores", 2.0 * n * k, (double)n * k * dtype_size(dt));
    DevBuf tmp;
    if (!d_rows) {
        tmp = DevBuf(c, (size_t)n * sizeof(double));
        d_rows = tmp.as<double>();
    }
    if (dt == BCUR_F32)
        k_row_sumsq<float><<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>((const float*)v, n, k, ld, d_rows);
    else
        k_row_sumsq<double><<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>((const double*)v, n, k, ld, d_rows);
    LAUNCH_CHECK(c);
    if (d_blocks) segment_sum(c, d_rows, d_offsets, G, d_blocks);
}

void segment_sum(Ctx* c, const double* x, const int64_t* d_offsets, int64_t G, double* d_out) {
    if (G <= 0) return;
    const int64_t threads = G * 32;
    k_segment_sum<<<(unsigned)((threads + 255) / 256), 256, 0, c->stream>>>(x, d_offsets, G, d_out);
    LAUNCH_CHECK(c);
}

void max_dev_identity(Ctx* c, const double* g, int64_t w, int64_t ld, double* d_out) {
    ProfScope prof(c, "max_dev", 0.0, 8.0 * w * w);
    CUDA_CHECK(cudaMemsetAsync(d_out, 0, sizeof(double), c->stream));
    if (w <= 0) return;
    const int blocks = (int)std::min<int64_t>((w + 7) / 8, 4LL * c->sm_count);
    k_max_dev_identity<<<blocks, 256, 0, c->stream>>>(g, (int)w, ld, reinterpret_cast<unsigned long long*>(d_out));
    LAUNCH_CHECK(c);
}

void block_spectral(Ctx* c, const double* v, int64_t ld, int64_t k, const int64_t* d_offsets, int64_t G, double* d_fro2,
                    double* d_spec2) {
    if (k > BS_KMAX) fail(BCUR_E_INVALID_ARGUMENT, "block_stable_rank: k <= 64 on this path");
    if (G <= 0 || k <= 0) return;
    k_block_spectral<<<(unsigned)G, BS_T, 0, c->stream>>>(v, ld, (int)k, d_offsets, d_fro2, d_spec2);
    LAUNCH_CHECK(c);
}

void max_row_sumsq(Ctx* c, const double* u, int64_t m, int64_t ld, int64_t k, double* d_out) {
    CUDA_CHECK(cudaMemsetAsync(d_out, 0, sizeof(double), c->stream));
    if (m <= 0 || k <= 0) return;
    const unsigned g = (unsigned)std::min<int64_t>((m + 255) / 256, 4LL * c->sm_count);
    k_max_row_sumsq<<<g, 256, 0, c->stream>>>(u, m, ld, (int)k, reinterpret_cast<unsigned long long*>(d_out));
    LAUNCH_CHECK(c);
}

void sum_vector(Ctx* c, const double* x, int64_t n, double* d_out) {
    k_sum_vector<<<1, 1024, 0, c->stream>>>(x, n, d_out);
    LAUNCH_CHECK(c);
}

void sumsq_vector(Ctx* c, const double* x, int64_t n, double* d_out) {
    constexpr int P = 128;
    DevBuf part(c, P * sizeof(double));
    k_sumsq_part<<<P, 256, 0, c->stream>>>(x, n, part.as<double>());
    LAUNCH_CHECK(c);
    sum_vector(c, part.as<double>(), P, d_out);
}

}  // namespace ops
}  // namespace bcur_b200
