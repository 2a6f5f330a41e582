// kernels_sample.cu — seeded block sampling and materialization.
//
//  * distribution_draw: ScoreVector::distribution (leverage.cpp:92-98),
//    require_distribution (sampler.cpp:16-31) and draw_blocks/categorical_draw
//    (sampler.cpp:35-50, 116-146) in one warp: each lane owns a contiguous chunk
//    of the G probabilities, chunk masses are warp-scanned, and the lane whose
//    range holds u = uniform·mass walks its chunk in index order.  One uniform
//    per draw, supplied by the caller's Rng, exactly as the reference consumes it.
//  * gather_blocks: materialize_columns (sampler.cpp:161-184) and its row-block
//    analogue (row blocks = column blocks of Aᵀ).
//  * argmax_masked: greedy selection criterion (ties → lowest index).
#include "ops.h"

namespace bcur_b200 {
namespace {

__device__ __forceinline__ double wsum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// p (workspace, G doubles) ; active flags in `act` (G bytes)
__global__ void __launch_bounds__(32) k_distribution_draw(const double* __restrict__ scores, int64_t G, int normalize,
                                                          int64_t g, int mode, const double* __restrict__ uniforms,
                                                          double* p, unsigned char* act,
                                                          bcur_block_draw* __restrict__ draws,
                                                          double* __restrict__ margins, int* status) {
    const int lane = threadIdx.x;
    // the working copies of p and the active flags live in shared memory when they fit: the draw
    // loop is one serial chain, and with the global workspace every step of it paid an L2 round
    // trip (81 µs for g = 32 draws over G = 512 blocks at c3, profiles/r02an/step_c3.txt)
    constexpr int SG = 4096;
    __shared__ double sp[SG];
    __shared__ unsigned char sa[SG];
    if (G <= SG) {
        p = sp;
        act = sa;
    }
    const int64_t chunk = (G + 31) / 32;
    const int64_t lo = imin64(G, lane * chunk), hi = imin64(G, lo + chunk);
    // total of scores (fixed order)
    double part = 0.0;
    for (int64_t i = lo; i < hi; ++i) part += scores[i];
    const double total = wsum(part);
    if (normalize && !(total > 0.0)) {
        if (lane == 0) *status = BCUR_E_ZERO_MATRIX;
        return;
    }
    int bad = 0;
    double psum = 0.0;
    int64_t positive = 0;
    for (int64_t i = lo; i < hi; ++i) {
        const double v = normalize ? scores[i] / total : scores[i];
        p[i] = v;
        act[i] = 1;
        if (!isfinite(v) || v < 0.0) bad = 1;
        psum += v;
        positive += v > 0.0 ? 1 : 0;
    }
    __syncwarp();  // p[] is read across lanes below (p[pick])
    bad = __any_sync(0xffffffffu, bad);
    psum = wsum(psum);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) positive += __shfl_xor_sync(0xffffffffu, positive, o);
    if (bad || fabs(psum - 1.0) > 1e-10) {
        if (lane == 0) *status = BCUR_E_DISTRIBUTION_INVALID;
        return;
    }
    if (mode == BCUR_WITHOUT_REPLACEMENT && g > positive) {
        if (lane == 0) *status = BCUR_E_NOT_ENOUGH_BLOCKS;
        return;
    }
    // chunk masses of active positive entries
    double mass_chunk = 0.0;
    for (int64_t i = lo; i < hi; ++i)
        if (p[i] > 0.0) mass_chunk += p[i];
    double mass = 1.0;
    double u_next = g > 0 ? uniforms[0] : 0.0;
    for (int64_t t = 0; t < g; ++t) {
        const double u = u_next * mass;
        if (t + 1 < g) u_next = uniforms[t + 1];  // (in flight during this draw)
        // inclusive scan of chunk masses
        double incl = mass_chunk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        double excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = 0.0;
        // owner: last lane with a nonempty chunk whose prefix ≤ u
        const unsigned cand = __ballot_sync(0xffffffffu, mass_chunk > 0.0 && excl <= u);
        const int owner = cand ? 31 - __clz(cand) : -1;
        int64_t pick = -1;
        double margin = 0.0;
        if (lane == owner) {
            double cum = excl;
            int64_t last = -1;
            for (int64_t i = lo; i < hi; ++i) {
                if (!act[i] || !(p[i] > 0.0)) continue;
                last = i;
                const double prev = cum;
                cum += p[i];
                if (cum > u) {
                    pick = i;
                    margin = fmin(u - prev, cum - u);
                    break;
                }
            }
            if (pick < 0) pick = last;  // fp guard: u on the top edge (sampler.cpp:49)
        }
        pick = __shfl_sync(0xffffffffu, pick, owner < 0 ? 0 : owner);
        margin = __shfl_sync(0xffffffffu, margin, owner < 0 ? 0 : owner);
        if (pick < 0) {
            if (lane == 0) *status = BCUR_E_DISTRIBUTION_INVALID;
            return;
        }
        const double pj = p[pick];
        if (lane == 0) {
            draws[t].block = pick;
            draws[t].probability = pj;
            draws[t].scale = 1.0 / sqrt((double)g * pj);
            if (margins) margins[t] = margin;
        }
        if (mode == BCUR_WITHOUT_REPLACEMENT) {
            if (lane == owner) {
                act[pick] = 0;
                mass_chunk = 0.0;
                for (int64_t i = lo; i < hi; ++i)
                    if (act[i] && p[i] > 0.0) mass_chunk += p[i];
            }
            mass -= pj;
        }
        __syncwarp();
    }
    if (lane == 0) *status = BCUR_OK;
}

// grid (ndraws, chunks); one CTA copies some columns (or row segments) of one draw
template <class TI, class TO>
__global__ void k_gather(const TI* __restrict__ a, int64_t m, int64_t n, int64_t lda, const int64_t* __restrict__ off,
                         const bcur_block_draw* __restrict__ draws, const int64_t* __restrict__ dst_off, int rows,
                         int scaled, TO* __restrict__ out, int64_t ldo) {
    const int64_t t = blockIdx.x;
    const int64_t b = draws[t].block;
    const double s = scaled ? draws[t].scale : 1.0;
    const int64_t beg = off[b], w = off[b + 1] - off[b];
    const int64_t d0 = dst_off[t];
    if (!rows) {
        // columns [beg, beg+w) → out columns [d0, d0+w)
        for (int64_t jj = blockIdx.y; jj < w; jj += gridDim.y) {
            const TI* src = a + (beg + jj) * lda;
            TO* dst = out + (d0 + jj) * ldo;
            for (int64_t i = threadIdx.x; i < m; i += blockDim.x) dst[i] = (TO)((double)src[i] * s);
        }
    } else {
        // rows [beg, beg+w) of every column → out rows [d0, d0+w)
        const int64_t total = w * n;
        for (int64_t e = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.y * blockDim.x) {
            const int64_t ii = e % w, j = e / w;
            out[d0 + ii + j * ldo] = (TO)((double)a[beg + ii + j * lda] * s);
        }
    }
}

__global__ void k_argmax(const double* __restrict__ x, const unsigned char* __restrict__ sel, int64_t G,
                         int64_t* out_idx, double* out_vals) {
    const int lane = threadIdx.x;
    double b1 = -INFINITY, b2 = -INFINITY;
    int64_t i1 = -1;
    for (int64_t i = lane; i < G; i += 32) {
        if (sel && sel[i]) continue;
        const double v = x[i];
        if (v > b1) { b2 = b1; b1 = v; i1 = i; }
        else if (v > b2) { b2 = v; }
    }
    // combine: greater value wins; equal values → lower index
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob1 = __shfl_xor_sync(0xffffffffu, b1, o);
        const double ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
        const int64_t oi1 = __shfl_xor_sync(0xffffffffu, i1, o);
        double n1, n2;
        int64_t ni;
        const bool other_wins = (ob1 > b1) || (ob1 == b1 && oi1 >= 0 && (i1 < 0 || oi1 < i1));
        if (other_wins) { n1 = ob1; ni = oi1; n2 = fmax(b1, ob2); }
        else { n1 = b1; ni = i1; n2 = fmax(ob1, b2); }
        b1 = n1; b2 = n2; i1 = ni;
    }
    if (lane == 0) {
        *out_idx = i1;
        out_vals[0] = b1;
        out_vals[1] = b2;
    }
}

// `count` successive masked argmax picks in one launch (the greedy's frozen tail: each pick only
// masks its block): out[t] = {index, best, second best} as k_argmax reports them, sel updated.
__global__ void k_argmax_seq(const double* __restrict__ x, unsigned char* sel, int64_t G, int count,
                             double* __restrict__ out) {
    const int lane = threadIdx.x;
    for (int t = 0; t < count; ++t) {
        double b1 = -INFINITY, b2 = -INFINITY;
        int64_t i1 = -1;
        for (int64_t i = lane; i < G; i += 32) {
            if (((volatile unsigned char*)sel)[i]) continue;
            const double v = x[i];
            if (v > b1) { b2 = b1; b1 = v; i1 = i; }
            else if (v > b2) { b2 = v; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {  // greater value wins; equal values → lower index
            const double ob1 = __shfl_xor_sync(0xffffffffu, b1, o);
            const double ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
            const int64_t oi1 = __shfl_xor_sync(0xffffffffu, i1, o);
            const bool other_wins = (ob1 > b1) || (ob1 == b1 && oi1 >= 0 && (i1 < 0 || oi1 < i1));
            const double n2 = other_wins ? fmax(b1, ob2) : fmax(ob1, b2);
            if (other_wins) { b1 = ob1; i1 = oi1; }
            b2 = n2;
        }
        if (lane == 0) {
            out[3 * t] = (double)i1;
            out[3 * t + 1] = b1;
            out[3 * t + 2] = b2;
            if (i1 >= 0) sel[i1] = 1;
        }
        __threadfence_block();
        __syncwarp();
    }
}

}  // namespace

namespace ops {

void argmax_masked_seq(Ctx* c, const double* x, unsigned char* mask_selected, int64_t G, int count, double* out3) {
    if (count <= 0) return;
    k_argmax_seq<<<1, 32, 0, c->stream>>>(x, mask_selected, G, count, out3);
    LAUNCH_CHECK(c);
}

void distribution_draw(Ctx* c, const double* d_scores, int64_t G, int normalize, int64_t g, int mode,
                       const double* d_uniforms, bcur_block_draw* d_draws, double* d_margins, int* d_status) {
    ProfScope prof(c, "draw", 0.0, 8.0 * G);
    DevBuf p(c, (size_t)G * sizeof(double)), act(c, (size_t)G);
    k_distribution_draw<<<1, 32, 0, c->stream>>>(d_scores, G, normalize, g, mode, d_uniforms, p.as<double>(),
                                                 act.as<unsigned char>(), d_draws, d_margins, d_status);
    LAUNCH_CHECK(c);
}

void gather_blocks(Ctx* c, const void* a, int dt, int64_t m, int64_t n, int64_t lda, const int64_t* d_offsets,
                   const bcur_block_draw* d_draws, const int64_t* d_dst_off, int64_t ndraws, int rows, int scaled,
                   void* out, int dto, int64_t ldo) {
    if (ndraws <= 0) return;
    ProfScope prof(c, "gather", 0.0, 0.0);
    dim3 grid((unsigned)ndraws, rows ? 64u : 32u);
#define BCUR_GATHER(TI, TO)                                                                                   \
    k_gather<TI, TO><<<grid, 256, 0, c->stream>>>((const TI*)a, m, n, lda, d_offsets, d_draws, d_dst_off, rows, \
                                                  scaled, (TO*)out, ldo)
    if (dt == BCUR_F32 && dto == BCUR_F32) BCUR_GATHER(float, float);
    else if (dt == BCUR_F32) BCUR_GATHER(float, double);
    else if (dto == BCUR_F32) BCUR_GATHER(double, float);
    else BCUR_GATHER(double, double);
#undef BCUR_GATHER
    LAUNCH_CHECK(c);
}

void argmax_masked(Ctx* c, const double* x, const unsigned char* mask_selected, int64_t G, int64_t* out_idx,
                   double* out_vals) {
    k_argmax<<<1, 32, 0, c->stream>>>(x, mask_selected, G, out_idx, out_vals);
    LAUNCH_CHECK(c);
}

}  // namespace ops
}  // namespace bcur_b200
