// kernels_umma.cu — the A-passes of the fp32 configs on 5th-gen tensor cores.
//
// fp32 accuracy from TF32 tensor cores with the 3×TF32 split (north star (1)):
//   a = a_hi + a_lo, x = x_hi + x_lo (a_hi, x_hi exactly representable in TF32)
//   a·x ≈ a_hi·x_hi + (a_hi·x_lo + a_lo·x_hi)          (3 tcgen05.mma kind::tf32)
//
//   AtX   Out(n×N) = Aᵀ·X   (Z = AᵀQ, Bᵀ = AᵀQ of the range finder; ‖Q_Cᵀ A_g‖² of the
//                          residual / greedy score via the ROWSQ epilogue — never stored)
//   AX    Out(m×N) = A·X    (Y = AΩ, Y = A·Z; split-K over the columns of A, fp64 partials)
//
// The tensor core's fp32 accumulate rounds toward zero at every MMA step (measured:
// a bias of ≈ steps·2⁻²⁴ relative), so the accumulator is never long-lived: the hi·hi
// and the small cross terms go to separate TMEM accumulators, which are double-buffered
// and drained every CH stages (K = CH·32) by the epilogue warps — into compensated fp32
// pairs (Fast2Sum on the FMA pipe, ≈ fp64-grade) — while the MMA warp fills the other buffer.
// Each k-step is one MMA spanning all NT N-tiles (N = NT·64, or 2·NT·64 for the fused
// a_hi·[x_hi | x_lo]) so the A tile is read from shared memory once per k-step.
//
// Warp roles (1 CTA/SM): warp 0 TMA producer (A tile + x_hi/x_lo tiles into an mbarrier
// stage ring); warp 1 TMEM allocator + single-lane UMMA issuer; warps 2,3 (+2 more when
// NT = 1) form a_lo = rn(a − trunc(a)) from the staged A tile (byte-image transform,
// swizzle-agnostic — the tensor core truncates the raw fp32 tile to a_hi itself); warps
// 4.. drain TMEM (tcgen05.ld 32x32b, lane quarter = warp % 4, one 64-column tile per warp)
// and run the fused epilogue.
// A (column-major) is a K-major operand for AtX (SW128) and an MN-major operand for AX
// (tf32 MN-major needs the 128B/32B-atom swizzle); x_hi/x_lo are K-major.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ops.h"
#include <cuda_fp16.h>

namespace bcur_b200 {
namespace {

constexpr int BM = 128, BK = 32, BN = 64, CH = 2;
__device__ int g_dbg_flags = 0;  // BCUR_UMMA_DEBUG: bit 0 skip a_lo transform, bit 1 skip drain, bit 2 skip MMAs (timing experiments)
bool g_wave_barrier_off = false;  // BCUR_UMMA_NO_WAVE_BARRIER=1 (experiments)
bool g_no_pair = false;           // BCUR_UMMA_NO_PAIR=1: single-CTA row-Σ² (experiments)
bool g_no_x3pair = true;          // BCUR_UMMA_X3_PAIR=1: CTA-pair 3×TF32 products (measured slower so far)
bool g_no_h3pair = false;         // BCUR_UMMA_NO_H3_PAIR=1: single-CTA 3×FP16 products (experiments)
bool g_no_hi_only = false;        // BCUR_UMMA_NO_HI_ONLY=1: GEMM_HI_ONLY products with all three MMAs (experiments)
bool g_no_fastacc = false;        // BCUR_UMMA_NO_FAST_ACC=1: GEMM_FAST_ACC products on the split accumulators (experiments)
int g_l2hint = 0;                 // BCUR_ROWSQ_L2HINT: row-Σ² TMA L2 hints, 1 = X evict-last, 2 = also A evict-first (experiments)
int g_pf = -1;                    // BCUR_UMMA_PF: A-tile L2 prefetch distance in stages (experiments)
constexpr uint32_t A_TILE = BM * BK * 4;  // 16 KB
constexpr uint32_t X_TILE = BN * BK * 4;  // 8 KB (one 64-column N tile)
// K elements per stage: tiles are 128-byte K rows (SWIZZLE_128B) — 32 tf32 or 64 fp16
// elements; every MMA consumes 32 bytes of K (8 tf32 / 16 fp16), so the byte geometry of
// stages, descriptors and tensor maps is the same for both kinds.
template <bool H> constexpr int bke() { return H ? 2 * BK : BK; }

// NT 64-column N tiles per CTA share every staged A tile (more N per CTA = fewer L2
// bytes per MMA).  Two precisions:
//  X3 (3×TF32): stage = {a_raw, a_lo, x_hi[NT], x_lo[NT]}; per tile a hi and a cross-term
//      accumulator, double-buffered in TMEM; drained into fp64 registers (1 tile/warp).
//  X1 (1×TF32, both operands rounded to nearest): stage = {rn(a) in place, x[NT]}; one
//      accumulator per tile; drained into fp32 (round-to-nearest) registers.
//      Only for sums of squared projections (ROWSQ): the unbiased rounding errors cancel
//      to ~1e-8 relative over the ~10⁸ terms.
//  H3 (3×FP16, H && X3): A and x both pre-split into fp16 hi + lo (exact power-of-two
//      scales per column, removed in the fp64 epilogue); stage = {a_hi, a_lo, x_hi[NT],
//      x_lo[NT]} all by TMA — no transform warps, and each kind::f16 MMA runs at twice the
//      TF32 rate.  hi + lo carry 22 significant bits, as the 3×TF32 split does.
template <int NT, bool X3, bool H = false>
struct Cfg {
    static constexpr bool H3 = H && X3;
    static constexpr int NACC = X3 ? 2 : 1;                                  // accumulators per tile
    static constexpr uint32_t BUFCOLS = NACC * BN * NT;                     // per drain buffer
    static constexpr int DCOLS = 64;                                         // output columns per drain warp
    // TMA stage = {a_raw, x_hi[NT], x_lo[NT] (X3)}; the a_lo split (3×TF32) lives in its own
    // LO_SLOTS-deep ring so the TMA ring keeps as many stages in flight as fit (the
    // HBM-bound passes need ≥ 6 × 16 KB of A in flight per SM).  H3 stages a_lo by TMA.
    static constexpr int LO_SLOTS = (X3 && !H3) ? 3 : 0;
    static constexpr uint32_t STAGE = (H3 ? 2 : 1) * A_TILE + (X3 ? 2 : 1) * NT * X_TILE;
    static constexpr int STAGES_FIT = (int)((232448u - 1280u - LO_SLOTS * A_TILE) / STAGE);
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
    static constexpr int LOR = H3 ? 0 : X3 ? LO_SLOTS : STAGES;  // lo_ready barriers
    static constexpr uint32_t SMEM_BYTES = STAGES * STAGE + LO_SLOTS * A_TILE + 1024 + 256;
    static constexpr uint32_t TMEM_USED = 2 * BUFCOLS;                      // ≤ 512
    static constexpr uint32_t TMEM_COLS = TMEM_USED <= 32 ? 32 : TMEM_USED <= 64 ? 64 : TMEM_USED <= 128 ? 128
                                        : TMEM_USED <= 256 ? 256 : 512;      // allocation: power of 2
    static constexpr int NDRAIN = 4 * NT * (BN / DCOLS);                     // drain warps
    // X3 runs whole warpgroups: WG0 = producer, MMA, 2 transform warps; NT drain warpgroups;
    // one more transform warpgroup (the a_lo split is the MMA's feeder).  The drain
    // warpgroups take the registers the others give up (setmaxnreg).  H3 keeps only WG0
    // (warps 2, 3 idle) and the drains.
    static constexpr int NTRANSFORM = H3 ? 2 : (X3 && NT == 1) ? 10 : 6;
    // register re-split (setmaxnreg) whenever the launch cap is below what the drains need
    static constexpr bool RESPLIT = (X3 && !(H3 && NT == 1)) || NT == 4;
    static constexpr int NTHREADS = 32 * (2 + NTRANSFORM + NDRAIN);
    static constexpr uint32_t REG_LOW = 56;
    // setmaxnreg moves registers only inside the CTA's launch allocation: every thread starts
    // with ptxas's cap R0 = ⌊65536 / NTHREADS⌋ (multiple of 8); the drains may grow by what the
    // other warpgroups release (an .inc that asks for more blocks forever).
    static constexpr uint32_t R0 = (65536u / NTHREADS) / 8 * 8;
    static constexpr uint32_t REG_DRAIN_FIT =
        R0 + ((NTHREADS - 32 * NDRAIN) * (R0 - REG_LOW) / (32 * NDRAIN)) / 8 * 8;
    static constexpr uint32_t REG_DRAIN = REG_DRAIN_FIT > 232 ? 232 : REG_DRAIN_FIT;
    static_assert(!RESPLIT || (NTHREADS % 128 == 0 && R0 > REG_LOW && REG_DRAIN > R0 &&
                          (NTHREADS - 32 * NDRAIN) * (R0 - REG_LOW) >= 32 * NDRAIN * (REG_DRAIN - R0)),
                  "X3 register split must fit the launch allocation");
    static_assert(TMEM_COLS <= 512, "TMEM budget");
};
// EPI_SPLIT / EPI_BASIS (3×FP16 A·X whose output is an orthonormal-basis candidate, |v| < 2):
//   SPLIT  the product written straight into the interleaved hi/lo layout of split_il (2M
//          halves per column, [hi 64 | lo 64] per 64-row chunk) with the fixed column scale
//          2^BASIS_E — the next products' A/X operand, with no fp64 copy and no split pass
//   BASIS  v + (the aux split, read back) written as the fp32 basis and its fp16·2^BASIS_E copy
//          (basis_out's layout): the CholQR2 correction Q = Q1 + Q1·(−F) and its output pass fused
enum { EPI_STORE = 0, EPI_ROWSQ = 1, EPI_RESID = 2, EPI_SPLIT = 3, EPI_BASIS = 4 };
constexpr int BASIS_E = 14;

// Round an fp32 value to the nearest TF32 (10-bit mantissa), ties to even.
__device__ __forceinline__ float rn_tf32(float x) {
    uint32_t u = __float_as_uint(x);
    u += 0xFFFu + ((u >> 13) & 1u);
    return __uint_as_float(u & 0xFFFFE000u);
}
// a_lo for a raw fp32 operand the tensor core truncates to TF32: the exact remainder,
// rounded to TF32 (ties away from zero) as the tensor core will read it.  The MMA ignores
// the 13 low mantissa bits of a kind::tf32 operand, so adding half an ulp is enough — the
// mask that would clear those bits is left to the hardware (a_lo is always finite).  Three
// ops per element: the transform warps run this on every A element of a 3×TF32 pass, and
// its op count sets the rate of the HBM-bound range-finder passes.
__device__ __forceinline__ float lo_of(float a) {
    const float r = a - __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
    return __uint_as_float(__float_as_uint(r) + 0x1000u);
}

// x rounded to the nearest TF32 (ties away) as the tensor core reads it: half an ulp added,
// the low bits left for the MMA to ignore (one op; for operands only an MMA consumes)
__device__ __forceinline__ float rn_mma(float x) { return __uint_as_float(__float_as_uint(x) + 0x1000u); }

// 2^e as a double (|e| < 1022): the exact scale of the split operands
__device__ __forceinline__ double exp2_int(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// ------------------------------------------------------------- PTX helpers
// Warp index broadcast from lane 0: ptxas then knows role branches on it are warp-uniform.
// With plain threadIdx.x >> 5 it must assume a role branch may split a warp, and wraps every
// tcgen05.mma in a BRA.DIV + ELECT + R2UR.BROADCAST waterfall (~24 SASS instructions per MMA,
// which made the small-N passes MMA-issue bound).
__device__ __forceinline__ int warp_index() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 0x989680;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
// L2 prefetch of a future A tile (no shared memory, no barrier): hides DRAM latency
// beyond what the shared-memory stage ring can keep in flight.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* tm, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(tm), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
        ::"r"(smem_u32(dst)), "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* tm, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];" ::"l"(tm), "r"(c0), "r"(c1), "r"(c2),
                 "r"(c3) : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* tm, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(tm), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// One A tile (A_TILE bytes) through f, NTT threads: every load of a thread is issued before
// its first store (the accesses are volatile asm, which the compiler keeps in order — a
// load/compute/store loop left each warp waiting out one shared-memory latency per float4).
template <int NTT, class F>
__device__ __forceinline__ void transform_tile(uint32_t src, uint32_t dst, int tid, F f) {
    constexpr int NV = (int)(A_TILE / 16), IT = (NV + NTT - 1) / NTT;
    float4 a[IT];
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        const int v = tid + j * NTT;
        if (NV % NTT == 0 || v < NV)
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(a[j].x), "=f"(a[j].y), "=f"(a[j].z), "=f"(a[j].w) : "r"(src + v * 16));
    }
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        const int v = tid + j * NTT;
        if (NV % NTT == 0 || v < NV)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + v * 16), "f"(f(a[j].x)),
                         "f"(f(a[j].y)), "f"(f(a[j].z)), "f"(f(a[j].w)) : "memory");
    }
}

// Shared-memory matrix descriptor (Blackwell version 1).  layout: 2 = SWIZZLE_128B
// (K-major operands), 1 = SWIZZLE_128B_BASE32B (MN-major 32-bit operands).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

// Whole-warp issue: every lane computes the same (uniform) descriptors and elect.sync
// picks the issuing lane inside the asm — a lane-0-only branch makes the compiler wrap
// each MMA in an ELECT/R2UR.BROADCAST waterfall (~56 cycles per instruction).
__device__ __forceinline__ void umma_tf32_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
        "}" ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_f16_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}" ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
template <bool H>
__device__ __forceinline__ void umma_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    if (H) umma_f16_warp(tmem_d, adesc, bdesc, idesc, accumulate);
    else umma_tf32_warp(tmem_d, adesc, bdesc, idesc, accumulate);
}
__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
        "}" ::"r"(smem_u32(bar)) : "memory");
}
#define TMEM_LD8(taddr, r)                                                                                         \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                            \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])     \
                 : "r"(taddr))

#define TMEM_LD16(taddr, r)                                                                                        \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),         \
                   "=r"(r[15])                                                                                     \
                 : "r"(taddr))

// Persistent tile schedule.  Tiles are (m_tile, n_tile, split); consecutive tiles walk
// group_n N tiles side by side, then the next M tile, so a wave of CTAs streams a band
// of A tiles and a band of X tiles together and both are served from L2 (a plain grid
// lets CTAs drift apart and re-streams the operands from HBM: 130 GB for a 4.3 GB pass).
//   sym:   Out = AᵀA — only tiles with n ≥ m (the upper triangle) are enumerated.
//   tri_x: X is upper triangular (X[k, j] = 0 for k > j) — each N tile stops at its diagonal.
//   wave_ctr: a wave barrier — a CTA's producer starts tile wave w+1 only after every CTA
//   has issued its wave-w loads, so a wave's CTAs stay in lockstep along K and share the
//   A and X bands through L2 (cooperative launch guarantees co-residency).
struct Sched {
    int m_tiles, n_tiles, splits, group_n, total;
    int k_tiles, kps, sym, tri_x;
    unsigned int* wave_ctr;
    int a_rn;  // X1: A already rounded to TF32 (no transform)
    int pf;    // A-tile L2 prefetch distance (stages)
    int x_il;  // H3: x_hi/x_lo come from one interleaved split (4-D map, part = hi|lo)
    int bke;   // K elements per k-tile (32 tf32, 64 fp16): the triangular-X limit is in these units
};
// CTAs that have a tile in waves 0..w
__device__ __forceinline__ unsigned int wave_arrivals(const Sched& sc, int w) {
    const int g = gridDim.x;
    unsigned int s = 0;
    for (int v = 0; v <= w; ++v) s += (unsigned int)max(0, min(g, sc.total - v * g));
    return s;
}
struct TileInfo {
    int m_tile, n_tile, split, kt0, nk;
};
template <int NT>
__device__ __forceinline__ TileInfo tile_info(const Sched& sc, int t) {
    TileInfo ti;
    const int per_split = sc.sym ? sc.n_tiles * (sc.n_tiles + 1) / 2 : sc.m_tiles * sc.n_tiles;
    ti.split = t / per_split;
    const int r = t - ti.split * per_split;
    if (sc.sym) {  // r = n(n+1)/2 + m, m ≤ n.  Integer search: a sqrtf (MUFU, vector
        // registers) here made the schedule look non-uniform to ptxas (see warp_index)
        int n = 0;
        while ((n + 1) * (n + 2) / 2 <= r) ++n;
        ti.n_tile = n;
        ti.m_tile = r - n * (n + 1) / 2;
    } else {
        const int gsz = sc.group_n * sc.m_tiles;
        const int g = r / gsz, first_n = g * sc.group_n;
        const int gn = min(sc.group_n, sc.n_tiles - first_n);
        const int rr = r - g * gsz;
        ti.n_tile = first_n + rr % gn;
        ti.m_tile = rr / gn;
        // triangular X: N tile j carries j + 1 diagonal blocks of K — walk the widest first so
        // the persistent CTAs end together (longest-processing-time order)
        if (sc.tri_x) ti.n_tile = sc.n_tiles - 1 - ti.n_tile;
    }
    ti.kt0 = ti.split * sc.kps;
    int kt1 = min(sc.k_tiles, ti.kt0 + sc.kps);
    if (sc.tri_x) kt1 = min(kt1, ((ti.n_tile + 1) * NT * BN + sc.bke - 1) / sc.bke);
    ti.nk = max(kt1 - ti.kt0, 0);
    return ti;
}

// Scales (H3): the fp64 result of output row r, column j is multiplied by
// 2^−(rexp[r] + cexp[j]) (either nullable) — the exact power-of-two scales of the split operands.
template <bool A_MN, int EPI, int NT, bool X3, bool H = false>
__global__ void __launch_bounds__(Cfg<NT, X3, H>::NTHREADS, 1)
k_umma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
       const __grid_constant__ CUtensorMap tmXl, const __grid_constant__ CUtensorMap tmAl, int M, int N,
       const Sched sc, double* __restrict__ out, int64_t ldo, double* __restrict__ partial, double alpha, double beta,
       const int* __restrict__ rexp, const int* __restrict__ cexp, const uint16_t* __restrict__ aux) {
    // instruction descriptor: fp32 accumulate, tf32 × tf32 (H: f16 × f16), B K-major,
    // N = n_cols, M = 128
    static_assert(!H || (X3 ? (EPI == EPI_STORE || (A_MN && (EPI == EPI_RESID || EPI == EPI_SPLIT || EPI == EPI_BASIS)))
                           : (EPI == EPI_ROWSQ && !A_MN)),
                  "fp16 operands: 3×FP16 products (stored, or the fused residual), or the pre-converted "
                  "row-sum-of-squares");
    constexpr bool H3 = H && X3;
    constexpr uint32_t FMT = H ? 0u : 2u;
    constexpr int BKE = bke<H>();
    auto idesc = [](uint32_t n_cols) -> uint32_t {
        return (1u << 4) | (FMT << 7) | (FMT << 10) | ((A_MN ? 1u : 0u) << 15) | ((n_cols >> 3) << 17) |
               ((uint32_t)(BM >> 4) << 24);
    };

    using CF = Cfg<NT, X3, H>;
    constexpr uint32_t BUFCOLS = CF::BUFCOLS;
    constexpr int STAGES = CF::STAGES;
    constexpr uint32_t STAGE = CF::STAGE, TMEM_COLS = CF::TMEM_COLS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    constexpr int LO_SLOTS = CF::LO_SLOTS, LOR = CF::LOR;
    uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE + LO_SLOTS * A_TILE);
    uint64_t* full = bars;                                   // [STAGES] TMA bytes landed
    uint64_t* empty = full + STAGES;                         // [STAGES] MMAs done with the stage
    uint64_t* lo_ready = empty + STAGES;                     // [LOR]   a_lo (X3) / rn (X1) written
    uint64_t* lo_empty = lo_ready + LOR;                     // [LO_SLOTS] MMAs done with the a_lo slot
    uint64_t* tfull = lo_empty + LO_SLOTS;                   // [2]
    uint64_t* tempty = tfull + 2;                            // [2]
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

    const int warp = warp_index(), lane = threadIdx.x & 31;
    // read once (a per-stage global load sat on the transform's critical path); broadcast so the
    // MMA guard below stays provably warp-uniform (see warp_index)
    const int dbg = __shfl_sync(0xffffffffu, g_dbg_flags, 0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < LOR; ++s) mbar_init(&lo_ready[s], 32 * CF::NTRANSFORM);
        for (int s = 0; s < LO_SLOTS; ++s) mbar_init(&lo_empty[s], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 32 * CF::NDRAIN);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmXh) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmXl) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // per stage: [a_raw][a_lo (H3)][x_hi tile 0..NT-1][x_lo tile 0..NT-1 (X3)]; then the a_lo slots
    constexpr uint32_t XOFF = (H3 ? 2 : 1) * A_TILE;
    auto a_raw = [&](int s) { return smem + s * STAGE; };
    auto x_hi = [&](int s) { return smem + s * STAGE + XOFF; };
    auto x_lo = [&](int s) { return smem + s * STAGE + XOFF + NT * X_TILE; };
    auto a_lo = [&](int l) { return smem + STAGES * STAGE + l * A_TILE; };

    // roles: branch per warpgroup first so the register re-split (X3) is warpgroup-uniform
    if (warp >= 4 && warp < 4 + CF::NDRAIN) {
        if (CF::RESPLIT) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CF::REG_DRAIN));
        // ------------------------------------------- TMEM drain + epilogue
        // warp → (TMEM lane quarter q, DC-column slice of the NT·64 output columns)
        constexpr int DC = CF::DCOLS;
        const int q = warp & 3;
        const int slice = (warp - 4) >> 2;
        const int ccol = slice * DC;                  // first output column (within the tile) of this warp
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        int gc = 0;  // chunks drained so far (all tiles)
        double rsum = 0.0;  // EPI_RESID: this thread's Σ (D − product)² over its rows of every tile
        for (int t = blockIdx.x; t < sc.total; t += gridDim.x) {
        const TileInfo ti = tile_info<NT>(sc, t);
        const int m_tile = ti.m_tile, n_tile = ti.n_tile, split = ti.split;
        const int nchunks = (ti.nk + CH - 1) / CH;
        const int row = m_tile * BM + q * 32 + lane;
        // X3: compensated fp32 sums on the FMA pipe (acc + cmp ≈ fp64 accuracy; the
        // fp32→fp64 converts of a plain fp64 drain saturate the XU pipe and stall the MMA)
        float acc[DC], cmp[X3 ? DC : 1];
#pragma unroll
        for (int j = 0; j < DC; ++j) acc[j] = 0.0f;
#pragma unroll
        for (int j = 0; j < (X3 ? DC : 1); ++j) cmp[j] = 0.0f;
        for (int c = 0; c < nchunks; ++c) {
            const int g = gc + c, b = g & 1;
            mbar_wait(&tfull[b], (uint32_t)(g / 2) & 1u);
            tc_fence_after();
            if (dbg & 2) {  // experiment switch: skip the drain (wrong results)
                tc_fence_before();
                mbar_arrive(&tempty[b]);
                continue;
            }
            const uint32_t t_hi = tmem + lane_off + (uint32_t)(b * BUFCOLS + ccol);
            const uint32_t t_lo = t_hi + NT * BN;
            constexpr int LDW = (X3 || NT == 4) ? 8 : 16;  // narrower loads keep acc(+cmp)+loads in registers
#pragma unroll
            for (int j0 = 0; j0 < DC; j0 += LDW) {
                uint32_t h[LDW], l[LDW];
                if (LDW == 8) {
                    TMEM_LD8(t_hi + j0, h);
                    if (X3) TMEM_LD8(t_lo + j0, l);
                } else {
                    TMEM_LD16(t_hi + j0, h);
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < LDW; ++j) {
                    const int e = j0 + j;
                    const float hsum = __uint_as_float(h[j]);
                    if (X3) {
                        // hi chunks through a compensated (Fast2Sum) sum; the cross terms
                        // (~2⁻¹¹ of hi) go straight into the compensation accumulator with the
                        // rounding error — both are small, so one fp32 sum of them is exact to
                        // ~2⁻³⁵ of the result: 5 FP ops per element (8 with the cross term
                        // folded into hi by a second Fast2Sum first)
                        const float hv = hsum;
                        const float sum = __fadd_rn(acc[e], hv);
                        const float z = __fsub_rn(sum, acc[e]);
                        cmp[e] = __fadd_rn(cmp[e], __fadd_rn(__fsub_rn(hv, z), __uint_as_float(l[j])));
                        acc[e] = sum;
                    } else {
                        acc[e] += hsum;
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[b]);
        }
        const int col0 = n_tile * NT * BN + ccol;
        if (EPI == EPI_RESID) {
            // fused explicit residual: D is the fp32 A (column-major, ld = ldo) passed as `out`;
            // lanes are consecutive rows, so each column's loads are one 128-byte line per warp
            if (row < M) {
                const float* D = reinterpret_cast<const float*>(out);
                const int ncol = min(DC, N - col0);
                const int re = (H3 && rexp) ? rexp[row] : 0;
                constexpr int EB = 16;
#pragma unroll
                for (int j0 = 0; j0 < DC; j0 += EB) {
                    float dv[EB];
#pragma unroll
                    for (int jj = 0; jj < EB; ++jj)
                        dv[jj] = (j0 + jj < ncol) ? __ldg(D + row + (int64_t)(col0 + j0 + jj) * ldo) : 0.0f;
#pragma unroll
                    for (int jj = 0; jj < EB; ++jj) {
                        const int j = j0 + jj;
                        if (j >= ncol) continue;
                        double v = X3 ? (double)acc[j] + (double)cmp[X3 ? j : 0] : (double)acc[j];
                        if (H3) v *= exp2_int(-(re + (cexp ? cexp[col0 + j] : 0)));
                        const double e = (double)dv[jj] - v;
                        rsum = fma(e, e, rsum);
                    }
                }
            }
        } else if (EPI == EPI_SPLIT || EPI == EPI_BASIS) {
            // lanes are consecutive rows of one 64-row chunk: each column's hi (and lo) stores are
            // one 64-byte run per warp
            if (row < M) {
                const int ncol = min(DC, N - col0);
                const int64_t r_il = (int64_t)(row >> 6) * 128 + (row & 63);
                uint16_t* o16 = reinterpret_cast<uint16_t*>(EPI == EPI_SPLIT ? out : partial);
                float* o32 = reinterpret_cast<float*>(out);
                // BASIS: the aux values of 8 columns are loaded together (one L2 round trip per
                // column made the epilogue, not the MMAs, bound the correction product)
                float ax8[8];
#pragma unroll
                for (int j = 0; j < DC; ++j) {
                    if (EPI == EPI_BASIS && (j & 7) == 0) {
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            ax8[jj] = 0.0f;
                            if (aux && j + jj < ncol) {
                                const int64_t o = (int64_t)(col0 + j + jj) * 2 * M + r_il;
                                const uint16_t hb = aux[o], lb = aux[o + 64];
                                ax8[jj] = __half2float(*reinterpret_cast<const __half*>(&hb)) +
                                          __half2float(*reinterpret_cast<const __half*>(&lb));  // exact in fp32
                            }
                        }
                    }
                    if (j >= ncol) continue;
                    const int col = col0 + j;
                    double v = (double)acc[j] + (double)cmp[X3 ? j : 0];
                    v *= alpha * exp2_int(-(cexp ? cexp[col] : 0));
                    if (EPI == EPI_SPLIT) {
                        const double sv = v * (double)(1 << BASIS_E);
                        const __half h = __double2half(sv);
                        const __half l = __double2half(sv - (double)__half2float(h));
                        o16[(int64_t)col * 2 * M + r_il] = *reinterpret_cast<const uint16_t*>(&h);
                        o16[(int64_t)col * 2 * M + r_il + 64] = *reinterpret_cast<const uint16_t*>(&l);
                    } else {
                        v += (double)ax8[j & 7] * (1.0 / (double)(1 << BASIS_E));
                        o32[row + (int64_t)col * ldo] = (float)v;
                        // the fp16 copy as the interleaved split of v·2^14: hi = the row-Σ² pass's
                        // operand, lo = its rounding error (the sketch correction's Δ)
                        const double sv = v * (double)(1 << BASIS_E);
                        const __half h = __double2half(sv);
                        const __half l = __double2half(sv - (double)__half2float(h));
                        o16[(int64_t)col * 2 * M + r_il] = *reinterpret_cast<const uint16_t*>(&h);
                        o16[(int64_t)col * 2 * M + r_il + 64] = *reinterpret_cast<const uint16_t*>(&l);
                    }
                }
            }
        } else if (EPI == EPI_ROWSQ) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < DC; ++j) {
                const double v = (double)acc[j];
                s = fma(v, v, s);  // columns ≥ N are exact zeros
            }
            // one partial row-sum per DC-column slice of the output
            if (row < M) partial[(int64_t)(col0 / DC) * M + row] = s;
        } else if (row < M) {
            // split-K partials (plain stores) or alpha·v + beta·out; lanes = consecutive rows
            double* dst = partial ? partial + (int64_t)split * M * N + row : out + row;
            const int64_t stride = partial ? (int64_t)M : ldo;
            const bool plain = partial != nullptr || beta == 0.0;
            const double a_ = partial ? 1.0 : alpha;
            const int ncol = min(DC, N - col0);
            const int re = (H3 && rexp && row < M) ? rexp[row] : 0;
            // β ≠ 0: the old values are loaded 16 at a time before any store (one
            // read-modify-write per column made each element a dependent load → store round
            // trip through L2: the Q1 + Q1·(−F) correction ran at half the C·R⁻¹ rate)
            constexpr int EB = 16;
#pragma unroll
            for (int j0 = 0; j0 < DC; j0 += EB) {
                double old[EB];
#pragma unroll
                for (int jj = 0; jj < EB; ++jj) {
                    const int j = j0 + jj;
                    old[jj] = (!plain && j < ncol) ? dst[(int64_t)(col0 + j) * stride] : 0.0;
                }
#pragma unroll
                for (int jj = 0; jj < EB; ++jj) {
                    const int j = j0 + jj;
                    double v = X3 ? (double)acc[j] + (double)cmp[X3 ? j : 0] : (double)acc[j];
                    if (H3) v *= exp2_int(-(re + ((cexp && j < ncol) ? cexp[col0 + j] : 0)));
                    if (j < ncol) dst[(int64_t)(col0 + j) * stride] = plain ? a_ * v : fma(beta, old[jj], a_ * v);
                }
            }
        }
        gc += nchunks;
        }
        if (EPI == EPI_RESID) partial[(int64_t)blockIdx.x * (32 * CF::NDRAIN) + (warp - 4) * 32 + lane] = rsum;
    } else {
        if (CF::RESPLIT) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(CF::REG_LOW));
        if (warp == 0) {
            // ------------------------------------------------------ TMA producer
            if (lane == 0) {
                const int PF = sc.pf;  // A-tile L2 prefetch distance (stages)
                int gi = 0;             // stages issued so far (all tiles)
                for (int t = blockIdx.x, w = 0; t < sc.total; t += gridDim.x, ++w) {
                    if (sc.wave_ctr && w > 0) {  // wave barrier (see Sched)
                        const unsigned int target = wave_arrivals(sc, w - 1);
                        unsigned int v;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sc.wave_ctr) : "memory");
                        } while (v < target);
                    }
                    const TileInfo ti = tile_info<NT>(sc, t);
                    const int kt0 = ti.kt0, nk = ti.nk, m_tile = ti.m_tile, n_tile = ti.n_tile;
                    constexpr int MNA = H ? 64 : 32;  // MN elements per 128-byte row (A_MN)
                    // H3: A is the interleaved hi/lo copy, a 4-D map (64, hi|lo, ...): one 256-byte
                    // run per column and 64 rows holds both operands (see block_sumsq)
                    auto prefetch_a = [&](int i) {
                        const int k0 = (kt0 + i) * BKE;
                        if (H3) {
                            for (int hl = 0; hl < 2; ++hl) {
                                if (A_MN) {
                                    tma_prefetch_4d(&tmA, 0, hl, m_tile * 2, k0);
                                    tma_prefetch_4d(&tmA, 0, hl, m_tile * 2 + 1, k0);
                                } else {
                                    tma_prefetch_4d(&tmA, 0, hl, k0 / 64, m_tile * BM);
                                }
                            }
                        } else if (A_MN) tma_prefetch_3d(&tmA, 0, k0, m_tile * (BM / MNA));
                        else if (H) tma_prefetch_4d(&tmA, 0, 0, k0 / 64, m_tile * BM);
                        else tma_prefetch_2d(&tmA, k0, m_tile * BM);
                    };
                    for (int i = 0; i < PF && i < nk; ++i) prefetch_a(i);
                    for (int i = 0; i < nk; ++i, ++gi) {
                        const int s = gi % STAGES;
                        if (i + PF < nk) prefetch_a(i + PF);
                        mbar_wait(&empty[s], ((uint32_t)(gi / STAGES) & 1u) ^ 1u);
                        mbar_expect_tx(&full[s], STAGE);
                        const int k0 = (kt0 + i) * BKE;
                        if (H3) {
                            for (int hl = 0; hl < 2; ++hl) {
                                if (A_MN) {  // two 64-row chunks (8 KB MN atoms) × 64 K rows
                                    tma_load_4d(a_raw(s) + hl * A_TILE, &tmA, &full[s], 0, hl, m_tile * 2, k0);
                                    tma_load_4d(a_raw(s) + hl * A_TILE + A_TILE / 2, &tmA, &full[s], 0, hl,
                                                m_tile * 2 + 1, k0);
                                } else {
                                    tma_load_4d(a_raw(s) + hl * A_TILE, &tmA, &full[s], 0, hl, k0 / 64, m_tile * BM);
                                }
                            }
                        } else if (A_MN) tma_load_3d(a_raw(s), &tmA, &full[s], 0, k0, m_tile * (BM / MNA));
                        else if (H) tma_load_4d(a_raw(s), &tmA, &full[s], 0, 0, k0 / 64, m_tile * BM);  // hi of the copy
                        else tma_load_2d(a_raw(s), &tmA, &full[s], k0, m_tile * BM);
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) {
                            const int xc = (n_tile * NT + nt) * BN;
                            if (H && sc.x_il) {
                                tma_load_4d(x_hi(s) + nt * X_TILE, &tmXh, &full[s], 0, 0, k0 / 64, xc);
                                if (X3) tma_load_4d(x_lo(s) + nt * X_TILE, &tmXh, &full[s], 0, 1, k0 / 64, xc);
                            } else {
                                tma_load_2d(x_hi(s) + nt * X_TILE, &tmXh, &full[s], k0, xc);
                                if (X3) tma_load_2d(x_lo(s) + nt * X_TILE, &tmXl, &full[s], k0, xc);
                            }
                        }
                    }
                    if (sc.wave_ctr) atomicAdd(sc.wave_ctr, 1u);
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------------ MMA issuer
            int gi = 0, gc = 0;  // stages / chunks consumed so far (all tiles)
            for (int t = blockIdx.x; t < sc.total; t += gridDim.x) {
                const int nk = tile_info<NT>(sc, t).nk;
                for (int i = 0; i < nk; ++i, ++gi) {
                    const int s = gi % STAGES;
                    const int c = gc + i / CH, b = c & 1;
                    const bool first = (i % CH) == 0;
                    if (first) mbar_wait(&tempty[b], ((uint32_t)(c / 2) & 1u) ^ 1u);
                    const uint32_t ph = (uint32_t)(gi / STAGES) & 1u;
                    const int lr = (X3 && !H3) ? gi % (LO_SLOTS > 0 ? LO_SLOTS : 1) : s;
                    mbar_wait(&full[s], ph);
                    if (!H3) mbar_wait(&lo_ready[lr], X3 ? (uint32_t)(gi / (LO_SLOTS > 0 ? LO_SLOTS : 1)) & 1u : ph);
                    tc_fence_after();
                    {  // whole warp (elect.sync inside the issue helpers)
                        const uint32_t ar = smem_u32(a_raw(s)), xh = smem_u32(x_hi(s));
                        const uint32_t al = H3 ? ar + A_TILE : smem_u32(a_lo(lr));
#pragma unroll
                        for (int k8 = 0; k8 < BK / 8; ++k8) {
                            uint64_t da_r, da_l;
                            if (A_MN && H) {  // [2 MN atoms of 64, 8 KB apart][64 K rows of 128 B, 8-row groups 1 KB apart]
                                da_r = sdesc(ar + k8 * 2048, 8192, 1024, 2);
                                da_l = sdesc(al + k8 * 2048, 8192, 1024, 2);
                            } else if (A_MN) {  // [4 MN atoms, 4 KB apart][32 K rows of 128 B, 4-row groups 512 B apart]
                                da_r = sdesc(ar + k8 * 1024, 4096, 512, 1);
                                da_l = sdesc(al + k8 * 1024, 4096, 512, 1);
                            } else {     // K-major rows of 128 B, 8-row groups 1 KB apart; K step = 32 B
                                da_r = sdesc(ar + k8 * 32, 16, 1024, 2);
                                da_l = sdesc(al + k8 * 32, 16, 1024, 2);
                            }
                            // one instruction spans all NT N-tiles (the A tile is read once per k-step);
                            // X3 fuses a_hi·[x_hi | x_lo] (x_lo tiles follow x_hi in the stage, and the lo
                            // accumulator follows the hi one in TMEM), then adds a_lo·x_hi into lo.
                            // (Rotating independent accumulators per k-step was measured slower:
                            // the extra drain loads cost more than the MMA-chain overlap gains.)
                            const uint64_t dxh = sdesc(xh + k8 * 32, 16, 1024, 2);
                            const uint32_t t_hi = tmem + (uint32_t)(b * BUFCOLS), t_lo = t_hi + NT * BN;
                            const uint32_t acc = (!first || k8 > 0) ? 1u : 0u;
                            if (!(dbg & 4)) {  // bit 2: skip the MMAs (timing experiments)
                                umma_warp<H>(t_hi, da_r, dxh, idesc((X3 ? 2 : 1) * NT * BN), acc);
                                if (X3) umma_warp<H>(t_lo, da_l, dxh, idesc(NT * BN), 1u);
                            }
                        }
                        umma_commit_warp(&empty[s]);
                        if (X3 && !H3) umma_commit_warp(&lo_empty[lr]);
                        if ((i % CH) == CH - 1 || i == nk - 1) umma_commit_warp(&tfull[b]);
                    }
                    __syncwarp();
                }
                gc += (nk + CH - 1) / CH;
            }
        } else if (!H3) {
            // ------------------------- a_lo transform (X3) / in-place rn_tf32 (X1)
            constexpr int NTT = 32 * CF::NTRANSFORM;
            const int tid = (warp < 4 ? warp - 2 : warp - (4 + CF::NDRAIN) + 2) * 32 + lane;  // 0..NTT-1
            int gi = 0;
            int nk = 0, tile = blockIdx.x - (int)gridDim.x, i = 0;
            for (;; ++i, ++gi) {
                while (i >= nk) {  // next tile with work
                    tile += gridDim.x;
                    if (tile >= sc.total) break;
                    nk = tile_info<NT>(sc, tile).nk;
                    i = 0;
                }
                if (tile >= sc.total) break;
                const int s = gi % STAGES;
                const int lr = (X3 && !H3) ? gi % (LO_SLOTS > 0 ? LO_SLOTS : 1) : s;
                mbar_wait(&full[s], (uint32_t)(gi / STAGES) & 1u);
                if (X3) mbar_wait(&lo_empty[lr], ((uint32_t)(gi / (LO_SLOTS > 0 ? LO_SLOTS : 1)) & 1u) ^ 1u);
                const uint32_t src = smem_u32(a_raw(s)), dst = X3 ? smem_u32(a_lo(lr)) : src;
                if ((dbg & 1) || (!X3 && sc.a_rn)) {  // pre-rounded A (or the experiment switch)
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_arrive(&lo_ready[lr]);
                    continue;
                }
                if (X3) transform_tile<NTT>(src, dst, tid, lo_of);
                else transform_tile<NTT>(src, dst, tid, rn_mma);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&lo_ready[lr]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// ---------------------------------------------------------------- helpers
// x (K × N fp64) → x_hi = rn_tf32(x), x_lo = rn_tf32(x − x_hi) (fp32, ld K).  x_hi = rn(x)
// makes x_lo sign-symmetric, so the dropped a_lo·x_lo term carries no bias.
template <class T>
__global__ void k_split_hilo(const T* __restrict__ x, int64_t K, int64_t N, int64_t ldx, float* __restrict__ hi,
                             float* __restrict__ lo) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= K * N) return;
    const int64_t i = e % K, j = e / K;
    const double xd = (double)x[i + j * ldx];
    const float h = rn_tf32((float)xd);
    hi[e] = h;
    lo[e] = rn_tf32((float)(xd - (double)h));
}

__global__ void k_reduce_splits(int64_t M, int64_t N, int splits, const double* __restrict__ partial,
                                double* __restrict__ out, int64_t ldo, double alpha, double beta) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M * N) return;
    const int64_t i = e % M, j = e / M;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * M * N + e];
    double* o = out + i + j * ldo;
    *o = beta == 0.0 ? alpha * s : fma(beta, *o, alpha * s);
}

__global__ void k_sum_tiles(int64_t M, int tiles, const double* __restrict__ partial, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    double s = 0.0;
    for (int t = 0; t < tiles; ++t) s += partial[(int64_t)t * M + i];
    out[i] = s;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) fail(BCUR_E_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// promo: L2 sector promotion.  256 B suits contiguous streams (the next K tile is adjacent);
// reads of the hi half of the interleaved copy use 128 B, or every hi run would pull its lo
// neighbour from DRAM as well.
CUtensorMap make_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                     const uint32_t* box, CUtensorMapSwizzle swz,
                     CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
    CUtensorMap m;
    uint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode_fn()(&m, dt, rank, const_cast<void*>(base), dims, strides_bytes,
                             box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(BCUR_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

// Persistent launch: one CTA per SM (or fewer when there are fewer tiles).
template <bool A_MN, int EPI, int NT, bool X3, bool H = false>
void launch_umma_nt(Ctx* c, Sched sc, const CUtensorMap& ta, const CUtensorMap& th, const CUtensorMap& tl, int M,
                    int N, double* out, int64_t ldo, double* partial, double alpha, double beta,
                    const CUtensorMap* tal = nullptr, const int* rexp = nullptr, const int* cexp = nullptr,
                    bool wave_barrier = true, const uint16_t* aux = nullptr) {
    using CF = Cfg<NT, X3, H>;
    auto kern = k_umma<A_MN, EPI, NT, X3, H>;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES));
        attr = true;
    }
    if (sc.total <= 0) return;
    const int grid = std::min(sc.total, c->sm_count);
    DevBuf ctr;
    if (grid < sc.total && !(g_wave_barrier_off) && wave_barrier) {
        ctr = DevBuf(c, 64);
        CUDA_CHECK(cudaMemsetAsync(ctr.ptr, 0, 4, c->stream));
        sc.wave_ctr = ctr.as<unsigned int>();
    } else {
        sc.wave_ctr = nullptr;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(CF::NTHREADS);
    cfg.dynamicSmemBytes = CF::SMEM_BYTES;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr_c[1];
    attr_c[0].id = cudaLaunchAttributeCooperative;
    attr_c[0].val.cooperative = sc.wave_ctr ? 1 : 0;
    cfg.attrs = attr_c;
    cfg.numAttrs = 1;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, ta, th, tl, tal ? *tal : ta, M, N, sc, out, ldo, partial, alpha, beta,
                                  rexp, cexp, aux));
    LAUNCH_CHECK(c);
}

// 3×TF32 with 1 or 2 N tiles per CTA
template <bool A_MN, int EPI>
void launch_umma(Ctx* c, int nt_per_cta, Sched sc, const CUtensorMap& ta, const CUtensorMap& th,
                 const CUtensorMap& tl, int M, int N, double* out, int64_t ldo, double* partial, double alpha,
                 double beta) {
    if (nt_per_cta == 2)
        launch_umma_nt<A_MN, EPI, 2, true>(c, sc, ta, th, tl, M, N, out, ldo, partial, alpha, beta);
    else
        launch_umma_nt<A_MN, EPI, 1, true>(c, sc, ta, th, tl, M, N, out, ldo, partial, alpha, beta);
}

Sched make_sched(int m_tiles, int n_tiles, int splits, int k_tiles, int kps, bool sym, bool tri_x) {
    Sched sc;
    sc.m_tiles = m_tiles;
    sc.n_tiles = n_tiles;
    sc.splits = splits;
    sc.group_n = std::min(8, n_tiles);  // a wave of 148 CTAs ≈ 8 N tiles × 18 M tiles
    sc.k_tiles = k_tiles;
    sc.kps = kps;
    sc.sym = sym ? 1 : 0;
    sc.tri_x = tri_x ? 1 : 0;
    sc.total = splits * (sym ? n_tiles * (n_tiles + 1) / 2 : m_tiles * n_tiles);
    sc.wave_ctr = nullptr;
    sc.a_rn = 0;
    sc.pf = g_pf >= 0 ? g_pf : 12;
    sc.x_il = 0;
    sc.bke = BK;
    return sc;
}

// ------------------------------------------------ CTA-pair row-Σ² (cta_group::2)
// rowsq[j] = Σ_c (AᵀX)_jc² on a pre-rounded A (1×TF32), one CTA pair per 256 A columns ×
// 256 X columns.  Each CTA TMA-loads its own 128-column A tile and HALF of the X tile
// (the 2-SM TMA form signals the leader's barrier); the leader issues M=256 × N=256 MMAs
// (tcgen05.mma.cta_group::2) that read A from each CTA's shared memory and B split across
// the two; each CTA's TMEM holds its 128 rows.  Per SM and stage this moves 32 KB into
// shared memory and 32 KB out to the tensor core, against 48 + 48 KB for a single-CTA
// N=256 tile — the single-CTA pass is bound by shared-memory bandwidth.
constexpr int P2_NDRAIN = 16;                                   // 4 lane quarters × 4 64-column tiles
constexpr int P2_THREADS = 32 * (4 + P2_NDRAIN);               // producer, MMA, 2 idle, drains
constexpr uint32_t P2_STAGE = A_TILE + 2 * X_TILE;              // own A tile + half of the X tile
constexpr int P2_STAGES = 6;
constexpr uint32_t P2_SMEM = P2_STAGES * P2_STAGE + 1024 + 256;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 2-SM TMA loads with an optional L2 eviction policy (the createpolicy encodings CUTLASS uses).
// Measured on the c3 row-Σ² pass (profiles/r02ad): A evict-first + X evict-last raised its DRAM
// reads from 7.9 to 9.8 GB (a wave's 8 X tiles share each A tile through L2), so the default is
// no hint
constexpr uint64_t L2_EVICT_FIRST = 0x12F0000000000000ull, L2_EVICT_LAST = 0x14F0000000000000ull;
__device__ __forceinline__ void tma2sm_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                          uint64_t pol) {
    if (pol)
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst), "l"(map), "r"(bar), "r"(c0), "r"(c1), "l"(pol) : "memory");
    else
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma2sm_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2,
                                          int c3, uint64_t pol) {
    if (pol)
        asm volatile(
            "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(dst), "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2),
            "r"(c3), "l"(pol) : "memory");
    else
        asm volatile(
            "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
            : "memory");
}

// pair tile t → (A column pair mp, X tile nt): groups of 8 X tiles × all pairs, so a wave
// of pairs shares A and X bands through L2 (as make_sched's raster)
__device__ __forceinline__ void pair_tile(int t, int m_pairs, int n_tiles, int* mp, int* nt) {
    const int gn0 = n_tiles < 8 ? n_tiles : 8, gsz = gn0 * m_pairs;
    const int g = t / gsz, first = g * gn0, gn = min(gn0, n_tiles - first), r = t - g * gsz;
    *nt = first + r % gn;
    *mp = r / gn;
}

template <bool H>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P2_THREADS, 1)
k_umma2_rowsq(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX, int M, int m_pairs,
              int n_tiles, int k_tiles, double* __restrict__ partial, unsigned int* __restrict__ wave_ctr, int x_il,
              const int* __restrict__ tiles, int ntiles, int l2hint) {
    // tiles (nullable): the 128-column M tiles to compute, pairs taken in list order (the others'
    // rows of `partial` are left untouched); a missing second tile reads as TMA zeros past M
    auto m_of = [&](int mp, uint32_t r) { const int i = 2 * mp + (int)r; return tiles ? (i < ntiles ? tiles[i] : (M + BM - 1) / BM) : i; };
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(smem + P2_STAGES * P2_STAGE);
    uint64_t* full = bars;                     // [STAGES] leader: both CTAs' bytes
    uint64_t* empty = full + P2_STAGES;        // [STAGES] each CTA: multicast MMA commit
    uint64_t* tfull = empty + P2_STAGES;       // [2]      each CTA: multicast MMA commit
    uint64_t* tempty = tfull + 2;              // [2]      leader: both CTAs' drains
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    const int warp = warp_index(), lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int total = m_pairs * n_tiles;
    constexpr int NTP = 4;                     // N tiles (of 64) per pair tile = 256 columns
    constexpr uint32_t FMT = H ? 0u : 2u;   // f16 / tf32 operands
    constexpr int BKE = bke<H>();
    constexpr uint32_t IDESC = (1u << 4) | (FMT << 7) | (FMT << 10) | ((uint32_t)((NTP * BN) >> 3) << 17) |
                               ((uint32_t)(2 * BM >> 4) << 24);   // M = 256, N = 256
    if (threadIdx.x == 0) {
        for (int s = 0; s < P2_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * P2_NDRAIN);  // one (remote) arrive per drain warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int dbg = __shfl_sync(0xffffffffu, g_dbg_flags, 0);

    if (warp == 0) {
        // ---------------------------------------------------------------- producer
        if (lane == 0) {
            const uint32_t full0 = map_to_rank(smem_u32(&full[0]), 0);  // leader's barriers
            int gi = 0;
            for (int t = pair, w = 0; t < total; t += npairs, ++w) {
                if (wave_ctr && w > 0) {  // wave barrier: every CTA issued wave w-1 (lockstep along K)
                    unsigned int target = 0;
                    for (int v = 0; v < w; ++v) target += 2u * (unsigned int)max(0, min(npairs, total - v * npairs));
                    unsigned int val;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(val) : "l"(wave_ctr) : "memory");
                    } while (val < target);
                }
                int mp, nt;
                pair_tile(t, m_pairs, n_tiles, &mp, &nt);
                const int m_tile = m_of(mp, rank);
                for (int i = 0; i < k_tiles; ++i, ++gi) {
                    const int s = gi % P2_STAGES;
                    mbar_wait(&empty[s], ((uint32_t)(gi / P2_STAGES) & 1u) ^ 1u);
                    if (rank == 0) mbar_expect_tx(&full[s], 2 * P2_STAGE);
                    const uint32_t fb = full0 + s * 8;
                    const int k0 = i * BKE;
                    uint8_t* st = smem + s * P2_STAGE;
                    const uint64_t pa = l2hint >= 2 ? L2_EVICT_FIRST : 0, px = l2hint >= 1 ? L2_EVICT_LAST : 0;
                    if (H)  // the interleaved hi/lo copy (4-D map; hi = part 0)
                        tma2sm_4d(smem_u32(st), &tmA, fb, 0, 0, k0 / 64, m_tile * BM, pa);
                    else
                        tma2sm_2d(smem_u32(st), &tmA, fb, k0, m_tile * BM, pa);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int xc = (nt * NTP + (int)rank * 2 + h) * BN;
                        if (x_il)  // hi of an interleaved split (4-D map, part 0)
                            tma2sm_4d(smem_u32(st + A_TILE + h * X_TILE), &tmX, fb, 0, 0, k0 / 64, xc, px);
                        else
                            tma2sm_2d(smem_u32(st + A_TILE + h * X_TILE), &tmX, fb, k0, xc, px);
                    }
                }
                if (wave_ctr) atomicAdd(wave_ctr, 1u);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------- MMA issuer (leader only)
        if (rank == 0) {
            int gi = 0, gc = 0;
            for (int t = pair; t < total; t += npairs) {
                for (int i = 0; i < k_tiles; ++i, ++gi) {
                    const int s = gi % P2_STAGES;
                    const int c = gc + i / CH, b = c & 1;
                    const bool first = (i % CH) == 0;
                    if (first) mbar_wait(&tempty[b], ((uint32_t)(c / 2) & 1u) ^ 1u);
                    mbar_wait(&full[s], (uint32_t)(gi / P2_STAGES) & 1u);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smem + s * P2_STAGE), x0 = a0 + A_TILE;
                    const uint32_t d = tmem + (uint32_t)(b * NTP * BN);
#pragma unroll
                    for (int k8 = 0; k8 < BK / 8; ++k8) {
                        const uint64_t da = sdesc(a0 + k8 * 32, 16, 1024, 2);
                        const uint64_t dx = sdesc(x0 + k8 * 32, 16, 1024, 2);
                        const uint32_t acc = (!first || k8 > 0) ? 1u : 0u;
                        if (!(dbg & 4) && H)
                            asm volatile(
                                "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(da),
                                "l"(dx), "r"(IDESC), "r"(acc));
                        else if (!(dbg & 4))
                            asm volatile(
                                "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(da),
                                "l"(dx), "r"(IDESC), "r"(acc));
                    }
                    asm volatile(
                        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                        " [%0], %1;\n\t}" ::"r"(smem_u32(&empty[s])), "h"((uint16_t)3) : "memory");
                    if ((i % CH) == CH - 1 || i == k_tiles - 1)
                        asm volatile(
                            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                            " [%0], %1;\n\t}" ::"r"(smem_u32(&tfull[b])), "h"((uint16_t)3) : "memory");
                    __syncwarp();
                }
                gc += (k_tiles + CH - 1) / CH;
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------- drain (both CTAs, own TMEM rows)
        const int q = warp & 3, tile = (warp - 4) >> 2;   // lane quarter, 64-column tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t tempty0 = map_to_rank(smem_u32(&tempty[0]), 0);
        int gc = 0;
        const int nchunks = (k_tiles + CH - 1) / CH;
        for (int t = pair; t < total; t += npairs) {
            int mp, nt;
            pair_tile(t, m_pairs, n_tiles, &mp, &nt);
            const int row = m_of(mp, rank) * BM + q * 32 + lane;
            float acc[BN];
#pragma unroll
            for (int j = 0; j < BN; ++j) acc[j] = 0.0f;
            for (int c = 0; c < nchunks; ++c) {
                const int g = gc + c, b = g & 1;
                mbar_wait(&tfull[b], (uint32_t)(g / 2) & 1u);
                tc_fence_after();
                if (!(dbg & 2)) {
                    const uint32_t t0 = tmem + lane_off + (uint32_t)(b * NTP * BN + tile * BN);
#pragma unroll
                    for (int j0 = 0; j0 < BN; j0 += 16) {
                        uint32_t h[16];
                        TMEM_LD16(t0 + j0, h);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc[j0 + j] += __uint_as_float(h[j]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0)  // default (cta-scope release) form: a .cluster-scope release is a GPU-wide MEMBAR
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(tempty0 + b * 8) : "memory");
            }
            gc += nchunks;
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < BN; ++j) {
                const double v = (double)acc[j];
                s = fma(v, v, s);  // columns ≥ N are exact zeros (TMA zero fill)
            }
            if (row < M) partial[(int64_t)(nt * NTP + tile) * M + row] = s;
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// ------------------------------------------- CTA-pair 3×TF32 product (cta_group::2)
// Out = alpha·op(A)·X + beta·Out with 3×TF32 operands (as k_umma X3), one CTA pair per
// 256 output rows × 128 output columns.  Each CTA stages its own 128-row A tile and HALF
// of x_hi and x_lo (32 KB per stage against 48 KB for a single-CTA N = 128 X3 stage), and
// computes a_lo = a − trunc(a) into its own ring; the leader issues three M = 256 × N = 128
// MMAs per k-step (a·x_hi → hi, a·x_lo → lo, a_lo·x_hi → lo) that read both CTAs' shared
// memory.  (The single-CTA kernel fuses a·[x_hi | x_lo] into one N = 256 instruction; with
// B split across the pair at equal offsets the lo half would not be contiguous.)
// Hand-off: a CTA's transform warps meet at a named barrier after their a_lo stores and
// one thread arrives (cluster-scope release) on the leader's lo_ready — that arrive also
// vouches for the CTA's TMA bytes, which the transform waited for.
struct PSched {
    int m_pairs, n_tiles, total, k_tiles, sym, tri_x;
    unsigned int* wave_ctr;
    int bke;   // K elements per k-tile (32 tf32, 64 fp16): the triangular-X limit is in these units
    int x_il;  // H3: x_hi/x_lo from one interleaved split (4-D map, part = hi|lo)
    int hi_only;  // k_umma2_h3m: a_hi·x_hi only (GEMM_HI_ONLY): the lo halves are neither loaded nor used
};
constexpr int X3P_NTRANSFORM = 6, X3P_NDRAIN = 8;
constexpr int X3P_THREADS = 32 * (2 + X3P_NTRANSFORM + X3P_NDRAIN);        // 512
constexpr uint32_t X3P_STAGE = A_TILE + 2 * X_TILE;                          // A + x_hi half + x_lo half
constexpr int X3P_LO = 3;
constexpr int X3P_STAGES = (int)((232448u - 1280u - X3P_LO * A_TILE) / X3P_STAGE);
constexpr uint32_t X3P_SMEM = X3P_STAGES * X3P_STAGE + X3P_LO * A_TILE + 1024 + 256;
constexpr uint32_t X3P_R0 = (65536u / X3P_THREADS) / 8 * 8;                  // 128
constexpr uint32_t X3P_REG_LOW = 56;
constexpr uint32_t X3P_REG_DRAIN_FIT =
    X3P_R0 + ((X3P_THREADS - 32 * X3P_NDRAIN) * (X3P_R0 - X3P_REG_LOW) / (32 * X3P_NDRAIN)) / 8 * 8;
constexpr uint32_t X3P_REG_DRAIN = X3P_REG_DRAIN_FIT > 232 ? 232 : X3P_REG_DRAIN_FIT;

// pair tile t → (row pair mp, 128-column tile nt, k stages).  sym: only tiles touching the
// upper triangle (256·mp ≤ 128·nt + 127), column by column.
__device__ __forceinline__ void x3p_tile(const PSched& sc, int t, int* mp, int* nt, int* nk) {
    if (sc.sym) {
        int n = 0;
        for (;; ++n) {
            const int cnt = min(n / 2, sc.m_pairs - 1) + 1;
            if (t < cnt) break;
            t -= cnt;
        }
        *nt = n;
        *mp = t;
    } else {
        pair_tile(t, sc.m_pairs, sc.n_tiles, mp, nt);
        // triangular X: N tile j carries j + 1 diagonal blocks of K — the widest group first
        // (with no wave barrier the short tiles of the last group fill the tail)
        if (sc.tri_x) *nt = sc.n_tiles - 1 - *nt;
    }
    *nk = sc.tri_x ? min(sc.k_tiles, ((*nt + 1) * 2 * BN + sc.bke - 1) / sc.bke) : sc.k_tiles;
}

template <bool A_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(X3P_THREADS, 1)
k_umma2_x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
           const __grid_constant__ CUtensorMap tmXl, int M, int N, const PSched sc, double* __restrict__ out,
           int64_t ldo, double alpha, double beta) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(smem + X3P_STAGES * X3P_STAGE + X3P_LO * A_TILE);
    uint64_t* full = bars;                       // [STAGES] own TMA bytes
    uint64_t* empty = full + X3P_STAGES;         // [STAGES] multicast MMA commit
    uint64_t* lo_ready = empty + X3P_STAGES;     // [LO]     leader: one arrive per CTA
    uint64_t* lo_empty = lo_ready + X3P_LO;      // [LO]     multicast MMA commit
    uint64_t* tfull = lo_empty + X3P_LO;         // [2]      multicast MMA commit
    uint64_t* tempty = tfull + 2;                // [2]      leader: both CTAs' drain warps
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    const int warp = warp_index(), lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    constexpr int NTP = 2;  // 64-column tiles per pair tile
    constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((A_MN ? 1u : 0u) << 15) |
                               ((uint32_t)((NTP * BN) >> 3) << 17) | ((uint32_t)(2 * BM >> 4) << 24);
    constexpr uint32_t BUF = 2 * NTP * BN;  // hi + lo columns per TMEM buffer
    if (threadIdx.x == 0) {
        for (int s = 0; s < X3P_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int l = 0; l < X3P_LO; ++l) {
            mbar_init(&lo_ready[l], 2);
            mbar_init(&lo_empty[l], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * X3P_NDRAIN);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmXh) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmXl) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    auto a_raw = [&](int s) { return smem + s * X3P_STAGE; };
    auto x_hi = [&](int s) { return smem + s * X3P_STAGE + A_TILE; };
    auto x_lo = [&](int s) { return smem + s * X3P_STAGE + A_TILE + X_TILE; };
    auto a_lo = [&](int l) { return smem + X3P_STAGES * X3P_STAGE + l * A_TILE; };

    if (warp >= 4 && warp < 4 + X3P_NDRAIN) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(X3P_REG_DRAIN));
        // ------------------------------------------- drain (both CTAs, own TMEM rows)
        const int q = warp & 3, tile = (warp - 4) >> 2;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t tempty0 = map_to_rank(smem_u32(&tempty[0]), 0);
        int gc = 0;
        for (int t = pair; t < sc.total; t += npairs) {
            int mp, nt, nk;
            x3p_tile(sc, t, &mp, &nt, &nk);
            const int nchunks = (nk + CH - 1) / CH;
            const int row = (2 * mp + (int)rank) * BM + q * 32 + lane;
            float acc[BN], cmp[BN];
#pragma unroll
            for (int j = 0; j < BN; ++j) acc[j] = cmp[j] = 0.0f;
            for (int c = 0; c < nchunks; ++c) {
                const int g = gc + c, b = g & 1;
                mbar_wait(&tfull[b], (uint32_t)(g / 2) & 1u);
                tc_fence_after();
                const uint32_t t_hi = tmem + lane_off + (uint32_t)(b * BUF + tile * BN), t_lo = t_hi + NTP * BN;
#pragma unroll
                for (int j0 = 0; j0 < BN; j0 += 8) {
                    uint32_t h[8], l[8];
                    TMEM_LD8(t_hi + j0, h);
                    TMEM_LD8(t_lo + j0, l);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int e = j0 + j;
                        const float hv = __uint_as_float(h[j]), lv = __uint_as_float(l[j]);
                        const float tt = __fadd_rn(hv, lv);
                        const float et = __fsub_rn(lv, __fsub_rn(tt, hv));  // Fast2Sum, |hi| ≥ |lo|
                        const float sum = __fadd_rn(acc[e], tt);
                        const float z = __fsub_rn(sum, acc[e]);
                        cmp[e] = __fadd_rn(cmp[e], __fadd_rn(__fsub_rn(tt, z), et));
                        acc[e] = sum;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0)  // default (cta-scope) form, as k_umma2_rowsq
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(tempty0 + b * 8) : "memory");
            }
            gc += nchunks;
            const int col0 = nt * NTP * BN + tile * BN;
            if (row < M) {
                const int ncol = min(BN, N - col0);
                double* dst = out + row;
#pragma unroll
                for (int j = 0; j < BN; ++j) {
                    const double v = (double)acc[j] + (double)cmp[j];
                    if (j < ncol) {
                        double* o = dst + (int64_t)(col0 + j) * ldo;
                        *o = beta == 0.0 ? alpha * v : fma(beta, *o, alpha * v);
                    }
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(X3P_REG_LOW));
        if (warp == 0) {
            // ---------------------------------------------------------------- producer
            if (lane == 0) {
                constexpr int PF = 12;
                int gi = 0;
                for (int t = pair, w = 0; t < sc.total; t += npairs, ++w) {
                    if (sc.wave_ctr && w > 0) {
                        unsigned int target = 0;
                        for (int v = 0; v < w; ++v)
                            target += 2u * (unsigned int)max(0, min(npairs, sc.total - v * npairs));
                        unsigned int val;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(val) : "l"(sc.wave_ctr) : "memory");
                        } while (val < target);
                    }
                    int mp, nt, nk;
                    x3p_tile(sc, t, &mp, &nt, &nk);
                    const int m_tile = 2 * mp + (int)rank, xc = (nt * NTP + (int)rank) * BN;
                    auto prefetch_a = [&](int i) {
                        if (A_MN) tma_prefetch_3d(&tmA, 0, i * BK, m_tile * (BM / 32));
                        else tma_prefetch_2d(&tmA, i * BK, m_tile * BM);
                    };
                    for (int i = 0; i < PF && i < nk; ++i) prefetch_a(i);
                    for (int i = 0; i < nk; ++i, ++gi) {
                        const int s = gi % X3P_STAGES;
                        if (i + PF < nk) prefetch_a(i + PF);
                        mbar_wait(&empty[s], ((uint32_t)(gi / X3P_STAGES) & 1u) ^ 1u);
                        mbar_expect_tx(&full[s], X3P_STAGE);
                        const int k0 = i * BK;
                        if (A_MN) tma_load_3d(a_raw(s), &tmA, &full[s], 0, k0, m_tile * (BM / 32));
                        else tma_load_2d(a_raw(s), &tmA, &full[s], k0, m_tile * BM);
                        tma_load_2d(x_hi(s), &tmXh, &full[s], k0, xc);
                        tma_load_2d(x_lo(s), &tmXl, &full[s], k0, xc);
                    }
                    if (sc.wave_ctr) atomicAdd(sc.wave_ctr, 1u);
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------- MMA issuer (leader only)
            if (rank == 0) {
                int gi = 0, gc = 0;
                for (int t = pair; t < sc.total; t += npairs) {
                    int mp, nt, nk;
                    x3p_tile(sc, t, &mp, &nt, &nk);
                    for (int i = 0; i < nk; ++i, ++gi) {
                        const int s = gi % X3P_STAGES, lr = gi % X3P_LO;
                        const int c = gc + i / CH, b = c & 1;
                        const bool first = (i % CH) == 0;
                        if (first) mbar_wait(&tempty[b], ((uint32_t)(c / 2) & 1u) ^ 1u);
                        mbar_wait(&lo_ready[lr], (uint32_t)(gi / X3P_LO) & 1u);
                        tc_fence_after();
                        const uint32_t ar = smem_u32(a_raw(s)), al = smem_u32(a_lo(lr));
                        const uint32_t xh = smem_u32(x_hi(s)), xl = smem_u32(x_lo(s));
                        const uint32_t d_hi = tmem + (uint32_t)(b * BUF), d_lo = d_hi + NTP * BN;
#pragma unroll
                        for (int k8 = 0; k8 < BK / 8; ++k8) {
                            uint64_t da_r, da_l;
                            if (A_MN) {
                                da_r = sdesc(ar + k8 * 1024, 4096, 512, 1);
                                da_l = sdesc(al + k8 * 1024, 4096, 512, 1);
                            } else {
                                da_r = sdesc(ar + k8 * 32, 16, 1024, 2);
                                da_l = sdesc(al + k8 * 32, 16, 1024, 2);
                            }
                            const uint64_t dxh = sdesc(xh + k8 * 32, 16, 1024, 2);
                            const uint64_t dxl = sdesc(xl + k8 * 32, 16, 1024, 2);
                            const uint32_t acc = (!first || k8 > 0) ? 1u : 0u;
                            asm volatile(
                                "{\n\t.reg .pred e, p, one;\n\telect.sync _|e, 0xffffffff;\n\t"
                                "setp.ne.b32 p, %7, 0;\n\tsetp.eq.b32 one, %7, %7;\n\t"
                                "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %2, %3, %6, p;\n\t"
                                "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], %2, %4, %6, p;\n\t"
                                "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], %5, %3, %6, one;\n\t}" ::"r"(d_hi),
                                "r"(d_lo), "l"(da_r), "l"(dxh), "l"(dxl), "l"(da_l), "r"(IDESC), "r"(acc));
                        }
                        asm volatile(
                            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                            " [%0], %2;\n\t"
                            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                            " [%1], %2;\n\t}" ::"r"(smem_u32(&empty[s])), "r"(smem_u32(&lo_empty[lr])),
                            "h"((uint16_t)3) : "memory");
                        if ((i % CH) == CH - 1 || i == nk - 1)
                            asm volatile(
                                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                                "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                                " [%0], %1;\n\t}" ::"r"(smem_u32(&tfull[b])), "h"((uint16_t)3) : "memory");
                        __syncwarp();
                    }
                    gc += (nk + CH - 1) / CH;
                }
            }
        } else {
            // ------------------------------------------- a_lo transform (both CTAs)
            constexpr int NTT = 32 * X3P_NTRANSFORM;
            const int tid = (warp < 4 ? warp - 2 : warp - (4 + X3P_NDRAIN) + 2) * 32 + lane;
            const uint32_t lo_ready0 = map_to_rank(smem_u32(&lo_ready[0]), 0);
            int gi = 0;
            for (int t = pair; t < sc.total; t += npairs) {
                int mp, nt, nk;
                x3p_tile(sc, t, &mp, &nt, &nk);
                for (int i = 0; i < nk; ++i, ++gi) {
                    const int s = gi % X3P_STAGES, lr = gi % X3P_LO;
                    mbar_wait(&full[s], (uint32_t)(gi / X3P_STAGES) & 1u);
                    mbar_wait(&lo_empty[lr], ((uint32_t)(gi / X3P_LO) & 1u) ^ 1u);
                    const uint32_t src = smem_u32(a_raw(s)), dst = smem_u32(a_lo(lr));
                    transform_tile<NTT>(src, dst, tid, lo_of);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile("bar.sync 1, %0;" ::"n"(NTT) : "memory");
                    if (tid == 0)
                        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(lo_ready0 + lr * 8)
                                     : "memory");
                }
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <bool A_MN>
void launch_umma2_x3(Ctx* c, PSched sc, const CUtensorMap& ta, const CUtensorMap& th, const CUtensorMap& tl, int M,
                     int N, double* out, int64_t ldo, double alpha, double beta) {
    auto kern = k_umma2_x3<A_MN>;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, X3P_SMEM));
        attr = true;
    }
    const int pairs = std::min(sc.total, c->sm_count / 2);
    DevBuf ctr;
    sc.wave_ctr = nullptr;
    if (pairs < sc.total && !g_wave_barrier_off) {  // ≤ 1 CTA per SM: all co-resident
        ctr = DevBuf(c, 64);
        CUDA_CHECK(cudaMemsetAsync(ctr.ptr, 0, 4, c->stream));
        sc.wave_ctr = ctr.as<unsigned int>();
    }
    kern<<<2 * pairs, X3P_THREADS, X3P_SMEM, c->stream>>>(ta, th, tl, M, N, sc, out, ldo, alpha, beta);
    LAUNCH_CHECK(c);
}
PSched make_psched(int mt, int nt, int k_tiles, bool sym, bool tri_x) {
    PSched sc;
    sc.m_pairs = (mt + 1) / 2;
    sc.n_tiles = nt;
    sc.k_tiles = k_tiles;
    sc.sym = sym ? 1 : 0;
    sc.tri_x = tri_x ? 1 : 0;
    sc.wave_ctr = nullptr;
    sc.bke = BK;
    sc.x_il = 0;
    sc.hi_only = 0;
    if (sym) {
        sc.total = 0;
        for (int n = 0; n < nt; ++n) sc.total += std::min(n / 2, sc.m_pairs - 1) + 1;
    } else {
        sc.total = sc.m_pairs * nt;
    }
    return sc;
}


// ------------------------------------------- CTA-pair 3×FP16 product (cta_group::2)
// The tensor-bound 3×FP16 products (Grams of C and Q1, C·R⁻¹, the CholQR2 correction, c4's
// Aᵀ·Q_C) on CTA pairs: one pair per 256 output rows × 128 output columns.  Each CTA stages
// its own 128-row a_hi/a_lo tile and HALF of x_hi/x_lo (48 KB per stage; both CTAs' TMA bytes
// land on the leader's barrier through the 2-SM TMA form), and the leader issues three M = 256
// × N = 128 MMAs per k-step (a_hi·x_hi → hi, a_hi·x_lo → lo, a_lo·x_hi → lo) that read both
// CTAs' shared memory.  Per SM and k-step that is 18 KB of operand reads + 12 KB of TMA writes
// for 2·786 K flop, against 20 + 16 KB for the single-CTA N = 128 H3 tile — the single-CTA
// kernel is bound by shared-memory bandwidth (0.67 of the f16 MMA rate measured, 0.67 modelled).
// Epilogues as k_umma's H3 forms: STORE (α, β, exact scale removal), SPLIT, BASIS.
constexpr int H2_NDRAIN = 8;                                  // 4 lane quarters × 2 64-column tiles
constexpr int H2_THREADS = 32 * (4 + H2_NDRAIN);              // producer, MMA, 2 idle, drains
constexpr uint32_t H2_STAGE = 2 * A_TILE + 2 * X_TILE;        // a_hi, a_lo, x_hi half, x_lo half
constexpr int H2_STAGES = (int)((232448u - 1280u) / H2_STAGE);
constexpr uint32_t H2_SMEM = H2_STAGES * H2_STAGE + 1024 + 256;
constexpr uint32_t H2_R0 = (65536u / H2_THREADS) / 8 * 8;     // 168
constexpr uint32_t H2_REG_LOW = 56;
constexpr uint32_t H2_REG_DRAIN_FIT = H2_R0 + ((H2_THREADS - 32 * H2_NDRAIN) * (H2_R0 - H2_REG_LOW) / (32 * H2_NDRAIN)) / 8 * 8;
constexpr uint32_t H2_REG_DRAIN = H2_REG_DRAIN_FIT > 232 ? 232 : H2_REG_DRAIN_FIT;

template <bool A_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(H2_THREADS, 1)
k_umma2_h3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
           const __grid_constant__ CUtensorMap tmXl, int M, int N, const PSched sc, void* __restrict__ out_v,
           int64_t ldo, double alpha, double beta, const int* __restrict__ rexp, const int* __restrict__ cexp,
           uint16_t* __restrict__ q16, const uint16_t* __restrict__ aux) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(smem + H2_STAGES * H2_STAGE);
    uint64_t* full = bars;                     // [STAGES] leader: both CTAs' bytes
    uint64_t* empty = full + H2_STAGES;        // [STAGES] each CTA: multicast MMA commit
    uint64_t* tfull = empty + H2_STAGES;       // [2]      each CTA: multicast MMA commit
    uint64_t* tempty = tfull + 2;              // [2]      leader: both CTAs' drain warps
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    const int warp = warp_index(), lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    constexpr int NTP = 2;                     // 64-column tiles per pair tile
    constexpr int BKH = bke<true>();
    constexpr uint32_t IDESC = (1u << 4) | ((A_MN ? 1u : 0u) << 15) | ((uint32_t)((NTP * BN) >> 3) << 17) |
                               ((uint32_t)(2 * BM >> 4) << 24);   // f16 × f16 → f32, M = 256, N = 128
    constexpr uint32_t BUF = 2 * NTP * BN;     // hi + lo columns per TMEM buffer
    if (threadIdx.x == 0) {
        for (int s = 0; s < H2_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * H2_NDRAIN);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmXh) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmXl) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    auto a_hi = [&](int s) { return smem + s * H2_STAGE; };
    auto x_hi = [&](int s) { return smem + s * H2_STAGE + 2 * A_TILE; };

    if (warp >= 4) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(H2_REG_DRAIN));
        // ------------------------------------------- drain (both CTAs, own TMEM rows)
        const int q = warp & 3, tile = (warp - 4) >> 2;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t tempty0 = map_to_rank(smem_u32(&tempty[0]), 0);
        int gc = 0;
        for (int t = pair; t < sc.total; t += npairs) {
            int mp, nt, nk;
            x3p_tile(sc, t, &mp, &nt, &nk);
            const int nchunks = (nk + CH - 1) / CH;
            const int row = (2 * mp + (int)rank) * BM + q * 32 + lane;
            float acc[BN], cmp[BN];
#pragma unroll
            for (int j = 0; j < BN; ++j) acc[j] = cmp[j] = 0.0f;
            for (int c = 0; c < nchunks; ++c) {
                const int g = gc + c, b = g & 1;
                mbar_wait(&tfull[b], (uint32_t)(g / 2) & 1u);
                tc_fence_after();
                const uint32_t t_hi = tmem + lane_off + (uint32_t)(b * BUF + tile * BN), t_lo = t_hi + NTP * BN;
#pragma unroll
                for (int j0 = 0; j0 < BN; j0 += 8) {
                    uint32_t h[8], l[8];
                    TMEM_LD8(t_hi + j0, h);
                    TMEM_LD8(t_lo + j0, l);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 8; ++j) {  // as k_umma's X3 drain: Fast2Sum of hi, cross terms into cmp
                        const int e = j0 + j;
                        const float hv = __uint_as_float(h[j]);
                        const float sum = __fadd_rn(acc[e], hv);
                        const float z = __fsub_rn(sum, acc[e]);
                        cmp[e] = __fadd_rn(cmp[e], __fadd_rn(__fsub_rn(hv, z), __uint_as_float(l[j])));
                        acc[e] = sum;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0)  // default (cta-scope) form, as k_umma2_rowsq
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(tempty0 + b * 8) : "memory");
            }
            gc += nchunks;
            const int col0 = nt * NTP * BN + tile * BN;
            if (row < M) {
                const int ncol = min(BN, N - col0);
                const int re = rexp ? rexp[row] : 0;
                if (EPI == EPI_STORE) {
                    double* dst = reinterpret_cast<double*>(out_v) + row;
                    constexpr int EB = 16;  // β ≠ 0: old values loaded 16 at a time before the stores
#pragma unroll
                    for (int j0 = 0; j0 < BN; j0 += EB) {
                        double old[EB];
#pragma unroll
                        for (int jj = 0; jj < EB; ++jj)
                            old[jj] = (beta != 0.0 && j0 + jj < ncol) ? dst[(int64_t)(col0 + j0 + jj) * ldo] : 0.0;
#pragma unroll
                        for (int jj = 0; jj < EB; ++jj) {
                            const int j = j0 + jj;
                            if (j >= ncol) continue;
                            double v = (double)acc[j] + (double)cmp[j];
                            v *= exp2_int(-(re + (cexp ? cexp[col0 + j] : 0)));
                            dst[(int64_t)(col0 + j) * ldo] = beta == 0.0 ? alpha * v : fma(beta, old[jj], alpha * v);
                        }
                    }
                } else {
                    const int64_t r_il = (int64_t)(row >> 6) * 128 + (row & 63);
                    float ax8[8];  // BASIS: 8 columns' aux values per round trip (see k_umma)
#pragma unroll
                    for (int j = 0; j < BN; ++j) {
                        if (EPI == EPI_BASIS && (j & 7) == 0) {
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj) {
                                ax8[jj] = 0.0f;
                                if (aux && j + jj < ncol) {
                                    const int64_t o = (int64_t)(col0 + j + jj) * 2 * M + r_il;
                                    const uint16_t hb = aux[o], lb = aux[o + 64];
                                    ax8[jj] = __half2float(*reinterpret_cast<const __half*>(&hb)) +
                                              __half2float(*reinterpret_cast<const __half*>(&lb));
                                }
                            }
                        }
                        if (j >= ncol) continue;
                        const int col = col0 + j;
                        double v = ((double)acc[j] + (double)cmp[j]) * (alpha * exp2_int(-(re + (cexp ? cexp[col] : 0))));
                        if (EPI == EPI_SPLIT) {
                            uint16_t* o16 = reinterpret_cast<uint16_t*>(out_v);
                            const double sv = v * (double)(1 << BASIS_E);
                            const __half h = __double2half(sv);
                            const __half l = __double2half(sv - (double)__half2float(h));
                            o16[(int64_t)col * 2 * M + r_il] = *reinterpret_cast<const uint16_t*>(&h);
                            o16[(int64_t)col * 2 * M + r_il + 64] = *reinterpret_cast<const uint16_t*>(&l);
                        } else {
                            v += (double)ax8[j & 7] * (1.0 / (double)(1 << BASIS_E));
                            reinterpret_cast<float*>(out_v)[row + (int64_t)col * ldo] = (float)v;
                            const double sv = v * (double)(1 << BASIS_E);  // interleaved hi/lo, as k_umma
                            const __half h = __double2half(sv);
                            const __half l = __double2half(sv - (double)__half2float(h));
                            q16[(int64_t)col * 2 * M + r_il] = *reinterpret_cast<const uint16_t*>(&h);
                            q16[(int64_t)col * 2 * M + r_il + 64] = *reinterpret_cast<const uint16_t*>(&l);
                        }
                    }
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(H2_REG_LOW));
        if (warp == 0) {
            // ---------------------------------------------------------------- producer
            if (lane == 0) {
                const uint32_t full0 = map_to_rank(smem_u32(&full[0]), 0);  // leader's barriers
                int gi = 0;
                for (int t = pair, w = 0; t < sc.total; t += npairs, ++w) {
                    if (sc.wave_ctr && w > 0) {  // wave barrier (see Sched)
                        unsigned int target = 0;
                        for (int v = 0; v < w; ++v)
                            target += 2u * (unsigned int)max(0, min(npairs, sc.total - v * npairs));
                        unsigned int val;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(val) : "l"(sc.wave_ctr) : "memory");
                        } while (val < target);
                    }
                    int mp, nt, nk;
                    x3p_tile(sc, t, &mp, &nt, &nk);
                    const int m_tile = 2 * mp + (int)rank, xc = (nt * NTP + (int)rank) * BN;
                    for (int i = 0; i < nk; ++i, ++gi) {
                        const int s = gi % H2_STAGES;
                        mbar_wait(&empty[s], ((uint32_t)(gi / H2_STAGES) & 1u) ^ 1u);
                        if (rank == 0) mbar_expect_tx(&full[s], 2 * H2_STAGE);
                        const uint32_t fb = full0 + s * 8;
                        const int k0 = i * BKH;
                        const uint32_t sa = smem_u32(a_hi(s)), sx = smem_u32(x_hi(s));
                        auto load4 = [&](uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3) {
                            asm volatile(
                                "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                                " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst), "l"(tm), "r"(fb), "r"(c0), "r"(c1),
                                "r"(c2), "r"(c3) : "memory");
                        };
#pragma unroll
                        for (int hl = 0; hl < 2; ++hl) {  // A: the interleaved hi/lo copy (4-D map)
                            if (A_MN) {  // two 64-row chunks (8 KB MN atoms) × 64 K rows
                                load4(sa + hl * A_TILE, &tmA, 0, hl, m_tile * 2, k0);
                                load4(sa + hl * A_TILE + A_TILE / 2, &tmA, 0, hl, m_tile * 2 + 1, k0);
                            } else {
                                load4(sa + hl * A_TILE, &tmA, 0, hl, k0 / 64, m_tile * BM);
                            }
                        }
                        if (sc.x_il) {
                            load4(sx, &tmXh, 0, 0, k0 / 64, xc);
                            load4(sx + X_TILE, &tmXh, 0, 1, k0 / 64, xc);
                        } else {
#pragma unroll
                            for (int hl = 0; hl < 2; ++hl)
                                asm volatile(
                                    "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                                    " [%0], [%1, {%3, %4}], [%2];" ::"r"(sx + hl * X_TILE), "l"(hl ? &tmXl : &tmXh),
                                    "r"(fb), "r"(k0), "r"(xc) : "memory");
                        }
                    }
                    if (sc.wave_ctr) atomicAdd(sc.wave_ctr, 1u);
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------- MMA issuer (leader only)
            if (rank == 0) {
                int gi = 0, gc = 0;
                for (int t = pair; t < sc.total; t += npairs) {
                    int mp, nt, nk;
                    x3p_tile(sc, t, &mp, &nt, &nk);
                    for (int i = 0; i < nk; ++i, ++gi) {
                        const int s = gi % H2_STAGES;
                        const int c = gc + i / CH, b = c & 1;
                        const bool first = (i % CH) == 0;
                        if (first) mbar_wait(&tempty[b], ((uint32_t)(c / 2) & 1u) ^ 1u);
                        mbar_wait(&full[s], (uint32_t)(gi / H2_STAGES) & 1u);
                        tc_fence_after();
                        const uint32_t ah = smem_u32(a_hi(s)), al = ah + A_TILE;
                        const uint32_t xh = smem_u32(x_hi(s)), xl = xh + X_TILE;
                        const uint32_t d_hi = tmem + (uint32_t)(b * BUF), d_lo = d_hi + NTP * BN;
#pragma unroll
                        for (int k8 = 0; k8 < BK / 8; ++k8) {
                            uint64_t dah, dal;
                            if (A_MN) {  // [2 MN atoms of 64, 8 KB apart][64 K rows of 128 B, 8-row groups 1 KB apart]
                                dah = sdesc(ah + k8 * 2048, 8192, 1024, 2);
                                dal = sdesc(al + k8 * 2048, 8192, 1024, 2);
                            } else {
                                dah = sdesc(ah + k8 * 32, 16, 1024, 2);
                                dal = sdesc(al + k8 * 32, 16, 1024, 2);
                            }
                            const uint64_t dxh = sdesc(xh + k8 * 32, 16, 1024, 2);
                            const uint64_t dxl = sdesc(xl + k8 * 32, 16, 1024, 2);
                            const uint32_t acc = (!first || k8 > 0) ? 1u : 0u;
                            asm volatile(
                                "{\n\t.reg .pred e, p, one;\n\telect.sync _|e, 0xffffffff;\n\t"
                                "setp.ne.b32 p, %7, 0;\n\tsetp.eq.b32 one, %7, %7;\n\t"
                                "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %6, p;\n\t"
                                "@e tcgen05.mma.cta_group::2.kind::f16 [%1], %2, %4, %6, p;\n\t"
                                "@e tcgen05.mma.cta_group::2.kind::f16 [%1], %5, %3, %6, one;\n\t}" ::"r"(d_hi),
                                "r"(d_lo), "l"(dah), "l"(dxh), "l"(dxl), "l"(dal), "r"(IDESC), "r"(acc));
                        }
                        asm volatile(
                            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                            " [%0], %1;\n\t}" ::"r"(smem_u32(&empty[s])), "h"((uint16_t)3) : "memory");
                        if ((i % CH) == CH - 1 || i == nk - 1)
                            asm volatile(
                                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                                "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                                " [%0], %1;\n\t}" ::"r"(smem_u32(&tfull[b])), "h"((uint16_t)3) : "memory");
                        __syncwarp();
                    }
                    gc += (nk + CH - 1) / CH;
                }
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <bool A_MN, int EPI>
void launch_umma2_h3(Ctx* c, PSched sc, const CUtensorMap& ta, const CUtensorMap& th, const CUtensorMap& tl, int M,
                     int N, void* out, int64_t ldo, double alpha, double beta, const int* rexp, const int* cexp,
                     uint16_t* q16, const uint16_t* aux) {
    auto kern = k_umma2_h3<A_MN, EPI>;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, H2_SMEM));
        attr = true;
    }
    if (sc.total <= 0) return;
    const int pairs = std::min(sc.total, c->sm_count / 2);
    DevBuf ctr;
    sc.wave_ctr = nullptr;
    // the wave barrier keeps a wave's pairs in lockstep along K (L2 sharing); with a triangular X
    // the tiles of a wave differ in length and every wave would wait for its longest tile
    if (pairs < sc.total && !g_wave_barrier_off && !sc.tri_x) {  // ≤ 1 CTA per SM: all co-resident
        ctr = DevBuf(c, 64);
        CUDA_CHECK(cudaMemsetAsync(ctr.ptr, 0, 4, c->stream));
        sc.wave_ctr = ctr.as<unsigned int>();
    }
    kern<<<2 * pairs, H2_THREADS, H2_SMEM, c->stream>>>(ta, th, tl, M, N, sc, out, ldo, alpha, beta, rexp, cexp, q16,
                                                         aux);
    LAUNCH_CHECK(c);
}

// ---------------- CTA-pair 3×FP16 product, one accumulator (M = 256 × N = 192 per pair)
// k_umma2_h3 with the three MMAs of a k-step (a_hi·x_hi, a_hi·x_lo, a_lo·x_hi) summed into ONE
// fp32 TMEM accumulator, which leaves room for N = 192 double-buffered (k_umma2_h3 keeps hi
// and cross terms apart: 2 × 128 columns per buffer).  Per SM and k-step: 21 KB of operand
// reads + 14 KB of TMA writes for 2·1.18 M flop (122 B/clk at the MMA rate, against 156 for
// k_umma2_h3's N = 128: the 128 B/clk shared-memory bound).  (N = 256 would need 16 drain warps
// of 64 fp32 accumulators each in a 96-register budget: they spilled in the drain loop.)  Accuracy: each 8-k-step chunk carries
// the tensor core's round-toward-zero bias over 24 accumulations (~7e-7 relative, systematic)
// and the chunks sum in plain fp32 — fp32-grade, not the ~2⁻²² of the split accumulators, so
// callers opt in (GEMM_FAST_ACC) where the product's error is corrected downstream or far
// inside its bar: c4's Q_CᵀA (U's 1e-4), the first CholQR pass's C·R⁻¹ and the second pass's
// small correction.
constexpr int HM_NTP = 3;                                      // 64-column tiles per pair tile (N = 192)
constexpr int HM_NDRAIN = 4 * HM_NTP;                          // 4 lane quarters × 3 64-column slices
constexpr int HM_THREADS = 32 * (4 + HM_NDRAIN);               // producer, MMA, 2 idle, drains
constexpr int HM_XR = HM_NTP * BN / 2;                         // B rows per CTA (96)
constexpr uint32_t HM_XT = HM_XR * 128;                        // bytes of one B part per stage (12 KB)
constexpr uint32_t HM_STAGE = 2 * A_TILE + 2 * HM_XT;          // a_hi, a_lo, x_hi part, x_lo part
constexpr int HM_STAGES = (int)((232448u - 1280u) / HM_STAGE);
constexpr uint32_t HM_SMEM = HM_STAGES * HM_STAGE + 1024 + 256;
constexpr uint32_t HM_R0 = (65536u / HM_THREADS) / 8 * 8;      // 96
constexpr uint32_t HM_REG_LOW = 56;
constexpr uint32_t HM_REG_DRAIN_FIT = HM_R0 + ((HM_THREADS - 32 * HM_NDRAIN) * (HM_R0 - HM_REG_LOW) / (32 * HM_NDRAIN)) / 8 * 8;

// pair tile t → (row pair mp, 192-column tile nt, k stages); tri_x: widest N group first
__device__ __forceinline__ void hm_tile(const PSched& sc, int t, int* mp, int* nt, int* nk) {
    pair_tile(t, sc.m_pairs, sc.n_tiles, mp, nt);
    if (sc.tri_x) *nt = sc.n_tiles - 1 - *nt;
    *nk = sc.tri_x ? min(sc.k_tiles, ((*nt + 1) * HM_NTP * BN + sc.bke - 1) / sc.bke) : sc.k_tiles;
}

template <bool A_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(HM_THREADS, 1)
k_umma2_h3m(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
            const __grid_constant__ CUtensorMap tmXl, int M, int N, const PSched sc, void* __restrict__ out_v,
            int64_t ldo, double alpha, double beta, const int* __restrict__ rexp, const int* __restrict__ cexp,
            uint16_t* __restrict__ q16, const uint16_t* __restrict__ aux) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(smem + HM_STAGES * HM_STAGE);
    uint64_t* full = bars;                     // [STAGES] leader: both CTAs' bytes
    uint64_t* empty = full + HM_STAGES;        // [STAGES] each CTA: multicast MMA commit
    uint64_t* tfull = empty + HM_STAGES;       // [2]      each CTA: multicast MMA commit
    uint64_t* tempty = tfull + 2;              // [2]      leader: both CTAs' drain warps
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    const int warp = warp_index(), lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    constexpr int NTP = HM_NTP;                // 64-column tiles per pair tile
    constexpr int BKH = bke<true>();
    constexpr uint32_t IDESC = (1u << 4) | ((A_MN ? 1u : 0u) << 15) | ((uint32_t)((NTP * BN) >> 3) << 17) |
                               ((uint32_t)(2 * BM >> 4) << 24);   // f16 × f16 → f32, M = 256, N = 192
    constexpr uint32_t BUF = 256;              // TMEM buffer stride (one N = 192 accumulator each)
    if (threadIdx.x == 0) {
        for (int s = 0; s < HM_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * HM_NDRAIN);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmXh) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmXl) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    auto a_hi = [&](int s) { return smem + s * HM_STAGE; };
    auto x_hi = [&](int s) { return smem + s * HM_STAGE + 2 * A_TILE; };

    if (warp >= 4) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(HM_REG_DRAIN_FIT));
        // ------------------------------------------- drain (both CTAs, own TMEM rows)
        const int q = warp & 3, slice = (warp - 4) >> 2;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t tempty0 = map_to_rank(smem_u32(&tempty[0]), 0);
        int gc = 0;
        for (int t = pair; t < sc.total; t += npairs) {
            int mp, nt, nk;
            hm_tile(sc, t, &mp, &nt, &nk);
            const int nchunks = (nk + CH - 1) / CH;
            const int row = (2 * mp + (int)rank) * BM + q * 32 + lane;
            float acc[BN];
#pragma unroll
            for (int j = 0; j < BN; ++j) acc[j] = 0.0f;
            for (int c = 0; c < nchunks; ++c) {
                const int g = gc + c, b = g & 1;
                mbar_wait(&tfull[b], (uint32_t)(g / 2) & 1u);
                tc_fence_after();
                const uint32_t t0 = tmem + lane_off + (uint32_t)(b * BUF + slice * BN);
#pragma unroll
                for (int j0 = 0; j0 < BN; j0 += 8) {
                    uint32_t h[8];
                    TMEM_LD8(t0 + j0, h);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j0 + j] += __uint_as_float(h[j]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0)  // default (cta-scope) form, as k_umma2_rowsq
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(tempty0 + b * 8) : "memory");
            }
            gc += nchunks;
            const int col0 = nt * NTP * BN + slice * BN;
            if (row < M) {
                const int ncol = min(BN, N - col0);
                const int re = rexp ? rexp[row] : 0;
                if (EPI == EPI_STORE) {
                    double* dst = reinterpret_cast<double*>(out_v) + row;
                    constexpr int EB = 8;  // β ≠ 0: old values loaded 8 at a time before the stores
#pragma unroll
                    for (int j0 = 0; j0 < BN; j0 += EB) {
                        double old[EB];
#pragma unroll
                        for (int jj = 0; jj < EB; ++jj)
                            old[jj] = (beta != 0.0 && j0 + jj < ncol) ? dst[(int64_t)(col0 + j0 + jj) * ldo] : 0.0;
#pragma unroll
                        for (int jj = 0; jj < EB; ++jj) {
                            const int j = j0 + jj;
                            if (j >= ncol) continue;
                            const double v = (double)acc[j] * exp2_int(-(re + (cexp ? cexp[col0 + j] : 0)));
                            dst[(int64_t)(col0 + j) * ldo] = beta == 0.0 ? alpha * v : fma(beta, old[jj], alpha * v);
                        }
                    }
                } else {
                    const int64_t r_il = (int64_t)(row >> 6) * 128 + (row & 63);
                    float ax8[8];  // BASIS: 8 columns' aux values per round trip (see k_umma)
#pragma unroll
                    for (int j = 0; j < BN; ++j) {
                        if (EPI == EPI_BASIS && (j & 7) == 0) {
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj) {
                                ax8[jj] = 0.0f;
                                if (aux && j + jj < ncol) {
                                    const int64_t o = (int64_t)(col0 + j + jj) * 2 * M + r_il;
                                    const uint16_t hb = aux[o], lb = aux[o + 64];
                                    ax8[jj] = __half2float(*reinterpret_cast<const __half*>(&hb)) +
                                              __half2float(*reinterpret_cast<const __half*>(&lb));
                                }
                            }
                        }
                        if (j >= ncol) continue;
                        const int col = col0 + j;
                        // fp32 from here on (this kernel's accumulator is one fp32 sum: GEMM_FAST_ACC).  The
                        // fp64 form — DMULs and three F2F.F16.F64 conversions per element on the XU pipe —
                        // left this epilogue exposed: the hi-only correction ran 19 % tensor-active, 13 % XU
                        // (profiles/r02ar/ncu_full_c3.md).  acc × 2^e is exact, and the split of an fp32
                        // value (hi = rn16(v·2¹⁴), lo = rn16(v·2¹⁴ − hi), the difference exact in fp32) is
                        // the one the fp64 form gave; BASIS adds the aux term with one fp32 rounding, the
                        // rounding of its fp32 output.
                        const float sc = (float)(alpha * exp2_int(-(re + (cexp ? cexp[col] : 0))));
                        float v = acc[j] * sc;
                        if (EPI == EPI_SPLIT) {
                            uint16_t* o16 = reinterpret_cast<uint16_t*>(out_v);
                            const float sv = v * (float)(1 << BASIS_E);
                            const __half h = __float2half_rn(sv);
                            const __half l = __float2half_rn(sv - __half2float(h));
                            o16[(int64_t)col * 2 * M + r_il] = *reinterpret_cast<const uint16_t*>(&h);
                            o16[(int64_t)col * 2 * M + r_il + 64] = *reinterpret_cast<const uint16_t*>(&l);
                        } else {
                            v = fmaf(ax8[j & 7], 1.0f / (float)(1 << BASIS_E), v);
                            reinterpret_cast<float*>(out_v)[row + (int64_t)col * ldo] = v;
                            const float sv = v * (float)(1 << BASIS_E);  // interleaved hi/lo, as k_umma
                            const __half h = __float2half_rn(sv);
                            const __half l = __float2half_rn(sv - __half2float(h));
                            q16[(int64_t)col * 2 * M + r_il] = *reinterpret_cast<const uint16_t*>(&h);
                            q16[(int64_t)col * 2 * M + r_il + 64] = *reinterpret_cast<const uint16_t*>(&l);
                        }
                    }
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(HM_REG_LOW));
        if (warp == 0) {
            // ---------------------------------------------------------------- producer
            if (lane == 0) {
                const uint32_t full0 = map_to_rank(smem_u32(&full[0]), 0);  // leader's barriers
                int gi = 0;
                for (int t = pair, w = 0; t < sc.total; t += npairs, ++w) {
                    if (sc.wave_ctr && w > 0) {  // wave barrier (see Sched)
                        unsigned int target = 0;
                        for (int v = 0; v < w; ++v)
                            target += 2u * (unsigned int)max(0, min(npairs, sc.total - v * npairs));
                        unsigned int val;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(val) : "l"(sc.wave_ctr) : "memory");
                        } while (val < target);
                    }
                    int mp, nt, nk;
                    hm_tile(sc, t, &mp, &nt, &nk);
                    const int m_tile = 2 * mp + (int)rank, xc = nt * NTP * BN + (int)rank * HM_XR;
                    for (int i = 0; i < nk; ++i, ++gi) {
                        const int s = gi % HM_STAGES;
                        mbar_wait(&empty[s], ((uint32_t)(gi / HM_STAGES) & 1u) ^ 1u);
                        if (rank == 0) mbar_expect_tx(&full[s], sc.hi_only ? 2 * (A_TILE + HM_XT) : 2 * HM_STAGE);
                        const uint32_t fb = full0 + s * 8;
                        const int k0 = i * BKH;
                        const uint32_t sa = smem_u32(a_hi(s)), sx = smem_u32(x_hi(s));
                        const int nhl = sc.hi_only ? 1 : 2;
                        auto load4 = [&](uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3) {
                            asm volatile(
                                "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                                " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst), "l"(tm), "r"(fb), "r"(c0), "r"(c1),
                                "r"(c2), "r"(c3) : "memory");
                        };
                        for (int hl = 0; hl < nhl; ++hl) {  // A: the interleaved hi/lo copy (4-D map)
                            if (A_MN) {
                                load4(sa + hl * A_TILE, &tmA, 0, hl, m_tile * 2, k0);
                                load4(sa + hl * A_TILE + A_TILE / 2, &tmA, 0, hl, m_tile * 2 + 1, k0);
                            } else {
                                load4(sa + hl * A_TILE, &tmA, 0, hl, k0 / 64, m_tile * BM);
                            }
                        }
                        // X: this CTA's 96 N rows, hi then lo, as three 32-row boxes each (the maps'
                        // boxes are 32 rows for this kernel)
                        for (int hl = 0; hl < nhl; ++hl)
#pragma unroll
                            for (int h3 = 0; h3 < 3; ++h3) {
                                const uint32_t dst = sx + hl * HM_XT + h3 * (HM_XT / 3);
                                if (sc.x_il)
                                    load4(dst, &tmXh, 0, hl, k0 / 64, xc + h3 * 32);
                                else
                                    asm volatile(
                                        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                                        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst), "l"(hl ? &tmXl : &tmXh), "r"(fb),
                                        "r"(k0), "r"(xc + h3 * 32) : "memory");
                            }
                    }
                    if (sc.wave_ctr) atomicAdd(sc.wave_ctr, 1u);
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------- MMA issuer (leader only)
            if (rank == 0) {
                int gi = 0, gc = 0;
                for (int t = pair; t < sc.total; t += npairs) {
                    int mp, nt, nk;
                    hm_tile(sc, t, &mp, &nt, &nk);
                    for (int i = 0; i < nk; ++i, ++gi) {
                        const int s = gi % HM_STAGES;
                        const int c = gc + i / CH, b = c & 1;
                        const bool first = (i % CH) == 0;
                        if (first) mbar_wait(&tempty[b], ((uint32_t)(c / 2) & 1u) ^ 1u);
                        mbar_wait(&full[s], (uint32_t)(gi / HM_STAGES) & 1u);
                        tc_fence_after();
                        const uint32_t ah = smem_u32(a_hi(s)), al = ah + A_TILE;
                        const uint32_t xh = smem_u32(x_hi(s)), xl = xh + HM_XT;
                        const uint32_t d = tmem + (uint32_t)(b * BUF);
#pragma unroll
                        for (int k8 = 0; k8 < BK / 8; ++k8) {
                            uint64_t dah, dal;
                            if (A_MN) {
                                dah = sdesc(ah + k8 * 2048, 8192, 1024, 2);
                                dal = sdesc(al + k8 * 2048, 8192, 1024, 2);
                            } else {
                                dah = sdesc(ah + k8 * 32, 16, 1024, 2);
                                dal = sdesc(al + k8 * 32, 16, 1024, 2);
                            }
                            const uint64_t dxh = sdesc(xh + k8 * 32, 16, 1024, 2);
                            const uint64_t dxl = sdesc(xl + k8 * 32, 16, 1024, 2);
                            const uint32_t acc = (!first || k8 > 0) ? 1u : 0u;
                            if (sc.hi_only)
                                asm volatile(
                                    "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\t"
                                    "setp.ne.b32 p, %4, 0;\n\t"
                                    "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                    "l"(dah), "l"(dxh), "r"(IDESC), "r"(acc));
                            else
                                asm volatile(
                                    "{\n\t.reg .pred e, p, one;\n\telect.sync _|e, 0xffffffff;\n\t"
                                    "setp.ne.b32 p, %6, 0;\n\tsetp.eq.b32 one, %6, %6;\n\t"
                                    "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %5, p;\n\t"
                                    "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %3, %5, one;\n\t"
                                    "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %4, %2, %5, one;\n\t}" ::"r"(d),
                                    "l"(dah), "l"(dxh), "l"(dxl), "l"(dal), "r"(IDESC), "r"(acc));
                        }
                        asm volatile(
                            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                            " [%0], %1;\n\t}" ::"r"(smem_u32(&empty[s])), "h"((uint16_t)3) : "memory");
                        if ((i % CH) == CH - 1 || i == nk - 1)
                            asm volatile(
                                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                                "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                                " [%0], %1;\n\t}" ::"r"(smem_u32(&tfull[b])), "h"((uint16_t)3) : "memory");
                        __syncwarp();
                    }
                    gc += (nk + CH - 1) / CH;
                }
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <bool A_MN, int EPI>
void launch_umma2_h3m(Ctx* c, PSched sc, const CUtensorMap& ta, const CUtensorMap& th, const CUtensorMap& tl, int M,
                      int N, void* out, int64_t ldo, double alpha, double beta, const int* rexp, const int* cexp,
                      uint16_t* q16, const uint16_t* aux) {
    auto kern = k_umma2_h3m<A_MN, EPI>;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, HM_SMEM));
        attr = true;
    }
    if (sc.total <= 0) return;
    const int pairs = std::min(sc.total, c->sm_count / 2);
    DevBuf ctr;
    sc.wave_ctr = nullptr;
    if (pairs < sc.total && !g_wave_barrier_off && !sc.tri_x) {
        ctr = DevBuf(c, 64);
        CUDA_CHECK(cudaMemsetAsync(ctr.ptr, 0, 4, c->stream));
        sc.wave_ctr = ctr.as<unsigned int>();
    }
    kern<<<2 * pairs, HM_THREADS, HM_SMEM, c->stream>>>(ta, th, tl, M, N, sc, out, ldo, alpha, beta, rexp, cexp, q16,
                                                         aux);
    LAUNCH_CHECK(c);
}

// ------------------------------------------------ fp16 operands (row-Σ² passes)
// max |x| over a K × N matrix into *mx (float bits; non-negative floats order as integers)
template <class T>
__global__ void k_absmax(const T* __restrict__ x, int64_t K, int64_t N, int64_t ldx, unsigned int* __restrict__ mx) {
    float m = 0.0f;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < K * N; e += (int64_t)gridDim.x * blockDim.x) {
        const float v = fabsf((float)x[e % K + (e / K) * ldx]);
        m = fmaxf(m, isfinite(v) ? v : 0.0f);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(mx, __float_as_uint(m));
}
// scale exponent q with max·2^q < 2^15 (as block_sumsq's per-column exponents)
__device__ __forceinline__ int f16_exp_of(unsigned int mxbits) {
    const float mx = __uint_as_float(mxbits);
    if (!(mx > 0.0f)) return 0;
    int e;
    frexpf(mx, &e);
    return 15 - e;
}
// x → fp16(x·2^q), K × N, ld K; q = f16_exp_of(*mx), also stored to *qout
template <class T>
__global__ void k_to_f16(const T* __restrict__ x, int64_t K, int64_t N, int64_t ldx, const unsigned int* __restrict__ mx,
                         uint16_t* __restrict__ out, int* __restrict__ qout) {
    const int q = f16_exp_of(*mx);
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e == 0) *qout = q;
    if (e >= K * N) return;
    const __half h = __float2half_rn(ldexpf((float)x[e % K + (e / K) * ldx], q));
    out[e] = *reinterpret_cast<const uint16_t*>(&h);
}
// out[i] = 2^(−2(colexp[i] + q)) · Σ_t partial[t·M + i]  (removes both exact scales)
__global__ void k_sum_tiles_scaled(int64_t M, int tiles, const double* __restrict__ partial, const int* __restrict__ colexp,
                                   const int* __restrict__ q, int qh, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    double s = 0.0;
    for (int t = 0; t < tiles; ++t) s += partial[(int64_t)t * M + i];
    out[i] = ldexp(s, -2 * (colexp[i] + (q ? *q : qh)));
}
// Q (fp64, K × N, ld ldq) → the fp32 basis and its fp16 copy for the row-Σ² passes, scaled by
// 2^14: entries of an orthonormal basis are ≤ 1 in magnitude, so no max pass is needed
__global__ void k_basis_out(const double* __restrict__ q, int64_t K, int64_t N, int64_t ldq, float* __restrict__ q32,
                            uint16_t* __restrict__ q16) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= K * N) return;
    const double v = q[e % K + (e / K) * ldq];
    q32[e] = (float)v;
    const __half h = __double2half(v * 16384.0);
    q16[e] = *reinterpret_cast<const uint16_t*>(&h);
}

// x (K × N, fp32 or fp64, ldx) → hi/lo fp32 (K × N, ld K)
void split_x(Ctx* c, const void* x, int dtx, int64_t K, int64_t N, int64_t ldx, DevBuf* hi, DevBuf* lo) {
    *hi = DevBuf(c, (size_t)K * N * 4);
    *lo = DevBuf(c, (size_t)K * N * 4);
    const unsigned g = (unsigned)((K * N + 255) / 256);
    if (dtx == BCUR_F32)
        k_split_hilo<float><<<g, 256, 0, c->stream>>>((const float*)x, K, N, ldx, hi->as<float>(), lo->as<float>());
    else
        k_split_hilo<double><<<g, 256, 0, c->stream>>>((const double*)x, K, N, ldx, hi->as<float>(), lo->as<float>());
    LAUNCH_CHECK(c);
}


// ------------------------------------------------ 3×FP16 operands (H3)
// x (K × N, fp32/fp64, ldx) → fp16 hi + lo (K × N, ld K), column j scaled by 2^q[j] with
// q[j] = f16 exponent of max_k |x[k,j]·2^−fold[k]| (fold nullable: the per-column exponents of
// the A operand of A·X, moved onto the rows of X so that A'X' = A·X·2^q exactly).
// One CTA per column; hi = rn16(x'), lo = rn16(x' − hi) (exact remainder in fp64).
template <class T, bool IL>
__global__ void __launch_bounds__(1024) k_split_f16(const T* __restrict__ x, int64_t K, int64_t ldx,
                                                   const int* __restrict__ fold, uint16_t* __restrict__ hi,
                                                   uint16_t* __restrict__ lo, int* __restrict__ q, int64_t ldo) {
    const int64_t j = blockIdx.x;
    const T* col = x + j * ldx;
    double mx = 0.0;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
        const double v = fabs((double)col[k]) * (fold ? exp2_int(-fold[k]) : 1.0);
        mx = v > mx ? v : mx;
    }
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
    int e = 0;
    if (mx > 0.0 && isfinite(mx)) frexp(mx, &e);
    const int qj = mx > 0.0 && isfinite(mx) ? 15 - e : 0;  // max·2^q < 2^15
    if (threadIdx.x == 0) q[j] = qj;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
        const double v = (double)col[k] * exp2_int(qj - (fold ? fold[k] : 0));
        const __half h = __double2half(v);
        const __half l = __double2half(v - (double)__half2float(h));
        // IL: the A-operand layout (block_sumsq's): per 64-row chunk [hi 64 | lo 64], 2K per column
        const int64_t ih = IL ? j * 2 * K + (k >> 6) * 128 + (k & 63) : j * ldo + k;
        hi[ih] = *reinterpret_cast<const uint16_t*>(&h);
        (IL ? hi : lo)[IL ? ih + 64 : ih] = *reinterpret_cast<const uint16_t*>(&l);
    }
}

// 3×FP16 tile counts: split K until the persistent waves are nearly full (a 3.46-wave pass
// idles 14% of the SMs in its last wave); partials are fp64, so fewer is cheaper.
int h3_splits(int tiles, int k_tiles, int sms) {
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 8 && (s == 1 || k_tiles / s >= 16); ++s) {
        const int64_t t = (int64_t)tiles * s;
        const double eff = (double)t / ((double)sms * (double)((t + sms - 1) / sms));
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            best = s;
        }
        if (eff >= 0.95) break;
    }
    return best;
}
}  // namespace

namespace ops {

bool umma_ok(int dta, int64_t m, int64_t lda, const void* a) {
    static int enabled = -1;
    if (enabled < 0) {
        const char* e = getenv("BCUR_DISABLE_UMMA");
        enabled = (e && e[0] == '1') ? 0 : 1;
        const char* wb = getenv("BCUR_UMMA_NO_WAVE_BARRIER");
        g_wave_barrier_off = wb && wb[0] == '1';
        const char* np_ = getenv("BCUR_UMMA_NO_PAIR");
        g_no_pair = np_ && np_[0] == '1';
        const char* nx = getenv("BCUR_UMMA_X3_PAIR");
        g_no_x3pair = !(nx && nx[0] == '1');
        const char* nh = getenv("BCUR_UMMA_NO_H3_PAIR");
        g_no_h3pair = nh && nh[0] == '1';
        const char* nf = getenv("BCUR_UMMA_NO_FAST_ACC");
        g_no_fastacc = nf && nf[0] == '1';
        const char* nho = getenv("BCUR_UMMA_NO_HI_ONLY");
        g_no_hi_only = nho && nho[0] == '1';
        const char* l2h = getenv("BCUR_ROWSQ_L2HINT");
        if (l2h) g_l2hint = atoi(l2h);
        const char* pf = getenv("BCUR_UMMA_PF");
        if (pf) g_pf = atoi(pf);
        const char* d = getenv("BCUR_UMMA_DEBUG");
        if (d) {
            const int f = atoi(d);
            CUDA_CHECK(cudaMemcpyToSymbol(g_dbg_flags, &f, sizeof f));
        }
    }
    return enabled && dta == BCUR_F32 && m % 32 == 0 && (lda * 4) % 16 == 0 && ((uintptr_t)a % 16) == 0 && m > 0 &&
           m < (1LL << 31);
}

// Out(n×N) = alpha·Aᵀ X + beta·Out  (A m×n fp32 col-major; X m×N fp32/fp64) → fp64 store,
// or rowsq[j] = Σ_c (AᵀX)_jc² (rowsq != nullptr; product never stored)
void umma_atx(Ctx* c, const float* A, int64_t m, int64_t n, int64_t lda, const void* X, int dtx, int64_t N,
              int64_t ldx, double alpha, double beta, double* out, int64_t ldo, double* rowsq, bool sym,
              bool a_rounded) {
    if (n <= 0 || N <= 0) {
        if (rowsq && n > 0) CUDA_CHECK(cudaMemsetAsync(rowsq, 0, n * sizeof(double), c->stream));
        return;
    }
    const int NT = N > BN ? 2 : 1;
    sym = sym && !rowsq && NT == 2 && n == N;  // Gram AᵀA: upper-triangle tiles only
    ProfScope prof(c, rowsq ? "umma_atx_rowsq" : "umma_atx_store", (sym ? 1.0 : 2.0) * n * N * m,
                   4.0 * m * n + (double)dtype_size(dtx) * m * N + (rowsq ? 8.0 * n : 8.0 * n * N));
    DevBuf xh, xl;
    split_x(c, X, dtx, m, N, ldx, &xh, &xl);
    const uint64_t dA[2] = {(uint64_t)m, (uint64_t)n}, sA[1] = {(uint64_t)lda * 4};
    const uint32_t bA[2] = {BK, BM};
    const uint64_t dX[2] = {(uint64_t)m, (uint64_t)N}, sX[1] = {(uint64_t)m * 4};
    const uint32_t bX[2] = {BK, BN};
    CUtensorMap ta = make_map(A, 2, dA, sA, bA, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap th = make_map(xh.ptr, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap tl = make_map(xl.ptr, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B);
    const int k_tiles = (int)((m + BK - 1) / BK);
    const int mt = (int)((n + BM - 1) / BM);
    if (rowsq) {
        // Σ of squared projections: 1×TF32 with both operands rounded to nearest (unbiased);
        // up to 4 N tiles (256 columns) per CTA share each A tile; narrow panels (greedy
        // steps) use fewer tiles and a deeper stage ring (HBM-bound regime).
        const int NTX = N <= BN ? 1 : N <= 2 * BN ? 2 : 4;
        const int nt = (int)((N + NTX * BN - 1) / (NTX * BN));
        Sched sc = make_sched(mt, nt, 1, k_tiles, k_tiles, false, false);
        sc.a_rn = a_rounded ? 1 : 0;
        DevBuf part(c, (size_t)nt * NTX * n * sizeof(double));
        if (NTX == 4 && a_rounded && mt >= 2 && !g_no_pair) {
            // CTA pairs: 256 A columns × 256 X columns per pair (see k_umma2_rowsq)
            static bool attr = false;
            if (!attr) {
                CUDA_CHECK(cudaFuncSetAttribute(k_umma2_rowsq<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, P2_SMEM));
                attr = true;
            }
            const int m_pairs = (mt + 1) / 2;
            const int pairs = std::min(m_pairs * nt, c->sm_count / 2);
            DevBuf ctr;
            unsigned int* wc = nullptr;
            if (pairs < m_pairs * nt && !g_wave_barrier_off) {  // ≤ 1 CTA per SM: all co-resident
                ctr = DevBuf(c, 64);
                CUDA_CHECK(cudaMemsetAsync(ctr.ptr, 0, 4, c->stream));
                wc = ctr.as<unsigned int>();
            }
            k_umma2_rowsq<false><<<2 * pairs, P2_THREADS, P2_SMEM, c->stream>>>(ta, th, (int)n, m_pairs, nt, k_tiles,
                                                                         part.as<double>(), wc, 0, nullptr, 0, g_l2hint);
            LAUNCH_CHECK(c);
        } else if (NTX == 1)
            launch_umma_nt<false, EPI_ROWSQ, 1, false>(c, sc, ta, th, th, (int)n, (int)N, nullptr, 0,
                                                       part.as<double>(), 1.0, 0.0);
        else if (NTX == 2)
            launch_umma_nt<false, EPI_ROWSQ, 2, false>(c, sc, ta, th, th, (int)n, (int)N, nullptr, 0,
                                                       part.as<double>(), 1.0, 0.0);
        else
            launch_umma_nt<false, EPI_ROWSQ, 4, false>(c, sc, ta, th, th, (int)n, (int)N, nullptr, 0,
                                                       part.as<double>(), 1.0, 0.0);
        k_sum_tiles<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(n, nt * NTX, part.as<double>(), rowsq);
        LAUNCH_CHECK(c);
        return;
    }
    const int nt = (int)((N + NT * BN - 1) / (NT * BN));
    // split K (the m rows) when there are fewer output tiles than SMs (a thin Q_Cᵀ·P of
    // the greedy CGS2 has ≤ 64 tiles of 2048 stages each); fp64 partials, ordered reduce
    const int tiles = sym ? nt * (nt + 1) / 2 : mt * nt;
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>((2LL * c->sm_count + tiles - 1) / tiles, k_tiles / 32));
    const int kps = (k_tiles + splits - 1) / splits;
    splits = (k_tiles + kps - 1) / kps;
    const Sched sc = make_sched(mt, nt, splits, k_tiles, kps, sym, false);
    if (splits == 1 && NT == 2 && mt >= 2 && !g_no_x3pair) {  // CTA pairs (see k_umma2_x3)
        const PSched ps = make_psched(mt, nt, k_tiles, sym, false);
        if (ps.total >= c->sm_count / 2) {
            launch_umma2_x3<false>(c, ps, ta, th, tl, (int)n, (int)N, out, ldo, alpha, beta);
            return;
        }
    }
    if (splits == 1) {
        launch_umma<false, EPI_STORE>(c, NT, sc, ta, th, tl, (int)n, (int)N, out, ldo, nullptr, alpha, beta);
        return;
    }
    DevBuf part(c, (size_t)splits * n * N * sizeof(double));
    if (sym) CUDA_CHECK(cudaMemsetAsync(part.ptr, 0, part.bytes, c->stream));  // skipped lower tiles
    launch_umma<false, EPI_STORE>(c, NT, sc, ta, th, tl, (int)n, (int)N, nullptr, 0, part.as<double>(), 1.0, 0.0);
    k_reduce_splits<<<(unsigned)((n * N + 255) / 256), 256, 0, c->stream>>>(n, N, splits, part.as<double>(), out, ldo,
                                                                            alpha, beta);
    LAUNCH_CHECK(c);
}

void basis_out(Ctx* c, const double* q, int64_t K, int64_t N, int64_t ldq, float* q32, uint16_t* q16) {
    if (K <= 0 || N <= 0) return;
    k_basis_out<<<(unsigned)((K * N + 255) / 256), 256, 0, c->stream>>>(q, K, N, ldq, q32, q16);
    LAUNCH_CHECK(c);
}

bool rowsq_tiles_ok(int64_t M, int64_t N) {
    (void)umma_ok(BCUR_F32, 32, 8, nullptr);  // reads the environment switches once
    return N > 2 * BN && (M + BM - 1) / BM >= 2 && !g_no_pair;
}

void gemm_rowsumsq_f16(Ctx* c, int64_t M, int64_t N, int64_t K, const uint16_t* A16, int64_t lda, const int* colexp,
                       const void* X, int dtx, int64_t ldx, double* rowsq, bool interleaved, const uint16_t* x16_pre,
                       int q_pre, bool x16_il, const int* d_tiles, int ntiles) {
    if (M <= 0) return;
    if (N <= 0 || K <= 0) {
        CUDA_CHECK(cudaMemsetAsync(rowsq, 0, M * sizeof(double), c->stream));
        return;
    }
    if (K % 64 != 0 || lda != K || ((uintptr_t)A16 % 16) != 0)
        fail(BCUR_E_INVALID_ARGUMENT, "gemm_rowsumsq_f16: the fp16 copy needs K % 64 == 0 (lda = K)");
    // the work of THIS launch: with a tile list only ntiles 128-row tiles of AᵀX are computed (the
    // selected blocks' columns are skipped by the caller, which adds their mass from the norms)
    const double Mw = (d_tiles && ntiles > 0) ? std::min<double>((double)M, 128.0 * ntiles) : (double)M;
    ProfScope prof(c, "umma_atx_rowsq", 2.0 * Mw * N * K, 2.0 * K * Mw + (double)dtype_size(dtx) * K * N + 8.0 * Mw);
    (void)umma_ok(BCUR_F32, K, lda, A16);  // reads the environment switches once
    // X → fp16 with one power-of-two scale from its max (device-side; no host sync), unless
    // the caller passes it pre-converted (x16_pre, scale 2^q_pre)
    DevBuf mx(c, 64), x16;
    int* q = reinterpret_cast<int*>(mx.as<unsigned int>() + 1);
    const unsigned gx = (unsigned)std::min<int64_t>((K * N + 255) / 256, 4LL * c->sm_count);
    const unsigned gc = (unsigned)((K * N + 255) / 256);
    if (x16_pre) {
        q = nullptr;
    } else if (dtx == BCUR_F32) {
        x16 = DevBuf(c, (size_t)K * N * 2);
        CUDA_CHECK(cudaMemsetAsync(mx.ptr, 0, 8, c->stream));
        k_absmax<float><<<gx, 256, 0, c->stream>>>((const float*)X, K, N, ldx, mx.as<unsigned int>());
        k_to_f16<float><<<gc, 256, 0, c->stream>>>((const float*)X, K, N, ldx, mx.as<unsigned int>(),
                                                   x16.as<uint16_t>(), q);
    } else {
        x16 = DevBuf(c, (size_t)K * N * 2);
        CUDA_CHECK(cudaMemsetAsync(mx.ptr, 0, 8, c->stream));
        k_absmax<double><<<gx, 256, 0, c->stream>>>((const double*)X, K, N, ldx, mx.as<unsigned int>());
        k_to_f16<double><<<gc, 256, 0, c->stream>>>((const double*)X, K, N, ldx, mx.as<unsigned int>(),
                                                    x16.as<uint16_t>(), q);
    }
    LAUNCH_CHECK(c);
    constexpr int BKH = bke<true>();
    // hi of the copy as (64 rows, hi|lo, K/64 chunks, M columns), box = one chunk × 128 columns;
    // the compact copy is the same map with one part per chunk
    const uint64_t dA[4] = {64, interleaved ? 2u : 1u, (uint64_t)(K / 64), (uint64_t)M};
    const uint64_t sA[3] = {128, interleaved ? 256u : 128u, (uint64_t)K * (interleaved ? 4 : 2)};
    const uint32_t bA[4] = {64, 1, 1, BM};
    const uint64_t dX[2] = {(uint64_t)K, (uint64_t)N}, sX[1] = {(uint64_t)K * 2};
    const uint32_t bX[2] = {BKH, BN};
    CUtensorMap ta = make_map(A16, 4, dA, sA, bA, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                              interleaved ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    const bool xil = x16_pre && x16_il;  // X = the hi part of an interleaved split (4-D map, part 0)
    const uint64_t dXi[4] = {64, 2, (uint64_t)(K / 64), (uint64_t)N}, sXi[3] = {128, 256, (uint64_t)K * 4};
    const uint32_t bXi[4] = {64, 1, 1, BN};
    CUtensorMap tx = xil ? make_map(x16_pre, 4, dXi, sXi, bXi, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B)
                         : make_map(x16_pre ? (const void*)x16_pre : x16.ptr, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    const int k_tiles = (int)((K + BKH - 1) / BKH);
    const int mt = (int)((M + BM - 1) / BM);
    const int NTX = N <= BN ? 1 : N <= 2 * BN ? 2 : 4;
    const int nt = (int)((N + NTX * BN - 1) / (NTX * BN));
    DevBuf part(c, (size_t)nt * NTX * M * sizeof(double));
    if (d_tiles) {  // only the listed tiles are computed: the rest of the row sums are zero
        if (!(NTX == 4 && mt >= 2 && !g_no_pair)) fail(BCUR_E_INVALID_ARGUMENT, "gemm_rowsumsq_f16: tile lists need the CTA-pair path");
        CUDA_CHECK(cudaMemsetAsync(part.ptr, 0, part.bytes, c->stream));
    }
    if (NTX == 4 && mt >= 2 && !g_no_pair) {
        static bool attr = false;
        if (!attr) {
            CUDA_CHECK(cudaFuncSetAttribute(k_umma2_rowsq<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, P2_SMEM));
            attr = true;
        }
        const int m_pairs = d_tiles ? (ntiles + 1) / 2 : (mt + 1) / 2;
        const int pairs = std::min(m_pairs * nt, c->sm_count / 2);
        DevBuf ctr;
        unsigned int* wc = nullptr;
        if (pairs < m_pairs * nt && !g_wave_barrier_off) {
            ctr = DevBuf(c, 64);
            CUDA_CHECK(cudaMemsetAsync(ctr.ptr, 0, 4, c->stream));
            wc = ctr.as<unsigned int>();
        }
        k_umma2_rowsq<true><<<2 * pairs, P2_THREADS, P2_SMEM, c->stream>>>(ta, tx, (int)M, m_pairs, nt, k_tiles,
                                                                           part.as<double>(), wc, xil ? 1 : 0,
                                                                           d_tiles, ntiles, g_l2hint);
        LAUNCH_CHECK(c);
    } else {
        Sched sc = make_sched(mt, nt, 1, k_tiles, k_tiles, false, false);
        sc.a_rn = 1;  // converted operands: no transform
        sc.pf = g_pf >= 0 ? g_pf : 0;  // no L2 prefetch on the fp16 copy (as the 3×FP16 passes)
        sc.x_il = xil ? 1 : 0;
        if (NTX == 1)
            launch_umma_nt<false, EPI_ROWSQ, 1, false, true>(c, sc, ta, tx, tx, (int)M, (int)N, nullptr, 0,
                                                             part.as<double>(), 1.0, 0.0);
        else if (NTX == 2)
            launch_umma_nt<false, EPI_ROWSQ, 2, false, true>(c, sc, ta, tx, tx, (int)M, (int)N, nullptr, 0,
                                                             part.as<double>(), 1.0, 0.0);
        else
            launch_umma_nt<false, EPI_ROWSQ, 4, false, true>(c, sc, ta, tx, tx, (int)M, (int)N, nullptr, 0,
                                                             part.as<double>(), 1.0, 0.0);
    }
    k_sum_tiles_scaled<<<(unsigned)((M + 255) / 256), 256, 0, c->stream>>>(M, nt * NTX, part.as<double>(), colexp, q,
                                                                           q_pre, rowsq);
    LAUNCH_CHECK(c);
}

// Out(m×N) = alpha·A X + beta·Out  (A m×n fp32; X n×N fp32/fp64), split-K over n with fp64
// partials.  x_upper_tri: X[k, j] = 0 for k > j (R⁻¹ of a Cholesky factor) — each N tile
// stops at its diagonal (half the MMAs).
void umma_ax(Ctx* c, const float* A, int64_t m, int64_t n, int64_t lda, const void* X, int dtx, int64_t N,
             int64_t ldx, double alpha, double beta, double* out, int64_t ldo, bool x_upper_tri, bool x1) {
    if (m <= 0 || N <= 0) return;
    ProfScope prof(c, x1 ? "umma_ax_x1" : "umma_ax", (x_upper_tri ? 1.0 : 2.0) * m * n * N,
                   4.0 * m * n + (double)dtype_size(dtx) * n * N + 8.0 * m * N);
    DevBuf xh, xl;
    split_x(c, X, dtx, n, N, ldx, &xh, &xl);
    // 3-D view of column-major A: (32 rows, n columns, m/32 row groups)
    const uint64_t dA[3] = {32, (uint64_t)n, (uint64_t)(m / 32)}, sA[2] = {(uint64_t)lda * 4, 128};
    const uint32_t bA[3] = {32, BK, BM / 32};
    const uint64_t dX[2] = {(uint64_t)n, (uint64_t)N}, sX[1] = {(uint64_t)n * 4};
    const uint32_t bX[2] = {BK, BN};
    CUtensorMap ta = make_map(A, 3, dA, sA, bA, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    CUtensorMap th = make_map(xh.ptr, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap tl = make_map(xl.ptr, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B);
    const int k_tiles = (int)((n + BK - 1) / BK);
    const int NT = x1 ? (N > 2 * BN ? 4 : N > BN ? 2 : 1) : (N > BN ? 2 : 1);
    const int mt = (int)((m + BM - 1) / BM), nt = (int)((N + NT * BN - 1) / (NT * BN));
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>((2LL * c->sm_count + mt * nt - 1) / (mt * nt),
                                                             k_tiles / 16));
    const int kps = (k_tiles + splits - 1) / splits;
    splits = (k_tiles + kps - 1) / kps;
    const Sched sc = make_sched(mt, nt, splits, k_tiles, kps, false, x_upper_tri);
    // 1×TF32 (both operands rounded to nearest) for small corrections: up to 4 N tiles per CTA
    auto launch = [&](double* o, int64_t lo, double* prt, double al, double be) {
        if (!x1) {
            launch_umma<true, EPI_STORE>(c, NT, sc, ta, th, tl, (int)m, (int)N, o, lo, prt, al, be);
        } else if (NT == 4) {
            launch_umma_nt<true, EPI_STORE, 4, false>(c, sc, ta, th, th, (int)m, (int)N, o, lo, prt, al, be);
        } else if (NT == 2) {
            launch_umma_nt<true, EPI_STORE, 2, false>(c, sc, ta, th, th, (int)m, (int)N, o, lo, prt, al, be);
        } else {
            launch_umma_nt<true, EPI_STORE, 1, false>(c, sc, ta, th, th, (int)m, (int)N, o, lo, prt, al, be);
        }
    };
    if (splits == 1 && !x1 && NT == 2 && mt >= 2 && !g_no_x3pair) {  // CTA pairs (see k_umma2_x3)
        const PSched ps = make_psched(mt, nt, k_tiles, false, x_upper_tri);
        if (ps.total >= c->sm_count / 2) {
            launch_umma2_x3<true>(c, ps, ta, th, tl, (int)m, (int)N, out, ldo, alpha, beta);
            return;
        }
    }
    if (splits == 1) {
        launch(out, ldo, nullptr, alpha, beta);
        return;
    }
    DevBuf part(c, (size_t)splits * m * N * sizeof(double));
    launch(nullptr, 0, part.as<double>(), 1.0, 0.0);
    k_reduce_splits<<<(unsigned)((m * N + 255) / 256), 256, 0, c->stream>>>(m, N, splits, part.as<double>(), out, ldo,
                                                                            alpha, beta);
    LAUNCH_CHECK(c);
}


// ---- 3×FP16 (H3) products -------------------------------------------------
// one CTA per column: few, tall columns (the range finder's 65536 × 60 operands) get 1024
// threads so the two passes over each column keep enough loads in flight
static unsigned split_threads(int64_t K, int64_t N, Ctx* c) {
    return (N < 2 * c->sm_count && K >= 8192) ? 1024u : 256u;
}
void split_f16(Ctx* c, const void* x, int dtx, int64_t K, int64_t N, int64_t ldx, const int* fold, SplitF16* out) {
    out->K = K;
    out->N = N;
    out->ld = (K + 7) / 8 * 8;
    out->hi = DevBuf(c, (size_t)std::max<int64_t>(out->ld * N, 1) * 2);
    out->lo = DevBuf(c, (size_t)std::max<int64_t>(out->ld * N, 1) * 2);
    out->exps = DevBuf(c, (size_t)std::max<int64_t>(N, 1) * sizeof(int));
    if (K <= 0 || N <= 0) return;
    ProfScope prof(c, "split_f16", 0.0, (double)K * N * (dtype_size(dtx) + 4));
    if (dtx == BCUR_F32)
        k_split_f16<float, false><<<(unsigned)N, split_threads(K, N, c), 0, c->stream>>>((const float*)x, K, ldx, fold,
                                                                     out->hi.as<uint16_t>(), out->lo.as<uint16_t>(),
                                                                     out->exps.as<int>(), out->ld);
    else
        k_split_f16<double, false><<<(unsigned)N, split_threads(K, N, c), 0, c->stream>>>((const double*)x, K, ldx, fold,
                                                                      out->hi.as<uint16_t>(), out->lo.as<uint16_t>(),
                                                                      out->exps.as<int>(), out->ld);
    LAUNCH_CHECK(c);
}

void split_il_into(Ctx* c, const void* a, int dta, int64_t m, int64_t n, int64_t lda, uint16_t* il, int* exps) {
    if (m % 64 != 0) fail(BCUR_E_INVALID_ARGUMENT, "split_il: needs m % 64 == 0");
    if (m <= 0 || n <= 0) return;
    ProfScope prof(c, "split_f16", 0.0, (double)m * n * (dtype_size(dta) + 4));
    if (dta == BCUR_F32)
        k_split_f16<float, true><<<(unsigned)n, split_threads(m, n, c), 0, c->stream>>>((const float*)a, m, lda, nullptr, il, nullptr,
                                                                    exps, 0);
    else
        k_split_f16<double, true><<<(unsigned)n, split_threads(m, n, c), 0, c->stream>>>((const double*)a, m, lda, nullptr, il, nullptr,
                                                                     exps, 0);
    LAUNCH_CHECK(c);
}

void split_il(Ctx* c, const void* a, int dta, int64_t m, int64_t n, int64_t lda, DevBuf* il, DevBuf* exps) {
    *il = DevBuf(c, (size_t)std::max<int64_t>(m * n, 1) * 4);
    *exps = DevBuf(c, (size_t)std::max<int64_t>(n, 1) * sizeof(int));
    split_il_into(c, a, dta, m, n, lda, il->as<uint16_t>(), exps->as<int>());
}

// A split on the fly (interleaved) and X split per column; the Gram form reads A's split as X too.
void gemm_h3(Ctx* c, bool a_mn, const void* A, int dta, int64_t m, int64_t n, int64_t lda, const void* X, int dtx,
             int64_t N, int64_t ldx, double alpha, double beta, double* out, int64_t ldo, int flags) {
    DevBuf il, ea;
    split_il(c, A, dta, m, n, lda, &il, &ea);
    if ((flags & GEMM_SYM_UPPER) && !a_mn) {  // X = A: its interleaved split serves both operands
        const F16View xv{il.as<uint16_t>(), nullptr, ea.as<int>(), m, n};
        umma_h3(c, false, il.as<uint16_t>(), ea.as<int>(), m, n, xv, alpha, beta, out, ldo, flags);
        return;
    }
    umma_h3(c, a_mn, il.as<uint16_t>(), ea.as<int>(), m, n, X, dtx, N, ldx, alpha, beta, out, ldo, flags);
}

bool h3_ok(int64_t m) {
    (void)umma_ok(BCUR_F32, 32, 8, nullptr);  // reads the environment switches once
    static int enabled = -1;
    if (enabled < 0) {
        const char* e = getenv("BCUR_DISABLE_H3");
        enabled = (e && e[0] == '1') ? 0 : 1;
    }
    return enabled && m > 0 && m % 64 == 0 && m < (1LL << 30);
}

// epi: EPI_STORE (out fp64), EPI_SPLIT (out = the uint16 interleaved split, a_mn), EPI_BASIS (out = fp32 q32,
// q16 = its fp16 copy, aux = the split added back, a_mn)
static void umma_h3_epi(Ctx* c, bool a_mn, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const F16View& X,
                        double alpha, double beta, void* out_v, int64_t ldo, int flags, int epi, uint16_t* q16,
                        const uint16_t* aux) {
    double* out = reinterpret_cast<double*>(out_v);
    const bool sym_req = (flags & GEMM_SYM_UPPER) != 0, tri = (flags & GEMM_B_UPPER) != 0 && a_mn;
    const int64_t M = a_mn ? m : n, K = a_mn ? n : m, N = X.N;
    if (M <= 0 || N <= 0) return;
    if (X.K != K) fail(BCUR_E_DIMENSION_MISMATCH, "umma_h3: X rows do not match the contraction");
    if (!h3_ok(m)) fail(BCUR_E_INVALID_ARGUMENT, "umma_h3: needs m % 64 == 0");
    const int NT = N > BN ? 2 : 1;
    const bool sym = sym_req && !a_mn && NT == 2 && M == N;
    ProfScope prof(c, a_mn ? "umma_ax_h3" : "umma_atx_h3", ((sym || tri) ? 1.0 : 2.0) * M * N * K,
                   4.0 * m * n + 4.0 * K * N + 8.0 * M * N);
    constexpr int BKH = bke<true>();
    // the interleaved copy: element (row r, column j, part hl) at j·2m + (r/64)·128 + hl·64 + r%64
    // 4-D view (64 rows, hi|lo, m/64 row chunks, n columns).  AᵀX (K = rows): box = one chunk ×
    // 128 columns.  A·X (K = columns): box = one chunk × 64 columns, loaded twice per stage
    // (the tile's two 64-row MN atoms).
    const uint64_t dA[4] = {64, 2, (uint64_t)(m / 64), (uint64_t)n};
    const uint64_t sA[3] = {128, 256, (uint64_t)m * 4};
    const uint32_t bA[4] = {64, 1, 1, a_mn ? (uint32_t)BKH : (uint32_t)BM};
    CUtensorMap ta = make_map(AL, 4, dA, sA, bA, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    CUtensorMap th, tl;
    if (X.lo) {  // separate hi, lo (K × N each, ld X.ld or K)
        const int64_t ldx = X.ld > 0 ? X.ld : K;
        if ((ldx * 2) % 16 != 0) fail(BCUR_E_INVALID_ARGUMENT, "umma_h3: X leading dimension must be a multiple of 8");
        const uint64_t dX[2] = {(uint64_t)K, (uint64_t)N}, sX[1] = {(uint64_t)ldx * 2};
        const uint32_t bX[2] = {BKH, BN};
        th = make_map(X.hi, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
        tl = make_map(X.lo, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    } else {     // interleaved (split_il layout, K % 64 == 0): one 4-D map, part 0 = hi, 1 = lo
        if (K % 64 != 0) fail(BCUR_E_INVALID_ARGUMENT, "umma_h3: an interleaved X needs K % 64 == 0");
        // X.part ≥ 0: that part alone — a one-part map based at it, so the kernel's load of the
        // other part falls outside the tensor and reads as zeros (TMA fill)
        const bool one = X.part >= 0;
        const uint64_t dX[4] = {64, one ? 1u : 2u, (uint64_t)(K / 64), (uint64_t)N}, sX[3] = {128, 256, (uint64_t)K * 4};
        const uint32_t bX[4] = {64, 1, 1, BN};
        th = make_map(one ? X.hi + 64 * X.part : X.hi, 4, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                      one ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
        tl = th;
    }
    const int k_tiles = (int)((K + BKH - 1) / BKH);
    const int mt = (int)((M + BM - 1) / BM), nt = (int)((N + NT * BN - 1) / (NT * BN));
    const int tiles = sym ? nt * (nt + 1) / 2 : mt * nt;
    // split-K fills the last persistent wave, but its fp64 partials cost (splits + 1)·M·N·8
    // bytes of traffic plus a reduce: for wide outputs (the 4096² Gram of C) that exceeded the
    // wave it saved, so only outputs below 8 M elements split
    int splits = (epi == EPI_STORE && (double)M * (double)N <= 8.0e6) ? h3_splits(tiles, k_tiles, c->sm_count) : 1;
    const int kps = (k_tiles + splits - 1) / splits;
    splits = (k_tiles + kps - 1) / kps;
    Sched sc = make_sched(mt, nt, splits, k_tiles, kps, sym, tri);
    // No L2 prefetch: with the stage ring alone the 3×FP16 passes stream at 5.7-6.2 TB/s; 12
    // stages of prefetch (57 MB of A in flight) dropped them to ~4 TB/s (L2 thrash)
    sc.pf = g_pf >= 0 ? g_pf : 0;
    sc.x_il = X.lo ? 0 : 1;
    sc.bke = BKH;  // fp16 k-tiles: the diagonal limit of a triangular X in 64-row units (was 2× too far)
    const int* rexp = a_mn ? nullptr : ea;
    const int* cexp = X.exps;
    if ((flags & GEMM_FAST_ACC) && NT == 2 && !sym && splits == 1 && M >= 2 * BM && !g_no_h3pair && !g_no_fastacc) {
        // one accumulator per pair tile of 256 × 192 (k_umma2_h3m); its X maps load 32-row boxes
        PSched ps = make_psched(mt, (int)((N + HM_NTP * BN - 1) / (HM_NTP * BN)), k_tiles, false, tri);
        ps.bke = BKH;
        ps.x_il = X.lo ? 0 : 1;
        ps.hi_only = (flags & GEMM_HI_ONLY) && !g_no_hi_only ? 1 : 0;
        if (X.lo) {
            const int64_t ldx = X.ld > 0 ? X.ld : K;
            const uint64_t dX[2] = {(uint64_t)K, (uint64_t)N}, sX[1] = {(uint64_t)ldx * 2};
            const uint32_t bX[2] = {BKH, 32};
            th = make_map(X.hi, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
            tl = make_map(X.lo, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
        } else {
            const bool one = X.part >= 0;
            const uint64_t dX[4] = {64, one ? 1u : 2u, (uint64_t)(K / 64), (uint64_t)N}, sX[3] = {128, 256, (uint64_t)K * 4};
            const uint32_t bX[4] = {64, 1, 1, 32};
            th = make_map(one ? X.hi + 64 * X.part : X.hi, 4, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                          one ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
            tl = th;
        }
        if (a_mn) {
            if (epi == EPI_SPLIT)
                launch_umma2_h3m<true, EPI_SPLIT>(c, ps, ta, th, tl, (int)M, (int)N, out_v, ldo, alpha, 0.0, rexp, cexp,
                                                  nullptr, nullptr);
            else if (epi == EPI_BASIS)
                launch_umma2_h3m<true, EPI_BASIS>(c, ps, ta, th, tl, (int)M, (int)N, out_v, ldo, alpha, 0.0, rexp, cexp,
                                                  q16, aux);
            else
                launch_umma2_h3m<true, EPI_STORE>(c, ps, ta, th, tl, (int)M, (int)N, out_v, ldo, alpha, beta, rexp,
                                                  cexp, nullptr, nullptr);
        } else {
            if (epi != EPI_STORE) fail(BCUR_E_INVALID_ARGUMENT, "umma_h3: split/basis output needs A·X");
            launch_umma2_h3m<false, EPI_STORE>(c, ps, ta, th, tl, (int)M, (int)N, out_v, ldo, alpha, beta, rexp, cexp,
                                               nullptr, nullptr);
        }
        return;
    }
    if (NT == 2 && splits == 1 && M >= 2 * BM && !g_no_h3pair) {
        // tensor-bound shapes: CTA pairs (k_umma2_h3)
        PSched ps = make_psched(mt, nt, k_tiles, sym, tri);
        ps.bke = BKH;
        ps.x_il = X.lo ? 0 : 1;
        // the A·X map's box is one 64-row chunk × 64 columns (two loads per tile), AᵀX one chunk × 128
        if (a_mn) {
            if (epi == EPI_SPLIT)
                launch_umma2_h3<true, EPI_SPLIT>(c, ps, ta, th, tl, (int)M, (int)N, out_v, ldo, alpha, 0.0, rexp, cexp,
                                                 nullptr, nullptr);
            else if (epi == EPI_BASIS)
                launch_umma2_h3<true, EPI_BASIS>(c, ps, ta, th, tl, (int)M, (int)N, out_v, ldo, alpha, 0.0, rexp, cexp,
                                                 q16, aux);
            else
                launch_umma2_h3<true, EPI_STORE>(c, ps, ta, th, tl, (int)M, (int)N, out_v, ldo, alpha, beta, rexp, cexp,
                                                 nullptr, nullptr);
        } else {
            if (epi != EPI_STORE) fail(BCUR_E_INVALID_ARGUMENT, "umma_h3: split/basis output needs A·X");
            launch_umma2_h3<false, EPI_STORE>(c, ps, ta, th, tl, (int)M, (int)N, out_v, ldo, alpha, beta, rexp, cexp,
                                              nullptr, nullptr);
        }
        return;
    }
    auto launch = [&](double* o, int64_t ldo_, double* prt, double al, double be) {
        if (epi == EPI_SPLIT || epi == EPI_BASIS) {
            if (!a_mn || NT != 2 || M % 64 != 0) fail(BCUR_E_INVALID_ARGUMENT, "umma_h3: split/basis output needs A·X, N > 64, M % 64 == 0");
            if (epi == EPI_SPLIT)
                launch_umma_nt<true, EPI_SPLIT, 2, true, true>(c, sc, ta, th, tl, (int)M, (int)N, o, ldo_, nullptr, al, 0.0,
                                                                nullptr, nullptr, cexp);
            else
                launch_umma_nt<true, EPI_BASIS, 2, true, true>(c, sc, ta, th, tl, (int)M, (int)N, o, ldo_,
                                                                reinterpret_cast<double*>(q16), al, 0.0, nullptr, nullptr,
                                                                cexp, true, aux);
            return;
        }
        if (a_mn) {
            if (NT == 2) launch_umma_nt<true, EPI_STORE, 2, true, true>(c, sc, ta, th, tl, (int)M, (int)N, o, ldo_, prt, al, be, nullptr, rexp, cexp);
            else launch_umma_nt<true, EPI_STORE, 1, true, true>(c, sc, ta, th, tl, (int)M, (int)N, o, ldo_, prt, al, be, nullptr, rexp, cexp);
        } else {
            if (NT == 2) launch_umma_nt<false, EPI_STORE, 2, true, true>(c, sc, ta, th, tl, (int)M, (int)N, o, ldo_, prt, al, be, nullptr, rexp, cexp);
            else launch_umma_nt<false, EPI_STORE, 1, true, true>(c, sc, ta, th, tl, (int)M, (int)N, o, ldo_, prt, al, be, nullptr, rexp, cexp);
        }
    };
    if (splits == 1) {
        launch(out, ldo, nullptr, alpha, beta);
        return;
    }
    DevBuf part(c, (size_t)splits * M * N * sizeof(double));
    if (sym || tri) CUDA_CHECK(cudaMemsetAsync(part.ptr, 0, part.bytes, c->stream));  // skipped tiles / k ranges
    launch(nullptr, 0, part.as<double>(), 1.0, 0.0);
    k_reduce_splits<<<(unsigned)((M * N + 255) / 256), 256, 0, c->stream>>>(M, N, splits, part.as<double>(), out, ldo,
                                                                            alpha, beta);
    LAUNCH_CHECK(c);
}

void umma_h3(Ctx* c, bool a_mn, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const F16View& X,
             double alpha, double beta, double* out, int64_t ldo, int flags) {
    umma_h3_epi(c, a_mn, AL, ea, m, n, X, alpha, beta, out, ldo, flags, EPI_STORE, nullptr, nullptr);
}

void umma_h3_to_split(Ctx* c, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const void* X, int dtx,
                      int64_t N, int64_t ldx, double alpha, uint16_t* out_il, int flags) {
    SplitF16 xs;
    split_f16(c, X, dtx, n, N, ldx, ea, &xs);
    umma_h3_epi(c, true, AL, ea, m, n, view(xs), alpha, 0.0, out_il, m, flags, EPI_SPLIT, nullptr, nullptr);
}

void umma_h3_basis(Ctx* c, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const void* X, int dtx, int64_t N,
                   int64_t ldx, double alpha, const uint16_t* addend_il, float* q32, uint16_t* q16, int flags) {
    SplitF16 xs;
    split_f16(c, X, dtx, n, N, ldx, ea, &xs);
    umma_h3_epi(c, true, AL, ea, m, n, view(xs), alpha, 0.0, q32, m, flags, EPI_BASIS, q16, addend_il);
}

__global__ void k_fill_int(int* p, int64_t count, int v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) p[i] = v;
}
void fill_basis_exps(Ctx* c, int* exps, int64_t n) {
    if (n <= 0) return;
    k_fill_int<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(exps, n, BASIS_E);
    LAUNCH_CHECK(c);
}

// Σ_ij (D − A·X)_ij² with A given as its interleaved split (m × n, column exponents ea), X fp64
// (n × N, ldx; split here with ea folded into its rows) and D fp32 (m × N, ldd) — the product
// is never stored (EPI_RESID); one fp64 partial per drain thread of each persistent CTA, summed
// in a fixed order (deterministic).
void umma_h3_resid(Ctx* c, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const void* X, int dtx, int64_t N,
                   int64_t ldx, const float* D, int64_t ldd, double* d_sum) {
    if (m <= 0 || N <= 0) return;
    if (!h3_ok(m)) fail(BCUR_E_INVALID_ARGUMENT, "umma_h3_resid: needs m % 64 == 0");
    SplitF16 xs;
    split_f16(c, X, dtx, n, N, ldx, ea, &xs);
    const int64_t M = m, K = n;
    const int NT = N > BN ? 2 : 1;
    ProfScope prof(c, "umma_resid_h3", 2.0 * M * N * K, 4.0 * m * n + 4.0 * K * N + 4.0 * M * N);
    constexpr int BKH = bke<true>();
    const uint64_t dA[4] = {64, 2, (uint64_t)(m / 64), (uint64_t)n};
    const uint64_t sA[3] = {128, 256, (uint64_t)m * 4};
    const uint32_t bA[4] = {64, 1, 1, (uint32_t)BKH};
    CUtensorMap ta = make_map(AL, 4, dA, sA, bA, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    const int64_t lx = xs.ld > 0 ? xs.ld : K;
    const uint64_t dX[2] = {(uint64_t)K, (uint64_t)N}, sX[1] = {(uint64_t)lx * 2};
    const uint32_t bX[2] = {BKH, BN};
    CUtensorMap th = make_map(xs.hi.ptr, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    CUtensorMap tl = make_map(xs.lo.ptr, 2, dX, sX, bX, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    const int k_tiles = (int)((K + BKH - 1) / BKH);
    const int mt = (int)((M + BM - 1) / BM), nt = (int)((N + NT * BN - 1) / (NT * BN));
    Sched sc = make_sched(mt, nt, 1, k_tiles, k_tiles, false, false);
    sc.pf = g_pf >= 0 ? g_pf : 0;
    sc.x_il = 0;
    sc.bke = BKH;
    const int grid = std::min(sc.total, c->sm_count);
    const int per = 32 * (NT == 2 ? Cfg<2, true, true>::NDRAIN : Cfg<1, true, true>::NDRAIN);
    DevBuf part(c, (size_t)grid * per * sizeof(double));
    double* dd = const_cast<double*>(reinterpret_cast<const double*>(D));  // read-only inside EPI_RESID
    if (NT == 2)
        launch_umma_nt<true, EPI_RESID, 2, true, true>(c, sc, ta, th, tl, (int)M, (int)N, dd, ldd, part.as<double>(), 1.0,
                                                       0.0, nullptr, nullptr, xs.exps.as<int>(), k_tiles >= 8);
    else
        launch_umma_nt<true, EPI_RESID, 1, true, true>(c, sc, ta, th, tl, (int)M, (int)N, dd, ldd, part.as<double>(), 1.0,
                                                       0.0, nullptr, nullptr, xs.exps.as<int>(), k_tiles >= 8);
    sum_vector(c, part.as<double>(), (int64_t)grid * per, d_sum);
}

void umma_h3(Ctx* c, bool a_mn, const uint16_t* AL, const int* ea, int64_t m, int64_t n, const void* X, int dtx,
             int64_t N, int64_t ldx, double alpha, double beta, double* out, int64_t ldo, int flags) {
    SplitF16 xs;
    split_f16(c, X, dtx, a_mn ? n : m, N, ldx, a_mn ? ea : nullptr, &xs);
    umma_h3(c, a_mn, AL, ea, m, n, view(xs), alpha, beta, out, ldo, flags);
}
}  // namespace ops
}  // namespace bcur_b200
