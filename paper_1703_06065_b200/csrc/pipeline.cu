// pipeline.cu — host orchestration of the Block-CUR hot path on one GPU (one
// column shard of A per rank; collectives through the context's bcur_comm).
//
//   range_finder   N1  (replaces truncate(svd(a),k), matcore.cpp:39-69)
//   block_css      R15 (sketch.cpp:68-82)
//   greedy_select  N3
//   block_cur      N4  (U = C⁺AR⁺; reference U = W⁺, blockcur.cpp:103)
//
// The numerical definitions (thresholds, orthonormalisation paths, residual
// rule) are shared with the oracle (oracle/bcur_oracle.py) and documented in
// DESIGN.md §Numerics.  Every floating-point operation runs on the device; the
// host only moves O(G)-sized decision data (draws, argmax, ranks, pivots).
// For fp32 inputs the factor bases are kept in fp32 so that every product with
// A or with a basis runs on the tcgen05 3×TF32 kernels (kernels_umma.cu).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <functional>

#include "pipeline.h"

namespace bcur_b200 {

using namespace ops;

// ------------------------------------------------------------- utilities
Mat64::Mat64(Ctx* c, int64_t m_, int64_t n_)
    : buf(c, (size_t)std::max<int64_t>(1, m_) * std::max<int64_t>(1, n_) * sizeof(double)),
      m(m_), n(n_), ld(std::max<int64_t>(1, m_)) {}

// (through the context's pinned read area: a copy into pageable memory — usually the caller's
// stack — is staged by the driver and costs more per read; c2's greedy makes ~40 of them)
template <class T>
static void d2h(Ctx* c, T* host, const T* dev, size_t count) {
    if (!count) return;
    c->read_later(host, dev, count * sizeof(T));
    c->read_all();
}
// host buffers may be stack-owned by the caller: small uploads go through the context's pinned
// ring (no synchronization), large ones synchronize
template <class T>
static void h2d(Ctx* c, T* dev, const T* host, size_t count) {
    if (!count) return;
    const void* src = c->stage_upload(host, count * sizeof(T));
    CUDA_CHECK(cudaMemcpyAsync(dev, src ? src : host, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    if (!src) c->sync();
}
// device → host read delivered by the next c->read_all() (one synchronization for several reads)
template <class T>
static void d2h_later(Ctx* c, T* host, const T* dev, size_t count) {
    c->read_later(host, dev, count * sizeof(T));
}
// drops undelivered reads when an operation ends (normally none are left; after a failure their
// host destinations may be gone)
struct ReadScope {
    Ctx* c;
    explicit ReadScope(Ctx* ctx) : c(ctx) {}
    ~ReadScope() {
        c->rd_items.clear();
        c->rd_off = 0;
    }
};

void allreduce(Ctx* c, double* d, int64_t count) {
    if (c->comm.world <= 1 || count <= 0) return;
    if (!c->comm.allreduce_f64) fail(BCUR_E_COMM, "allreduce requested but no callback installed");
    const int rc = c->comm.allreduce_f64(c->comm.user, d, count, c->stream);
    if (rc != 0) fail(BCUR_E_COMM, "allreduce callback failed with code " + std::to_string(rc));
}

// In-place broadcast of `bytes` bytes from rank `root` (the host's bcur_comm.broadcast).
static void broadcast(Ctx* c, void* buf, int64_t bytes, int root) {
    if (c->comm.world <= 1 || bytes <= 0) return;
    if (!c->comm.broadcast) fail(BCUR_E_COMM, "broadcast requested but no callback installed");
    const int rc = c->comm.broadcast(c->comm.user, buf, bytes, root, c->stream);
    if (rc != 0) fail(BCUR_E_COMM, "broadcast callback failed with code " + std::to_string(rc));
}
static bool can_broadcast(const Ctx* c) { return c->comm.world > 1 && c->comm.broadcast != nullptr; }

double tau_chol(int dt) { return dt == BCUR_F32 ? 1e-2 : 1e-5; }
double tau_rank(int dt) { return dt == BCUR_F32 ? 1e-5 : 1e-7; }
double theta_explicit(int dt) { return dt == BCUR_F32 ? 0.1 : 1e-6; }
double tau_saturate(int dt) { return dt == BCUR_F32 ? 1e-6 : 1e-12; }

Shard shard_of(const DMat* a, const int64_t* offsets, int64_t G) {
    Shard s;
    s.G = G;
    s.n_global = a->n_global > 0 ? a->n_global : a->n;
    s.col0 = a->col0;
    if (G < 1) fail(BCUR_E_INVALID_ARGUMENT, "partition must have at least one block");
    if (offsets[0] != 0 || offsets[G] != s.n_global)
        fail(BCUR_E_DIMENSION_MISMATCH, "partition does not cover the columns of A");
    for (int64_t g = 0; g < G; ++g)
        if (offsets[g + 1] <= offsets[g]) fail(BCUR_E_INVALID_ARGUMENT, "partition blocks must be non-empty and ordered");
    s.g0 = -1;
    s.g1 = -1;
    for (int64_t g = 0; g <= G; ++g) {
        if (offsets[g] == s.col0) s.g0 = g;
        if (offsets[g] == s.col0 + a->n) s.g1 = g;
    }
    if (s.g0 < 0 || s.g1 < 0 || s.g1 < s.g0)
        fail(BCUR_E_DIMENSION_MISMATCH, "column shard is not aligned to block boundaries");
    s.off_global.assign(offsets, offsets + G + 1);
    std::vector<int64_t> local(s.g1 - s.g0 + 1);
    for (int64_t g = s.g0; g <= s.g1; ++g) local[g - s.g0] = offsets[g] - s.col0;
    s.d_local = DevBuf(a->ctx, local.size() * sizeof(int64_t));
    h2d(a->ctx, s.d_local.as<int64_t>(), local.data(), local.size());
    Ctx* c = a->ctx;
    s.owner.assign(G, c->comm.rank);
    if (c->comm.world > 1) {  // which rank holds each block (shards need not be equal)
        std::vector<double> own(G, 0.0);
        for (int64_t g = s.g0; g < s.g1; ++g) own[g] = c->comm.rank + 1.0;
        DevBuf d(c, G * sizeof(double));
        h2d(c, d.as<double>(), own.data(), G);
        allreduce(c, d.as<double>(), G);
        d2h(c, own.data(), d.as<double>(), G);
        for (int64_t g = 0; g < G; ++g) {
            s.owner[g] = (int)own[g] - 1;
            if (s.owner[g] < 0 || s.owner[g] >= c->comm.world)
                fail(BCUR_E_DIMENSION_MISMATCH, "column shards do not tile the partition exactly once");
        }
    }
    return s;
}

// Gather a G-vector whose shard-local part [g0, g1) lives on each rank (zero-padded allreduce).
static void gather_blocks_vec(Ctx* c, const Shard& s, const double* d_local, double* d_global) {
    if (c->comm.world <= 1) {
        CUDA_CHECK(cudaMemcpyAsync(d_global, d_local, s.G * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    fill_f64(c, d_global, s.G, 0.0);
    CUDA_CHECK(cudaMemcpyAsync(d_global + s.g0, d_local, (s.g1 - s.g0) * sizeof(double), cudaMemcpyDeviceToDevice,
                               c->stream));
    allreduce(c, d_global, s.G);
}

// ------------------------------------------------- factorizations of any size
struct CholInfo {
    int info;
    double mindiag, maxdiag;
};

static void tri_inv_any(Ctx* c, const double* R, int64_t w, double* X, const double* dinv = nullptr);

// Recursive Cholesky with the inverse alongside (fp64, all on the device):
//   chol_inv([G11 G12; · G22]) :  (R11, X11) = chol_inv(G11)
//                                 R12 = X11ᵀ·G12                 (DMMA, op(A) lower)
//                                 G22 −= R12ᵀ·R12                (DMMA, upper tiles only)
//                                 (R22, X22) = chol_inv(G22)
//                                 X12 = −(X11·R12)·X22           (X11·R12 on a side stream,
//                                                                 overlapping the G22 branch)
// down to ≤ 128-wide leaves factored and inverted by one CTA each (kernels_dmma.cu).  The
// critical path is the 32 leaves of a 4096-wide Gram and the big products between them; no
// host round trip until the final status read (the blocked right-looking chain it replaces
// issued ~6 small dependent kernels per 128 columns).
struct CholRec {
    Ctx* c;
    double *W, *R, *X;
    int64_t w;
    int* st;
    cudaStream_t main_s, side_s;
    bool tc;  // products of ≥ 512-wide blocks on the tcgen05 3×FP16 kernels (fp32-class Grams)
    bool want_r;  // the caller reads R (its diagonal blocks are never read inside the recursion)
    size_t ev = 0;
};

// op(A)·X product of the recursion: DMMA fp64, or — `tc`, both block sides ≥ 512 — the 3×FP16
// tensor-core kernels (the Gram of an fp32 basis carries ~2⁻²² relative error already; the
// first CholQR pass only needs R to ~1e-5, the second pass restores orthonormality).
static void rec_gemm(CholRec& S, bool tc, Op ta, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                     const double* X, double beta, double* C, int flags) {
    Ctx* c = S.c;
    if (tc) {
        // gemm_h3: a_mn → Out(M×N) = A(M×K)·X(K×N); else Out(M×N) = Aᵀ·X with A K×M
        if (ta == OP_N)
            gemm_h3(c, true, A, BCUR_F64, M, K, S.w, X, BCUR_F64, N, S.w, alpha, beta, C, S.w, flags & GEMM_B_UPPER);
        else
            gemm_h3(c, false, A, BCUR_F64, K, M, S.w, X, BCUR_F64, N, S.w, alpha, beta, C, S.w, 0);
        return;
    }
    dgemm(c, ta, OP_N, M, N, K, alpha, A, BCUR_F64, S.w, X, BCUR_F64, S.w, beta, C, S.w, flags);
}

static void chol_rec(CholRec& S, int64_t o, int64_t n) {
    Ctx* c = S.c;
    const int64_t w = S.w;
    auto at = [&](double* p, int64_t i, int64_t j) { return p + i + j * w; };
    if (n <= 128) {
        // R and X were zeroed by chol_enqueue: the leaf writes the upper triangles only
        chol_inv_leaf(c, at(S.W, o, o), n, w, at(S.R, o, o), w, at(S.X, o, o), w, S.st,
                      reinterpret_cast<double*>(S.st) + 1, o, (S.want_r ? 0 : 1) | 2);
        return;
    }
    const int64_t nl = (n + 127) / 128, n1 = (nl + 1) / 2 * 128, n2 = n - n1, o2 = o + n1;
    const bool tc = S.tc && n1 >= 512 && n2 >= 256;
    chol_rec(S, o, n1);
    // R12 = X11ᵀ·G12
    rec_gemm(S, tc, OP_T, n1, n2, n1, 1.0, at(S.X, o, o), at(S.W, o, o2), 0.0, at(S.R, o, o2), GEMM_A_LOWER);
    const cudaEvent_t e_r12 = c->sync_event(S.ev++), e_t = c->sync_event(S.ev++);
    CUDA_CHECK(cudaEventRecord(e_r12, S.main_s));
    CUDA_CHECK(cudaStreamWaitEvent(S.side_s, e_r12, 0));
    c->waited(S.main_s, S.side_s);
    c->stream = S.side_s;  // T = X11·R12 into G12's place (G12 is consumed)
    rec_gemm(S, tc, OP_N, n1, n2, n1, 1.0, at(S.X, o, o), at(S.R, o, o2), 0.0, at(S.W, o, o2), GEMM_A_UPPER);
    CUDA_CHECK(cudaEventRecord(e_t, S.side_s));
    c->stream = S.main_s;
    // Schur complement G22 −= R12ᵀ·R12 (upper triangle; the tensor-core form writes it whole)
    rec_gemm(S, tc, OP_T, n2, n2, n1, -1.0, at(S.R, o, o2), at(S.R, o, o2), 1.0, at(S.W, o2, o2), GEMM_SYM_UPPER);
    chol_rec(S, o2, n2);
    CUDA_CHECK(cudaStreamWaitEvent(S.main_s, e_t, 0));
    c->waited(S.side_s, S.main_s);
    // X12 = −T·X22
    rec_gemm(S, tc, OP_N, n1, n2, n2, -1.0, at(S.W, o, o2), at(S.X, o2, o2), 0.0, at(S.X, o, o2), GEMM_B_UPPER);
}

// G (w×w SPD, fp64, upper triangle read) → R upper (w×w, ld w, lower zero) with G = RᵀR, and
// (Rinv nullable) X = R⁻¹ (upper, ld w).  info != 0: the pivot info − 1 failed (R, X invalid).
// Enqueue the factorization (no host round trip): st (64 bytes) receives {info, pad, min diag(R),
// max diag(G)} (chol_status_init's layout).
// want_r = false: R's diagonal blocks are not written (R still holds the off-diagonal blocks).
static void chol_enqueue(Ctx* c, const double* G, int64_t w, int64_t ldg, double* R, double* X, bool tc, int* st,
                         bool want_r = true) {
    chol_status_init(c, G, w, ldg, st);
    if (w <= 128) {
        chol_inv_leaf(c, G, w, ldg, R, w, X, w, st, reinterpret_cast<double*>(st) + 1, 0, want_r ? 0 : 1);
        return;
    }
    // the persistent kernel streams its operands in 16-byte pairs: even widths (odd ones, and
    // BCUR_CHOL_REC=1 for experiments, take the launch-per-product recursion below; at w = 200
    // both take ~0.17 ms, c1's C basis, profiles/r02af)
    static const bool rec = getenv("BCUR_CHOL_REC") != nullptr;
    // Wide fp32-class Grams: one level of the recursion around two persistent launches.  The
    // persistent kernel's cost is its serial chain (~80 µs per 128 columns up to w = 2048, ~107 µs
    // at 4096 where the DMMA bulk outgrows the FACT window: profiles/r02x/chol_bench.log), so the
    // two half-width chains cost what the whole one does and the off-diagonal quarter — three
    // quarters of the bulk flops — moves to four tcgen05 3×FP16 products (~0.05 ms each).
    static const int64_t hyb_min = getenv("BCUR_CHOL_HYBRID") ? atoll(getenv("BCUR_CHOL_HYBRID")) : 3072;
    if (!rec && w % 2 == 0 && tc && hyb_min > 0 && w >= hyb_min) {
        const int64_t n1 = ((w + 127) / 128 + 1) / 2 * 128, n2 = w - n1;
        Mat64 W(c, w, w), Xs(c, n1, n1), Rs;
        if (want_r) Rs = Mat64(c, n1, n1);
        copy_f64(c, G, w, w, ldg, W.p(), w);
        // zeros only where nothing is written below: X's lower-left quarter (the diagonal halves
        // arrive as full squares, X12 whole); R the same, and only when the caller reads it
        CUDA_CHECK(cudaMemset2DAsync(X + n1, w * sizeof(double), 0, n2 * sizeof(double), n1, c->stream));
        if (want_r) CUDA_CHECK(cudaMemset2DAsync(R + n1, w * sizeof(double), 0, n2 * sizeof(double), n1, c->stream));
        cudaStream_t main_s = c->stream, side_s = c->side_stream();
        c->order(main_s, side_s, 0);
        CholRec S{c, W.p(), R, X, w, st, main_s, side_s, true, want_r};
        auto at = [&](double* p, int64_t i, int64_t j) { return p + i + j * w; };
        // a diagonal half: the persistent kernel works on compact n × n outputs (ld n)
        auto half = [&](int64_t o, int64_t n) {
            if (!want_r) Rs = Mat64(c, n, n);  // (R's off-diagonal 128-blocks still land here; not read)
            chol_persistent(c, at(W.p(), o, o), n, w, Rs.p(), Xs.p(), st, want_r);
            CUDA_CHECK(cudaMemcpy2DAsync(at(X, o, o), w * sizeof(double), Xs.p(), n * sizeof(double), n * sizeof(double),
                                         n, cudaMemcpyDeviceToDevice, c->stream));
            if (want_r)
                CUDA_CHECK(cudaMemcpy2DAsync(at(R, o, o), w * sizeof(double), Rs.p(), n * sizeof(double),
                                             n * sizeof(double), n, cudaMemcpyDeviceToDevice, c->stream));
        };
        half(0, n1);
        rec_gemm(S, true, OP_T, n1, n2, n1, 1.0, at(X, 0, 0), at(W.p(), 0, n1), 0.0, at(R, 0, n1), GEMM_A_LOWER);
        const cudaEvent_t e_r12 = c->sync_event(S.ev++), e_t = c->sync_event(S.ev++);
        CUDA_CHECK(cudaEventRecord(e_r12, main_s));
        CUDA_CHECK(cudaStreamWaitEvent(side_s, e_r12, 0));
        c->waited(main_s, side_s);
        c->stream = side_s;  // T = X11·R12 into G12's place, beside the G22 branch
        rec_gemm(S, true, OP_N, n1, n2, n1, 1.0, at(X, 0, 0), at(R, 0, n1), 0.0, at(W.p(), 0, n1), GEMM_A_UPPER);
        CUDA_CHECK(cudaEventRecord(e_t, side_s));
        c->stream = main_s;
        rec_gemm(S, true, OP_T, n2, n2, n1, -1.0, at(R, 0, n1), at(R, 0, n1), 1.0, at(W.p(), n1, n1), GEMM_SYM_UPPER);
        half(n1, n2);
        CUDA_CHECK(cudaStreamWaitEvent(main_s, e_t, 0));
        c->waited(side_s, main_s);
        rec_gemm(S, true, OP_N, n1, n2, n2, -1.0, at(W.p(), 0, n1), at(X, n1, n1), 0.0, at(X, 0, n1), GEMM_B_UPPER);
        c->order(side_s, main_s, 1);
        return;
    }
    if (!rec && w % 2 == 0) {
        chol_persistent(c, G, w, ldg, R, X, st, want_r);
        return;
    }
    ProfScope prof(c, "chol_inv", 2.0 * w * w * w / 3.0, 8.0 * 4 * w * w);
    Mat64 W(c, w, w);
    copy_f64(c, G, w, w, ldg, W.p(), w);
    CUDA_CHECK(cudaMemsetAsync(R, 0, (size_t)w * w * sizeof(double), c->stream));
    CUDA_CHECK(cudaMemsetAsync(X, 0, (size_t)w * w * sizeof(double), c->stream));
    cudaStream_t main_s = c->stream, side_s = c->side_stream();
    c->order(main_s, side_s, 0);
    CholRec S{c, W.p(), R, X, w, st, main_s, side_s, tc, want_r};
    chol_rec(S, 0, w);
    c->stream = main_s;
    c->order(side_s, main_s, 1);
}

static CholInfo chol_any(Ctx* c, const double* G, int64_t w, int64_t ldg, double* R, double* Rinv = nullptr,
                         bool tc = false, bool want_r = true) {
    DevBuf st(c, 64);
    struct { int info; int pad; double mindiag, maxdiag; } hs;
    Mat64 Xown;
    double* X = Rinv;
    if (!X) {
        Xown = Mat64(c, w, w);
        X = Xown.p();
    }
    chol_enqueue(c, G, w, ldg, R, X, tc, st.as<int>(), want_r);
    c->read_later(&hs, st.ptr, sizeof hs);
    c->read_all();
    return {hs.info, hs.info ? 0.0 : hs.mindiag, hs.maxdiag};
}

// chol_any without the synchronization: the status is delivered into *hs by the next
// c->read_all() (callers enqueue speculative work behind the factorization meanwhile)
struct CholStat {
    int info, pad;
    double mindiag, maxdiag;
};
static void chol_later(Ctx* c, const double* G, int64_t w, int64_t ldg, double* R, double* Rinv, bool tc, bool want_r,
                       CholStat* hs) {
    DevBuf st(c, 64);
    chol_enqueue(c, G, w, ldg, R, Rinv, tc, st.as<int>(), want_r);
    c->read_later(hs, st.ptr, sizeof *hs);
}
static CholInfo chol_info(const CholStat& hs) { return {hs.info, hs.info ? 0.0 : hs.mindiag, hs.maxdiag}; }

int cholesky_inverse(Ctx* c, const double* G, int64_t w, int64_t ldg, double* R, double* Rinv, double* mindiag) {
    // BCUR_CHOL_TC=1 (tests): the path the fp32 pipelines take for their bases' Grams — off-diagonal
    // products on tcgen05 3×FP16, and for w ≥ 3072 the hybrid around two persistent launches
    const bool tc = getenv("BCUR_CHOL_TC") != nullptr && w % 128 == 0;
    const CholInfo ci = chol_any(c, G, w, ldg, R, Rinv, tc);
    if (mindiag) *mindiag = ci.mindiag;
    return ci.info;
}

// X = R⁻¹ for upper-triangular R (w×w, ld w).  Blocked back-substitution by block rows.
static void tri_inv_any(Ctx* c, const double* R, int64_t w, double* X, const double* dinv) {
    constexpr int64_t B = 128;  // single-CTA shared-memory inverse of ≤128-wide diagonal blocks
    if (w <= B) {
        tri_inv_upper(c, R, w, w, X, w);
        return;
    }
    if (w <= 144) dinv = nullptr;  // chol_any factored it in one piece (no blocks kept)
    fill_f64(c, X, w * w, 0.0);
    Mat64 T(c, B, w);
    const int64_t nb = (w + B - 1) / B;
    for (int64_t bi = nb - 1; bi >= 0; --bi) {
        const int64_t r0 = bi * B, rb = std::min(B, w - r0), c0 = r0 + rb, rest = w - c0;
        double* Xii = X + r0 + r0 * w;
        if (dinv) copy_f64(c, dinv + r0 * B, rb, rb, B, Xii, w);
        else tri_inv_upper(c, R + r0 + r0 * w, rb, w, Xii, w);
        if (rest > 0) {
            // X[r0, c0:] = −Rii⁻¹ · (R[r0, c0:] · X[c0:, c0:])
            gemm(c, OP_N, OP_N, rb, rest, rest, 1.0, R + r0 + c0 * w, BCUR_F64, w, X + c0 + c0 * w, BCUR_F64, w, 0.0,
                 T.p(), B);
            gemm(c, OP_N, OP_N, rb, rest, rb, -1.0, Xii, BCUR_F64, w, T.p(), BCUR_F64, B, 0.0, X + r0 + c0 * w, w);
        }
    }
}

// ------------------------------------------------------------------ orth
// X (rows × w, fp64) → Q (rows × r, fp64) with X ≈ Q·T.  Grams allreduced when dist.
// ref < 0 → ref = max column norm of X.  Mirrors oracle.orth.
int64_t orth(Ctx* c, const double* X, int64_t rows, int64_t w, int64_t ldx, double ref, int dt, double* Q,
             int64_t ldq, bool dist, Mat64* T_out, int* path_out) {
    if (w == 0) return 0;
    Mat64 G(c, w, w), R(c, w, w), Ri(c, w, w), Q1(c, rows, w);
    gemm(c, OP_T, OP_N, w, w, rows, 1.0, X, BCUR_F64, ldx, X, BCUR_F64, ldx, 0.0, G.p(), G.ld);
    if (dist) allreduce(c, G.p(), w * w);
    const CholInfo ci = chol_any(c, G.p(), w, G.ld, R.p(), Ri.p(), false, T_out != nullptr);
    if (ref < 0) ref = std::sqrt(std::max(ci.maxdiag, 0.0));
    int64_t r = w;
    const bool chol_ok = ci.info == 0 && std::isfinite(ci.mindiag) && ci.mindiag > tau_chol(dt) * ref;
    Mat64 Wr, sig;
    std::vector<double> sig_h;
    if (chol_ok) {
        gemm(c, OP_N, OP_N, rows, w, w, 1.0, X, BCUR_F64, ldx, Ri.p(), BCUR_F64, Ri.ld, 0.0, Q1.p(), Q1.ld);
    } else {
        // σ_max(X) ≤ ‖X‖_F ≤ sqrt(w·max diag G): below the rank cut every σ is, so the
        // eig path would keep nothing — skip the eigensolver (e.g. a panel already in span).
        if (std::sqrt((double)w * std::max(ci.maxdiag, 0.0)) <= tau_rank(dt) * ref) {
            if (path_out) *path_out = 1;
            if (T_out) *T_out = Mat64(c, 0, w);
            return 0;
        }
        if (!dist && rows < w) {
            // wide panel (e.g. 64 × 100 biometric blocks): the same nonzero spectrum from the
            // rows × rows Gram X·Xᵀ, whose eigenvectors are the orthonormal basis directly
            Mat64 Gr(c, rows, rows), lam(c, rows, 1), U(c, rows, rows);
            gemm(c, OP_N, OP_T, rows, rows, w, 1.0, X, BCUR_F64, ldx, X, BCUR_F64, ldx, 0.0, Gr.p(), Gr.ld);
            {   // safely full row rank → range(X) = ℝ^rows: Q = I, T = X (no eigensolve)
                Mat64 Rr(c, rows, rows);
                const CholInfo cr = chol_any(c, Gr.p(), rows, Gr.ld, Rr.p(), nullptr, false, false);
                if (cr.info == 0 && std::isfinite(cr.mindiag) && cr.mindiag > tau_chol(dt) * ref) {
                    fill_f64(c, Q1.p(), rows * rows, 0.0);
                    Mat64 one(c, rows, 1);
                    fill_f64(c, one.p(), rows, 1.0);
                    CUDA_CHECK(cudaMemcpy2DAsync(Q1.p(), (Q1.ld + 1) * sizeof(double), one.p(), sizeof(double),
                                                 sizeof(double), rows, cudaMemcpyDeviceToDevice, c->stream));
                    copy_f64(c, Q1.p(), rows, rows, Q1.ld, Q, ldq);
                    if (T_out) {
                        Mat64 T(c, rows, w);
                        copy_f64(c, X, rows, w, ldx, T.p(), T.ld);
                        *T_out = std::move(T);
                    }
                    if (path_out) *path_out = 1;
                    return rows;
                }
            }
            sym_eig(c, Gr.p(), rows, Gr.ld, lam.p(), U.p());
            std::vector<double> lh(rows);
            d2h(c, lh.data(), lam.p(), rows);
            r = 0;
            for (int64_t i = 0; i < rows; ++i)
                if (std::sqrt(std::max(lh[i], 0.0)) > tau_rank(dt) * ref) ++r;
            if (r == 0) {
                if (path_out) *path_out = 1;
                if (T_out) *T_out = Mat64(c, 0, w);
                return 0;
            }
            copy_f64(c, U.p(), rows, r, U.ld, Q1.p(), Q1.ld);
            Mat64 G2(c, r, r), R2(c, r, r), R2i(c, r, r);
            gemm(c, OP_T, OP_N, r, r, rows, 1.0, Q1.p(), BCUR_F64, Q1.ld, Q1.p(), BCUR_F64, Q1.ld, 0.0, G2.p(), G2.ld);
            const CholInfo c2 = chol_any(c, G2.p(), r, G2.ld, R2.p(), R2i.p(), false, T_out != nullptr);
            if (c2.info != 0) fail(BCUR_E_ITERATION_FAILURE, "orth: second CholQR pass failed");
            gemm(c, OP_N, OP_N, rows, r, r, 1.0, Q1.p(), BCUR_F64, Q1.ld, R2i.p(), BCUR_F64, R2i.ld, 0.0, Q, ldq);
            if (T_out) {  // T = R2 · (Q1ᵀ X)
                Mat64 QX(c, r, w), T(c, r, w);
                gemm(c, OP_T, OP_N, r, w, rows, 1.0, Q1.p(), BCUR_F64, Q1.ld, X, BCUR_F64, ldx, 0.0, QX.p(), QX.ld);
                gemm(c, OP_N, OP_N, r, w, r, 1.0, R2.p(), BCUR_F64, R2.ld, QX.p(), BCUR_F64, QX.ld, 0.0, T.p(), T.ld);
                *T_out = std::move(T);
            }
            if (path_out) *path_out = 1;
            return r;
        }
        Mat64 lam(c, w, 1), V(c, w, w);
        sym_eig(c, G.p(), w, G.ld, lam.p(), V.p());
        std::vector<double> lh(w);
        d2h(c, lh.data(), lam.p(), w);
        r = 0;
        for (int64_t i = 0; i < w; ++i) {
            const double s = std::sqrt(std::max(lh[i], 0.0));
            if (s > tau_rank(dt) * ref) ++r;
        }
        if (r == 0) {
            if (path_out) *path_out = 1;
            if (T_out) *T_out = Mat64(c, 0, w);
            return 0;
        }
        sig_h.resize(r);
        std::vector<double> inv(r);
        for (int64_t i = 0; i < r; ++i) {
            sig_h[i] = std::sqrt(lh[i]);
            inv[i] = 1.0 / sig_h[i];
        }
        Wr = Mat64(c, w, r);
        copy_f64(c, V.p(), w, r, V.ld, Wr.p(), Wr.ld);
        Mat64 dinv(c, r, 1);
        h2d(c, dinv.p(), inv.data(), r);
        Mat64 F(c, w, r);
        copy_f64(c, Wr.p(), w, r, Wr.ld, F.p(), F.ld);
        scale_columns(c, F.p(), w, r, F.ld, dinv.p());
        gemm(c, OP_N, OP_N, rows, r, w, 1.0, X, BCUR_F64, ldx, F.p(), BCUR_F64, F.ld, 0.0, Q1.p(), Q1.ld);
        sig = Mat64(c, r, 1);
        h2d(c, sig.p(), sig_h.data(), r);
    }
    // second pass: CholQR of the well-conditioned Q1
    Mat64 G2(c, r, r), R2(c, r, r), R2i(c, r, r);
    gemm(c, OP_T, OP_N, r, r, rows, 1.0, Q1.p(), BCUR_F64, Q1.ld, Q1.p(), BCUR_F64, Q1.ld, 0.0, G2.p(), G2.ld);
    if (dist) allreduce(c, G2.p(), r * r);
    const CholInfo c2 = chol_any(c, G2.p(), r, G2.ld, R2.p(), R2i.p(), false, T_out != nullptr);
    if (c2.info != 0) fail(BCUR_E_ITERATION_FAILURE, "orth: second CholQR pass failed");
    gemm(c, OP_N, OP_N, rows, r, r, 1.0, Q1.p(), BCUR_F64, Q1.ld, R2i.p(), BCUR_F64, R2i.ld, 0.0, Q, ldq);
    if (T_out) {
        Mat64 T(c, r, w);
        if (chol_ok) {
            gemm(c, OP_N, OP_N, r, w, r, 1.0, R2.p(), BCUR_F64, R2.ld, R.p(), BCUR_F64, R.ld, 0.0, T.p(), T.ld);
        } else {
            Mat64 R2s(c, r, r);
            copy_f64(c, R2.p(), r, r, R2.ld, R2s.p(), R2s.ld);
            scale_columns(c, R2s.p(), r, r, R2s.ld, sig.p());
            gemm(c, OP_N, OP_T, r, w, r, 1.0, R2s.p(), BCUR_F64, R2s.ld, Wr.p(), BCUR_F64, Wr.ld, 0.0, T.p(), T.ld);
        }
        *T_out = std::move(T);
    }
    if (path_out) *path_out = chol_ok ? 0 : 1;
    return r;
}

// Power-iteration orthonormalization (range finder, q ≥ 1): only span(Q) = span(X) matters
// there — the next product re-mixes the columns — so one CholQR pass Q = X·R⁻¹ suffices
// whenever orth's own CholQR test passes (min R_ii > τ_chol·ref ⇒ κ(X) < 1/τ_chol and
// ‖QᵀQ − I‖ ≲ κ²·u); the test runs on the device (*flag = 1 when it fails, and the caller
// redoes the range finder through orth), so no host round trip is needed.
static void orth_span(Ctx* c, const double* X, int64_t rows, int64_t w, int64_t ldx, double tau, double* Q,
                      int64_t ldq, bool dist, int* flag) {
    Mat64 G(c, w, w), R(c, w, w), Ri(c, w, w);
    DevBuf st(c, 64);
    gemm(c, OP_T, OP_N, w, w, rows, 1.0, X, BCUR_F64, ldx, X, BCUR_F64, ldx, 0.0, G.p(), G.ld, GEMM_SYM_UPPER);
    if (dist) allreduce(c, G.p(), w * w);
    chol_enqueue(c, G.p(), w, G.ld, R.p(), Ri.p(), false, st.as<int>(), false);
    chol_flag(c, st.as<int>(), tau, flag);
    gemm(c, OP_N, OP_N, rows, w, w, 1.0, X, BCUR_F64, ldx, Ri.p(), BCUR_F64, Ri.ld, 0.0, Q, ldq, GEMM_B_UPPER);
}

// ----------------------------------------------------------------- bases
// Orthonormal basis kept in fp32 (fp32 inputs: every product with it runs on the
// tensor cores) or fp64 (fp64 inputs).
struct Basis {
    DevBuf buf;
    int dt = BCUR_F64;
    int64_t rows = 0, cap = 0, rank = 0;
    void init(Ctx* c, int dt_, int64_t rows_, int64_t cap_, bool zero = true) {
        dt = dt_;
        rows = rows_;
        cap = std::max<int64_t>(cap_, 1);
        rank = 0;
        buf = DevBuf(c, (size_t)std::max<int64_t>(rows, 1) * cap * dtype_size(dt));
        if (zero) CUDA_CHECK(cudaMemsetAsync(buf.ptr, 0, buf.bytes, c->stream));
    }
    void* col(int64_t j) const { return (char*)buf.ptr + (size_t)j * rows * dtype_size(dt); }
    // optional 3×FP16 form of the fp32 basis (the interleaved hi/lo A operand, kept in step
    // with every append): the greedy CGS2 products run on it (kernels_umma.cu, H3)
    DevBuf il, iexps;
    bool h3() const { return il.ptr != nullptr; }
    // whole-C CholQR2 (fp32, 3×FP16): C = Q·R with R⁻¹ = rinv1·rinv2 (rinv1 = R1⁻¹ of the first
    // pass, rinv2 = I − F or the full R2⁻¹ of the second), kept for U = C⁺AR⁺ (block_cur)
    Mat64 rinv1, rinv2;
    bool has_rinv() const { return rinv1.m > 0 && rinv1.m == rank; }
    // the basis scaled by 2^14 (entries ≤ 1) as an interleaved fp16 hi/lo split (2·rows halves per
    // column): hi is the row-Σ² passes' X operand, lo its rounding error (sketch_correction);
    // x16e = the split's column exponents (all 14)
    DevBuf x16, x16e;
    void enable_h3(Ctx* c) {
        if (dt != BCUR_F32 || !h3_ok(rows)) return;
        il = DevBuf(c, (size_t)rows * cap * 4);
        iexps = DevBuf(c, (size_t)cap * sizeof(int));
    }
};

// Block CGS2 of panel P (rows × w, fp64, overwritten) against the basis; the new
// orthonormal columns are appended to it.  Returns the rank added.
static int64_t cgs2_append(Ctx* c, Basis* B, double* P, int64_t w, int64_t ldp, double ref, int dt, bool dist) {
    const int64_t rows = B->rows, cur = B->rank;
    if (cur > 0) {
        Mat64 X(c, cur, w);
        for (int pass = 0; pass < 2; ++pass) {
            if (B->h3())
                umma_h3(c, false, B->il.as<uint16_t>(), B->iexps.as<int>(), rows, cur, P, BCUR_F64, w, ldp, 1.0, 0.0,
                        X.p(), X.ld);
            else
                gemm(c, OP_T, OP_N, cur, w, rows, 1.0, B->buf.ptr, B->dt, rows, P, BCUR_F64, ldp, 0.0, X.p(), X.ld);
            if (dist) allreduce(c, X.p(), cur * w);
            if (B->h3())
                umma_h3(c, true, B->il.as<uint16_t>(), B->iexps.as<int>(), rows, cur, X.p(), BCUR_F64, w, X.ld, -1.0,
                        1.0, P, ldp);
            else
                gemm(c, OP_N, OP_N, rows, w, cur, -1.0, B->buf.ptr, B->dt, rows, X.p(), BCUR_F64, X.ld, 1.0, P, ldp);
        }
    }
    int64_t r;
    if (B->dt == BCUR_F64) {
        r = orth(c, P, rows, w, ldp, ref, dt, (double*)B->col(cur), rows, dist, nullptr, nullptr);
    } else {
        Mat64 Qn(c, rows, w);
        r = orth(c, P, rows, w, ldp, ref, dt, Qn.p(), Qn.ld, dist, nullptr, nullptr);
        convert(c, Qn.p(), BCUR_F64, rows, r, Qn.ld, B->col(cur), B->dt, rows);
        if (B->h3() && r > 0)
            split_il_into(c, B->col(cur), B->dt, rows, r, rows, B->il.as<uint16_t>() + (size_t)cur * 2 * rows,
                          B->iexps.as<int>() + cur);
    }
    B->rank += r;
    return r;
}

// Whole-matrix CholQR2 of C (rows × cc; fp32 on the tensor cores, fp64 on DGEMM), written
// to B.  Returns false (B untouched) when C is not safely full rank (oracle.cholqr2_whole).
// fp32 C on the 3×FP16 tensor-core path: every operand split once — C (Gram and C·R⁻¹ read
// one interleaved split), Q1 straight from fp64 (Gram and the correction) — and the products
// issued directly (a split per gemm() call re-split C and Q1, and Q1 went through fp32 first).
// cil_pre (nullable): C already split (gathered from A's interleaved copy with its exponents).
static bool cholqr2_whole_h3(Ctx* c, const void* C, int64_t rows, int64_t cc, bool dist, int dt, Basis* B,
                             bool keep_rinv, DevBuf* cil_pre = nullptr, DevBuf* ce_pre = nullptr) {
    Mat64 G(c, cc, cc), R(c, cc, cc), Ri(c, cc, cc), R1i;
    DevBuf cil, ce;
    if (cil_pre) {
        cil = std::move(*cil_pre);
        ce = std::move(*ce_pre);
    } else {
        split_il(c, C, BCUR_F32, rows, cc, rows, &cil, &ce);
    }
    const F16View cx{cil.as<uint16_t>(), nullptr, ce.as<int>(), rows, cc};
    umma_h3(c, false, cil.as<uint16_t>(), ce.as<int>(), rows, cc, cx, 1.0, 0.0, G.p(), G.ld, GEMM_SYM_UPPER);
    if (dist) allreduce(c, G.p(), cc * cc);
    // The factorization's status and the second pass's ‖Q1ᵀQ1 − I‖ come back in ONE read: Q1 and
    // its Gram are enqueued behind the factorization before its status is known (when it failed
    // they are garbage and discarded with the path)
    CholStat hs1{};
    chol_later(c, G.p(), cc, G.ld, R.p(), Ri.p(), true, false, &hs1);
    // Q1 = C·R⁻¹ written straight into its interleaved split (fixed column exponent: the columns
    // of Q1 have norm ≈ 1) — the operand of the Gram Q1ᵀQ1 and of the second-pass product, with
    // no fp64 Q1 and no split pass
    DevBuf qil(c, (size_t)rows * cc * 4), qe(c, (size_t)cc * sizeof(int));
    fill_basis_exps(c, qe.as<int>(), cc);
    // (one-accumulator products: a ~1e-6 error in Q1 is a column scaling or a random rotation
    // whose first-order effect on the captured mass vanishes, and the second pass measures Q1)
    umma_h3_to_split(c, cil.as<uint16_t>(), ce.as<int>(), rows, cc, Ri.p(), BCUR_F64, cc, Ri.ld, 1.0,
                     qil.as<uint16_t>(), GEMM_B_UPPER | GEMM_FAST_ACC);
    cil = DevBuf();
    if (keep_rinv) {
        R1i = Mat64(c, cc, cc);
        copy_f64(c, Ri.p(), cc, cc, Ri.ld, R1i.p(), cc);
    }
    const F16View qx{qil.as<uint16_t>(), nullptr, qe.as<int>(), rows, cc};
    umma_h3(c, false, qil.as<uint16_t>(), qe.as<int>(), rows, cc, qx, 1.0, 0.0, G.p(), G.ld, GEMM_SYM_UPPER);
    if (dist) allreduce(c, G.p(), cc * cc);
    // second pass as cholqr2_whole: near identity → Q = Q1 + Q1·(−F), else a full factorization
    Mat64 dev(c, 1, 1);
    max_dev_identity(c, G.p(), cc, G.ld, dev.p());
    double hdev = 1.0;
    d2h_later(c, &hdev, dev.p(), 1);
    c->read_all();
    const CholInfo ci = chol_info(hs1);
    const double ref = std::sqrt(std::max(ci.maxdiag, 0.0));
    if (!(ci.info == 0 && std::isfinite(ci.mindiag) && ci.mindiag > tau_chol(dt) * ref)) return false;
    const bool near = hdev < 1e-4;
    if (near) {
        near_identity_rinv(c, G.p(), cc, G.ld, Ri.p(), true);
    } else {
        const CholInfo c2 = chol_any(c, G.p(), cc, G.ld, R.p(), Ri.p(), true, false);
        if (c2.info != 0) return false;
    }
    B->init(c, BCUR_F32, rows, cc, false);  // every column is written below
    B->x16 = DevBuf(c, (size_t)rows * cc * 4);
    B->x16e = DevBuf(c, (size_t)cc * sizeof(int));
    fill_basis_exps(c, B->x16e.as<int>(), cc);
    // the second-pass product and the basis output in one pass: Q = Q1·X2 (+ Q1 read back from
    // its split when X2 = −F), written as the fp32 basis and its fp16·2^14 copy
    umma_h3_basis(c, qil.as<uint16_t>(), qe.as<int>(), rows, cc, Ri.p(), BCUR_F64, cc, Ri.ld, 1.0,
                  near ? qil.as<uint16_t>() : nullptr, B->buf.as<float>(), B->x16.as<uint16_t>(),
                  GEMM_B_UPPER | (near ? GEMM_FAST_ACC | GEMM_HI_ONLY : 0));  // near: a ≲1e-4-sized correction
    B->rank = cc;
    if (keep_rinv) {
        B->rinv1 = std::move(R1i);
        B->rinv2 = Mat64(c, cc, cc);
        if (near) near_identity_rinv(c, G.p(), cc, G.ld, B->rinv2.p(), false);  // I − F (Ri held −F)
        else copy_f64(c, Ri.p(), cc, cc, Ri.ld, B->rinv2.p(), cc);
    }
    return true;
}

static bool cholqr2_whole(Ctx* c, const void* C, int cdt, int64_t rows, int64_t cc, bool dist, int dt, Basis* B,
                          bool keep_rinv = false) {
    if (cc == 0 || rows < cc) return false;
    if (cdt == BCUR_F32 && h3_ok(rows) && cc >= 128) return cholqr2_whole_h3(c, C, rows, cc, dist, dt, B, keep_rinv);
    Mat64 G(c, cc, cc), R(c, cc, cc), Ri(c, cc, cc), Q1(c, rows, cc);
    // Grams: upper triangles only (every consumer — Cholesky, max|G−I|, I−F — reads the upper)
    gemm(c, OP_T, OP_N, cc, cc, rows, 1.0, C, cdt, rows, C, cdt, rows, 0.0, G.p(), G.ld, GEMM_SYM_UPPER);
    if (dist) allreduce(c, G.p(), cc * cc);
    // one read for the factorization's status and ‖Q1ᵀQ1 − I‖ (Q1 and its Gram speculative, as
    // cholqr2_whole_h3)
    CholStat hs1{};
    chol_later(c, G.p(), cc, G.ld, R.p(), Ri.p(), false, false, &hs1);
    gemm(c, OP_N, OP_N, rows, cc, cc, 1.0, C, cdt, rows, Ri.p(), BCUR_F64, Ri.ld, 0.0, Q1.p(), Q1.ld,
         GEMM_B_UPPER);
    // Q1 in the basis dtype (fp32 → every later product with it runs on the tensor cores)
    DevBuf q1f;
    const void* q1 = Q1.p();
    if (cdt == BCUR_F32) {
        q1f = DevBuf(c, (size_t)rows * cc * 4);
        convert(c, Q1.p(), BCUR_F64, rows, cc, Q1.ld, q1f.ptr, BCUR_F32, rows);
        q1 = q1f.ptr;
    }
    gemm(c, OP_T, OP_N, cc, cc, rows, 1.0, q1, cdt, rows, q1, cdt, rows, 0.0, G.p(), G.ld, GEMM_SYM_UPPER);
    if (dist) allreduce(c, G.p(), cc * cc);
    // Second pass.  Q1ᵀQ1 = I + E with ‖E‖ ~ 1e-7·κ(C)²; when ‖E‖_max < 1e-4 the Cholesky
    // factor is R2 = I + F + O(‖E‖²), F = strict_upper(E) + diag(E)/2, so R2⁻¹ = I − F to
    // ~1e-8 — no second factorization needed.  Otherwise: full Cholesky + inverse.
    Mat64 dev(c, 1, 1);
    max_dev_identity(c, G.p(), cc, G.ld, dev.p());
    double hdev = 1.0;
    d2h_later(c, &hdev, dev.p(), 1);
    c->read_all();
    const CholInfo ci = chol_info(hs1);
    const double ref = std::sqrt(std::max(ci.maxdiag, 0.0));
    if (!(ci.info == 0 && std::isfinite(ci.mindiag) && ci.mindiag > tau_chol(dt) * ref)) return false;
    const bool near = hdev < 1e-4;
    if (near) {
        // fp32: Q = Q1 + Q1·(−F) — the product is a ~1e-7-sized correction, so one rounded TF32
        // pass is exact to ~1e-11; fp64: Q = Q1·(I − F) on DGEMM
        near_identity_rinv(c, G.p(), cc, G.ld, Ri.p(), cdt == BCUR_F32);
    } else {
        const CholInfo c2 = chol_any(c, G.p(), cc, G.ld, R.p(), Ri.p(), false, false);
        if (c2.info != 0) return false;
    }
    B->init(c, cdt, rows, cc);
    if (cdt == BCUR_F32) {
        if (near)
            gemm(c, OP_N, OP_N, rows, cc, cc, 1.0, q1, cdt, rows, Ri.p(), BCUR_F64, Ri.ld, 1.0, Q1.p(), Q1.ld,
                 GEMM_B_UPPER | GEMM_X1);
        else
            gemm(c, OP_N, OP_N, rows, cc, cc, 1.0, q1, cdt, rows, Ri.p(), BCUR_F64, Ri.ld, 0.0, Q1.p(), Q1.ld,
                 GEMM_B_UPPER);
        convert(c, Q1.p(), BCUR_F64, rows, cc, Q1.ld, B->buf.ptr, BCUR_F32, rows);
    } else {
        gemm(c, OP_N, OP_N, rows, cc, cc, 1.0, q1, cdt, rows, Ri.p(), BCUR_F64, Ri.ld, 0.0, (double*)B->buf.ptr,
             rows, GEMM_B_UPPER);
    }
    B->rank = cc;
    return true;
}

// ---------------------------------------------------------- range finder
// A·X (trans = false) or AᵀX of the range finder: 3×FP16 from the norms pass's split of A
// when present, else the fp32 A path (3×TF32 on the tensor cores / fp64)
static void a_product(Ctx* c, const DMat* a, const RoundedA* ra, bool trans, int64_t N, const void* X, int dtx,
                      int64_t ldx, double* out, int64_t ldo, int flags = 0) {
    if (ra && ra->has_lo()) {
        umma_h3(c, !trans, ra->il.as<uint16_t>(), ra->exps.as<int>(), a->m, a->n, X, dtx, N, ldx, 1.0, 0.0, out,
                ldo, flags);
        return;
    }
    if (trans)
        gemm(c, OP_T, OP_N, a->n, N, a->m, 1.0, a->ptr, a->dtype, a->ld, X, dtx, ldx, 0.0, out, ldo);
    else
        gemm(c, OP_N, OP_N, a->m, N, a->n, 1.0, a->ptr, a->dtype, a->ld, X, dtx, ldx, 0.0, out, ldo);
}

// fast: every orthonormalization is one orth_span CholQR pass (no host round trips; the power
// iterations need only the span, the final basis passes the stricter κ < 100 test); returns
// false when a device-side CholQR test failed — the caller then reruns with fast = false
// (orth's CholQR2 / SVQB paths, identical to the oracle's).
static bool range_finder_impl(Ctx* c, const DMat* a, int64_t k, int64_t p, int64_t q, uint64_t key, Subspace* out,
                              bool rank_floor, const RoundedA* ra, bool fast, const std::function<void()>* after_read) {
    const int64_t m = a->m, nl = a->n;
    const int64_t ng = a->n_global > 0 ? a->n_global : a->n;
    const int64_t l = std::min(k + p, std::min(m, ng));
    const int dt = a->dtype;
    Mat64 Om(c, nl, l), Y(c, m, l);
    omega(c, key, nl, a->col0, l, Om.p(), Om.ld);
    a_product(c, a, ra, false, l, Om.p(), BCUR_F64, Om.ld, Y.p(), Y.ld);
    allreduce(c, Y.p(), m * l);
    Mat64 Qy(c, m, l);
    DevBuf flag(c, 64);
    if (fast) CUDA_CHECK(cudaMemsetAsync(flag.ptr, 0, sizeof(int), c->stream));
    int64_t r = l;
    for (int64_t it = 0; it < q; ++it) {
        if (fast) orth_span(c, Y.p(), m, r, Y.ld, tau_chol(dt), Qy.p(), Qy.ld, false, flag.as<int>());
        else r = orth(c, Y.p(), m, r, Y.ld, -1.0, dt, Qy.p(), Qy.ld, false, nullptr, nullptr);
        if (r == 0) fail(BCUR_E_ZERO_MATRIX, "range_finder: A is identically zero");
        Mat64 Z(c, nl, r), Qz(c, nl, r);
        a_product(c, a, ra, true, r, Qy.p(), BCUR_F64, Qy.ld, Z.p(), Z.ld);
        if (fast) orth_span(c, Z.p(), nl, r, Z.ld, tau_chol(dt), Qz.p(), Qz.ld, true, flag.as<int>());
        else r = orth(c, Z.p(), nl, r, Z.ld, -1.0, dt, Qz.p(), Qz.ld, true, nullptr, nullptr);
        if (r == 0) fail(BCUR_E_ZERO_MATRIX, "range_finder: A is identically zero");
        a_product(c, a, ra, false, r, Qz.p(), BCUR_F64, Qz.ld, Y.p(), Y.ld);
        allreduce(c, Y.p(), m * r);
    }
    // The final basis: one CholQR pass as well when κ(Y) < 100 (min R_ii > 1e-2·ref): then
    // ‖QᵀQ − I‖ ≲ 1e4·u ≈ 1e-12 and B = QᵀA has the singular subspace of the CholQR2 basis to
    // that accuracy.  Otherwise (the flag) the whole range finder reruns through orth.
    if (fast) orth_span(c, Y.p(), m, r, Y.ld, std::max(tau_chol(dt), 1e-2), Qy.p(), Qy.ld, false, flag.as<int>());
    else r = orth(c, Y.p(), m, r, Y.ld, -1.0, dt, Qy.p(), Qy.ld, false, nullptr, nullptr);
    if (r == 0) fail(BCUR_E_ZERO_MATRIX, "range_finder: A is identically zero");
    // Bᵀ = Aᵀ·Q (n_local × r); B·Bᵀ = Σ_ranks Bᵀ_sᵀ Bᵀ_s
    Mat64 Bt(c, nl, r), Gb(c, r, r), lam(c, r, 1), Ut(c, r, r);
    a_product(c, a, ra, true, r, Qy.p(), BCUR_F64, Qy.ld, Bt.p(), Bt.ld);
    gemm(c, OP_T, OP_N, r, r, nl, 1.0, Bt.p(), BCUR_F64, Bt.ld, Bt.p(), BCUR_F64, Bt.ld, 0.0, Gb.p(), Gb.ld);
    allreduce(c, Gb.p(), r * r);
    sym_eig(c, Gb.p(), r, Gb.ld, lam.p(), Ut.p());
    int hflag = 0;
    std::vector<double> lh(r);
    if (fast) d2h_later(c, &hflag, flag.as<int>(), 1);
    d2h_later(c, lh.data(), lam.p(), r);
    c->read_all();  // (also delivers the caller's earlier reads, which after_read checks)
    if (after_read && *after_read) (*after_read)();
    if (hflag) return false;  // a failed CholQR test: Q (and everything after) is unusable
    std::vector<double> sg(r);
    for (int64_t i = 0; i < r; ++i) sg[i] = std::sqrt(std::max(lh[i], 0.0));
    if (!(sg[0] > 0.0)) fail(BCUR_E_ZERO_MATRIX, "range_finder: A is identically zero");
    // the reference's rank cut (matcore.cpp:35-49); the working-precision floor is opt-in
    double tol = 1e-12 * (double)std::max(m, ng) * sg[0];
    if (rank_floor) tol = std::max(tol, tau_rank(dt) * sg[0]);
    int64_t rank = 0;
    while (rank < r && sg[rank] > tol) ++rank;
    const int64_t ke = std::min(k, rank);
    std::vector<double> inv(ke);
    for (int64_t i = 0; i < ke; ++i) inv[i] = 1.0 / sg[i];
    Mat64 Wm(c, r, ke), dinv(c, ke, 1);
    copy_f64(c, Ut.p(), r, ke, Ut.ld, Wm.p(), Wm.ld);
    h2d(c, dinv.p(), inv.data(), ke);
    scale_columns(c, Wm.p(), r, ke, Wm.ld, dinv.p());
    out->v = Mat64(c, nl, ke);
    gemm(c, OP_N, OP_N, nl, ke, r, 1.0, Bt.p(), BCUR_F64, Bt.ld, Wm.p(), BCUR_F64, Wm.ld, 0.0, out->v.p(), out->v.ld);
    out->u = Mat64(c, m, ke);
    gemm(c, OP_N, OP_N, m, ke, r, 1.0, Qy.p(), BCUR_F64, Qy.ld, Ut.p(), BCUR_F64, Ut.ld, 0.0, out->u.p(), out->u.ld);
    // require_orthonormal evidence: V_kᵀV_k = Wmᵀ (B Bᵀ) Wm
    Mat64 T1(c, r, ke), Vg(c, ke, ke), dev(c, 1, 1);
    gemm(c, OP_N, OP_N, r, ke, r, 1.0, Gb.p(), BCUR_F64, Gb.ld, Wm.p(), BCUR_F64, Wm.ld, 0.0, T1.p(), T1.ld);
    gemm(c, OP_T, OP_N, ke, ke, r, 1.0, Wm.p(), BCUR_F64, Wm.ld, T1.p(), BCUR_F64, T1.ld, 0.0, Vg.p(), Vg.ld);
    max_dev_identity(c, Vg.p(), ke, Vg.ld, dev.p());
    d2h_later(c, &out->orth_dev, dev.p(), 1);  // delivered by the caller's next read_all()
    out->k_eff = ke;
    out->l = l;
    out->sigma.assign(sg.begin(), sg.begin() + rank);
    return true;
}

void range_finder(Ctx* c, const DMat* a, int64_t k, int64_t p, int64_t q, uint64_t key, Subspace* out,
                  bool rank_floor, const RoundedA* ra, const std::function<void()>* after_read, bool defer) {
    if (k < 1) fail(BCUR_E_INVALID_ARGUMENT, "range_finder: k must be >= 1");
    if (p < 0 || q < 0) fail(BCUR_E_INVALID_ARGUMENT, "range_finder: p and q must be >= 0");
    static const bool no_fast = getenv("BCUR_RF_SAFE") != nullptr;  // experiments: orth everywhere
    if (no_fast || !range_finder_impl(c, a, k, p, q, key, out, rank_floor, ra, true, after_read)) {
        c->read_all();
        if (after_read && *after_read) (*after_read)();
        range_finder_impl(c, a, k, p, q, key, out, rank_floor, ra, false, nullptr);
    }
    if (!defer) c->read_all();  // out->orth_dev
}

// ------------------------------------------------------------- helpers
static std::vector<int64_t> unique_in_order(const std::vector<int64_t>& v) {
    std::vector<int64_t> out;
    for (int64_t b : v)
        if (std::find(out.begin(), out.end(), b) == out.end()) out.push_back(b);
    return out;
}

// Replicate column block b of A (owned by one rank) as an fp64 rows × w panel.  The block
// travels in its stored dtype (fp32: half the bytes of the fp64 panel) through the host's
// broadcast; without one, as a zero-padded fp64 allreduce.
static void block_panel(Ctx* c, const DMat* a, const Shard& s, int64_t b, double* P) {
    const int64_t w = s.off_global[b + 1] - s.off_global[b];
    const bool mine = b >= s.g0 && b < s.g1;
    if (can_broadcast(c)) {
        const size_t es = dtype_size(a->dtype);
        DevBuf blk(c, (size_t)a->m * w * es);
        if (mine)
            CUDA_CHECK(cudaMemcpy2DAsync(blk.ptr, a->m * es, (const char*)a->ptr + (size_t)(s.off_global[b] - s.col0) * a->ld * es,
                                         a->ld * es, a->m * es, w, cudaMemcpyDeviceToDevice, c->stream));
        broadcast(c, blk.ptr, (int64_t)(a->m * w * es), s.owner[b]);
        convert_to_f64(c, blk.ptr, a->dtype, a->m, w, a->m, P, a->m);
        return;
    }
    if (mine) {
        const size_t es = dtype_size(a->dtype);
        convert_to_f64(c, (const char*)a->ptr + (size_t)(s.off_global[b] - s.col0) * a->ld * es, a->dtype, a->m, w,
                       a->ld, P, a->m);
    } else {
        fill_f64(c, P, a->m * w, 0.0);
    }
    allreduce(c, P, a->m * w);  // broadcast from the owner
}

// Orthonormal basis of the selected (unique, in order) column blocks of A:
// whole-C CholQR2 on the tensor cores for fp32 when safely full rank, else block
// CGS2 panels with per-panel rank revealing (oracle.column_basis).
static void column_basis(Ctx* c, const DMat* a, const Shard& s, const std::vector<int64_t>& blocks,
                         const std::vector<double>& bn2, Basis* B, bool keep_rinv = false,
                         const RoundedA* ra = nullptr) {
    const int64_t m = a->m;
    int64_t cap = 0;
    for (int64_t b : blocks) cap += s.off_global[b + 1] - s.off_global[b];
    bool tried = false;
    // every rank must take the same path: with several ranks, the split path needs the
    // broadcast and the interleaved copy on all of them
    bool split_ok = cap >= 128 && cap <= m && ra && ra->has_lo();
    if (c->comm.world > 1) {
        split_ok = split_ok && can_broadcast(c);
        Mat64 f(c, 1, 1);
        fill_f64(c, f.p(), 1, split_ok ? 1.0 : 0.0);
        allreduce(c, f.p(), 1);
        double h = 0.0;
        d2h(c, &h, f.p(), 1);
        split_ok = h == (double)c->comm.world;
    }
    if (split_ok) {
        // C's 3×FP16 split is a gather of A's interleaved copy (2m halves and one exponent per
        // column): no fp32 C, no split pass.  Several ranks: each block is broadcast by its
        // owner in that form (4 bytes per element, the fp32 size) and C is replicated.
        DevBuf cil(c, (size_t)m * cap * 4), ce(c, (size_t)cap * sizeof(int));
        int64_t at = 0;
        if (c->comm.world <= 1) {  // one launch for every block and its exponents
            std::vector<CopySeg> segs;
            size_t mx = 0;
            for (int64_t b : blocks) {
                const int64_t w = s.off_global[b + 1] - s.off_global[b], j0 = s.off_global[b] - s.col0;
                segs.push_back({ra->il.as<uint16_t>() + (size_t)j0 * 2 * m, cil.as<uint16_t>() + (size_t)at * 2 * m,
                                (size_t)w * m * 4});
                segs.push_back({ra->exps.as<int>() + j0, ce.as<int>() + at, (size_t)w * sizeof(int)});
                mx = std::max(mx, (size_t)w * m * 4);
                at += w;
            }
            DevBuf dsegs(c, segs.size() * sizeof(CopySeg));
            h2d(c, dsegs.as<CopySeg>(), segs.data(), segs.size());
            copy_segments(c, dsegs.as<CopySeg>(), (int)segs.size(), mx);
        }
        else for (int64_t b : blocks) {
            const int64_t w = s.off_global[b + 1] - s.off_global[b], j0 = s.off_global[b] - s.col0;
            uint16_t* dst = cil.as<uint16_t>() + (size_t)at * 2 * m;
            if (b >= s.g0 && b < s.g1) {
                CUDA_CHECK(cudaMemcpyAsync(dst, ra->il.as<uint16_t>() + (size_t)j0 * 2 * m, (size_t)w * m * 4,
                                           cudaMemcpyDeviceToDevice, c->stream));
                CUDA_CHECK(cudaMemcpyAsync(ce.as<int>() + at, ra->exps.as<int>() + j0, (size_t)w * sizeof(int),
                                           cudaMemcpyDeviceToDevice, c->stream));
            }
            broadcast(c, dst, (int64_t)w * m * 4, s.owner[b]);
            broadcast(c, ce.as<int>() + at, (int64_t)w * (int64_t)sizeof(int), s.owner[b]);
            at += w;
        }
        if (cholqr2_whole_h3(c, nullptr, m, cap, false, a->dtype, B, keep_rinv, &cil, &ce)) return;
        tried = true;
    }
    if (cap > 0 && cap <= m && !tried) {  // whole-C CholQR2 first (oracle.column_basis)
        const int cdt = a->dtype;
        const size_t es = dtype_size(cdt);
        DevBuf cf(c, (size_t)m * cap * es);
        int64_t at = 0;
        if (c->comm.world <= 1 && a->ld == m) {  // contiguous blocks: one launch for all of them
            std::vector<CopySeg> segs;
            size_t mx = 0;
            for (int64_t b : blocks) {
                const int64_t w = s.off_global[b + 1] - s.off_global[b];
                segs.push_back({(const char*)a->ptr + (size_t)(s.off_global[b] - s.col0) * a->ld * es,
                                (char*)cf.ptr + (size_t)at * m * es, (size_t)w * m * es});
                mx = std::max(mx, (size_t)w * m * es);
                at += w;
            }
            DevBuf dsegs(c, segs.size() * sizeof(CopySeg));
            h2d(c, dsegs.as<CopySeg>(), segs.data(), segs.size());
            copy_segments(c, dsegs.as<CopySeg>(), (int)segs.size(), mx);
        }
        else for (int64_t b : blocks) {
            const int64_t w = s.off_global[b + 1] - s.off_global[b];
            char* dst = (char*)cf.ptr + (size_t)at * m * es;
            if (c->comm.world <= 1) {
                convert(c, (const char*)a->ptr + (size_t)(s.off_global[b] - s.col0) * a->ld * es, cdt, m, w, a->ld, dst,
                        cdt, m);
            } else {
                Mat64 P(c, m, w);
                block_panel(c, a, s, b, P.p());
                convert(c, P.p(), BCUR_F64, m, w, m, dst, cdt, m);
            }
            at += w;
        }
        if (cholqr2_whole(c, cf.ptr, cdt, m, cap, false, a->dtype, B, keep_rinv)) return;
    }
    B->init(c, a->dtype == BCUR_F32 ? BCUR_F32 : BCUR_F64, m, cap);
    for (int64_t b : blocks) {
        const int64_t w = s.off_global[b + 1] - s.off_global[b];
        Mat64 P(c, m, w);
        block_panel(c, a, s, b, P.p());
        cgs2_append(c, B, P.p(), w, P.ld, std::sqrt(std::max(bn2[b], 0.0)), a->dtype, false);
    }
}

// block_sumsq's fp16 copy of an fp32 A (RoundedA, pipeline.h).  with_lo: the interleaved
// hi/lo form (range finder on 3×FP16) when it fits, else the compact hi copy.
static void make_rounded(Ctx* c, const DMat* a, RoundedA* ra, bool with_lo) {
    if (a->dtype != BCUR_F32 || !h3_ok(a->m) || a->n <= 0 || !umma_ok(a->dtype, a->m, a->ld, a->ptr)) return;
    const size_t one = (size_t)a->m * (size_t)a->n * 2;
    const size_t headroom = (size_t)8 << 30;  // the rest of the pipeline's workspace
    size_t need = with_lo ? 2 * one : one;
    // a cached interleaved-size block is reused for the compact copy too (a block_css and a
    // greedy_select on the same A alternate between the two: re-allocating ~70 GB per call
    // at c5 cost more than every kernel of the step)
    size_t alloc = (!with_lo && c->cached(2 * one)) ? 2 * one : need;
    if (!c->cached(alloc)) {  // first call for this shape (cudaMemGetInfo is not free: not per step)
        size_t freeb = 0, totalb = 0;
        CUDA_CHECK(cudaMemGetInfo(&freeb, &totalb));
        if (need + headroom > freeb + c->pooled_bytes) need = one;  // no room for lo
        if (need + headroom > freeb + c->pooled_bytes) return;      // does not fit: fp32 A paths
        if (need + headroom > freeb) c->trim();                      // make room from the workspace cache
        alloc = need;
    }
    ra->il = DevBuf(c, alloc);
    ra->interleaved = need > one;
    ra->exps = DevBuf(c, (size_t)a->n * sizeof(int));
}
// rows[j] = Σ_c (AᵀX)_jc² over the shard's columns: from the fp16 copy when present
static void rowsq_pass(Ctx* c, const DMat* a, const RoundedA* ra, int64_t N, const void* X, int dtx, int64_t ldx,
                       double* rows, const uint16_t* x16 = nullptr, const int* d_tiles = nullptr, int ntiles = 0) {
    if (ra && ra->ok())
        gemm_rowsumsq_f16(c, a->n, N, a->m, ra->il.as<uint16_t>(), a->m, ra->exps.as<int>(), X, dtx, ldx, rows,
                          ra->interleaved, (x16 && ldx == a->m) ? x16 : nullptr, 14, true, d_tiles, ntiles);
    else
        gemm_rowsumsq(c, OP_T, OP_N, a->n, N, a->m, a->ptr, a->dtype, a->ld, X, dtx, ldx, rows);
}

// Columns whose projection onto the basis is known exactly: the selected blocks themselves (A_g
// lies in span(C) = span(Q), so ‖QᵀA_g‖² = ‖A_g‖², their norms-pass value).  The row-Σ² pass
// skips the 128-column tiles they cover whole (c3: 32 of 512) — for full-rank whole-C bases on
// the CTA-pair path.
struct KnownCols {
    std::vector<int> keep;      // tiles the pass computes
    DevBuf d_keep;
    std::vector<int64_t> cols;  // skipped local column ranges [c0, c1) (pairs)
    double mass = 0.0;          // Σ ‖A_g‖² over the skipped blocks (shard-local)
    bool active() const { return !cols.empty(); }
};
static KnownCols known_columns(Ctx* c, const DMat* a, const Shard& s, const Basis& B,
                               const std::vector<int64_t>& blocks, const std::vector<double>& bn2, const RoundedA* ra) {
    KnownCols k;
    const int64_t nl = a->n, mt = (nl + 127) / 128;
    int64_t width = 0;
    for (int64_t g : blocks) width += s.off_global[g + 1] - s.off_global[g];
    static const bool off = getenv("BCUR_NO_KNOWN_COLS") != nullptr;  // experiments
    if (off || !ra || !ra->ok() || B.rank != width || !rowsq_tiles_ok(nl, B.rank) || !B.x16.ptr) return k;
    std::vector<char> skip(mt, 0);
    for (int64_t g : blocks) {
        if (g < s.g0 || g >= s.g1) continue;
        const int64_t c0 = s.off_global[g] - s.col0, c1 = s.off_global[g + 1] - s.col0;
        if (c0 % 128 != 0 || (c1 - c0) % 128 != 0) continue;  // whole tiles only
        for (int64_t t = c0 / 128; t < c1 / 128; ++t) skip[t] = 1;
        k.cols.push_back(c0);
        k.cols.push_back(c1);
        k.mass += bn2[g];
    }
    if (k.cols.empty()) return k;
    for (int64_t t = 0; t < mt; ++t)
        if (!skip[t]) k.keep.push_back((int)t);
    k.d_keep = DevBuf(c, std::max<size_t>(1, k.keep.size()) * sizeof(int));
    if (!k.keep.empty()) h2d(c, k.d_keep.as<int>(), k.keep.data(), k.keep.size());
    return k;
}

// Σ_g ‖Qᵀ A_g‖² (shard-local per-block values in d_blk_local, allreduced total); with `known`,
// the skipped blocks contribute their exact ‖A_g‖² to the total (not to d_blk_local)
static void projected_mass_later(Ctx* c, const DMat* a, const Shard& s, const Basis& B, double* d_blk_local,
                                 const RoundedA* ra, const KnownCols* known, double* h2);
static double projected_mass(Ctx* c, const DMat* a, const Shard& s, const Basis& B, double* d_blk_local,
                             const RoundedA* ra = nullptr, const KnownCols* known = nullptr) {
    double h[2] = {0.0, 0.0};
    projected_mass_later(c, a, s, B, d_blk_local, ra, known, h);
    c->read_all();
    return h[0] + h[1];
}
// the same, its two parts {Σ‖QᵀA_g‖² computed, known mass} delivered into h2 by c->read_all()
static void projected_mass_later(Ctx* c, const DMat* a, const Shard& s, const Basis& B, double* d_blk_local,
                                 const RoundedA* ra, const KnownCols* known, double* h2) {
    const int64_t nl = a->n;
    Mat64 rows(c, nl, 1), tot(c, 1, 1);
    const bool kn = known && known->active();
    rowsq_pass(c, a, ra, B.rank, B.buf.ptr, B.dt, B.rows, rows.p(), B.x16.as<uint16_t>(),
               kn ? known->d_keep.as<int>() : nullptr, kn ? (int)known->keep.size() : 0);
    Mat64 blk(c, std::max<int64_t>(1, s.g1 - s.g0), 1), tot2(c, 2, 1);
    double* b = d_blk_local ? d_blk_local : blk.p();
    segment_sum(c, rows.p(), s.d_local.as<int64_t>(), s.g1 - s.g0, b);
    sum_vector(c, b, s.g1 - s.g0, tot2.p());
    const double km = kn ? known->mass : 0.0;
    h2d(c, tot2.p() + 1, &km, 1);
    allreduce(c, tot2.p(), 2);
    d2h_later(c, h2, tot2.p(), 2);
}

// First-order correction of the row-Σ² pass's fp16 basis copy along the sketch's top-k
// directions.  The pass reads Q̃ = rn16(Q·2¹⁴)·2⁻¹⁴ (11 significant bits): along a direction u
// that carries a large share of ‖A‖² (the low-rank signal), ‖Q̃ᵀu‖² differs from ‖Qᵀu‖² by a
// random ~2⁻¹¹/√(3m) relative error that does not average out over the columns of A (measured
// 4e-6 of ‖QᵀA‖² at 2048 × 8192; profiles/r02b/diag_rowsq.log).  With U_kΣ_k from the range
// finder (A ≈ U_kΣ_kV_kᵀ + the rest),  Σ_k σ_k²(‖Qᵀu_k‖² − ‖Q̃ᵀu_k‖²)  restores those
// directions; what remains is spread over many directions and averages out (~1e-7).  Two
// thin DMMA products (r × k).
// h2 (delivered by c->read_all()): {‖W_hi + W_lo‖², ‖W_hi‖²}, the correction is h2[0] − h2[1];
// both stay 0 when there is nothing to correct
static void sketch_correction_later(Ctx* c, const Basis& B, const Subspace& sub, const KnownCols* known, double* h2) {
    const int64_t m = B.rows, r = B.rank, ke = sub.k_eff;
    if (r <= 0 || ke <= 0 || !B.x16.ptr || B.dt != BCUR_F32 || !h3_ok(m)) return;
    // W_hi = (UΣ)ᵀQ̃ and W_lo = (UΣ)ᵀΔ from the two parts of the basis's fp16 split (Q̃ = hi,
    // Δ = lo, Q = Q̃ + Δ to 22 bits): 3×FP16 products with UΣ split once, reading only the
    // 2-byte parts — no fp32 copy of Q̃ and no pass over the fp32 Q:
    //   Σ_k σ_k²(‖Qᵀu_k‖² − ‖Q̃ᵀu_k‖²) = ‖W_hi + W_lo‖² − ‖W_hi‖²
    // (W_lo is 2⁻¹¹ of W_hi: the fp64 difference keeps ~13 digits of the correction)
    Mat64 US(c, m, ke), sg(c, ke, 1), W(c, ke, 3 * r), tot(c, 2, 1);
    copy_f64(c, sub.u.p(), m, ke, sub.u.ld, US.p(), US.ld);
    h2d(c, sg.p(), sub.sigma.data(), ke);
    if (known && known->active()) {
        // the pass skipped the known columns (their exact mass is used): only the share
        // 1 − Σ_{j known} v_jk² of each component went through the fp16 basis copy
        Mat64 lev(c, ke, 1), w(c, ke, 1);
        DevBuf dr(c, known->cols.size() * sizeof(int64_t));
        h2d(c, dr.as<int64_t>(), known->cols.data(), known->cols.size());
        colsumsq_ranges(c, sub.v.p(), sub.v.ld, ke, dr.as<int64_t>(), (int)(known->cols.size() / 2), lev.p());
        allreduce(c, lev.p(), ke);
        sigma_weights(c, sg.p(), lev.p(), ke, w.p());
        scale_columns(c, US.p(), m, ke, US.ld, w.p());
    } else {
        scale_columns(c, US.p(), m, ke, US.ld, sg.p());
    }
    DevBuf uil, ue;
    split_il(c, US.p(), BCUR_F64, m, ke, US.ld, &uil, &ue);
    double* blk[3] = {W.p(), W.p() + r * W.ld, W.p() + 2 * r * W.ld};  // W_hi | −W_lo | W_hi + W_lo
    for (int part = 0; part < 2; ++part) {
        F16View xv{B.x16.as<uint16_t>(), nullptr, B.x16e.as<int>(), m, r};
        xv.part = part;
        umma_h3(c, false, uil.as<uint16_t>(), ue.as<int>(), m, ke, xv, part ? -1.0 : 1.0, 0.0, blk[part], W.ld);
    }
    copy_f64(c, blk[0], ke, r, W.ld, blk[2], W.ld);
    axpy_neg(c, blk[1], blk[2], ke * r);
    sumsq_vector(c, blk[2], ke * r, tot.p());  // the blocks are contiguous (ld = ke)
    sumsq_vector(c, blk[0], ke * r, tot.p() + 1);
    d2h_later(c, h2, tot.p(), 2);
}

// ‖A − Q Qᵀ A‖² (streamed: X = QᵀA, then Σ (A − Q X)² tile by tile; blockcur.cpp:46's
// ‖A − C(UR)‖ with C·U·R = P_C A).  fp32 A with its interleaved 3×FP16 copy: both products on
// tcgen05 — X = QᵀA reads that copy as its X operand (no new split of A), the second product
// runs with the subtraction and the square-sum fused into its epilogue (EPI_RESID: A·X never
// stored) — over column chunks of A that bound X to ~1 GB.  Otherwise DMMA fp64.
static double explicit_residual(Ctx* c, const DMat* a, const Basis& B, const RoundedA* ra = nullptr) {
    const int64_t m = a->m, nl = a->n, r = B.rank;
    Mat64 tot(c, 1, 1);
    if (r > 0 && B.dt == BCUR_F32 && a->dtype == BCUR_F32 && ra && ra->has_lo() && h3_ok(m)) {
        DevBuf qil, qe;
        split_il(c, B.buf.ptr, BCUR_F32, m, r, B.rows, &qil, &qe);
        const int64_t nc = std::max<int64_t>(128, std::min<int64_t>(nl, ((int64_t)1 << 30) / (8 * r) / 128 * 128));
        const int64_t nchunks = (nl + nc - 1) / nc;
        Mat64 X(c, r, std::min(nc, nl)), parts(c, nchunks, 1);
        for (int64_t ci = 0; ci < nchunks; ++ci) {
            const int64_t j0 = ci * nc, w = std::min(nc, nl - j0);
            const F16View av{ra->il.as<uint16_t>() + (size_t)j0 * 2 * m, nullptr, ra->exps.as<int>() + j0, m, w};
            umma_h3(c, false, qil.as<uint16_t>(), qe.as<int>(), m, r, av, 1.0, 0.0, X.p(), r);
            umma_h3_resid(c, qil.as<uint16_t>(), qe.as<int>(), m, r, X.p(), BCUR_F64, w, r,
                          (const float*)a->ptr + (size_t)j0 * a->ld, a->ld, parts.p() + ci);
        }
        sum_vector(c, parts.p(), nchunks, tot.p());
        allreduce(c, tot.p(), 1);
        double h = 0.0;
        d2h(c, &h, tot.p(), 1);
        return h;
    }
    Mat64 X(c, std::max<int64_t>(r, 1), nl);
    if (r > 0)
        gemm(c, OP_T, OP_N, r, nl, m, 1.0, B.buf.ptr, B.dt, B.rows, a->ptr, a->dtype, a->ld, 0.0, X.p(), X.ld);
    else
        fill_f64(c, X.p(), nl, 0.0);
    gemm_resid_sumsq(c, OP_N, OP_N, m, nl, std::max<int64_t>(r, 1), B.buf.ptr, B.dt, B.rows, X.p(), BCUR_F64, X.ld,
                     a->ptr, a->dtype, a->ld, tot.p());
    allreduce(c, tot.p(), 1);
    double h = 0.0;
    d2h(c, &h, tot.p(), 1);
    return h;
}

// global per-block ‖A_g‖² (host copy) and ‖A‖²
static void block_norms_later(Ctx* c, const DMat* a, const Shard& s, std::vector<double>* bn2, Mat64* d_global,
                              double* a2, RoundedA* ra = nullptr, bool with_lo = true);
static double block_norms(Ctx* c, const DMat* a, const Shard& s, std::vector<double>* bn2, Mat64* d_global,
                          RoundedA* ra = nullptr, bool with_lo = true) {
    double h = 0.0;
    block_norms_later(c, a, s, bn2, d_global, &h, ra, with_lo);
    c->read_all();
    return h;
}
// the same, *bn2 and *a2 delivered by c->read_all()
static void block_norms_later(Ctx* c, const DMat* a, const Shard& s, std::vector<double>* bn2, Mat64* d_global,
                              double* a2, RoundedA* ra, bool with_lo) {
    Mat64 loc(c, std::max<int64_t>(1, s.g1 - s.g0), 1);
    *d_global = Mat64(c, s.G, 1);
    if (ra) make_rounded(c, a, ra, with_lo);
    const bool f16 = ra && ra->ok();
    block_sumsq(c, a->ptr, a->dtype, a->m, a->ld, s.d_local.as<int64_t>(), s.g1 - s.g0, loc.p(), nullptr, a->m,
                f16 && !ra->interleaved ? ra->il.as<uint16_t>() : nullptr, f16 ? ra->exps.as<int>() : nullptr,
                f16 && ra->interleaved ? ra->il.as<uint16_t>() : nullptr);
    gather_blocks_vec(c, s, loc.p(), d_global->p());
    Mat64 tot(c, 1, 1);
    sum_vector(c, d_global->p(), s.G, tot.p());
    bn2->assign(s.G, 0.0);
    d2h_later(c, bn2->data(), d_global->p(), s.G);
    d2h_later(c, a2, tot.p(), 1);
}

// scores (global G, device) from the shard-local rows of V
static void block_scores(Ctx* c, const Shard& s, const Mat64& v, int64_t nl, double* d_global) {
    Mat64 loc(c, std::max<int64_t>(1, s.g1 - s.g0), 1);
    row_sumsq_blocks(c, v.p(), BCUR_F64, nl, v.n, v.ld, s.d_local.as<int64_t>(), s.g1 - s.g0, nullptr, loc.p());
    gather_blocks_vec(c, s, loc.p(), d_global);
}

static void draw_on_device(Ctx* c, const double* d_scores, int64_t G, int64_t g, int mode, const double* uniforms,
                           std::vector<bcur_block_draw>* draws, std::vector<double>* margins) {
    Mat64 du(c, std::max<int64_t>(g, 1), 1), dm(c, std::max<int64_t>(g, 1), 1);
    DevBuf dd(c, (size_t)std::max<int64_t>(g, 1) * sizeof(bcur_block_draw)), st(c, 16);
    h2d(c, du.p(), uniforms, g);
    distribution_draw(c, d_scores, G, 1, g, mode, du.p(), dd.as<bcur_block_draw>(), dm.p(), st.as<int>());
    int status = 0;
    draws->resize(g);
    margins->resize(g);
    d2h_later(c, &status, st.as<int>(), 1);
    d2h_later(c, draws->data(), dd.as<bcur_block_draw>(), g);
    d2h_later(c, margins->data(), dm.p(), g);
    c->read_all();  // (with the caller's pending reads)
    if (status == BCUR_E_ZERO_MATRIX) fail(BCUR_E_ZERO_MATRIX, "ScoreVector::distribution: scores sum to zero");
    if (status == BCUR_E_DISTRIBUTION_INVALID) fail(BCUR_E_DISTRIBUTION_INVALID, "draw_blocks: invalid distribution");
    if (status == BCUR_E_NOT_ENOUGH_BLOCKS)
        fail(BCUR_E_NOT_ENOUGH_BLOCKS, "draw_blocks: more distinct blocks requested than have positive probability");
    if (status != BCUR_OK) fail(BCUR_E_CUDA, "draw_blocks: kernel status " + std::to_string(status));
}

// ------------------------------------------------------------- block CSS
void block_css(Ctx* c, const DMat* a, const int64_t* offsets, int64_t G, const bcur_options& o, const double* uniforms,
               CssOut* out) {
    if (o.k < 1) fail(BCUR_E_INVALID_ARGUMENT, "block_css: k must be >= 1");
    if (o.g < 1) fail(BCUR_E_INVALID_ARGUMENT, "draw_blocks: g must be >= 1");
    // Host round trips: the range finder's eigenvalues (which also deliver ‖A‖² and the block
    // norms), the draws (with the scores and orth_dev), the basis path decision, the residual.
    ReadScope rs(c);
    std::unique_ptr<ProfScope> ph(new ProfScope(c, "phase:1 norms", 0, 0));
    Shard s = shard_of(a, offsets, G);
    std::vector<double> bn2;
    Mat64 dbn;
    RoundedA ra;
    double a2 = 0.0;
    block_norms_later(c, a, s, &bn2, &dbn, &a2, &ra);
    const std::function<void()> check_a = [&]() {
        if (!std::isfinite(a2)) fail(BCUR_E_INVALID_ARGUMENT, "block_css: matrix contains NaN or Inf");  // require_finite
        if (!(a2 > 0.0)) fail(BCUR_E_ZERO_MATRIX, "block_css: A is identically zero");
    };
    ph.reset(new ProfScope(c, "phase:2 range_finder", 0, 0));
    Subspace sub;
    range_finder(c, a, o.k, o.p, o.q, bcur_omega_key(o.seed), &sub, o.rank_floor != 0, &ra, &check_a, true);
    ph.reset(new ProfScope(c, "phase:3 scores+draw", 0, 0));
    Mat64 sc(c, G, 1);
    block_scores(c, s, sub.v, a->n, sc.p());
    out->scores.resize(G);
    d2h_later(c, out->scores.data(), sc.p(), G);
    out->normalizer = (double)sub.k_eff;
    draw_on_device(c, sc.p(), G, o.g, o.mode, uniforms, &out->draws, &out->margins);
    std::vector<int64_t> blocks;
    for (auto& d : out->draws) blocks.push_back(d.block);
    ph.reset(new ProfScope(c, "phase:4 basis", 0, 0));
    Basis B;
    column_basis(c, a, s, unique_in_order(blocks), bn2, &B, false, &ra);
    ph.reset(new ProfScope(c, "phase:5 residual", 0, 0));
    double res2 = 0.0;
    if (o.residual != BCUR_RESID_EXPLICIT) {  // Pythagoras first (AUTO falls back to explicit when small)
        const KnownCols known = known_columns(c, a, s, B, unique_in_order(blocks), bn2, &ra);
        double pm[2] = {0.0, 0.0}, sk[2] = {0.0, 0.0};  // one read for the pass and its correction
        projected_mass_later(c, a, s, B, nullptr, &ra, &known, pm);
        if (ra.ok() && B.x16.ptr) sketch_correction_later(c, B, sub, &known, sk);
        c->read_all();
        res2 = a2 - (pm[0] + pm[1]) - (sk[0] - sk[1]);
    }
    ph.reset();
    int path = 0;
    if (o.residual == BCUR_RESID_EXPLICIT || (o.residual == BCUR_RESID_AUTO && res2 < theta_explicit(a->dtype) * a2)) {
        res2 = explicit_residual(c, a, B, &ra);
        path = 1;
    }
    out->rep = bcur_report{};
    out->rep.abs_err = std::sqrt(std::max(res2, 0.0));
    out->rep.a_norm = std::sqrt(a2);
    out->rep.rel_err = out->rep.abs_err / out->rep.a_norm;
    out->rep.k_eff = sub.k_eff;
    out->rep.rank_c = B.rank;
    out->rep.residual_path = path;
    out->rep.orth_dev = sub.orth_dev;
}

// ------------------------------------------------------- Algorithm 1 (reference)
// Thin SVD pieces of a small fp64 matrix X (rows × cols) through the Gram of its shorter
// side (eig on the device): σ descending, the rank by rank_tolerance (matcore.cpp:35-49),
// and the singular vectors on the Gram side.  right = true: Gram XᵀX (cols × cols), vectors
// are V; else XXᵀ, vectors are U.
struct SmallSvd {
    Mat64 vec;  // side × rank
    std::vector<double> sigma;
    int64_t rank = 0;
};
static SmallSvd small_svd(Ctx* c, const double* X, int64_t rows, int64_t cols, int64_t ldx, bool right,
                          double tol_override = -1.0) {
    const int64_t w = right ? cols : rows;
    if (w > 512) fail(BCUR_E_INVALID_ARGUMENT, "block_cur: the small SVD side must be <= 512");
    Mat64 Gm(c, w, w), lam(c, w, 1), V(c, w, w);
    if (right)
        gemm(c, OP_T, OP_N, w, w, rows, 1.0, X, BCUR_F64, ldx, X, BCUR_F64, ldx, 0.0, Gm.p(), Gm.ld);
    else
        gemm(c, OP_N, OP_T, w, w, cols, 1.0, X, BCUR_F64, ldx, X, BCUR_F64, ldx, 0.0, Gm.p(), Gm.ld);
    sym_eig(c, Gm.p(), w, Gm.ld, lam.p(), V.p());
    std::vector<double> lh(w);
    d2h(c, lh.data(), lam.p(), w);
    SmallSvd out;
    for (double l : lh) out.sigma.push_back(std::sqrt(std::max(l, 0.0)));
    const double tol = tol_override >= 0.0 ? tol_override
                       : out.sigma.empty() ? 0.0 : 1e-12 * (double)std::max(rows, cols) * out.sigma[0];
    while (out.rank < w && out.sigma[out.rank] > tol && out.sigma[out.rank] > 0.0) ++out.rank;
    out.vec = Mat64(c, w, std::max<int64_t>(out.rank, 1));
    if (out.rank > 0) copy_f64(c, V.p(), w, out.rank, V.ld, out.vec.p(), out.vec.ld);
    return out;
}

// X⁺ (cols × rows) of a small fp64 X and its numerical rank (matcore.cpp:85-91).  Full rank
// (the usual case): CholQR2 of X's tall orientation, tall = Q·T, so X⁺ = T⁻¹·Qᵀ (X tall) or
// Q·T⁻ᵀ (Xᵀ tall) — forward error ~u·κ(X).  Otherwise the Gram of the shorter side with the
// reference's rank rule (error ~u·κ(X)² on the kept range).
// tol_scale: the rank cut is tol_scale·σ₁ (default 1e-12·max(rows, cols), matcore.cpp:35-37)
static int64_t pinv_small(Ctx* c, const double* Xp, int64_t rows, int64_t cols, int64_t ldx, Mat64* out,
                          double tol_scale = -1.0) {
    *out = Mat64(c, cols, rows);
    const bool right = cols <= rows;
    {
        const int64_t tall = std::max(rows, cols), wide = std::min(rows, cols);
        Mat64 X(c, tall, wide), Q(c, tall, wide), T;
        if (right) copy_f64(c, Xp, rows, cols, ldx, X.p(), X.ld);
        else transpose(c, Xp, BCUR_F64, rows, cols, ldx, X.p(), BCUR_F64, X.ld);
        int path = -1;
        const int64_t got = orth(c, X.p(), tall, wide, X.ld, -1.0, BCUR_F64, Q.p(), Q.ld, false, &T, &path);
        if (path == 0 && got == wide && T.m == wide && T.n == wide) {
            Mat64 Ti(c, wide, wide);
            tri_inv_any(c, T.p(), wide, Ti.p(), nullptr);
            if (right)
                gemm(c, OP_N, OP_T, cols, rows, cols, 1.0, Ti.p(), BCUR_F64, Ti.ld, Q.p(), BCUR_F64, Q.ld, 0.0,
                     out->p(), out->ld);
            else
                gemm(c, OP_N, OP_T, cols, rows, rows, 1.0, Q.p(), BCUR_F64, Q.ld, Ti.p(), BCUR_F64, Ti.ld, 0.0,
                     out->p(), out->ld);
            return wide;
        }
    }
    SmallSvd sw = small_svd(c, Xp, rows, cols, ldx, right);
    if (tol_scale >= 0.0 && !sw.sigma.empty()) {  // re-cut with the caller's tolerance
        const double tol = tol_scale * sw.sigma[0];
        int64_t k = 0;
        while (k < (int64_t)sw.sigma.size() && sw.sigma[k] > tol && sw.sigma[k] > 0.0) ++k;
        sw.rank = std::min<int64_t>(k, sw.vec.n);
    }
    if (sw.rank == 0) {
        fill_f64(c, out->p(), cols * rows, 0.0);
        return 0;
    }
    const int64_t rw = sw.rank, side = right ? cols : rows;
    std::vector<double> inv2(rw);
    for (int64_t i = 0; i < rw; ++i) inv2[i] = 1.0 / (sw.sigma[i] * sw.sigma[i]);
    Mat64 d2(c, rw, 1), Vs(c, side, rw), P(c, side, side);
    h2d(c, d2.p(), inv2.data(), rw);
    copy_f64(c, sw.vec.p(), side, rw, sw.vec.ld, Vs.p(), Vs.ld);
    scale_columns(c, Vs.p(), side, rw, Vs.ld, d2.p());
    gemm(c, OP_N, OP_T, side, side, rw, 1.0, Vs.p(), BCUR_F64, Vs.ld, sw.vec.p(), BCUR_F64, sw.vec.ld, 0.0, P.p(), P.ld);
    if (right)  // X⁺ = (XᵀX)⁺ Xᵀ
        gemm(c, OP_N, OP_T, cols, rows, cols, 1.0, P.p(), BCUR_F64, P.ld, Xp, BCUR_F64, ldx, 0.0, out->p(), out->ld);
    else        // X⁺ = Xᵀ (XXᵀ)⁺
        gemm(c, OP_T, OP_N, cols, rows, rows, 1.0, Xp, BCUR_F64, ldx, P.p(), BCUR_F64, P.ld, 0.0, out->p(), out->ld);
    return rw;
}

void block_cur_alg1(Ctx* c, const DMat* a, const int64_t* offsets, int64_t G, int64_t k, const bcur_row_draw* rows,
                    int64_t r, bool scaled_rows, int64_t g, int block_mode, const double* uniforms, Alg1Out* out) {
    const int64_t m = a->m, n = a->n;
    if (c->comm.world > 1) fail(BCUR_E_INVALID_ARGUMENT, "block_cur (Algorithm 1): single device");
    if (k < 1 || k > std::min(m, n)) fail(BCUR_E_INVALID_ARGUMENT, "block_cur: need 1 <= k <= min(m, n)");
    if (r < 1 || g < 1) fail(BCUR_E_INVALID_ARGUMENT, "block_cur: r and g must be >= 1");
    Shard s = shard_of(a, offsets, G);
    std::vector<double> bn2;
    Mat64 dbn;
    const double a2 = block_norms(c, a, s, &bn2, &dbn);
    if (!std::isfinite(a2)) fail(BCUR_E_INVALID_ARGUMENT, "block_cur: matrix contains NaN or Inf");
    // R = the drawn rows (materialize_rows, sampler.cpp:186-202): unit row blocks of A
    for (int64_t t = 0; t < r; ++t)
        if (rows[t].row < 0 || rows[t].row >= m) fail(BCUR_E_DIMENSION_MISMATCH, "materialize_rows: row index out of range");
    Mat64 R(c, r, n);
    {
        std::vector<int64_t> unit(m + 1), dst(r);
        for (int64_t i = 0; i <= m; ++i) unit[i] = i;
        std::vector<bcur_block_draw> dr(r);
        for (int64_t t = 0; t < r; ++t) {
            dr[t] = {rows[t].row, rows[t].probability, scaled_rows ? rows[t].scale : 1.0};
            dst[t] = t;
        }
        DevBuf du(c, unit.size() * sizeof(int64_t)), dd(c, dr.size() * sizeof(bcur_block_draw)), ds(c, r * sizeof(int64_t));
        h2d(c, du.as<int64_t>(), unit.data(), unit.size());
        h2d(c, dd.as<bcur_block_draw>(), dr.data(), dr.size());
        h2d(c, ds.as<int64_t>(), dst.data(), dst.size());
        gather_blocks(c, a->ptr, a->dtype, m, n, a->ld, du.as<int64_t>(), dd.as<bcur_block_draw>(), ds.as<int64_t>(), r, 1,
                      1, R.p(), BCUR_F64, R.ld);
    }
    // approximate block leverage of R (leverage.cpp:155-164): all rank(R) right singular
    // vectors.  The row space and rank of R are those of its distinct rows (a row drawn
    // twice with replacement is an exact copy); the Gram of the distinct rows cannot show
    // the copies' zero singular values as rounding-level ones (~1e-8·σ₁ through a Gram,
    // above the 1e-12·max(r, n)·σ₁ rank cut).  σ₁ of the cut is R's own.
    std::vector<int64_t> urow;
    for (int64_t t = 0; t < r; ++t)
        if (std::find(urow.begin(), urow.end(), rows[t].row) == urow.end()) urow.push_back(rows[t].row);
    const int64_t ru = (int64_t)urow.size();
    Mat64 Ru(c, ru, n);
    {
        std::vector<int64_t> unit(m + 1), dst(ru);
        for (int64_t i = 0; i <= m; ++i) unit[i] = i;
        std::vector<bcur_block_draw> dr(ru);
        for (int64_t t = 0; t < ru; ++t) {
            dr[t] = {urow[t], 0.0, scaled_rows ? rows[0].scale : 1.0};
            dst[t] = t;
        }
        DevBuf du(c, unit.size() * sizeof(int64_t)), dd(c, dr.size() * sizeof(bcur_block_draw)), ds(c, ru * sizeof(int64_t));
        h2d(c, du.as<int64_t>(), unit.data(), unit.size());
        h2d(c, dd.as<bcur_block_draw>(), dr.data(), dr.size());
        h2d(c, ds.as<int64_t>(), dst.data(), dst.size());
        gather_blocks(c, a->ptr, a->dtype, m, n, a->ld, du.as<int64_t>(), dd.as<bcur_block_draw>(), ds.as<int64_t>(), ru,
                      1, 1, Ru.p(), BCUR_F64, Ru.ld);
    }
    double sigma1 = 0.0;
    {
        Mat64 Gr(c, r, r), lam(c, r, 1), Vr(c, r, r);
        gemm(c, OP_N, OP_T, r, r, n, 1.0, R.p(), BCUR_F64, R.ld, R.p(), BCUR_F64, R.ld, 0.0, Gr.p(), Gr.ld);
        sym_eig(c, Gr.p(), r, Gr.ld, lam.p(), Vr.p());
        double l0 = 0.0;
        d2h(c, &l0, lam.p(), 1);
        sigma1 = std::sqrt(std::max(l0, 0.0));
    }
    SmallSvd sr = small_svd(c, Ru.p(), ru, n, Ru.ld, false, 1e-12 * (double)std::max(r, n) * sigma1);
    if (sr.rank == 0 || !(sigma1 > 0.0))  // R·Rᵀ = 0 ⇔ R = 0 (blockcur.cpp:94-96)
        fail(BCUR_E_DEGENERATE_R, "block_cur: sampled row matrix R is identically zero");
    const int64_t rk = sr.rank;
    Mat64 V(c, n, rk), Vraw(c, n, rk), Ws(c, ru, rk), dinv(c, rk, 1), sc(c, G, 1);
    {
        std::vector<double> inv(rk);
        for (int64_t i = 0; i < rk; ++i) inv[i] = 1.0 / sr.sigma[i];
        h2d(c, dinv.p(), inv.data(), rk);
        copy_f64(c, sr.vec.p(), ru, rk, sr.vec.ld, Ws.p(), Ws.ld);
        scale_columns(c, Ws.p(), ru, rk, Ws.ld, dinv.p());
        gemm(c, OP_T, OP_N, n, rk, ru, 1.0, Ru.p(), BCUR_F64, Ru.ld, Ws.p(), BCUR_F64, Ws.ld, 0.0, Vraw.p(), Vraw.ld);
        // Rᵀ·Ũ·Σ⁻¹ carries the Gram's κ(R)² error in its orthonormality, not in its span (the
        // row space): CholQR2 of it gives the right-singular subspace to fp64 accuracy, and
        // block leverage depends on the subspace only
        const int64_t got = orth(c, Vraw.p(), n, rk, Vraw.ld, -1.0, BCUR_F64, V.p(), V.ld, false, nullptr, nullptr);
        if (got != rk) {
            std::string sv;
            for (int64_t i = 0; i < (int64_t)sr.sigma.size(); ++i) sv += " " + std::to_string(sr.sigma[i]);
            fail(BCUR_E_ITERATION_FAILURE, "block_cur: row-space basis lost rank (" + std::to_string(got) + " of " +
                                               std::to_string(rk) + "; sigma" + sv + ")");
        }
    }
    block_scores(c, s, V, n, sc.p());
    out->scores.resize(G);
    d2h(c, out->scores.data(), sc.p(), G);
    out->normalizer = (double)rk;
    draw_on_device(c, sc.p(), G, g, block_mode, uniforms, &out->draws, &out->margins);
    // C = A·S (m × cc), scaled (materialize_columns); W = R·S enters through its distinct part
    int64_t cc = 0;
    std::vector<int64_t> dst;
    for (auto& d : out->draws) {
        dst.push_back(cc);
        cc += offsets[d.block + 1] - offsets[d.block];
    }
    Mat64 C(c, m, cc);
    {
        DevBuf dd(c, out->draws.size() * sizeof(bcur_block_draw)), ds(c, dst.size() * sizeof(int64_t));
        h2d(c, dd.as<bcur_block_draw>(), out->draws.data(), out->draws.size());
        h2d(c, ds.as<int64_t>(), dst.data(), dst.size());
        gather_blocks(c, a->ptr, a->dtype, m, n, a->ld, s.d_local.as<int64_t>(), dd.as<bcur_block_draw>(),
                      ds.as<int64_t>(), g, 0, 1, C.p(), BCUR_F64, C.ld);
    }
    // U = W⁺ (matcore.cpp:85-91).  W's repeated rows (a row drawn twice) and repeated column
    // blocks (a block drawn twice with replacement) are exact copies: W = P·W_u·Qᵀ with P, Q
    // 0/1 selections.  With D_r, D_c the multiplicities, P·D_r^-½ and Q·D_c^-½ have orthonormal
    // columns, so W = (P·D_r^-½)·X·(Q·D_c^-½)ᵀ with X = D_r^½·W_u·D_c^½ and, exactly,
    // W⁺ = Q·D_c^-½ · X⁺ · D_r^-½·Pᵀ — same singular values, same rank rule.  (A Gram of W
    // itself would show the copies' zero singular values as ~1e-8·σ₁ ones.)
    std::vector<int64_t> ublk;
    for (auto& d : out->draws)
        if (std::find(ublk.begin(), ublk.end(), d.block) == ublk.end()) ublk.push_back(d.block);
    int64_t cu = 0;
    std::vector<int64_t> ustart;
    for (int64_t b : ublk) {
        ustart.push_back(cu);
        cu += offsets[b + 1] - offsets[b];
    }
    Mat64 Wu(c, ru, cu);
    {
        std::vector<bcur_block_draw> ud;
        for (int64_t b : ublk)
            for (auto& d : out->draws)
                if (d.block == b) {
                    ud.push_back(d);
                    break;
                }
        DevBuf dd(c, ud.size() * sizeof(bcur_block_draw)), ds(c, ustart.size() * sizeof(int64_t));
        h2d(c, dd.as<bcur_block_draw>(), ud.data(), ud.size());
        h2d(c, ds.as<int64_t>(), ustart.data(), ustart.size());
        gather_blocks(c, Ru.p(), BCUR_F64, ru, n, Ru.ld, s.d_local.as<int64_t>(), dd.as<bcur_block_draw>(),
                      ds.as<int64_t>(), (int64_t)ud.size(), 0, 1, Wu.p(), BCUR_F64, Wu.ld);
    }
    std::vector<double> mrow(ru, 0.0), mcol(cu, 0.0);
    for (int64_t t = 0; t < r; ++t) mrow[std::find(urow.begin(), urow.end(), rows[t].row) - urow.begin()] += 1.0;
    for (auto& d : out->draws) {
        const int64_t ui = std::find(ublk.begin(), ublk.end(), d.block) - ublk.begin();
        for (int64_t x = 0; x < offsets[d.block + 1] - offsets[d.block]; ++x) mcol[ustart[ui] + x] += 1.0;
    }
    {
        std::vector<double> sr_(ru), sc_(cu);
        for (int64_t i = 0; i < ru; ++i) sr_[i] = std::sqrt(mrow[i]);
        for (int64_t j = 0; j < cu; ++j) sc_[j] = std::sqrt(mcol[j]);
        Mat64 dr(c, ru, 1), dc(c, cu, 1);
        h2d(c, dr.p(), sr_.data(), ru);
        h2d(c, dc.p(), sc_.data(), cu);
        scale_rows(c, Wu.p(), ru, cu, Wu.ld, dr.p());
        scale_columns(c, Wu.p(), ru, cu, Wu.ld, dc.p());
    }
    Mat64 Wup;  // X⁺ (cu × ru), rank cut of W's own shape
    out->rep.rank_w = pinv_small(c, Wu.p(), ru, cu, Wu.ld, &Wup, 1e-12 * (double)std::max(r, cc));
    out->u = Mat64(c, cc, r);
    {
        // Qs (cc × cu): column j of C → its distinct column, weight 1/multiplicity of its block;
        // Ps (ru × r): distinct row u → drawn row t, weight 1/multiplicity of the row
        std::vector<double> qs((size_t)cc * cu, 0.0), ps((size_t)ru * r, 0.0);
        int64_t j = 0;
        for (auto& d : out->draws) {
            const int64_t w = offsets[d.block + 1] - offsets[d.block];
            const int64_t ui = std::find(ublk.begin(), ublk.end(), d.block) - ublk.begin();
            for (int64_t x = 0; x < w; ++x, ++j)
                qs[(size_t)j + (size_t)(ustart[ui] + x) * cc] = 1.0 / std::sqrt(mcol[ustart[ui] + x]);
        }
        for (int64_t t = 0; t < r; ++t) {
            const int64_t ui = std::find(urow.begin(), urow.end(), rows[t].row) - urow.begin();
            ps[(size_t)ui + (size_t)t * ru] = 1.0 / std::sqrt(mrow[ui]);
        }
        Mat64 Qs(c, cc, cu), Ps(c, ru, r), T(c, cu, r);
        h2d(c, Qs.p(), qs.data(), qs.size());
        h2d(c, Ps.p(), ps.data(), ps.size());
        gemm(c, OP_N, OP_N, cu, r, ru, 1.0, Wup.p(), BCUR_F64, Wup.ld, Ps.p(), BCUR_F64, Ps.ld, 0.0, T.p(), T.ld);
        gemm(c, OP_N, OP_N, cc, r, cu, 1.0, Qs.p(), BCUR_F64, Qs.ld, T.p(), BCUR_F64, T.ld, 0.0, out->u.p(),
             out->u.ld);
    }
    // ‖A − C (U R)‖_F explicitly (error_report, blockcur.cpp:33-52), for U and U_k
    auto resid = [&](const Mat64& U) {
        Mat64 X(c, cc, n), tot(c, 1, 1);
        gemm(c, OP_N, OP_N, cc, n, r, 1.0, U.p(), BCUR_F64, U.ld, R.p(), BCUR_F64, R.ld, 0.0, X.p(), X.ld);
        gemm_resid_sumsq(c, OP_N, OP_N, m, n, cc, C.p(), BCUR_F64, C.ld, X.p(), BCUR_F64, X.ld, a->ptr, a->dtype, a->ld,
                         tot.p());
        double h = 0.0;
        d2h(c, &h, tot.p(), 1);
        return std::sqrt(std::max(h, 0.0));
    };
    out->rep.abs_err_u = resid(out->u);
    // U_k = best_rank_k(U, k) = U·V_k·V_kᵀ with V_k the top-k right singular vectors of U
    {
        SmallSvd su = small_svd(c, out->u.p(), cc, r, out->u.ld, true);
        const int64_t kk = std::min<int64_t>(k, su.rank);
        Mat64 Uk(c, cc, r);
        if (kk == 0) {
            fill_f64(c, Uk.p(), cc * r, 0.0);
        } else {
            Mat64 Pk(c, r, r);
            gemm(c, OP_N, OP_T, r, r, kk, 1.0, su.vec.p(), BCUR_F64, su.vec.ld, su.vec.p(), BCUR_F64, su.vec.ld, 0.0,
                 Pk.p(), Pk.ld);
            gemm(c, OP_N, OP_N, cc, r, r, 1.0, out->u.p(), BCUR_F64, out->u.ld, Pk.p(), BCUR_F64, Pk.ld, 0.0, Uk.p(),
                 Uk.ld);
        }
        out->rep.abs_err_uk = resid(Uk);
    }
    out->rep.a_norm = std::sqrt(a2);
    out->rep.rank_r = rk;
}

// ---------------------------------------------------------------- greedy
void greedy_select(Ctx* c, const DMat* a, const int64_t* offsets, int64_t G, const bcur_options& o, GreedyOut* out) {
    if (o.g < 1 || o.g > G) fail(BCUR_E_INVALID_ARGUMENT, "greedy_select: need 1 <= g <= number of blocks");
    Shard s = shard_of(a, offsets, G);
    std::vector<double> bn2;
    Mat64 res;
    RoundedA ra;
    // res starts as ‖A_g‖²; the greedy scores need only hi (compact copy: half the bytes per pass)
    const double a2 = block_norms(c, a, s, &bn2, &res, &ra, false);
    if (!std::isfinite(a2)) fail(BCUR_E_INVALID_ARGUMENT, "greedy_select: matrix contains NaN or Inf");  // require_finite
    if (!(a2 > 0.0)) fail(BCUR_E_ZERO_MATRIX, "greedy_select: A is identically zero");
    const int dt = a->dtype;
    const int64_t m = a->m;
    int64_t cap = 0;
    {
        std::vector<int64_t> w(G);
        for (int64_t g = 0; g < G; ++g) w[g] = offsets[g + 1] - offsets[g];
        std::sort(w.begin(), w.end(), std::greater<int64_t>());
        for (int64_t t = 0; t < o.g; ++t) cap += w[t];
    }
    Basis B;
    B.init(c, dt == BCUR_F32 ? BCUR_F32 : BCUR_F64, m, cap);
    B.enable_h3(c);
    DevBuf sel(c, (size_t)G);
    CUDA_CHECK(cudaMemsetAsync(sel.ptr, 0, G, c->stream));
    DevBuf didx(c, 64);
    Mat64 lev;
    bool have_lev = false;
    Mat64 loc(c, std::max<int64_t>(1, s.g1 - s.g0), 1), upd(c, G, 1), rows(c, a->n, 1);
    out->steps.clear();
    // Once the basis spans all m rows nothing can be added and no residual changes: a step that is
    // saturated then stays saturated (the maximum runs over fewer blocks), so such steps reduce to
    // the leverage argmax — one host read each — with the frozen residuals read once.  (c2, m = 64:
    // seven of its eight steps; each used to run the two CGS2 passes, a Gram and a 100-wide
    // Cholesky to find rank 0, ~185 µs and three reads per step: profiles/r02ax/step_c2.txt.)
    bool frozen = false;
    std::vector<double> res_frozen, picks;
    int64_t pick0 = 0;
    for (int64_t t = 0; t < o.g; ++t) {
        struct { int64_t idx; double v1, v2; } hm;
        bcur_greedy_step st{};
        if (!frozen) {
            argmax_masked(c, res.p(), sel.as<unsigned char>(), G, didx.as<int64_t>(), didx.as<double>() + 1);
            d2h(c, reinterpret_cast<char*>(&hm), reinterpret_cast<const char*>(didx.ptr), 24);
            st.block = hm.idx;
            st.score = hm.v1;
            st.margin = hm.v1 - hm.v2;
            st.saturated = hm.v1 <= tau_saturate(dt) * a2 ? 1 : 0;
        } else {
            st.saturated = 1;
        }
        if (frozen) {
            if (picks.empty()) {  // every remaining pick in one launch and one read
                const int count = (int)(o.g - t);
                Mat64 dp(c, 3, count);
                argmax_masked_seq(c, lev.p(), sel.as<unsigned char>(), G, count, dp.p());
                picks.resize((size_t)3 * count);
                d2h(c, picks.data(), dp.p(), picks.size());
                pick0 = t;
            }
            const double* pk = picks.data() + 3 * (t - pick0);
            st.block = (int64_t)pk[0];
            st.margin = pk[1] - pk[2];
            st.score = res_frozen[st.block];
            st.rank_added = 0;
            out->steps.push_back(st);
            continue;  // (sel was updated on the device; nothing is added and no residual changes)
        } else if (st.saturated) {
            if (!have_lev) {
                Subspace sub;
                range_finder(c, a, o.k, o.p, o.q, bcur_omega_key(o.seed), &sub, o.rank_floor != 0);
                lev = Mat64(c, G, 1);
                block_scores(c, s, sub.v, a->n, lev.p());
                have_lev = true;
            }
            argmax_masked(c, lev.p(), sel.as<unsigned char>(), G, didx.as<int64_t>(), didx.as<double>() + 1);
            d2h(c, reinterpret_cast<char*>(&hm), reinterpret_cast<const char*>(didx.ptr), 24);
            st.block = hm.idx;
            st.margin = hm.v1 - hm.v2;
            double rv = 0.0;
            d2h(c, &rv, res.p() + hm.idx, 1);
            st.score = rv;
        }
        const int64_t b = st.block;
        const unsigned char one = 1;
        h2d(c, sel.as<unsigned char>() + b, &one, 1);
        const int64_t w = offsets[b + 1] - offsets[b];
        const int64_t cur = B.rank;
        int64_t r = 0;
        if (B.rank < m) {  // (a basis of all m rows: every further panel has rank 0 against it)
            Mat64 P(c, m, w);
            block_panel(c, a, s, b, P.p());
            r = cgs2_append(c, &B, P.p(), w, P.ld, std::sqrt(std::max(bn2[b], 0.0)), dt, false);
        }
        if (r > 0) {
            // res_g −= ‖Q_newᵀ A_g‖²
            rowsq_pass(c, a, &ra, r, B.col(cur), B.dt, B.rows, rows.p());
            segment_sum(c, rows.p(), s.d_local.as<int64_t>(), s.g1 - s.g0, loc.p());
            gather_blocks_vec(c, s, loc.p(), upd.p());
            axpy_neg(c, upd.p(), res.p(), G);
        }
        if (st.saturated && B.rank >= m && have_lev && !frozen) {  // (after this step's update, if any)
            frozen = true;
            res_frozen.resize(G);
            d2h(c, res_frozen.data(), res.p(), G);
        }
        st.rank_added = r;
        out->steps.push_back(st);
    }
    out->residuals.resize(G);
    d2h(c, out->residuals.data(), res.p(), G);
    Mat64 tot(c, 1, 1);
    sum_vector(c, res.p(), G, tot.p());
    double res2 = 0.0;
    d2h(c, &res2, tot.p(), 1);
    int path = 0;
    if (o.residual == BCUR_RESID_EXPLICIT || (o.residual == BCUR_RESID_AUTO && res2 < theta_explicit(dt) * a2)) {
        res2 = explicit_residual(c, a, B);
        path = 1;
    }
    out->rep = bcur_report{};
    out->rep.abs_err = std::sqrt(std::max(res2, 0.0));
    out->rep.a_norm = std::sqrt(a2);
    out->rep.rel_err = out->rep.abs_err / out->rep.a_norm;
    out->rep.rank_c = B.rank;
    out->rep.residual_path = path;
}

// ------------------------------------------------------------ block CUR
void block_cur(Ctx* c, const DMat* a, const int64_t* coff, int64_t Gc, const int64_t* roff, int64_t Gr,
               const bcur_options& o, const double* uniforms, bool want_u, CurOut* out) {
    const int64_t m = a->m, nl = a->n;
    const int dt = a->dtype;
    const int bdt = dt == BCUR_F32 ? BCUR_F32 : BCUR_F64;
    const bool dist = c->comm.world > 1;
    if (o.g < 1 || o.g_rows < 1) fail(BCUR_E_INVALID_ARGUMENT, "block_cur: g and g_rows must be >= 1");
    if (Gr < 1 || roff[0] != 0 || roff[Gr] != m) fail(BCUR_E_DIMENSION_MISMATCH, "block_cur: row partition does not match A");
    Shard s = shard_of(a, coff, Gc);
    std::vector<double> bn2;
    Mat64 dbn;
    RoundedA ra;
    const double a2 = block_norms(c, a, s, &bn2, &dbn, &ra);
    if (!std::isfinite(a2)) fail(BCUR_E_INVALID_ARGUMENT, "block_cur: matrix contains NaN or Inf");  // require_finite
    if (!(a2 > 0.0)) fail(BCUR_E_ZERO_MATRIX, "block_cur: A is identically zero");
    Subspace sub;
    range_finder(c, a, o.k, o.p, o.q, bcur_omega_key(o.seed), &sub, o.rank_floor != 0, &ra);
    Mat64 csc(c, Gc, 1), rsc(c, Gr, 1);
    block_scores(c, s, sub.v, nl, csc.p());
    DevBuf droff(c, (Gr + 1) * sizeof(int64_t));
    h2d(c, droff.as<int64_t>(), roff, Gr + 1);
    row_sumsq_blocks(c, sub.u.p(), BCUR_F64, m, sub.u.n, sub.u.ld, droff.as<int64_t>(), Gr, nullptr, rsc.p());
    out->col_scores.resize(Gc);
    out->row_scores.resize(Gr);
    d2h(c, out->col_scores.data(), csc.p(), Gc);
    d2h(c, out->row_scores.data(), rsc.p(), Gr);
    std::vector<double> mc, mr;
    draw_on_device(c, csc.p(), Gc, o.g, o.mode, uniforms, &out->col_draws, &mc);
    draw_on_device(c, rsc.p(), Gr, o.g_rows, o.mode, uniforms + o.g, &out->row_draws, &mr);
    std::vector<int64_t> cb, rb;
    for (auto& d : out->col_draws) cb.push_back(d.block);
    for (auto& d : out->row_draws) rb.push_back(d.block);
    cb = unique_in_order(cb);
    rb = unique_in_order(rb);
    // Q_C (m × rc), replicated
    Basis QC;
    column_basis(c, a, s, cb, bn2, &QC, want_u, &ra);
    // Q_R (n_local × rr): basis of the selected row blocks of A (column blocks of Aᵀ),
    // row-distributed over ranks.  Rᵀ_u = unscaled selected rows, transposed.
    int64_t ru = 0;
    std::vector<int64_t> dst_u;
    for (int64_t h : rb) { dst_u.push_back(ru); ru += roff[h + 1] - roff[h]; }
    DevBuf rtu(c, (size_t)nl * std::max<int64_t>(ru, 1) * dtype_size(bdt));
    {
        std::vector<bcur_block_draw> dr;
        for (int64_t h : rb) dr.push_back({h, 0.0, 1.0});
        DevBuf dd(c, dr.size() * sizeof(bcur_block_draw)), dds(c, dst_u.size() * sizeof(int64_t));
        h2d(c, dd.as<bcur_block_draw>(), dr.data(), dr.size());
        h2d(c, dds.as<int64_t>(), dst_u.data(), dst_u.size());
        DevBuf rr_(c, (size_t)std::max<int64_t>(ru, 1) * nl * dtype_size(bdt));
        gather_blocks(c, a->ptr, dt, m, nl, a->ld, droff.as<int64_t>(), dd.as<bcur_block_draw>(), dds.as<int64_t>(),
                      (int64_t)dr.size(), 1, 0, rr_.ptr, bdt, ru);
        transpose(c, rr_.ptr, bdt, ru, nl, ru, rtu.ptr, bdt, nl);
    }
    std::vector<double> rbn2(Gr, 0.0);
    {
        // ‖A_h‖² for the selected row blocks, from the columns of Rᵀ_u (allreduced over shards)
        std::vector<int64_t> lo(dst_u);
        lo.push_back(ru);
        DevBuf dlo(c, lo.size() * sizeof(int64_t));
        h2d(c, dlo.as<int64_t>(), lo.data(), lo.size());
        Mat64 t(c, std::max<int64_t>((int64_t)rb.size(), 1), 1);
        block_sumsq(c, rtu.ptr, bdt, nl, nl, dlo.as<int64_t>(), (int64_t)rb.size(), t.p());
        allreduce(c, t.p(), (int64_t)rb.size());
        std::vector<double> th(rb.size());
        d2h(c, th.data(), t.p(), rb.size());
        for (size_t i = 0; i < rb.size(); ++i) rbn2[rb[i]] = th[i];
    }
    Basis QR;
    bool whole = false;
    if (ru > 0) whole = cholqr2_whole(c, rtu.ptr, bdt, nl, ru, dist, dt, &QR, want_u);
    if (!whole) {
        QR.init(c, bdt, nl, ru);
        for (size_t i = 0; i < rb.size(); ++i) {
            const int64_t h = rb[i], w = roff[h + 1] - roff[h];
            Mat64 P(c, nl, w);
            convert(c, (const char*)rtu.ptr + (size_t)dst_u[i] * nl * dtype_size(bdt), bdt, nl, w, nl, P.p(),
                    BCUR_F64, P.ld);
            cgs2_append(c, &QR, P.p(), w, P.ld, std::sqrt(std::max(rbn2[h], 0.0)), dt, dist);
        }
    }
    out->rank_r = QR.rank;
    const int64_t rc = QC.rank, rr = QR.rank;
    // M = Q_Cᵀ A Q_R:  Xᵀ = A_sᵀ Q_C (n_local × rc), Mᵀ = Σ_s Q_R,sᵀ Xᵀ (rr × rc)
    Mat64 Xt(c, nl, std::max<int64_t>(rc, 1)), Mt(c, std::max<int64_t>(rr, 1), std::max<int64_t>(rc, 1));
    Mat64 M(c, std::max<int64_t>(rc, 1), std::max<int64_t>(rr, 1));
    // one-accumulator product (~1e-6 relative, against U's 1e-4 and the error's ~1e-7 here)
    a_product(c, a, &ra, true, rc, QC.buf.ptr, QC.dt, QC.rows, Xt.p(), Xt.ld, GEMM_FAST_ACC);
    gemm(c, OP_T, OP_N, rr, rc, nl, 1.0, QR.buf.ptr, QR.dt, QR.rows, Xt.p(), BCUR_F64, Xt.ld, 0.0, Mt.p(), Mt.ld);
    allreduce(c, Mt.p(), rr * rc);
    transpose(c, Mt.p(), BCUR_F64, rr, rc, Mt.ld, M.p(), BCUR_F64, M.ld);
    Mat64 tot(c, 1, 1);
    {
        Mat64 rows2(c, std::max<int64_t>(rc, 1), 1);
        row_sumsq_blocks(c, M.p(), BCUR_F64, rc, rr, M.ld, nullptr, 0, rows2.p(), nullptr);
        sum_vector(c, rows2.p(), rc, tot.p());
    }
    double mm = 0.0;
    d2h(c, &mm, tot.p(), 1);
    double res2 = a2 - mm;
    int path = 0;
    if (o.residual == BCUR_RESID_EXPLICIT || (o.residual == BCUR_RESID_AUTO && res2 < theta_explicit(dt) * a2)) {
        // Σ (A_s − Q_C (M Q_R,sᵀ))²
        Mat64 Bm(c, std::max<int64_t>(rc, 1), nl);
        Mat64 qr64(c, nl, std::max<int64_t>(rr, 1));
        convert(c, QR.buf.ptr, QR.dt, nl, rr, nl, qr64.p(), BCUR_F64, qr64.ld);
        gemm(c, OP_N, OP_T, rc, nl, rr, 1.0, M.p(), BCUR_F64, M.ld, qr64.p(), BCUR_F64, qr64.ld, 0.0, Bm.p(), Bm.ld);
        gemm_resid_sumsq(c, OP_N, OP_N, m, nl, rc, QC.buf.ptr, QC.dt, QC.rows, Bm.p(), BCUR_F64, Bm.ld, a->ptr, dt,
                         a->ld, tot.p());
        allreduce(c, tot.p(), 1);
        d2h(c, &res2, tot.p(), 1);
        path = 1;
    }
    out->u_valid = false;
    // Fast U: with distinct draws and full-rank whole-C bases, C = Q_C·R_C·D_C and
    // Rᵀ = Q_R·R_R·D_R (D = the draws' sampling scales), so
    //   U = C⁺ A R⁺ = D_C⁻¹ · R_C⁻¹ · M · R_R⁻ᵀ · D_R⁻¹
    // from the inverse factors the CholQR2 already holds (R⁻¹ = rinv1·rinv2) — four fp64
    // products instead of gathering C and Rᵀ, forming T = QᵀC and two pseudo-inverses.
    int64_t ccw = 0, crw = 0;
    for (auto& d : out->col_draws) ccw += coff[d.block + 1] - coff[d.block];
    for (auto& d : out->row_draws) crw += roff[d.block + 1] - roff[d.block];
    if (want_u && rc > 0 && rr > 0 && cb.size() == out->col_draws.size() && rb.size() == out->row_draws.size() &&
        QC.has_rinv() && QR.has_rinv() && rc == ccw && rr == crw) {
        std::vector<double> sc, sr;
        for (auto& d : out->col_draws)
            for (int64_t j = coff[d.block]; j < coff[d.block + 1]; ++j) sc.push_back(1.0 / d.scale);
        for (auto& d : out->row_draws)
            for (int64_t j = roff[d.block]; j < roff[d.block + 1]; ++j) sr.push_back(1.0 / d.scale);
        Mat64 dsc(c, ccw, 1), dsr(c, crw, 1), T1(c, ccw, crw), T2(c, ccw, crw);
        h2d(c, dsc.p(), sc.data(), ccw);
        h2d(c, dsr.p(), sr.data(), crw);
        out->u = Mat64(c, ccw, crw);
        if (dt == BCUR_F32 && h3_ok(ccw) && h3_ok(crw)) {
            // fp32 inputs: the four triangular products on the tcgen05 3×FP16 kernels (~2⁻²²
            // relative, against U's 1e-4 bar; on DMMA they were ~9 ms of c4's step):
            //   V = R_C⁻¹·M = rinv1·(rinv2·M),  Uᵀ = R_R⁻¹·Vᵀ = rinv1_R·(rinv2_R·Vᵀ)
            Mat64 Vt(c, crw, ccw), W1(c, crw, ccw);
            gemm_h3(c, true, QC.rinv2.p(), BCUR_F64, ccw, ccw, QC.rinv2.ld, M.p(), BCUR_F64, crw, M.ld, 1.0, 0.0, T1.p(),
                    T1.ld, 0);
            gemm_h3(c, true, QC.rinv1.p(), BCUR_F64, ccw, ccw, QC.rinv1.ld, T1.p(), BCUR_F64, crw, T1.ld, 1.0, 0.0, T2.p(),
                    T2.ld, 0);
            transpose(c, T2.p(), BCUR_F64, ccw, crw, T2.ld, Vt.p(), BCUR_F64, Vt.ld);
            gemm_h3(c, true, QR.rinv2.p(), BCUR_F64, crw, crw, QR.rinv2.ld, Vt.p(), BCUR_F64, ccw, Vt.ld, 1.0, 0.0, W1.p(),
                    W1.ld, 0);
            gemm_h3(c, true, QR.rinv1.p(), BCUR_F64, crw, crw, QR.rinv1.ld, W1.p(), BCUR_F64, ccw, W1.ld, 1.0, 0.0, Vt.p(),
                    Vt.ld, 0);
            transpose(c, Vt.p(), BCUR_F64, crw, ccw, Vt.ld, out->u.p(), BCUR_F64, out->u.ld);
        } else {
            gemm(c, OP_N, OP_N, ccw, crw, ccw, 1.0, QC.rinv2.p(), BCUR_F64, QC.rinv2.ld, M.p(), BCUR_F64, M.ld, 0.0,
                 T1.p(), T1.ld);
            gemm(c, OP_N, OP_N, ccw, crw, ccw, 1.0, QC.rinv1.p(), BCUR_F64, QC.rinv1.ld, T1.p(), BCUR_F64, T1.ld, 0.0,
                 T2.p(), T2.ld);
            gemm(c, OP_N, OP_T, ccw, crw, crw, 1.0, T2.p(), BCUR_F64, T2.ld, QR.rinv2.p(), BCUR_F64, QR.rinv2.ld, 0.0,
                 T1.p(), T1.ld);
            gemm(c, OP_N, OP_T, ccw, crw, crw, 1.0, T1.p(), BCUR_F64, T1.ld, QR.rinv1.p(), BCUR_F64, QR.rinv1.ld, 0.0,
                 out->u.p(), out->u.ld);
        }
        scale_rows(c, out->u.p(), ccw, crw, out->u.ld, dsc.p());
        scale_columns(c, out->u.p(), ccw, crw, out->u.ld, dsr.p());
        out->u_valid = true;
    } else if (want_u && rc > 0 && rr > 0) {
        // C (m × cc) and Rᵀ (n_local × cr) with their sampling scales
        int64_t cc = 0, cr = 0;
        std::vector<int64_t> dco, dro;
        for (auto& d : out->col_draws) { dco.push_back(cc); cc += coff[d.block + 1] - coff[d.block]; }
        for (auto& d : out->row_draws) { dro.push_back(cr); cr += roff[d.block + 1] - roff[d.block]; }
        DevBuf Cm(c, (size_t)m * cc * dtype_size(bdt)), Rt(c, (size_t)nl * cr * dtype_size(bdt));
        {
            Mat64 C64(c, m, cc);
            fill_f64(c, C64.p(), m * cc, 0.0);
            std::vector<bcur_block_draw> mine;
            std::vector<int64_t> dst;
            for (size_t t = 0; t < out->col_draws.size(); ++t) {
                const int64_t b = out->col_draws[t].block;
                if (b >= s.g0 && b < s.g1) {
                    bcur_block_draw d = out->col_draws[t];
                    d.block = b - s.g0;
                    mine.push_back(d);
                    dst.push_back(dco[t]);
                }
            }
            if (!mine.empty()) {
                DevBuf dd(c, mine.size() * sizeof(bcur_block_draw)), ddst(c, dst.size() * sizeof(int64_t));
                h2d(c, dd.as<bcur_block_draw>(), mine.data(), mine.size());
                h2d(c, ddst.as<int64_t>(), dst.data(), dst.size());
                gather_blocks(c, a->ptr, dt, m, nl, a->ld, s.d_local.as<int64_t>(), dd.as<bcur_block_draw>(),
                              ddst.as<int64_t>(), (int64_t)mine.size(), 0, 1, C64.p(), BCUR_F64, C64.ld);
            }
            allreduce(c, C64.p(), m * cc);
            convert(c, C64.p(), BCUR_F64, m, cc, C64.ld, Cm.ptr, bdt, m);
        }
        {
            DevBuf dd(c, out->row_draws.size() * sizeof(bcur_block_draw)), ddst(c, dro.size() * sizeof(int64_t));
            h2d(c, dd.as<bcur_block_draw>(), out->row_draws.data(), out->row_draws.size());
            h2d(c, ddst.as<int64_t>(), dro.data(), dro.size());
            DevBuf Rm(c, (size_t)cr * nl * dtype_size(bdt));
            gather_blocks(c, a->ptr, dt, m, nl, a->ld, droff.as<int64_t>(), dd.as<bcur_block_draw>(), ddst.as<int64_t>(),
                          (int64_t)out->row_draws.size(), 1, 1, Rm.ptr, bdt, cr);
            transpose(c, Rm.ptr, bdt, cr, nl, cr, Rt.ptr, bdt, nl);
        }
        // T_C = Q_Cᵀ C (rc × cc), T_R = Q_Rᵀ Rᵀ (rr × cr)
        Mat64 TC(c, rc, cc), TR(c, rr, cr);
        gemm(c, OP_T, OP_N, rc, cc, m, 1.0, QC.buf.ptr, QC.dt, QC.rows, Cm.ptr, bdt, m, 0.0, TC.p(), TC.ld);
        gemm(c, OP_T, OP_N, rr, cr, nl, 1.0, QR.buf.ptr, QR.dt, QR.rows, Rt.ptr, bdt, nl, 0.0, TR.p(), TR.ld);
        allreduce(c, TR.p(), rr * cr);
        // T⁺ = Tᵀ (T Tᵀ)⁻¹ ; (T Tᵀ)⁻¹ = R⁻¹ R⁻ᵀ with T Tᵀ = RᵀR
        auto pinv_rows = [&](const Mat64& T, int64_t rk, int64_t cols, Mat64* out_p) {
            Mat64 G(c, rk, rk), R(c, rk, rk), Ri(c, rk, rk), Gi(c, rk, rk);
            gemm(c, OP_N, OP_T, rk, rk, cols, 1.0, T.p(), BCUR_F64, T.ld, T.p(), BCUR_F64, T.ld, 0.0, G.p(), G.ld);
            const CholInfo ci = chol_any(c, G.p(), rk, G.ld, R.p(), Ri.p(), false, false);
            if (ci.info != 0) fail(BCUR_E_ITERATION_FAILURE, "block_cur: factor Gram is not positive definite");
            gemm(c, OP_N, OP_T, rk, rk, rk, 1.0, Ri.p(), BCUR_F64, Ri.ld, Ri.p(), BCUR_F64, Ri.ld, 0.0, Gi.p(), Gi.ld);
            *out_p = Mat64(c, cols, rk);
            gemm(c, OP_T, OP_N, cols, rk, rk, 1.0, T.p(), BCUR_F64, T.ld, Gi.p(), BCUR_F64, Gi.ld, 0.0, out_p->p(),
                 out_p->ld);
        };
        Mat64 TCp, TRp;
        pinv_rows(TC, rc, cc, &TCp);  // cc × rc
        pinv_rows(TR, rr, cr, &TRp);  // cr × rr
        Mat64 T2(c, cc, rr);
        gemm(c, OP_N, OP_N, cc, rr, rc, 1.0, TCp.p(), BCUR_F64, TCp.ld, M.p(), BCUR_F64, M.ld, 0.0, T2.p(), T2.ld);
        out->u = Mat64(c, cc, cr);
        gemm(c, OP_N, OP_T, cc, cr, rr, 1.0, T2.p(), BCUR_F64, T2.ld, TRp.p(), BCUR_F64, TRp.ld, 0.0, out->u.p(),
             out->u.ld);
        out->u_valid = true;
    }
    out->rep = bcur_report{};
    out->rep.abs_err = std::sqrt(std::max(res2, 0.0));
    out->rep.a_norm = std::sqrt(a2);
    out->rep.rel_err = out->rep.abs_err / out->rep.a_norm;
    out->rep.k_eff = sub.k_eff;
    out->rep.rank_c = rc;
    out->rep.rank_r = rr;
    out->rep.residual_path = path;
    out->rep.orth_dev = sub.orth_dev;
}

}  // namespace bcur_b200
