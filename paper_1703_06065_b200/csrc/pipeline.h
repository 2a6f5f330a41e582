// pipeline.h — hot-path orchestration (pipeline.cu) used by the C ABI (capi.cu).
#pragma once
#include <functional>

#include <vector>

#include "ops.h"

namespace bcur_b200 {

// fp64 device matrix in pooled memory (column-major, ld = max(1, m)).
struct Mat64 {
    DevBuf buf;
    int64_t m = 0, n = 0, ld = 1;
    Mat64() = default;
    Mat64(Ctx* c, int64_t m_, int64_t n_);
    double* p() const { return buf.as<double>(); }
};

// Column shard of A against a global block partition.
struct Shard {
    int64_t G = 0, g0 = 0, g1 = 0, col0 = 0, n_global = 0;
    std::vector<int64_t> off_global;  // G+1
    DevBuf d_local;                   // (g1-g0+1) offsets relative to the shard's first column
    std::vector<int> owner;           // G: the rank holding each block
};

struct Subspace {
    Mat64 v;  // n_local × k_eff
    Mat64 u;  // m × k_eff
    std::vector<double> sigma;
    int64_t k_eff = 0, l = 0;
    double orth_dev = 0.0;
};

struct CssOut {
    std::vector<double> scores, margins;
    double normalizer = 0.0;
    std::vector<bcur_block_draw> draws;
    bcur_report rep{};
};

struct GreedyOut {
    std::vector<bcur_greedy_step> steps;
    std::vector<double> residuals;
    bcur_report rep{};
};

struct CurOut {
    std::vector<double> col_scores, row_scores;
    std::vector<bcur_block_draw> col_draws, row_draws;
    Mat64 qr, u;
    int64_t rank_r = 0;
    bool u_valid = false;
    bcur_report rep{};
};

// fp16 copy of an fp32 A written by the norms pass (block_sumsq): column j scaled by 2^exps[j]
// (exact), hi = rn16(a·2^e) — the row-Σ² passes' operand (kind::f16, the same 11-bit
// significands as a round-to-nearest TF32 copy) — either alone (compact: m halves per column)
// or interleaved per 64-row chunk with lo = rn16(a·2^e − hi) ([hi 64 | lo 64], 2m halves per
// column): hi + lo is the A operand of the 3×FP16 range-finder products.  Empty when A is fp64,
// m % 64 != 0, or it does not fit.
struct RoundedA {
    DevBuf il, exps;
    bool interleaved = false;
    bool ok() const { return il.ptr != nullptr; }
    bool has_lo() const { return ok() && interleaved; }
};

struct Alg1Out {
    std::vector<double> scores, margins;
    double normalizer = 0.0;
    std::vector<bcur_block_draw> draws;
    Mat64 u;  // c × r
    bcur_alg1_report rep{};
};

Shard shard_of(const DMat* a, const int64_t* offsets, int64_t G);
// G (w×w SPD, upper read) → R (w×w, ld w, upper) with G = RᵀR and Rinv = R⁻¹ (nullable, ld w);
// returns 0 or the failed pivot + 1 (recursive, DMMA products, ≤128-wide fused leaves)
int cholesky_inverse(Ctx* c, const double* G, int64_t w, int64_t ldg, double* R, double* Rinv, double* mindiag);
void allreduce(Ctx* c, double* d, int64_t count);
int64_t orth(Ctx* c, const double* X, int64_t rows, int64_t w, int64_t ldx, double ref, int dt, double* Q,
             int64_t ldq, bool dist, Mat64* T_out, int* path_out);
// after_read (nullable): run right after the first stream synchronization (the caller's
// deferred reads — e.g. ‖A‖² — are then delivered and can be checked before any of the range
// finder's own decisions); defer: out->orth_dev is delivered by the caller's next read_all()
void range_finder(Ctx* c, const DMat* a, int64_t k, int64_t p, int64_t q, uint64_t key, Subspace* out,
                  bool rank_floor, const RoundedA* ra = nullptr, const std::function<void()>* after_read = nullptr,
                  bool defer = false);
void block_css(Ctx* c, const DMat* a, const int64_t* offsets, int64_t G, const bcur_options& o, const double* uniforms,
               CssOut* out);
void greedy_select(Ctx* c, const DMat* a, const int64_t* offsets, int64_t G, const bcur_options& o, GreedyOut* out);
void block_cur_alg1(Ctx* c, const DMat* a, const int64_t* offsets, int64_t G, int64_t k, const bcur_row_draw* rows,
                    int64_t r, bool scaled_rows, int64_t g, int block_mode, const double* uniforms, Alg1Out* out);
void block_cur(Ctx* c, const DMat* a, const int64_t* coff, int64_t Gc, const int64_t* roff, int64_t Gr,
               const bcur_options& o, const double* uniforms, bool want_u, CurOut* out);

}  // namespace bcur_b200
