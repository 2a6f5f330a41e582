/*
 * bcur_b200.h — C ABI of the B200-native Block-CUR hot path.
 *
 * Drop-in boundary for the reference's hot path (/root/reference/proj/include/bcur):
 * every entry point below names the reference interface it replaces.  Plain
 * pointers and sizes only; host arrays are caller-owned, device objects
 * (bcur_ctx, bcur_dmat) are library-owned and released with *_destroy.
 * A context is used by one host thread at a time.  All compute runs on the
 * GPU (sm_100a); there is no CPU fallback — without a usable device every
 * compute call returns BCUR_E_CUDA.
 *
 * Matrices are column-major with a leading dimension (Eigen's default,
 * matcore.hpp:10), fp32 or fp64.  Block partitions are passed as G+1 strictly
 * increasing column offsets covering [0, n) (BlockPartition, leverage.hpp:18-48).
 */
#ifndef BCUR_B200_H
#define BCUR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.hpp:9-57 → status codes (C++ mirror maps them back to exceptions). */
typedef enum {
    BCUR_OK = 0,
    BCUR_E_INVALID_ARGUMENT = 1,   /* std::invalid_argument */
    BCUR_E_OUT_OF_RANGE = 2,       /* std::out_of_range */
    BCUR_E_DIMENSION_MISMATCH = 3, /* DimensionMismatch */
    BCUR_E_INVALID_BASIS = 4,      /* InvalidBasis */
    BCUR_E_ZERO_BLOCK = 5,         /* ZeroBlock */
    BCUR_E_ZERO_MATRIX = 6,        /* ZeroMatrix */
    BCUR_E_DISTRIBUTION_INVALID = 7,
    BCUR_E_NOT_ENOUGH_BLOCKS = 8,
    BCUR_E_DEGENERATE_R = 9,
    BCUR_E_ITERATION_FAILURE = 10,
    BCUR_E_PARSE = 11,
    BCUR_E_CUDA = 12,              /* device error / no device */
    BCUR_E_COMM = 13               /* collective callback failed */
} bcur_status;

typedef enum { BCUR_F32 = 0, BCUR_F64 = 1 } bcur_dtype;

/* sampler.hpp:11 SamplingMode */
typedef enum { BCUR_WITH_REPLACEMENT = 0, BCUR_WITHOUT_REPLACEMENT = 1 } bcur_sampling_mode;

typedef enum { BCUR_RESID_AUTO = -1, BCUR_RESID_PYTHAGORAS = 0, BCUR_RESID_EXPLICIT = 1 } bcur_residual_mode;

typedef struct bcur_ctx_s* bcur_ctx;
typedef struct bcur_dmat_s* bcur_dmat;
typedef struct bcur_rng_s* bcur_rng;

/* sampler.hpp:17-21 BlockDraw */
typedef struct {
    int64_t block;
    double probability; /* original p_j */
    double scale;       /* 1/sqrt(g·p_j) */
} bcur_block_draw;

/* ---------------------------------------------------------------- context */
bcur_status bcur_ctx_create(int device, bcur_ctx* out);
bcur_status bcur_ctx_destroy(bcur_ctx ctx);
/* Run on a caller-owned cudaStream_t (NULL → library-owned stream). */
bcur_status bcur_ctx_set_stream(bcur_ctx ctx, void* cuda_stream);
void* bcur_ctx_stream(bcur_ctx ctx);
bcur_status bcur_ctx_synchronize(bcur_ctx ctx);
/* Number of kernels this context has launched so far (bench evidence). */
int64_t bcur_ctx_launch_count(bcur_ctx ctx);
/* Per-kernel-class accounting with CUDA events on the context stream.
 * enable=1 clears and starts recording; bcur_ctx_profile_dump synchronizes and
 * writes JSON {"tag": {"scopes": n, "ms": t, "flops": f, "bytes": b}, ...}
 * (algorithmic flops/bytes) into buf; returns the needed length. */
bcur_status bcur_ctx_profile(bcur_ctx ctx, int enable);
int64_t bcur_ctx_profile_dump(bcur_ctx ctx, char* buf, int64_t cap);

/* Multi-GPU plumbing: one process (context) per GPU; the host supplies the
 * collectives (e.g. torch.distributed over NCCL).  Callbacks run on the
 * calling thread and must enqueue on `stream` (or complete before returning). */
typedef struct {
    int rank;
    int world;
    void* user;
    /* in-place sum of `count` doubles at device pointer `buf` */
    int (*allreduce_f64)(void* user, double* buf, int64_t count, void* stream);
    /* broadcast of `bytes` bytes at device pointer `buf` from rank `root` (nullable: the
     * library then emulates it with a zero-padded allreduce_f64 of fp64 data).  Selected
     * column blocks of A travel through it in their stored form — fp32, or the fp16 hi/lo
     * split of the 3×FP16 path (4 bytes per element) — not as fp64. */
    int (*broadcast)(void* user, void* buf, int64_t bytes, int root, void* stream);
} bcur_comm;
bcur_status bcur_ctx_set_comm(bcur_ctx ctx, const bcur_comm* comm); /* NULL → single rank */

/* --------------------------------------------------------------- matrices */
bcur_status bcur_dmat_create(bcur_ctx ctx, int dtype, int64_t m, int64_t n, bcur_dmat* out);
/* Copies m×n column-major host data (leading dimension ld_host ≥ m). */
bcur_status bcur_dmat_upload(bcur_ctx ctx, bcur_dmat a, const void* host, int64_t ld_host);
/* The same copy enqueued on the context's upload stream, returning at once: the next call that
 * uses `a` waits for it on the device (so an upload of the next input overlaps the current
 * decomposition).  The copy first waits for the uses of `a` already enqueued.  `host` must stay
 * valid and unmodified until then (pinned memory makes the copy asynchronous). */
bcur_status bcur_dmat_upload_async(bcur_ctx ctx, bcur_dmat a, const void* host, int64_t ld_host);
bcur_status bcur_dmat_download(bcur_ctx ctx, bcur_dmat a, void* host, int64_t ld_host);
/* Page-locked host memory for inputs and result buffers (the reference returns its results by
 * value, blockcur.hpp:44-58; here large ones — U of bcur_block_cur — land in caller-owned host
 * memory, and a pinned destination takes one DMA copy where a pageable one is staged). */
bcur_status bcur_host_alloc(size_t bytes, void** out);
bcur_status bcur_host_free(void* p);
/* Wraps caller-owned device memory (no copy, not freed by destroy). */
bcur_status bcur_dmat_wrap(bcur_ctx ctx, int dtype, int64_t m, int64_t n, void* dev_ptr, int64_t ld,
                           bcur_dmat* out);
bcur_status bcur_dmat_info(bcur_dmat a, int* dtype, int64_t* m, int64_t* n, int64_t* ld, void** dev_ptr);
/* Column shard: this matrix holds global columns [col0, col0+n) of an n_global-column matrix. */
bcur_status bcur_dmat_set_shard(bcur_dmat a, int64_t col0, int64_t n_global);
bcur_status bcur_dmat_destroy(bcur_dmat a);

/* ------------------------------------------------------- synthetic inputs */
typedef enum { BCUR_GEN_LOWRANK = 0, BCUR_GEN_BIOMETRIC = 1 } bcur_gen_kind;
typedef struct {
    int kind;            /* bcur_gen_kind */
    int dtype;           /* bcur_dtype */
    int64_t m, n;
    int64_t rank;        /* LOWRANK: number of singular triples */
    const double* sigma; /* LOWRANK: rank values */
    double noise;        /* LOWRANK: iid N(0, noise²) */
    uint64_t seed;
    int64_t col0;        /* first global column to generate (column shards) */
    int64_t n_global;    /* global column count (0 → n) */
} bcur_gen_spec;
/* A = U·diag(σ)·Vᵀ + ν·E (U, V Gaussian-then-orthonormalised) or the config-2
 * biometric surrogate; Philox counters, so shards are independent of the split. */
bcur_status bcur_dmat_generate(bcur_ctx ctx, const bcur_gen_spec* spec, bcur_dmat* out);

/* ------------------------------------------------------------------- Rng */
/* rng.hpp:13-63 (std::mt19937_64 + the reference's hand-written conversions). */
bcur_status bcur_rng_create(uint64_t seed, bcur_rng* out);
bcur_status bcur_rng_destroy(bcur_rng r);
uint64_t bcur_rng_seed(bcur_rng r);
uint64_t bcur_rng_next_u64(bcur_rng r);
double bcur_rng_uniform01(bcur_rng r);
uint64_t bcur_rng_below(bcur_rng r, uint64_t bound);
double bcur_rng_normal(bcur_rng r);
uint64_t bcur_rng_split_seed(bcur_rng r, uint64_t stream);
/* Sketch key used by the pipelines: Rng(seed).split(0x6F6D656761).seed(). */
uint64_t bcur_omega_key(uint64_t seed);

/* ------------------------------------------------------ hot-path kernels */
/* matcore.cpp:93-95 frobenius_norm */
bcur_status bcur_frobenius_norm(bcur_ctx ctx, bcur_dmat a, double* out);
/* per-block ‖A_g‖_F² (sketch.cpp:21-26 middleCols(..).squaredNorm()) */
bcur_status bcur_block_sq_norms(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G, double* out);
/* leverage.cpp:108-121 block_leverage (+ require_orthonormal, leverage.cpp:11-23;
 * tol < 0 → 1e-8 for fp64 input, 1e-4 for fp32). */
bcur_status bcur_block_leverage(bcur_ctx ctx, bcur_dmat v_k, const int64_t* offsets, int64_t G, double tol,
                                double* scores, double* normalizer);
/* leverage.cpp:123-153 score diagnostics: per-block stable ranks ‖V_g‖_F²/‖V_g‖_2² of the row
 * blocks of V_k (k ≤ 64), their minimum (block_stable_rank) and the incoherence
 * (m/k)·max_i ‖U_kᵀe_i‖² (u_k nullable).  Outputs are written before a zero-mass block is
 * reported as BCUR_E_ZERO_BLOCK (its stable rank is NaN). */
bcur_status bcur_block_diagnostics(bcur_ctx ctx, bcur_dmat v_k, bcur_dmat u_k, const int64_t* offsets, int64_t G,
                                   double* stable_ranks, double* block_stable_rank, double* incoherence);
/* leverage.cpp:100-106 column_leverage */
bcur_status bcur_column_leverage(bcur_ctx ctx, bcur_dmat v_k, double tol, double* scores, double* normalizer);
/* N1: randomized range finder replacing truncate(svd(a), k) (matcore.cpp:39-69).
 * Returns V_k (n×k_eff) and U_k (m×k_eff) fp64 device matrices (either out may be NULL),
 * sigma (k_eff values, host, nullable). */
bcur_status bcur_range_finder(bcur_ctx ctx, bcur_dmat a, int64_t k, int64_t p, int64_t q, uint64_t key,
                              bcur_dmat* v_out, bcur_dmat* u_out, double* sigma_out, int64_t* k_eff);
/* The sketch products of the range finder on the hot-path kernels (tcgen05 3×TF32 for
 * fp32 A, fp64 SIMT otherwise): out (fp64) = A·X (transpose=0, X n×N) or Aᵀ·X
 * (transpose=1, X m×N).  X is fp64.  rows_out (nullable, host, length n) with
 * transpose=1 receives Σ_c (AᵀX)_jc² instead of storing the product (out may be NULL). */
bcur_status bcur_sketch_product(bcur_ctx ctx, bcur_dmat a, bcur_dmat x, int transpose, bcur_dmat out,
                                double* rows_out);
/* Structured forms of the same products (diagnostics and tests; the pipelines use them for
 * the basis Grams and Q = C·R⁻¹):
 *   BCUR_PRODUCT_GRAM      out = AᵀA, upper triangle only (x must be NULL, transpose = 1)
 *   BCUR_PRODUCT_X_UPPER   X is upper triangular (zero below its diagonal; the tcgen05 path
 *                          skips that part of the product)
 *   BCUR_PRODUCT_ROWSQ_F16 out (n × 1) = Σ_c (AᵀX)_jc² through the pipelines' fp16 path
 *                          (fp32 A with m % 64 == 0; transpose = 1)
 *   BCUR_PRODUCT_H3        A·X, AᵀX or (with GRAM) AᵀA through the pipelines' 3×FP16 form: A
 *                          split into fp16 hi + lo by the norms pass (fp32 A; m % 64 == 0 for
 *                          A·X, m % 8 == 0 for AᵀX)
 *   BCUR_PRODUCT_FAST_ACC  with H3: the three MMAs of a k-step into one fp32 accumulator (CTA pairs,
 *                          ~1e-6 relative instead of ~2⁻²²; the pipelines' C·R⁻¹ and c4's Q_CᵀA)
 *   BCUR_PRODUCT_HI_ONLY   with FAST_ACC: the a_hi·x_hi MMA alone (2⁻¹¹ relative; the pipelines'
 *                          CholQR2 second-pass correction Q1·(−F), ‖F‖ ≲ 1e-4)
 */
enum { BCUR_PRODUCT_GRAM = 1, BCUR_PRODUCT_X_UPPER = 2, BCUR_PRODUCT_ROWSQ_F16 = 4, BCUR_PRODUCT_H3 = 8,
       BCUR_PRODUCT_FAST_ACC = 16, BCUR_PRODUCT_HI_ONLY = 32 };
bcur_status bcur_sketch_product_ex(bcur_ctx ctx, bcur_dmat a, bcur_dmat x, int transpose, int flags, bcur_dmat out);
/* The factorization behind every orthonormal basis of the path (CholQR2 of the sketch, of C,
 * of Rᵀ — the reference's pseudoinverse, matcore.cpp:85-91, and svd, :39-56, are never
 * formed): g (w×w fp64, upper triangle read) → r_out = R (upper, zero below) with G = RᵀR and
 * rinv_out = R⁻¹ (nullable).  Recursive on the device: ≤128-wide leaves factored and inverted
 * by one CTA, DMMA products between them.  *info = 0, or j + 1 when pivot j is not positive
 * (R, R⁻¹ then undefined).  min_diag (nullable) = min diag(R). */
bcur_status bcur_cholesky(bcur_ctx ctx, bcur_dmat g, bcur_dmat r_out, bcur_dmat rinv_out, int* info, double* min_diag);
/* blockcur.cpp:54-109 block_cur — the reference's default Algorithm 1 (row_sampling =
 * uniform): R = the caller's row draws of A (sampler.cpp:54-95, drawn from its Rng; scaled
 * unless distinct), approximate block leverage of R (all rank(R) right singular vectors,
 * leverage.cpp:155-164), g block draws with the caller's uniforms (one per draw, drawn after
 * the rows), C = A·S, W = R·S, U = W⁺ (matcore.cpp:85-91), and ‖A − C·U·R‖_F for U and for
 * its rank-k truncation (matcore.cpp:81-83).  Single device.  u_out (nullable) receives U,
 * c × r with ld c (c = the drawn blocks' total width; size it for the g widest blocks). */
typedef struct {
    int64_t row;
    double probability; /* 1/m */
    double scale;       /* 1/sqrt(r·p) (applied when scaled_rows) */
} bcur_row_draw;
typedef struct {
    double abs_err_u;   /* ‖A − C·U·R‖_F      (metrics_u) */
    double abs_err_uk;  /* ‖A − C·U_k·R‖_F    (metrics_uk) */
    double a_norm;      /* ‖A‖_F */
    int64_t rank_r;     /* rank(R) = the scores' normalizer */
    int64_t rank_w;     /* numerical rank of W */
} bcur_alg1_report;
bcur_status bcur_block_cur_alg1(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G, int64_t k,
                                const bcur_row_draw* rows, int64_t r, int scaled_rows, int64_t g, int block_mode,
                                const double* uniforms, double* scores_out, double* normalizer_out,
                                bcur_block_draw* draws_out, double* margins_out, double* u_out,
                                bcur_alg1_report* report);
/* io.cpp:105-137 load_matrix_binary / save_matrix_binary: the reference's ".bcur" format
 * (magic "BCUR", u64 rows, u64 cols, f64 row-major).  The loader streams row chunks through
 * pinned staging into a column-major device matrix of the requested dtype; columns
 * [col0, col0 + ncols) select a shard (ncols = -1: to the end).  Missing magic, truncated
 * header or data, unreasonable dimensions and NaN/Inf entries return BCUR_E_PARSE.
 * bcur_bcur_header reads only the dimensions (to plan shards). */
bcur_status bcur_bcur_header(const char* path, int64_t* rows, int64_t* cols);
bcur_status bcur_dmat_load_bcur(bcur_ctx ctx, const char* path, int dtype, int64_t col0, int64_t ncols,
                                bcur_dmat* out);
bcur_status bcur_dmat_save_bcur(bcur_ctx ctx, bcur_dmat a, const char* path);
/* sampler.cpp:116-146 draw_blocks (probabilities on the host, one uniform per draw
 * drawn by the caller from its Rng; margins_out[t] = distance of u_t to the nearest
 * CDF edge, nullable). */
bcur_status bcur_draw_blocks(bcur_ctx ctx, const double* probs, int64_t G, int64_t g, int mode,
                             const double* uniforms, uint64_t seed, bcur_block_draw* out, double* margins_out);
/* sampler.cpp:161-184 materialize_columns; row blocks = column blocks of Aᵀ. */
bcur_status bcur_materialize_columns(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G,
                                     const bcur_block_draw* draws, int64_t ndraws, bcur_dmat* out);
bcur_status bcur_materialize_row_blocks(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G,
                                        const bcur_block_draw* draws, int64_t ndraws, bcur_dmat* out);
/* blockcur.cpp:33-52 error_report: abs_err = ‖A − C(UR)‖_F, a_norm = ‖A‖_F. */
bcur_status bcur_error_report(bcur_ctx ctx, bcur_dmat a, bcur_dmat c, bcur_dmat u, bcur_dmat r, double* abs_err,
                              double* a_norm);

/* ------------------------------------------------------- whole pipelines */
typedef struct {
    int64_t k, p, q;    /* range finder: rank, oversampling, power iterations */
    int64_t g;          /* blocks to select (column blocks for CUR) */
    int64_t g_rows;     /* CUR: row blocks to select */
    int mode;           /* bcur_sampling_mode */
    int residual;       /* bcur_residual_mode */
    uint64_t seed;      /* Rng seed: sketch key = bcur_omega_key(seed) */
    int rank_floor;     /* 0 (default): the sketch's numerical rank is the reference's
                           (σ > 1e-12·max(m,n)·σ₁, matcore.cpp:35-49); 1: also drop
                           σ ≤ τ_rank·σ₁ (1e-5 fp32, 1e-7 fp64: near the working precision) */
} bcur_options;

typedef struct {
    double abs_err;     /* ‖A − C C⁺ A‖_F  (CUR: ‖A − C U R‖_F) */
    double a_norm;      /* ‖A‖_F */
    double rel_err;     /* abs_err / a_norm */
    int64_t k_eff;      /* rank of the subspace used for scores */
    int64_t rank_c;     /* numerical rank of C (CUR: of C) */
    int64_t rank_r;     /* CUR: numerical rank of R */
    int residual_path;  /* 0 Pythagoras, 1 explicit */
    double orth_dev;    /* max |V_kᵀV_k − I| (require_orthonormal evidence) */
} bcur_report;

/* R15 block_css (sketch.cpp:68-82): scores → draws (uniforms[g] from the caller's
 * Rng) → C → ‖A − CC⁺A‖_F.  scores_out[G], draws_out[g], margins_out[g] nullable. */
bcur_status bcur_block_css(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G, const bcur_options* opt,
                           const double* uniforms, double* scores_out, double* normalizer_out,
                           bcur_block_draw* draws_out, double* margins_out, bcur_report* rep);

/* N3 greedy deterministic selection. */
typedef struct {
    int64_t block;
    double score;       /* residual ‖(I−P_C)A_g‖² at pick time (or leverage if saturated) */
    double margin;      /* top1 − top2 of the criterion */
    int saturated;
    int64_t rank_added;
} bcur_greedy_step;
bcur_status bcur_greedy_select(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G, const bcur_options* opt,
                               bcur_greedy_step* steps_out, double* residuals_out, bcur_report* rep);

/* N4 block CUR with row and column blocks, U = C⁺AR⁺ (uniforms: g column draws
 * then g_rows row draws).  u_out (c×r column-major, ldu) nullable. */
bcur_status bcur_block_cur(bcur_ctx ctx, bcur_dmat a, const int64_t* col_offsets, int64_t Gc,
                           const int64_t* row_offsets, int64_t Gr, const bcur_options* opt, const double* uniforms,
                           double* col_scores, double* row_scores, bcur_block_draw* col_draws,
                           bcur_block_draw* row_draws, double* u_out, int64_t ldu, bcur_report* rep);

/* Thread-local message of the last failing call. */
const char* bcur_last_error(void);
const char* bcur_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BCUR_B200_H */
