// bcur_b200.hpp — header-only C++ mirror of the reference API (proj/include/bcur/*.hpp)
// over the C ABI in bcur_b200.h.  Same namespace (`bcur`), type names, function names,
// argument meaning and exception types as the reference, so a caller of the hot path
// (bcur_main.cpp:115-170, bench.cpp:217-347, the unit tests) switches by changing the
// include and linking libbcur_b200.so instead of the Eigen build.  Differences, by design:
//   * Matrix / Vector are small column-major value types (Eigen is not a dependency);
//     they expose rows()/cols()/operator()(i,j)/data() like Eigen::MatrixXd.
//   * Large inputs stay on the GPU: every entry point also accepts a DeviceMatrix.
//   * block_css's rank-k subspace comes from the randomized range finder (p, q in
//     CssOptions; defaults p=10, q=2) instead of a full SVD of A (matcore.cpp:39-56).
//   * error_report fills rel_to_best_k only when an ErrorBaseline is passed (the
//     reference computes it from a full SVD of A, which this path never runs).
// All compute runs on the device; there is no CPU fallback.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bcur_b200.h"

namespace bcur {

using Index = std::ptrdiff_t;

// ------------------------------------------------------------------ errors.hpp:9-57
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IterationFailure : Error { using Error::Error; };
struct InvalidBasis : Error { using Error::Error; };
struct ZeroBlock : Error { using Error::Error; };
struct ZeroMatrix : Error { using Error::Error; };
struct DistributionInvalid : Error { using Error::Error; };
struct NotEnoughBlocks : Error { using Error::Error; };
struct DegenerateR : Error { using Error::Error; };
struct DimensionMismatch : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA / collective failure (no reference analogue)

namespace detail {
inline void check(bcur_status st) {
    if (st == BCUR_OK) return;
    const char* m = bcur_last_error();
    const std::string msg = m ? m : "bcur_b200 error";
    switch (st) {
        case BCUR_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case BCUR_E_OUT_OF_RANGE: throw std::out_of_range(msg);
        case BCUR_E_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case BCUR_E_INVALID_BASIS: throw InvalidBasis(msg);
        case BCUR_E_ZERO_BLOCK: throw ZeroBlock(msg);
        case BCUR_E_ZERO_MATRIX: throw ZeroMatrix(msg);
        case BCUR_E_DISTRIBUTION_INVALID: throw DistributionInvalid(msg);
        case BCUR_E_NOT_ENOUGH_BLOCKS: throw NotEnoughBlocks(msg);
        case BCUR_E_DEGENERATE_R: throw DegenerateR(msg);
        case BCUR_E_ITERATION_FAILURE: throw IterationFailure(msg);
        case BCUR_E_PARSE: throw ParseError(msg);
        default: throw DeviceError(msg);
    }
}
}  // namespace detail

// ------------------------------------------------------------ matcore.hpp:10-12
class Vector {
public:
    Vector() = default;
    explicit Vector(Index n, double v = 0.0) : d_(static_cast<std::size_t>(n), v) {}
    explicit Vector(std::vector<double> v) : d_(std::move(v)) {}
    Index size() const { return static_cast<Index>(d_.size()); }
    double& operator()(Index i) { return d_[static_cast<std::size_t>(i)]; }
    double operator()(Index i) const { return d_[static_cast<std::size_t>(i)]; }
    double& operator[](Index i) { return (*this)(i); }
    double operator[](Index i) const { return (*this)(i); }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }
    double sum() const {
        double s = 0.0;
        for (double x : d_) s += x;
        return s;
    }
    Vector operator/(double x) const {
        Vector o(*this);
        for (double& v : o.d_) v /= x;
        return o;
    }

private:
    std::vector<double> d_;
};

class Matrix {  // column-major, ld = rows (Eigen::MatrixXd default)
public:
    Matrix() = default;
    Matrix(Index rows, Index cols) : r_(rows), c_(cols), d_(static_cast<std::size_t>(rows * cols), 0.0) {}
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(i + j * r_)]; }
    double operator()(Index i, Index j) const { return d_[static_cast<std::size_t>(i + j * r_)]; }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }

private:
    Index r_ = 0, c_ = 0;
    std::vector<double> d_;
};

// -------------------------------------------------------------- device context
// One context per host thread (the reference has none; its functions are pure).
class Device {
public:
    explicit Device(int device = 0) { detail::check(bcur_ctx_create(device, &h_)); }
    ~Device() {
        if (h_) bcur_ctx_destroy(h_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    bcur_ctx handle() const { return h_; }
    static Device& current() {
        thread_local std::unique_ptr<Device> dev;
        if (!dev) dev = std::make_unique<Device>(0);
        return *dev;
    }

private:
    bcur_ctx h_ = nullptr;
};

// A column-major fp32/fp64 matrix resident in HBM (optionally one column shard).
class DeviceMatrix {
public:
    DeviceMatrix() = default;
    explicit DeviceMatrix(bcur_dmat h) : h_(h) {}
    static DeviceMatrix upload(const Matrix& a, Device& dev = Device::current()) {
        bcur_dmat h = nullptr;
        detail::check(bcur_dmat_create(dev.handle(), BCUR_F64, a.rows(), a.cols(), &h));
        DeviceMatrix m(h);
        detail::check(bcur_dmat_upload(dev.handle(), h, a.data(), std::max<Index>(a.rows(), 1)));
        return m;
    }
    static DeviceMatrix upload_f32(const float* colmajor, Index rows, Index cols, Device& dev = Device::current()) {
        bcur_dmat h = nullptr;
        detail::check(bcur_dmat_create(dev.handle(), BCUR_F32, rows, cols, &h));
        DeviceMatrix m(h);
        detail::check(bcur_dmat_upload(dev.handle(), h, colmajor, std::max<Index>(rows, 1)));
        return m;
    }
    // io.cpp:105-137 load_matrix_binary, streamed into HBM: columns [col0, col0 + ncols) of a
    // ".bcur" file (ncols = -1: to the end) as fp64 or fp32; ParseError as in the reference
    static DeviceMatrix load_binary(const std::string& path, int dtype = BCUR_F64, Index col0 = 0, Index ncols = -1,
                                    Device& dev = Device::current()) {
        bcur_dmat h = nullptr;
        detail::check(bcur_dmat_load_bcur(dev.handle(), path.c_str(), dtype, col0, ncols, &h));
        return DeviceMatrix(h);
    }
    void save_binary(const std::string& path, Device& dev = Device::current()) const {
        detail::check(bcur_dmat_save_bcur(dev.handle(), h_, path.c_str()));
    }
    static DeviceMatrix generate(const bcur_gen_spec& spec, Device& dev = Device::current()) {
        bcur_dmat h = nullptr;
        detail::check(bcur_dmat_generate(dev.handle(), &spec, &h));
        return DeviceMatrix(h);
    }
    DeviceMatrix(DeviceMatrix&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    DeviceMatrix& operator=(DeviceMatrix&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    ~DeviceMatrix() {
        if (h_) bcur_dmat_destroy(h_);
    }
    bcur_dmat handle() const { return h_; }
    Index rows() const { return info().m; }
    Index cols() const { return info().n; }
    Matrix download(Device& dev = Device::current()) const {  // fp32 data is widened to fp64
        const Info i = info();
        Matrix out(i.m, i.n);
        if (i.dtype == BCUR_F64) {
            detail::check(bcur_dmat_download(dev.handle(), h_, out.data(), std::max<int64_t>(i.m, 1)));
        } else {
            std::vector<float> tmp(static_cast<std::size_t>(i.m * i.n));
            detail::check(bcur_dmat_download(dev.handle(), h_, tmp.data(), std::max<int64_t>(i.m, 1)));
            for (std::size_t e = 0; e < tmp.size(); ++e) out.data()[e] = tmp[e];
        }
        return out;
    }

private:
    struct Info { int dtype; int64_t m, n, ld; };
    Info info() const {
        Info i{};
        void* p = nullptr;
        detail::check(bcur_dmat_info(h_, &i.dtype, &i.m, &i.n, &i.ld, &p));
        return i;
    }
    bcur_dmat h_ = nullptr;
};

// -------------------------------------------------------------- rng.hpp:13-63
class Rng {  // the library's mt19937_64 stream with the reference's conversions
public:
    explicit Rng(std::uint64_t seed) { detail::check(bcur_rng_create(seed, &h_)); }
    ~Rng() {
        if (h_) bcur_rng_destroy(h_);
    }
    Rng(Rng&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    Rng(const Rng&) = delete;
    std::uint64_t seed() const { return bcur_rng_seed(h_); }
    std::uint64_t next_u64() { return bcur_rng_next_u64(h_); }
    double uniform01() { return bcur_rng_uniform01(h_); }
    std::uint64_t below(std::uint64_t bound) { return bcur_rng_below(h_, bound); }
    double normal() { return bcur_rng_normal(h_); }
    Rng split(std::uint64_t stream) const { return Rng(bcur_rng_split_seed(h_, stream)); }

private:
    bcur_rng h_ = nullptr;
};

// ------------------------------------------------------- leverage.hpp:11-82
struct BlockRange {
    Index begin = 0;
    Index end = 0;
    Index width() const { return end - begin; }
};

class BlockPartition {
public:
    static BlockPartition equal_blocks(Index n, Index block_size) {  // leverage.cpp:29-41
        if (n < 1 || block_size < 1) throw std::invalid_argument("equal_blocks: n and block size must be >= 1");
        std::vector<BlockRange> r;
        for (Index b = 0; b < n; b += block_size) r.push_back({b, std::min(n, b + block_size)});
        BlockPartition p(n, std::move(r));
        p.nominal_s_ = block_size;
        return p;
    }
    static BlockPartition from_boundaries(Index n, std::span<const Index> cuts) {  // leverage.cpp:43-56
        std::vector<BlockRange> r;
        Index prev = 0;
        for (Index c : cuts) {
            if (c <= prev || c >= n) throw std::invalid_argument("from_boundaries: cuts must be increasing in (0, n)");
            r.push_back({prev, c});
            prev = c;
        }
        r.push_back({prev, n});
        return BlockPartition(n, std::move(r));
    }
    BlockPartition(Index n, std::vector<BlockRange> ranges) : n_(n), ranges_(std::move(ranges)) {
        Index at = 0;
        for (const auto& r : ranges_) {
            if (r.begin != at || r.end <= r.begin)
                throw std::invalid_argument("BlockPartition: ranges must be contiguous, disjoint and non-empty");
            at = r.end;
        }
        if (at != n_ || ranges_.empty()) throw std::invalid_argument("BlockPartition: ranges must cover [0, n)");
        nominal_s_ = max_width();
    }
    Index num_columns() const { return n_; }
    Index num_blocks() const { return static_cast<Index>(ranges_.size()); }
    const BlockRange& range(Index g) const { return ranges_.at(static_cast<std::size_t>(g)); }
    Index width(Index g) const { return range(g).width(); }
    Index max_width() const {
        Index w = 0;
        for (const auto& r : ranges_) w = std::max(w, r.width());
        return w;
    }
    Index nominal_block_size() const { return nominal_s_; }
    const std::vector<BlockRange>& ranges() const { return ranges_; }
    Index block_of_column(Index j) const {  // leverage.cpp:82-90
        if (j < 0 || j >= n_) throw std::out_of_range("block_of_column: column out of range");
        Index lo = 0, hi = num_blocks() - 1;
        while (lo < hi) {
            const Index mid = (lo + hi + 1) / 2;
            if (ranges_[static_cast<std::size_t>(mid)].begin <= j) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    }
    std::vector<int64_t> offsets() const {  // the ABI's G+1 offsets
        std::vector<int64_t> o;
        for (const auto& r : ranges_) o.push_back(r.begin);
        o.push_back(n_);
        return o;
    }

private:
    Index n_ = 0;
    Index nominal_s_ = 0;
    std::vector<BlockRange> ranges_;
};

struct ScoreVector {
    Vector scores;
    double normalizer = 1.0;
    Vector probabilities() const { return scores / normalizer; }
    Vector distribution() const {  // leverage.cpp:92-98
        const double s = scores.sum();
        if (!(s > 0.0)) throw ZeroMatrix("ScoreVector::distribution: scores sum to zero");
        return scores / s;
    }
};

namespace detail {
inline ScoreVector leverage(const DeviceMatrix& v, const BlockPartition* part, double tol) {
    Device& dev = Device::current();
    ScoreVector out;
    if (part) {
        const auto off = part->offsets();
        out.scores = Vector(part->num_blocks());
        check(bcur_block_leverage(dev.handle(), v.handle(), off.data(), part->num_blocks(), tol, out.scores.data(),
                                  &out.normalizer));
    } else {
        out.scores = Vector(v.rows());
        check(bcur_column_leverage(dev.handle(), v.handle(), tol, out.scores.data(), &out.normalizer));
    }
    return out;
}
}  // namespace detail

// leverage.cpp:100-106 — score_j = ‖row j of V_k‖², normalizer k (V_k must be orthonormal)
inline ScoreVector column_leverage(const Matrix& v_k) {
    return detail::leverage(DeviceMatrix::upload(v_k), nullptr, -1.0);
}
// leverage.cpp:108-121 — ℓ_g = ‖V_kᵀE_g‖_F²
inline ScoreVector block_leverage(const Matrix& v_k, const BlockPartition& part) {
    return detail::leverage(DeviceMatrix::upload(v_k), &part, -1.0);
}
inline ScoreVector block_leverage(const DeviceMatrix& v_k, const BlockPartition& part) {
    return detail::leverage(v_k, &part, -1.0);
}

// -------------------------------------------------------- sampler.hpp:11-72
enum class SamplingMode { with_replacement, without_replacement };
inline const char* to_string(SamplingMode m) {
    return m == SamplingMode::with_replacement ? "with_replacement" : "without_replacement";
}
struct BlockDraw {
    Index block = 0;
    double probability = 0.0;
    double scale = 0.0;
};
struct SamplingPlan {
    std::vector<BlockDraw> draws;
    SamplingMode mode = SamplingMode::with_replacement;
    std::uint64_t seed = 0;
    std::vector<double> margins;  // D14 near-tie record (not in the reference)
    Index num_draws() const { return static_cast<Index>(draws.size()); }
};

namespace detail {
inline int mode_code(SamplingMode m) {
    return m == SamplingMode::with_replacement ? BCUR_WITH_REPLACEMENT : BCUR_WITHOUT_REPLACEMENT;
}
inline std::vector<double> uniforms(Rng& rng, Index g) {  // one uniform01 per draw (sampler.cpp:36)
    std::vector<double> u(static_cast<std::size_t>(g));
    for (auto& x : u) x = rng.uniform01();
    return u;
}
inline SamplingPlan plan_from(const std::vector<bcur_block_draw>& d, const std::vector<double>& margins,
                              SamplingMode mode, std::uint64_t seed) {
    SamplingPlan p;
    p.mode = mode;
    p.seed = seed;
    p.margins = margins;
    for (const auto& x : d) p.draws.push_back({x.block, x.probability, x.scale});
    return p;
}
inline std::vector<bcur_block_draw> to_c(const SamplingPlan& p) {
    std::vector<bcur_block_draw> d;
    for (const auto& x : p.draws) d.push_back({x.block, x.probability, x.scale});
    return d;
}
}  // namespace detail

// sampler.cpp:116-146
inline SamplingPlan draw_blocks(const Vector& probs, Index g, SamplingMode mode, Rng& rng) {
    if (g < 1) throw std::invalid_argument("draw_blocks: g must be >= 1");
    const std::uint64_t seed = rng.seed();
    const auto u = detail::uniforms(rng, g);
    std::vector<bcur_block_draw> d(static_cast<std::size_t>(g));
    std::vector<double> margins(static_cast<std::size_t>(g));
    detail::check(bcur_draw_blocks(Device::current().handle(), probs.data(), probs.size(), g, detail::mode_code(mode),
                                   u.data(), seed, d.data(), margins.data()));
    return detail::plan_from(d, margins, mode, seed);
}
// sampler.cpp:148-159
inline SamplingPlan identity_plan(const BlockPartition& part) {
    SamplingPlan p;
    for (Index g = 0; g < part.num_blocks(); ++g) p.draws.push_back({g, 1.0, 1.0});
    return p;
}
// sampler.cpp:161-184 — C = A S
inline Matrix materialize_columns(const Matrix& a, const BlockPartition& part, const SamplingPlan& plan) {
    if (a.cols() != part.num_columns()) throw DimensionMismatch("materialize_columns: partition does not match A");
    Device& dev = Device::current();
    DeviceMatrix da = DeviceMatrix::upload(a, dev);
    const auto off = part.offsets();
    const auto d = detail::to_c(plan);
    bcur_dmat h = nullptr;
    detail::check(bcur_materialize_columns(dev.handle(), da.handle(), off.data(), part.num_blocks(), d.data(),
                                           static_cast<int64_t>(d.size()), &h));
    return DeviceMatrix(h).download(dev);
}

// -------------------------------------------------------- matcore.hpp:46
inline double frobenius_norm(const DeviceMatrix& a) {
    double v = 0.0;
    detail::check(bcur_frobenius_norm(Device::current().handle(), a.handle(), &v));
    return v;
}
inline double frobenius_norm(const Matrix& a) { return frobenius_norm(DeviceMatrix::upload(a)); }

// ------------------------------------------------------ blockcur.hpp:19-76
enum class UVariant { full, rank_k };
struct ErrorReport {
    double abs_err = 0.0;
    double rel_to_a = 0.0;
    std::optional<double> rel_to_best_k;
    Index k = 0;
    UVariant variant = UVariant::full;
};
struct ErrorBaseline {
    double a_norm = 0.0;
    double best_k_residual = 0.0;
    Index k = 0;
};
// blockcur.cpp:33-52 — ‖A − C(UR)‖_F
inline ErrorReport error_report(const Matrix& a, const Matrix& c, const Matrix& u, const Matrix& r, Index k,
                                UVariant variant = UVariant::full, const ErrorBaseline* baseline = nullptr) {
    Device& dev = Device::current();
    auto da = DeviceMatrix::upload(a, dev), dc = DeviceMatrix::upload(c, dev), du = DeviceMatrix::upload(u, dev),
         dr = DeviceMatrix::upload(r, dev);
    ErrorReport rep;
    double a_norm = 0.0;
    detail::check(bcur_error_report(dev.handle(), da.handle(), dc.handle(), du.handle(), dr.handle(), &rep.abs_err,
                                    &a_norm));
    rep.rel_to_a = a_norm > 0.0 ? rep.abs_err / a_norm : 0.0;
    if (baseline && baseline->best_k_residual >= 1e-12) rep.rel_to_best_k = rep.abs_err / baseline->best_k_residual;
    rep.k = k;
    rep.variant = variant;
    return rep;
}

// ------------------------------ blockcur.hpp:36-76 — the reference's Algorithm 1
enum class RowSampling { uniform, leverage };
struct RowDraw {
    Index row;
    double probability, scale;
};
struct RowPlan {
    std::vector<RowDraw> draws;
    Index source_rows = 0;
    SamplingMode mode = SamplingMode::with_replacement;
    std::uint64_t seed = 0;
    Index num_draws() const { return static_cast<Index>(draws.size()); }
};
// sampler.cpp:54-95 — uniform row draws from the caller's Rng (one below() per draw)
inline RowPlan draw_rows(Index m, Index r, Rng& rng) {
    if (r < 1) throw std::invalid_argument("draw_rows: r must be >= 1");
    if (m < 1) throw std::invalid_argument("draw_rows: m must be >= 1");
    RowPlan plan{{}, m, SamplingMode::with_replacement, rng.seed()};
    const double p = 1.0 / static_cast<double>(m), scale = 1.0 / std::sqrt(static_cast<double>(r) * p);
    for (Index t = 0; t < r; ++t) plan.draws.push_back({static_cast<Index>(rng.below(static_cast<std::uint64_t>(m))), p, scale});
    return plan;
}
inline RowPlan draw_rows_distinct(Index m, Index r, Rng& rng) {
    if (r < 1 || m < 1) throw std::invalid_argument("draw_rows_distinct: m and r must be >= 1");
    if (r > m) throw std::invalid_argument("draw_rows_distinct: r must be <= m");
    std::vector<Index> pool(static_cast<std::size_t>(m));
    for (Index i = 0; i < m; ++i) pool[static_cast<std::size_t>(i)] = i;
    RowPlan plan{{}, m, SamplingMode::without_replacement, rng.seed()};
    const double p = 1.0 / static_cast<double>(m), scale = 1.0 / std::sqrt(static_cast<double>(r) * p);
    for (Index t = 0; t < r; ++t) {
        const auto pick = static_cast<Index>(rng.below(static_cast<std::uint64_t>(m - t)));
        std::swap(pool[static_cast<std::size_t>(t + pick)], pool[static_cast<std::size_t>(t)]);
        plan.draws.push_back({pool[static_cast<std::size_t>(t)], p, scale});
    }
    return plan;
}
struct CurOptions {
    SamplingMode block_mode = SamplingMode::with_replacement;
    RowSampling row_sampling = RowSampling::uniform;  // leverage rows: not on this path
    bool distinct_rows = false;
};
struct CurResult {  // C, R and W stay on the device: materialize_columns / rows on demand
    Matrix u;       // c × r, U = W⁺
    RowPlan row_plan;
    SamplingPlan block_plan;
    ScoreVector block_scores;  // approximate block leverage of R (normalizer = rank R)
    ErrorReport metrics_u, metrics_uk;
    std::vector<double> trial_errors;
};
// blockcur.cpp:54-109 — rows → R, approximate block leverage of R, g blocks → C, W,
// U = W⁺, ‖A − CUR‖_F for U and U_k; everything after the row draws runs on the GPU
inline CurResult block_cur(const DeviceMatrix& a, const BlockPartition& part, Index k, Index r, Index g,
                           const CurOptions& opts, Rng& rng, const ErrorBaseline* baseline = nullptr) {
    if (opts.row_sampling != RowSampling::uniform)
        throw std::invalid_argument("block_cur: leverage row sampling needs the exact SVD of A (not on this path)");
    if (r < 1 || g < 1) throw std::invalid_argument("block_cur: r and g must be >= 1");
    Device& dev = Device::current();
    const Index m = a.rows();
    CurResult res;
    res.row_plan = opts.distinct_rows ? draw_rows_distinct(m, r, rng) : draw_rows(m, r, rng);
    std::vector<bcur_row_draw> rd;
    for (const RowDraw& d : res.row_plan.draws) rd.push_back({d.row, d.probability, d.scale});
    const std::uint64_t seed = rng.seed();
    const auto u = detail::uniforms(rng, g);
    const auto off = part.offsets();
    const Index G = part.num_blocks();
    std::vector<Index> widths;
    for (Index b = 0; b < G; ++b) widths.push_back(off[static_cast<std::size_t>(b) + 1] - off[static_cast<std::size_t>(b)]);
    std::sort(widths.begin(), widths.end(), std::greater<Index>());
    Index cap = 0;
    for (Index t = 0; t < g && t < G; ++t) cap += widths[static_cast<std::size_t>(t)];
    std::vector<double> ubuf(static_cast<std::size_t>(std::max<Index>(cap * r, 1)));
    res.block_scores.scores = Vector(G);
    std::vector<bcur_block_draw> d(static_cast<std::size_t>(g));
    std::vector<double> margins(static_cast<std::size_t>(g));
    bcur_alg1_report rep{};
    detail::check(bcur_block_cur_alg1(dev.handle(), a.handle(), off.data(), G, k,
                                      rd.data(), r, opts.distinct_rows ? 0 : 1, g, detail::mode_code(opts.block_mode),
                                      u.data(), res.block_scores.scores.data(), &res.block_scores.normalizer, d.data(),
                                      margins.data(), ubuf.data(), &rep));
    res.block_plan = detail::plan_from(d, margins, opts.block_mode, seed);
    Index cc = 0;
    for (const auto& x : d) cc += off[static_cast<std::size_t>(x.block) + 1] - off[static_cast<std::size_t>(x.block)];
    res.u = Matrix(cc, r);
    std::copy(ubuf.begin(), ubuf.begin() + cc * r, res.u.data());
    for (ErrorReport* e : {&res.metrics_u, &res.metrics_uk}) {
        e->abs_err = e == &res.metrics_u ? rep.abs_err_u : rep.abs_err_uk;
        e->rel_to_a = rep.a_norm > 0.0 ? e->abs_err / rep.a_norm : 0.0;
        if (baseline && baseline->k == k && baseline->best_k_residual >= 1e-12)
            e->rel_to_best_k = e->abs_err / baseline->best_k_residual;
        e->k = k;
        e->variant = e == &res.metrics_u ? UVariant::full : UVariant::rank_k;
    }
    res.trial_errors = {res.metrics_u.abs_err};
    return res;
}
inline CurResult block_cur(const Matrix& a, const BlockPartition& part, Index k, Index r, Index g,
                           const CurOptions& opts, Rng& rng, const ErrorBaseline* baseline = nullptr) {
    return block_cur(DeviceMatrix::upload(a), part, k, r, g, opts, rng, baseline);
}
// blockcur.cpp:111-133 — t independent trials on one Rng stream, the lowest ‖A − CUR‖ kept
inline CurResult block_cur_boosted(const DeviceMatrix& a, const BlockPartition& part, Index k, Index r, Index g,
                                   Index t, const CurOptions& opts, Rng& rng, const ErrorBaseline* baseline = nullptr) {
    if (t < 1) throw std::invalid_argument("block_cur_boosted: t must be >= 1");
    CurResult best;
    std::vector<double> errors;
    for (Index trial = 0; trial < t; ++trial) {
        CurResult cur = block_cur(a, part, k, r, g, opts, rng, baseline);
        errors.push_back(cur.metrics_u.abs_err);
        if (trial == 0 || cur.metrics_u.abs_err < best.metrics_u.abs_err) best = std::move(cur);
    }
    best.trial_errors = std::move(errors);
    return best;
}

// ----------------------------------------------------------- sketch.hpp:32-39
struct CssOptions {
    Index p = 10, q = 2;  // range finder oversampling / power iterations
    SamplingMode mode = SamplingMode::with_replacement;  // reference default (sketch.cpp:78)
    bool materialize_c = true;
};
struct CssResult {
    Matrix c;
    double projection_error = 0.0;  // ‖A − C C⁺ A‖_F
    SamplingPlan plan;
    // beyond the reference: the scores and the run report
    ScoreVector scores;
    bcur_report report{};
};

inline CssResult block_css(const DeviceMatrix& a, const BlockPartition& part, Index k, Index g, Rng& rng,
                           const CssOptions& o = {}) {
    if (k < 1) throw std::invalid_argument("block_css: k must be >= 1");
    if (g < 1) throw std::invalid_argument("draw_blocks: g must be >= 1");
    Device& dev = Device::current();
    const auto off = part.offsets();
    const Index G = part.num_blocks();
    const std::uint64_t seed = rng.seed();
    const auto u = detail::uniforms(rng, g);
    bcur_options opt{k, o.p, o.q, g, 0, detail::mode_code(o.mode), BCUR_RESID_AUTO, seed};
    CssResult res;
    res.scores.scores = Vector(G);
    std::vector<bcur_block_draw> d(static_cast<std::size_t>(g));
    std::vector<double> margins(static_cast<std::size_t>(g));
    detail::check(bcur_block_css(dev.handle(), a.handle(), off.data(), G, &opt, u.data(), res.scores.scores.data(),
                                 &res.scores.normalizer, d.data(), margins.data(), &res.report));
    res.plan = detail::plan_from(d, margins, o.mode, seed);
    res.projection_error = res.report.abs_err;
    if (o.materialize_c) {
        bcur_dmat h = nullptr;
        detail::check(bcur_materialize_columns(dev.handle(), a.handle(), off.data(), G, d.data(), g, &h));
        res.c = DeviceMatrix(h).download(dev);
    }
    return res;
}
// sketch.hpp:39 — block column subset selection with g blocks at rank k
inline CssResult block_css(const Matrix& a, const BlockPartition& part, Index k, Index g, Rng& rng,
                           const CssOptions& o = {}) {
    return block_css(DeviceMatrix::upload(a), part, k, g, rng, o);
}

// ------------------------------------- north star (3): greedy deterministic selection
struct GreedyResult {
    std::vector<bcur_greedy_step> steps;
    Vector residuals;  // final ‖(I−P_C)A_g‖² per block
    bcur_report report{};
    std::vector<Index> blocks() const {
        std::vector<Index> b;
        for (const auto& s : steps) b.push_back(s.block);
        return b;
    }
};
inline GreedyResult greedy_select(const DeviceMatrix& a, const BlockPartition& part, Index k, Index g,
                                  std::uint64_t seed, Index p = 5, Index q = 0) {
    Device& dev = Device::current();
    const auto off = part.offsets();
    bcur_options opt{k, p, q, g, 0, BCUR_WITHOUT_REPLACEMENT, BCUR_RESID_AUTO, seed};
    GreedyResult r;
    r.steps.resize(static_cast<std::size_t>(g));
    r.residuals = Vector(part.num_blocks());
    detail::check(bcur_greedy_select(dev.handle(), a.handle(), off.data(), part.num_blocks(), &opt, r.steps.data(),
                                     r.residuals.data(), &r.report));
    return r;
}

// ------------------------------ north star (4): block CUR with row and column blocks, U = C⁺AR⁺
struct CurRowsColsResult {
    SamplingPlan col_plan, row_plan;
    ScoreVector col_scores, row_scores;
    Matrix u;  // c × r
    bcur_report report{};
};
inline CurRowsColsResult block_cur_rows_cols(const DeviceMatrix& a, const BlockPartition& col_part,
                                             const BlockPartition& row_part, Index k, Index gc, Index gr, Rng& rng,
                                             Index p = 10, Index q = 0,
                                             SamplingMode mode = SamplingMode::without_replacement) {
    Device& dev = Device::current();
    const auto co = col_part.offsets(), ro = row_part.offsets();
    const std::uint64_t seed = rng.seed();
    const auto u = detail::uniforms(rng, gc + gr);  // column draws, then row draws
    bcur_options opt{k, p, q, gc, gr, detail::mode_code(mode), BCUR_RESID_AUTO, seed};
    CurRowsColsResult r;
    r.col_scores.scores = Vector(col_part.num_blocks());
    r.row_scores.scores = Vector(row_part.num_blocks());
    std::vector<bcur_block_draw> cd(static_cast<std::size_t>(gc)), rd(static_cast<std::size_t>(gr));
    Matrix umax(gc * col_part.max_width(), gr * row_part.max_width());
    detail::check(bcur_block_cur(dev.handle(), a.handle(), co.data(), col_part.num_blocks(), ro.data(),
                                 row_part.num_blocks(), &opt, u.data(), r.col_scores.scores.data(),
                                 r.row_scores.scores.data(), cd.data(), rd.data(), umax.data(), umax.rows(),
                                 &r.report));
    r.col_plan = detail::plan_from(cd, {}, mode, seed);
    r.row_plan = detail::plan_from(rd, {}, mode, seed);
    Index cw = 0, rw = 0;
    for (const auto& x : cd) cw += col_part.width(x.block);
    for (const auto& x : rd) rw += row_part.width(x.block);
    r.u = Matrix(cw, rw);
    for (Index j = 0; j < rw; ++j)
        for (Index i = 0; i < cw; ++i) r.u(i, j) = umax(i, j);
    r.col_scores.normalizer = r.row_scores.normalizer = static_cast<double>(r.report.k_eff);
    return r;
}

}  // namespace bcur
