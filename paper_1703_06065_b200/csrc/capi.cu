// capi.cu — the C ABI (include/bcur_b200.h).  Validates arguments with the
// reference's error semantics (errors.hpp:9-57, sampler.cpp, leverage.cpp,
// blockcur.cpp), converts exceptions to bcur_status + a thread-local message,
// and forwards to the device pipeline.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "pipeline.h"

using namespace bcur_b200;

namespace {

thread_local std::string g_last_error;

bcur_status set_error(bcur_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

#define API_BEGIN try {
#define API_END                                                                  \
    return BCUR_OK;                                                              \
    }                                                                            \
    catch (const Failure& f) { return set_error(f.status, f.what()); }           \
    catch (const std::bad_alloc&) { return set_error(BCUR_E_CUDA, "host allocation failed"); } \
    catch (const std::exception& e) { return set_error(BCUR_E_INVALID_ARGUMENT, e.what()); }

Ctx* C(bcur_ctx c) {
    if (!c) fail(BCUR_E_INVALID_ARGUMENT, "null context");
    CUDA_CHECK(cudaSetDevice(c->device));
    return c;
}
DMat* M(bcur_dmat a) {
    if (!a) fail(BCUR_E_INVALID_ARGUMENT, "null matrix");
    if (a->pending) {  // an asynchronous upload into it: order the compute stream after the copy
        CUDA_CHECK(cudaStreamWaitEvent(a->ctx->stream, a->ready, 0));
        a->pending = false;
    }
    return a;
}

void check_dtype(int dt) {
    if (dt != BCUR_F32 && dt != BCUR_F64) fail(BCUR_E_INVALID_ARGUMENT, "dtype must be BCUR_F32 or BCUR_F64");
}

void check_partition(const int64_t* off, int64_t G, int64_t n, const char* what) {
    if (!off || G < 1) fail(BCUR_E_INVALID_ARGUMENT, std::string(what) + ": at least one block required");
    if (off[0] != 0) fail(BCUR_E_INVALID_ARGUMENT, std::string(what) + ": ranges must start at 0");
    for (int64_t g = 0; g < G; ++g)
        if (off[g + 1] <= off[g])
            fail(BCUR_E_INVALID_ARGUMENT, std::string(what) + ": ranges must be contiguous, non-empty, and ordered");
    if (n >= 0 && off[G] != n) fail(BCUR_E_DIMENSION_MISMATCH, std::string(what) + ": partition does not match matrix");
}

bcur_dmat new_dmat(Ctx* c, int dt, int64_t m, int64_t n) {
    auto* d = new bcur_dmat_s();
    d->ctx = c;
    d->dtype = dt;
    d->m = m;
    d->n = n;
    d->ld = std::max<int64_t>(m, 1);
    d->owned = true;
    const size_t bytes = (size_t)d->ld * (size_t)std::max<int64_t>(n, 1) * dtype_size(dt);
    cudaError_t e = cudaMalloc(&d->ptr, bytes);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        c->trim();
        e = cudaMalloc(&d->ptr, bytes);
        if (e != cudaSuccess) {
            delete d;
            fail(BCUR_E_CUDA, std::string("cudaMalloc of matrix failed: ") + cudaGetErrorString(e));
        }
    }
    return d;
}

bcur_dmat from_mat64(Ctx* c, const Mat64& x, int64_t m, int64_t n) {
    bcur_dmat d = new_dmat(c, BCUR_F64, m, n);
    if (m * n > 0)
        CUDA_CHECK(cudaMemcpy2DAsync(d->ptr, d->ld * 8, x.p(), x.ld * 8, m * 8, n, cudaMemcpyDeviceToDevice, c->stream));
    c->sync();
    return d;
}

double sumsq(Ctx* c, const DMat* a) {
    if (a->m * a->n == 0) return 0.0;
    const int64_t off[2] = {0, a->n};
    DevBuf d_off(c, sizeof off), out(c, sizeof(double));
    CUDA_CHECK(cudaMemcpyAsync(d_off.ptr, off, sizeof off, cudaMemcpyHostToDevice, c->stream));
    ops::block_sumsq(c, a->ptr, a->dtype, a->m, a->ld, d_off.as<int64_t>(), 1, out.as<double>());
    if (a->n_global > a->n) allreduce(c, out.as<double>(), 1);
    double h = 0.0;
    CUDA_CHECK(cudaMemcpyAsync(&h, out.ptr, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    return h;
}

// require_orthonormal (leverage.cpp:11-23) on the device Gram VᵀV.
void require_orthonormal(Ctx* c, const DMat* v, double tol, const char* what) {
    if (v->m < 1 || v->n < 1) fail(BCUR_E_INVALID_BASIS, std::string(what) + ": basis must be non-empty");
    if (v->m < v->n) fail(BCUR_E_INVALID_BASIS, std::string(what) + ": more columns than rows cannot be orthonormal");
    if (tol < 0) tol = v->dtype == BCUR_F32 ? 1e-4 : 1e-8;
    Mat64 g(c, v->n, v->n), dev(c, 1, 1);
    ops::gemm(c, ops::OP_T, ops::OP_N, v->n, v->n, v->m, 1.0, v->ptr, v->dtype, v->ld, v->ptr, v->dtype, v->ld, 0.0,
              g.p(), g.ld);
    ops::max_dev_identity(c, g.p(), v->n, g.ld, dev.p());
    double h = 0.0;
    CUDA_CHECK(cudaMemcpyAsync(&h, dev.p(), sizeof h, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (!(h <= tol))
        fail(BCUR_E_INVALID_BASIS, std::string(what) + ": column Gram deviates from identity by " + std::to_string(h));
}

void upload_draws(Ctx* c, const bcur_block_draw* draws, int64_t nd, const int64_t* off, int64_t G, int64_t* total,
                  DevBuf* d_draws, DevBuf* d_dst, DevBuf* d_off) {
    std::vector<int64_t> dst(nd);
    int64_t t = 0;
    for (int64_t i = 0; i < nd; ++i) {
        if (draws[i].block < 0 || draws[i].block >= G)
            fail(BCUR_E_DIMENSION_MISMATCH, "materialize: plan references block " + std::to_string(draws[i].block) +
                                                " outside the partition");
        dst[i] = t;
        t += off[draws[i].block + 1] - off[draws[i].block];
    }
    *total = t;
    *d_draws = DevBuf(c, nd * sizeof(bcur_block_draw));
    *d_dst = DevBuf(c, nd * sizeof(int64_t));
    *d_off = DevBuf(c, (G + 1) * sizeof(int64_t));
    CUDA_CHECK(cudaMemcpyAsync(d_draws->ptr, draws, nd * sizeof(bcur_block_draw), cudaMemcpyHostToDevice, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(d_dst->ptr, dst.data(), nd * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(d_off->ptr, off, (G + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    c->sync();
}

}  // namespace

struct bcur_rng_s {
    uint64_t seed;
    std::mt19937_64 engine;
    double spare = 0.0;
    bool has_spare = false;
    explicit bcur_rng_s(uint64_t s) : seed(s), engine(s) {}
    double uniform01() { return (double)(engine() >> 11) * 0x1.0p-53; }  // rng.hpp:22
};

extern "C" {

const char* bcur_last_error(void) { return g_last_error.c_str(); }
const char* bcur_version(void) { return "bcur_b200 0.1.0 (sm_100a)"; }

// ------------------------------------------------------------- context
bcur_status bcur_ctx_create(int device, bcur_ctx* out) {
    API_BEGIN
    if (!out) fail(BCUR_E_INVALID_ARGUMENT, "null output");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        (void)cudaGetLastError();
        fail(BCUR_E_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= count) fail(BCUR_E_INVALID_ARGUMENT, "device index out of range");
    CUDA_CHECK(cudaSetDevice(device));
    auto* c = new bcur_ctx_s();
    c->device = device;
    CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    CUDA_CHECK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    *out = c;
    API_END
}

bcur_status bcur_ctx_destroy(bcur_ctx ctx) {
    API_BEGIN
    if (!ctx) return BCUR_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->trim();
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->up_ring) cudaFreeHost(ctx->up_ring);
    if (ctx->rd_area) cudaFreeHost(ctx->rd_area);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
        cudaStreamSynchronize(ctx->side2);
        cudaStreamDestroy(ctx->side2);
        cudaStreamSynchronize(ctx->hp);
        cudaStreamDestroy(ctx->hp);
        cudaStreamSynchronize(ctx->side3);
        cudaStreamDestroy(ctx->side3);
        for (auto e : ctx->side_ev) cudaEventDestroy(e);
    }
    if (ctx->up) {
        cudaStreamSynchronize(ctx->up);
        cudaStreamDestroy(ctx->up);
    }
    delete ctx;
    API_END
}

bcur_status bcur_ctx_set_stream(bcur_ctx ctx, void* s) {
    API_BEGIN
    Ctx* c = C(ctx);
    c->sync();
    if (c->own_stream) cudaStreamDestroy(c->stream);
    if (s) {
        c->stream = (cudaStream_t)s;
        c->own_stream = false;
    } else {
        CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    API_END
}

void* bcur_ctx_stream(bcur_ctx ctx) { return ctx ? (void*)ctx->stream : nullptr; }

bcur_status bcur_ctx_synchronize(bcur_ctx ctx) {
    API_BEGIN
    C(ctx)->sync();
    API_END
}

int64_t bcur_ctx_launch_count(bcur_ctx ctx) { return ctx ? ctx->launches : 0; }

bcur_status bcur_ctx_profile(bcur_ctx ctx, int enable) {
    API_BEGIN
    Ctx* c = C(ctx);
    c->sync();
    for (auto& r : c->prof_recs) {
        c->ev_pool.push_back(r.e0);
        c->ev_pool.push_back(r.e1);
    }
    c->prof_recs.clear();
    c->prof = enable != 0;
    c->allocs_mark = c->allocs;
    API_END
}

int64_t bcur_ctx_profile_dump(bcur_ctx ctx, char* buf, int64_t cap) {
    if (!ctx) return -1;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    struct Acc { int64_t n = 0; double ms = 0, flops = 0, bytes = 0; };
    std::map<std::string, Acc> acc;
    for (auto& r : ctx->prof_recs) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) {
            (void)cudaGetLastError();
            continue;
        }
        Acc& a = acc[r.tag];
        a.n++;
        a.ms += ms;
        a.flops += r.flops;
        a.bytes += r.bytes;
    }
    std::string s = "{";
    bool first = true;
    char tmp[512];
    for (auto& kv : acc) {
        std::snprintf(tmp, sizeof tmp, "%s\"%s\": {\"scopes\": %lld, \"ms\": %.6f, \"flops\": %.6e, \"bytes\": %.6e}",
                      first ? "" : ", ", kv.first.c_str(), (long long)kv.second.n, kv.second.ms, kv.second.flops,
                      kv.second.bytes);
        s += tmp;
        first = false;
    }
    std::snprintf(tmp, sizeof tmp, "%s\"_cudaMalloc\": {\"scopes\": %lld, \"ms\": 0, \"flops\": 0, \"bytes\": 0}",
                  first ? "" : ", ", (long long)(ctx->allocs - ctx->allocs_mark));
    s += tmp;
    s += "}";
    if (buf && cap > 0) {
        std::strncpy(buf, s.c_str(), (size_t)cap - 1);
        buf[cap - 1] = 0;
    }
    return (int64_t)s.size() + 1;
}

bcur_status bcur_ctx_set_comm(bcur_ctx ctx, const bcur_comm* comm) {
    API_BEGIN
    Ctx* c = C(ctx);
    if (!comm) {
        c->comm = bcur_comm{0, 1, nullptr, nullptr, nullptr};
    } else {
        if (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world)
            fail(BCUR_E_INVALID_ARGUMENT, "bcur_comm: invalid rank/world");
        if (comm->world > 1 && !comm->allreduce_f64) fail(BCUR_E_INVALID_ARGUMENT, "bcur_comm: allreduce_f64 required");
        c->comm = *comm;
    }
    API_END
}

// -------------------------------------------------------------- matrices
bcur_status bcur_dmat_create(bcur_ctx ctx, int dtype, int64_t m, int64_t n, bcur_dmat* out) {
    API_BEGIN
    Ctx* c = C(ctx);
    check_dtype(dtype);
    if (m < 0 || n < 0 || !out) fail(BCUR_E_INVALID_ARGUMENT, "bcur_dmat_create: bad shape");
    *out = new_dmat(c, dtype, m, n);
    API_END
}

bcur_status bcur_dmat_upload(bcur_ctx ctx, bcur_dmat a, const void* host, int64_t ld_host) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    if (ld_host < d->m) fail(BCUR_E_INVALID_ARGUMENT, "bcur_dmat_upload: ld_host < m");
    const size_t es = dtype_size(d->dtype);
    if (d->m * d->n > 0)
        CUDA_CHECK(cudaMemcpy2DAsync(d->ptr, d->ld * es, host, ld_host * es, d->m * es, d->n, cudaMemcpyHostToDevice,
                                     c->stream));
    c->sync();
    API_END
}

bcur_status bcur_dmat_upload_async(bcur_ctx ctx, bcur_dmat a, const void* host, int64_t ld_host) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    if (ld_host < d->m) fail(BCUR_E_INVALID_ARGUMENT, "bcur_dmat_upload_async: ld_host < m");
    if (!c->up) CUDA_CHECK(cudaStreamCreateWithFlags(&c->up, cudaStreamNonBlocking));
    if (!d->ready) CUDA_CHECK(cudaEventCreateWithFlags(&d->ready, cudaEventDisableTiming));
    // the copy overwrites `a`: it waits for every use of `a` already enqueued on the compute stream
    CUDA_CHECK(cudaEventRecord(d->ready, c->stream));
    CUDA_CHECK(cudaStreamWaitEvent(c->up, d->ready, 0));
    const size_t es = dtype_size(d->dtype);
    if (d->m * d->n > 0) {
        if (ld_host == d->m && d->ld == d->m)  // contiguous on both sides: one linear copy
            CUDA_CHECK(cudaMemcpyAsync(d->ptr, host, (size_t)d->m * d->n * es, cudaMemcpyHostToDevice, c->up));
        else
            CUDA_CHECK(cudaMemcpy2DAsync(d->ptr, d->ld * es, host, ld_host * es, d->m * es, d->n, cudaMemcpyHostToDevice,
                                         c->up));
    }
    CUDA_CHECK(cudaEventRecord(d->ready, c->up));
    d->pending = true;
    API_END
}

// ---------------------------------------------------------------- .bcur files
// io.cpp:105-137 (load_matrix_binary) / save_matrix_binary: magic "BCUR", u64 rows, u64 cols
// (little-endian), rows·cols f64 row-major.  Streamed in row chunks through two pinned
// staging buffers (disk read of chunk i+1 overlaps the copy and device transpose of chunk
// i) straight into a column-major device matrix of either dtype; a column range selects a
// shard (one contiguous run per row).  Errors are ParseError as in the reference.
namespace {
struct BcurHeader {
    uint64_t rows = 0, cols = 0;
};
BcurHeader read_bcur_header(FILE* f, const std::string& path) {
    char magic[4] = {0, 0, 0, 0};
    if (fread(magic, 1, 4, f) != 4 || memcmp(magic, "BCUR", 4) != 0) fail(BCUR_E_PARSE, path + ": missing BCUR magic");
    BcurHeader h;
    if (fread(&h.rows, 8, 1, f) != 1 || fread(&h.cols, 8, 1, f) != 1) fail(BCUR_E_PARSE, path + ": truncated header");
    constexpr uint64_t kMaxDim = 1ull << 31;
    if (h.rows == 0 || h.cols == 0 || h.rows >= kMaxDim || h.cols >= kMaxDim)
        fail(BCUR_E_PARSE, path + ": unreasonable dimensions " + std::to_string(h.rows) + "x" + std::to_string(h.cols));
    return h;
}
struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) fclose(f);
    }
};
}  // namespace

bcur_status bcur_bcur_header(const char* path, int64_t* rows, int64_t* cols) {
    API_BEGIN
    if (!path || !rows || !cols) fail(BCUR_E_INVALID_ARGUMENT, "bcur_bcur_header: null argument");
    File fh;
    fh.f = fopen(path, "rb");
    if (!fh.f) fail(BCUR_E_PARSE, std::string("cannot open ") + path);
    const BcurHeader h = read_bcur_header(fh.f, path);
    *rows = (int64_t)h.rows;
    *cols = (int64_t)h.cols;
    API_END
}

bcur_status bcur_dmat_load_bcur(bcur_ctx ctx, const char* path, int dtype, int64_t col0, int64_t ncols,
                                bcur_dmat* out) {
    API_BEGIN
    Ctx* c = C(ctx);
    check_dtype(dtype);
    if (!path || !out) fail(BCUR_E_INVALID_ARGUMENT, "bcur_dmat_load_bcur: null argument");
    File fh;
    fh.f = fopen(path, "rb");
    if (!fh.f) fail(BCUR_E_PARSE, std::string("cannot open ") + path);
    const BcurHeader h = read_bcur_header(fh.f, path);
    const int64_t m = (int64_t)h.rows, n = (int64_t)h.cols;
    if (ncols < 0) ncols = n - col0;
    if (col0 < 0 || ncols < 1 || col0 + ncols > n)
        fail(BCUR_E_OUT_OF_RANGE, "bcur_dmat_load_bcur: column range outside the file's " + std::to_string(n) + " columns");
    // entry data must be complete (the reference reads all rows·cols and reports truncation)
    const long long data0 = 4 + 16;
    if (fseeko(fh.f, 0, SEEK_END) != 0) fail(BCUR_E_PARSE, std::string(path) + ": cannot seek");
    const long long size = ftello(fh.f);
    if (size < data0 + (long long)(m * n * 8)) fail(BCUR_E_PARSE, std::string(path) + ": truncated entry data");
    bcur_dmat d = new_dmat(c, dtype, ncols, m);  // staged as its transpose's shape, fixed below
    d->m = m;
    d->n = ncols;
    d->ld = std::max<int64_t>(m, 1);
    const int64_t chunk_rows = std::max<int64_t>(1, std::min<int64_t>(m, ((int64_t)64 << 20) / (8 * ncols)));
    const size_t chunk_bytes = (size_t)chunk_rows * ncols * 8;
    void* pin[2] = {nullptr, nullptr};
    cudaEvent_t done[2];
    for (int b = 0; b < 2; ++b) {
        CUDA_CHECK(cudaHostAlloc(&pin[b], chunk_bytes, cudaHostAllocDefault));
        CUDA_CHECK(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
    }
    struct Cleanup {
        void** pin;
        cudaEvent_t* done;
        ~Cleanup() {
            for (int b = 0; b < 2; ++b) {
                cudaEventSynchronize(done[b]);
                cudaFreeHost(pin[b]);
                cudaEventDestroy(done[b]);
            }
        }
    } cleanup{pin, done};
    try {
        DevBuf stage(c, chunk_bytes), flag(c, 16);
        CUDA_CHECK(cudaMemsetAsync(flag.ptr, 0, 4, c->stream));
        int64_t r0 = 0;
        for (int b = 0; r0 < m; r0 += chunk_rows, b ^= 1) {
            const int64_t rr = std::min(chunk_rows, m - r0);
            CUDA_CHECK(cudaEventSynchronize(done[b]));  // the copy that last used this staging buffer
            char* dst = (char*)pin[b];
            if (col0 == 0 && ncols == n) {
                if (fseeko(fh.f, data0 + (long long)(r0 * n * 8), SEEK_SET) != 0 ||
                    fread(dst, 8, (size_t)(rr * n), fh.f) != (size_t)(rr * n))
                    fail(BCUR_E_PARSE, std::string(path) + ": truncated entry data");
            } else {
                for (int64_t i = 0; i < rr; ++i) {
                    if (fseeko(fh.f, data0 + (long long)(((r0 + i) * n + col0) * 8), SEEK_SET) != 0 ||
                        fread(dst + (size_t)i * ncols * 8, 8, (size_t)ncols, fh.f) != (size_t)ncols)
                        fail(BCUR_E_PARSE, std::string(path) + ": truncated entry data");
                }
            }
            CUDA_CHECK(cudaMemcpyAsync(stage.ptr, dst, (size_t)rr * ncols * 8, cudaMemcpyHostToDevice, c->stream));
            CUDA_CHECK(cudaEventRecord(done[b], c->stream));
            ops::flag_nonfinite(c, stage.as<double>(), rr * ncols, flag.as<unsigned int>());
            // the chunk is row-major rr × ncols = column-major ncols × rr: transpose into rows r0.. of A
            ops::transpose(c, stage.ptr, BCUR_F64, ncols, rr, ncols, (char*)d->ptr + (size_t)r0 * dtype_size(dtype),
                           dtype, d->ld);
        }
        unsigned int bad = 0;
        CUDA_CHECK(cudaMemcpyAsync(&bad, flag.ptr, 4, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (bad) fail(BCUR_E_PARSE, std::string(path) + ": matrix contains NaN or Inf");  // make_dense → require_finite
    } catch (...) {
        cudaStreamSynchronize(c->stream);
        cudaFree(d->ptr);
        delete d;
        throw;
    }
    *out = d;
    API_END
}

bcur_status bcur_dmat_save_bcur(bcur_ctx ctx, bcur_dmat a, const char* path) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    if (!path) fail(BCUR_E_INVALID_ARGUMENT, "bcur_dmat_save_bcur: null path");
    if (d->m < 1 || d->n < 1) fail(BCUR_E_INVALID_ARGUMENT, "bcur_dmat_save_bcur: empty matrix");
    // row-major fp64 on the device (transpose + widen), then one download
    DevBuf rm(c, (size_t)d->m * d->n * 8);
    ops::transpose(c, d->ptr, d->dtype, d->m, d->n, d->ld, rm.ptr, BCUR_F64, d->n);
    std::vector<double> host((size_t)d->m * d->n);
    CUDA_CHECK(cudaMemcpyAsync(host.data(), rm.ptr, host.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    File fh;
    fh.f = fopen(path, "wb");
    if (!fh.f) fail(BCUR_E_PARSE, std::string("cannot write ") + path);
    const uint64_t rows = (uint64_t)d->m, cols = (uint64_t)d->n;
    if (fwrite("BCUR", 1, 4, fh.f) != 4 || fwrite(&rows, 8, 1, fh.f) != 1 || fwrite(&cols, 8, 1, fh.f) != 1 ||
        fwrite(host.data(), 8, host.size(), fh.f) != host.size())
        fail(BCUR_E_PARSE, std::string("cannot write ") + path);
    API_END
}

// Device → host copy of a result matrix (width_bytes × cols, pitched on both sides), synchronous.
// Pinned (or registered) destinations take one DMA copy.  A pageable destination made the driver
// stage the copy itself at ~4.7 GB/s — c4's 75 MB U took 16 ms of its 55 ms step
// (profiles/r02aw/step_c4.txt) — so it goes through two pinned staging buffers instead: the
// DMA of chunk i + 1 runs while the host copies chunk i into the caller's memory.
static void download_2d(Ctx* c, void* host, size_t host_pitch, const void* dev, size_t dev_pitch, size_t width_bytes,
                        size_t cols) {
    if (!width_bytes || !cols) return;
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, host) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();  // (an unregistered pointer reports an error on older drivers)
    const size_t total = width_bytes * cols;
    if (pinned || total <= ((size_t)1 << 20)) {
        CUDA_CHECK(cudaMemcpy2DAsync(host, host_pitch, dev, dev_pitch, width_bytes, cols, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        return;
    }
    constexpr size_t CHUNK = (size_t)8 << 20;
    static thread_local char* stage[2] = {nullptr, nullptr};
    static thread_local cudaEvent_t done[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; ++b)
        if (!stage[b]) {
            CUDA_CHECK(cudaMallocHost(&stage[b], CHUNK));
            CUDA_CHECK(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
        }
    const size_t cols_per = std::max<size_t>(1, CHUNK / width_bytes);
    if (width_bytes > CHUNK) {  // one column exceeds a chunk: the plain copy
        CUDA_CHECK(cudaMemcpy2DAsync(host, host_pitch, dev, dev_pitch, width_bytes, cols, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        return;
    }
    const size_t nchunks = (cols + cols_per - 1) / cols_per;
    auto issue = [&](size_t i) {
        const size_t c0 = i * cols_per, nc = std::min(cols_per, cols - c0);
        CUDA_CHECK(cudaMemcpy2DAsync(stage[i & 1], width_bytes, (const char*)dev + c0 * dev_pitch, dev_pitch, width_bytes,
                                     nc, cudaMemcpyDeviceToHost, c->stream));
        CUDA_CHECK(cudaEventRecord(done[i & 1], c->stream));
    };
    issue(0);
    for (size_t i = 0; i < nchunks; ++i) {
        CUDA_CHECK(cudaEventSynchronize(done[i & 1]));
        if (i + 1 < nchunks) issue(i + 1);  // (the other buffer: its chunk i − 1 was copied out below)
        const size_t c0 = i * cols_per, nc = std::min(cols_per, cols - c0);
        for (size_t j = 0; j < nc; ++j)
            std::memcpy((char*)host + (c0 + j) * host_pitch, stage[i & 1] + j * width_bytes, width_bytes);
    }
    c->sync();
}

bcur_status bcur_host_alloc(size_t bytes, void** out) {
    API_BEGIN
    if (!out) fail(BCUR_E_INVALID_ARGUMENT, "bcur_host_alloc: null output");
    *out = nullptr;
    if (bytes) CUDA_CHECK(cudaMallocHost(out, bytes));
    API_END
}

bcur_status bcur_host_free(void* p) {
    API_BEGIN
    if (p) CUDA_CHECK(cudaFreeHost(p));
    API_END
}

bcur_status bcur_dmat_download(bcur_ctx ctx, bcur_dmat a, void* host, int64_t ld_host) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    if (ld_host < d->m) fail(BCUR_E_INVALID_ARGUMENT, "bcur_dmat_download: ld_host < m");
    const size_t es = dtype_size(d->dtype);
    if (d->m * d->n > 0) download_2d(c, host, ld_host * es, d->ptr, d->ld * es, d->m * es, d->n);
    else c->sync();
    API_END
}

bcur_status bcur_dmat_wrap(bcur_ctx ctx, int dtype, int64_t m, int64_t n, void* dev_ptr, int64_t ld, bcur_dmat* out) {
    API_BEGIN
    Ctx* c = C(ctx);
    check_dtype(dtype);
    if (m < 0 || n < 0 || ld < std::max<int64_t>(m, 1) || !out) fail(BCUR_E_INVALID_ARGUMENT, "bcur_dmat_wrap: bad shape");
    auto* d = new bcur_dmat_s();
    d->ctx = c;
    d->dtype = dtype;
    d->m = m;
    d->n = n;
    d->ld = ld;
    d->ptr = dev_ptr;
    d->owned = false;
    *out = d;
    API_END
}

bcur_status bcur_dmat_info(bcur_dmat a, int* dtype, int64_t* m, int64_t* n, int64_t* ld, void** dev_ptr) {
    API_BEGIN
    DMat* d = M(a);
    if (dtype) *dtype = d->dtype;
    if (m) *m = d->m;
    if (n) *n = d->n;
    if (ld) *ld = d->ld;
    if (dev_ptr) *dev_ptr = d->ptr;
    API_END
}

bcur_status bcur_dmat_set_shard(bcur_dmat a, int64_t col0, int64_t n_global) {
    API_BEGIN
    DMat* d = M(a);
    if (col0 < 0 || n_global < col0 + d->n) fail(BCUR_E_INVALID_ARGUMENT, "bcur_dmat_set_shard: bad shard");
    d->col0 = col0;
    d->n_global = n_global;
    API_END
}

bcur_status bcur_dmat_destroy(bcur_dmat a) {
    API_BEGIN
    if (!a) return BCUR_OK;
    if (a->ready) {
        cudaEventSynchronize(a->ready);
        cudaEventDestroy(a->ready);
    }
    if (a->owned && a->ptr) {
        cudaSetDevice(a->ctx->device);
        cudaStreamSynchronize(a->ctx->stream);
        cudaFree(a->ptr);
    }
    delete a;
    API_END
}

bcur_status bcur_dmat_generate(bcur_ctx ctx, const bcur_gen_spec* spec, bcur_dmat* out) {
    API_BEGIN
    Ctx* c = C(ctx);
    if (!spec || !out) fail(BCUR_E_INVALID_ARGUMENT, "null spec/output");
    check_dtype(spec->dtype);
    const int64_t m = spec->m, n = spec->n;
    const int64_t ng = spec->n_global > 0 ? spec->n_global : n;
    if (m < 1 || n < 1 || spec->col0 < 0 || spec->col0 + n > ng) fail(BCUR_E_INVALID_ARGUMENT, "generate: bad shape");
    bcur_dmat d = new_dmat(c, spec->dtype, m, n);
    try {
        if (spec->kind == BCUR_GEN_LOWRANK) {
            const int64_t r = spec->rank;
            if (r < 1 || r > std::min(m, ng) || !spec->sigma) fail(BCUR_E_INVALID_ARGUMENT, "generate: need 1 <= rank <= min(m, n)");
            // Gaussian factors → orthonormal (positive-diagonal CholQR2), U scaled by σ
            Mat64 U0(c, m, r), V0(c, ng, r), U(c, m, r), V(c, ng, r), sg(c, r, 1);
            ops::gaussian_matrix(c, spec->seed, 1, m, r, U0.p(), U0.ld);
            ops::gaussian_matrix(c, spec->seed, 2, ng, r, V0.p(), V0.ld);
            if (orth(c, U0.p(), m, r, U0.ld, -1.0, BCUR_F64, U.p(), U.ld, false, nullptr, nullptr) != r ||
                orth(c, V0.p(), ng, r, V0.ld, -1.0, BCUR_F64, V.p(), V.ld, false, nullptr, nullptr) != r)
                fail(BCUR_E_ITERATION_FAILURE, "generate: factor orthonormalisation lost rank");
            CUDA_CHECK(cudaMemcpyAsync(sg.p(), spec->sigma, r * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            ops::scale_columns(c, U.p(), m, r, U.ld, sg.p());
            ops::lowrank_assemble(c, U.p(), V.p(), m, n, r, spec->col0, ng, spec->noise, spec->seed, d->ptr, d->dtype,
                                  d->ld);
        } else if (spec->kind == BCUR_GEN_BIOMETRIC) {
            ops::biometric(c, m, n, spec->col0, ng, spec->seed, d->ptr, d->dtype, d->ld);
        } else {
            fail(BCUR_E_INVALID_ARGUMENT, "generate: unknown kind");
        }
        c->sync();
    } catch (...) {
        bcur_dmat_destroy(d);
        throw;
    }
    d->col0 = spec->col0;
    d->n_global = ng;
    *out = d;
    API_END
}

// ------------------------------------------------------------------- Rng
bcur_status bcur_rng_create(uint64_t seed, bcur_rng* out) {
    API_BEGIN
    if (!out) fail(BCUR_E_INVALID_ARGUMENT, "null output");
    *out = new bcur_rng_s(seed);
    API_END
}
bcur_status bcur_rng_destroy(bcur_rng r) {
    delete r;
    return BCUR_OK;
}
uint64_t bcur_rng_seed(bcur_rng r) { return r->seed; }
uint64_t bcur_rng_next_u64(bcur_rng r) { return r->engine(); }
double bcur_rng_uniform01(bcur_rng r) { return r->uniform01(); }
uint64_t bcur_rng_below(bcur_rng r, uint64_t bound) {  // rng.hpp:25-32
    const uint64_t limit = bound * (UINT64_MAX / bound);
    uint64_t x = r->engine();
    while (x >= limit) x = r->engine();
    return x % bound;
}
double bcur_rng_normal(bcur_rng r) {  // rng.hpp:35-47
    if (r->has_spare) {
        r->has_spare = false;
        return r->spare;
    }
    const double u1 = 1.0 - r->uniform01();
    const double u2 = r->uniform01();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    r->spare = radius * std::sin(angle);
    r->has_spare = true;
    return radius * std::cos(angle);
}
static uint64_t split_seed(uint64_t seed, uint64_t stream) {  // rng.hpp:51-56
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t bcur_rng_split_seed(bcur_rng r, uint64_t stream) { return split_seed(r->seed, stream); }
uint64_t bcur_omega_key(uint64_t seed) { return split_seed(seed, 0x6F6D656761ULL); }

// ---------------------------------------------------------------- kernels
bcur_status bcur_frobenius_norm(bcur_ctx ctx, bcur_dmat a, double* out) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    if (!out) fail(BCUR_E_INVALID_ARGUMENT, "null output");
    *out = std::sqrt(sumsq(c, d));
    API_END
}

bcur_status bcur_block_sq_norms(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G, double* out) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    check_partition(offsets, G, d->n, "block_sq_norms");
    DevBuf off(c, (G + 1) * sizeof(int64_t)), res(c, G * sizeof(double));
    CUDA_CHECK(cudaMemcpyAsync(off.ptr, offsets, (G + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    ops::block_sumsq(c, d->ptr, d->dtype, d->m, d->ld, off.as<int64_t>(), G, res.as<double>());
    CUDA_CHECK(cudaMemcpyAsync(out, res.ptr, G * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    API_END
}

bcur_status bcur_block_leverage(bcur_ctx ctx, bcur_dmat v_k, const int64_t* offsets, int64_t G, double tol,
                                double* scores, double* normalizer) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* v = M(v_k);
    require_orthonormal(c, v, tol, "block_leverage");
    check_partition(offsets, G, -1, "block_leverage");
    if (offsets[G] != v->m) fail(BCUR_E_DIMENSION_MISMATCH, "block_leverage: partition size does not match V_k rows");
    DevBuf off(c, (G + 1) * sizeof(int64_t)), res(c, G * sizeof(double));
    CUDA_CHECK(cudaMemcpyAsync(off.ptr, offsets, (G + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    ops::row_sumsq_blocks(c, v->ptr, v->dtype, v->m, v->n, v->ld, off.as<int64_t>(), G, nullptr, res.as<double>());
    CUDA_CHECK(cudaMemcpyAsync(scores, res.ptr, G * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (normalizer) *normalizer = (double)v->n;
    API_END
}

bcur_status bcur_block_diagnostics(bcur_ctx ctx, bcur_dmat v_k, bcur_dmat u_k, const int64_t* offsets, int64_t G,
                                   double* stable_ranks, double* block_stable_rank, double* incoherence) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* V = M(v_k);
    if (V->dtype != BCUR_F64) fail(BCUR_E_INVALID_ARGUMENT, "block_stable_rank: V_k must be fp64");
    check_partition(offsets, G, V->m, "block_stable_rank");
    require_orthonormal(c, V, 1e-6, "block_stable_rank");  // range-finder bases of fp32 A: ~1e-7
    DevBuf doff(c, (G + 1) * sizeof(int64_t)), fro(c, G * sizeof(double)), spec(c, G * sizeof(double));
    CUDA_CHECK(cudaMemcpyAsync(doff.ptr, offsets, (G + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    ops::block_spectral(c, (const double*)V->ptr, V->ld, V->n, doff.as<int64_t>(), G, fro.as<double>(), spec.as<double>());
    std::vector<double> hf(G), hs(G);
    CUDA_CHECK(cudaMemcpyAsync(hf.data(), fro.ptr, G * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(hs.data(), spec.ptr, G * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    double mn = INFINITY;
    bool zero = false;
    for (int64_t g = 0; g < G; ++g) {
        const double sr = hf[g] > 0.0 ? hf[g] / hs[g] : NAN;  // leverage.cpp:128-139: ZeroBlock
        if (!(hf[g] > 0.0)) zero = true;
        if (stable_ranks) stable_ranks[g] = sr;
        mn = std::min(mn, sr);
    }
    if (block_stable_rank) *block_stable_rank = zero ? NAN : mn;
    if (incoherence && u_k) {  // leverage.cpp:148-153: (m/k)·max_i ‖U_kᵀ e_i‖²
        DMat* U = M(u_k);
        if (U->dtype != BCUR_F64) fail(BCUR_E_INVALID_ARGUMENT, "incoherence: U_k must be fp64");
        require_orthonormal(c, U, 1e-6, "incoherence");
        DevBuf mx(c, sizeof(double));
        ops::max_row_sumsq(c, (const double*)U->ptr, U->m, U->ld, U->n, mx.as<double>());
        double h = 0.0;
        CUDA_CHECK(cudaMemcpyAsync(&h, mx.ptr, sizeof h, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        *incoherence = (double)U->m / (double)U->n * h;
    }
    if (zero) fail(BCUR_E_ZERO_BLOCK, "column_block_stable_ranks: a block has zero Frobenius mass");
    API_END
}

bcur_status bcur_column_leverage(bcur_ctx ctx, bcur_dmat v_k, double tol, double* scores, double* normalizer) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* v = M(v_k);
    require_orthonormal(c, v, tol, "column_leverage");
    DevBuf res(c, v->m * sizeof(double));
    ops::row_sumsq_blocks(c, v->ptr, v->dtype, v->m, v->n, v->ld, nullptr, 0, res.as<double>(), nullptr);
    CUDA_CHECK(cudaMemcpyAsync(scores, res.ptr, v->m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (normalizer) *normalizer = (double)v->n;
    API_END
}

bcur_status bcur_range_finder(bcur_ctx ctx, bcur_dmat a, int64_t k, int64_t p, int64_t q, uint64_t key,
                              bcur_dmat* v_out, bcur_dmat* u_out, double* sigma_out, int64_t* k_eff) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    if (d->m < 1 || d->n < 1) fail(BCUR_E_INVALID_ARGUMENT, "range_finder: matrix must be non-empty");
    Subspace s;
    range_finder(c, d, k, p, q, key, &s, false);
    if (v_out) *v_out = from_mat64(c, s.v, d->n, s.k_eff);
    if (u_out) *u_out = from_mat64(c, s.u, d->m, s.k_eff);
    if (sigma_out) std::memcpy(sigma_out, s.sigma.data(), s.k_eff * sizeof(double));
    if (k_eff) *k_eff = s.k_eff;
    API_END
}

bcur_status bcur_cholesky(bcur_ctx ctx, bcur_dmat g, bcur_dmat r_out, bcur_dmat rinv_out, int* info, double* min_diag) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat *G = M(g), *R = M(r_out), *X = rinv_out ? M(rinv_out) : nullptr;
    const int64_t w = G->m;
    if (G->dtype != BCUR_F64 || R->dtype != BCUR_F64 || (X && X->dtype != BCUR_F64))
        fail(BCUR_E_INVALID_ARGUMENT, "cholesky: matrices must be fp64");
    if (G->n != w || R->m != w || R->n != w || (X && (X->m != w || X->n != w)) || R->ld != w || (X && X->ld != w))
        fail(BCUR_E_DIMENSION_MISMATCH, "cholesky: G, R, R^-1 must be w x w (R and R^-1 with ld = w)");
    if (w < 1) fail(BCUR_E_INVALID_ARGUMENT, "cholesky: empty matrix");
    const int st = cholesky_inverse(c, (const double*)G->ptr, w, G->ld, (double*)R->ptr, X ? (double*)X->ptr : nullptr,
                                    min_diag);
    if (info) *info = st;
    c->sync();
    API_END
}

bcur_status bcur_sketch_product(bcur_ctx ctx, bcur_dmat a, bcur_dmat x, int transpose, bcur_dmat out,
                                double* rows_out) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat *A = M(a), *X = M(x);
    if (X->dtype != BCUR_F64) fail(BCUR_E_INVALID_ARGUMENT, "sketch_product: X must be fp64");
    const int64_t K = transpose ? A->m : A->n, rows = transpose ? A->n : A->m;
    if (X->m != K) fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product: inner dimensions differ");
    if (rows_out) {
        if (!transpose) fail(BCUR_E_INVALID_ARGUMENT, "sketch_product: row sums need transpose=1");
        Mat64 r(c, rows, 1);
        ops::gemm_rowsumsq(c, ops::OP_T, ops::OP_N, rows, X->n, K, A->ptr, A->dtype, A->ld, X->ptr, BCUR_F64, X->ld,
                           r.p());
        CUDA_CHECK(cudaMemcpyAsync(rows_out, r.p(), rows * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    } else {
        DMat* O = M(out);
        if (O->dtype != BCUR_F64 || O->m != rows || O->n != X->n)
            fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product: output must be fp64 rows × N");
        ops::gemm(c, transpose ? ops::OP_T : ops::OP_N, ops::OP_N, rows, X->n, K, 1.0, A->ptr, A->dtype, A->ld,
                  X->ptr, BCUR_F64, X->ld, 0.0, (double*)O->ptr, O->ld);
    }
    c->sync();
    API_END
}

bcur_status bcur_sketch_product_ex(bcur_ctx ctx, bcur_dmat a, bcur_dmat x, int transpose, int flags, bcur_dmat out) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat *A = M(a), *O = M(out);
    if (flags & ~(BCUR_PRODUCT_GRAM | BCUR_PRODUCT_X_UPPER | BCUR_PRODUCT_ROWSQ_F16 | BCUR_PRODUCT_H3 |
                  BCUR_PRODUCT_FAST_ACC | BCUR_PRODUCT_HI_ONLY))
        fail(BCUR_E_INVALID_ARGUMENT, "sketch_product_ex: bad flags");
    if (flags & BCUR_PRODUCT_H3) {
        // the pipelines' 3×FP16 form: A split once by the norms pass into fp16 hi + lo
        DMat* X = x ? M(x) : nullptr;
        const bool gram = (flags & BCUR_PRODUCT_GRAM) != 0;
        if (flags & BCUR_PRODUCT_ROWSQ_F16) fail(BCUR_E_INVALID_ARGUMENT, "sketch_product_ex: H3 has no row-sum form");
        if (A->dtype != BCUR_F32 || A->ld % 4 != 0 || ((uintptr_t)A->ptr % 16) != 0 || !ops::h3_ok(A->m))
            fail(BCUR_E_INVALID_ARGUMENT, "sketch_product_ex: H3 needs fp32 A with m % 64 == 0");
        if (gram ? (x || !transpose) : !X) fail(BCUR_E_INVALID_ARGUMENT, "sketch_product_ex: bad H3 operands");
        const int64_t K = transpose ? A->m : A->n, rows = transpose ? A->n : A->m, N = gram ? A->n : X->n;
        if (!gram && (X->dtype != BCUR_F64 || X->m != K)) fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product_ex: bad X");
        if (O->dtype != BCUR_F64 || O->m != rows || O->n != N)
            fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product_ex: output must be fp64 rows × N");
        DevBuf il(c, (size_t)A->m * A->n * 4), exps(c, (size_t)A->n * sizeof(int)),
            off(c, 2 * sizeof(int64_t)), tot(c, sizeof(double));
        const int64_t h_off[2] = {0, A->n};
        CUDA_CHECK(cudaMemcpyAsync(off.ptr, h_off, sizeof h_off, cudaMemcpyHostToDevice, c->stream));
        ops::block_sumsq(c, A->ptr, A->dtype, A->m, A->ld, off.as<int64_t>(), 1, tot.as<double>(), nullptr, A->m,
                         nullptr, exps.as<int>(), il.as<uint16_t>());
        const int fl = (gram ? ops::GEMM_SYM_UPPER : (flags & BCUR_PRODUCT_X_UPPER) ? ops::GEMM_B_UPPER : 0) |
                       ((flags & BCUR_PRODUCT_FAST_ACC) ? ops::GEMM_FAST_ACC : 0) |
                       ((flags & BCUR_PRODUCT_HI_ONLY) ? ops::GEMM_HI_ONLY : 0);
        if (gram) {  // X = the same matrix, split on its own (K-major X operand)
            ops::SplitF16 xs;
            ops::split_f16(c, A->ptr, A->dtype, A->m, A->n, A->ld, nullptr, &xs);
            ops::umma_h3(c, false, il.as<uint16_t>(), exps.as<int>(), A->m, A->n, ops::view(xs), 1.0, 0.0,
                         (double*)O->ptr, O->ld, fl);
        } else {
            ops::umma_h3(c, !transpose, il.as<uint16_t>(), exps.as<int>(), A->m, A->n, X->ptr, X->dtype, X->n, X->ld,
                         1.0, 0.0, (double*)O->ptr, O->ld, fl);
        }
        c->sync();
        return BCUR_OK;
    }
    if (flags & BCUR_PRODUCT_ROWSQ_F16) {
        DMat* X = x ? M(x) : nullptr;
        if (flags != BCUR_PRODUCT_ROWSQ_F16 || !X || !transpose)
            fail(BCUR_E_INVALID_ARGUMENT, "sketch_product_ex: the fp16 row-sum form takes X and transpose = 1");
        if (A->dtype != BCUR_F32 || A->m % 64 != 0 || A->ld % 4 != 0 || ((uintptr_t)A->ptr % 16) != 0)
            fail(BCUR_E_INVALID_ARGUMENT, "sketch_product_ex: the fp16 row-sum form needs fp32 A with m % 64 == 0");
        if (X->m != A->m) fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product_ex: inner dimensions differ");
        if (O->dtype != BCUR_F64 || O->m != A->n || O->n != 1)
            fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product_ex: row sums go to an fp64 n × 1 output");
        DevBuf a16(c, (size_t)A->m * A->n * 4), exps(c, (size_t)A->n * sizeof(int)), off(c, 2 * sizeof(int64_t)),
            tot(c, sizeof(double));
        const int64_t h_off[2] = {0, A->n};
        CUDA_CHECK(cudaMemcpyAsync(off.ptr, h_off, sizeof h_off, cudaMemcpyHostToDevice, c->stream));
        ops::block_sumsq(c, A->ptr, A->dtype, A->m, A->ld, off.as<int64_t>(), 1, tot.as<double>(), nullptr, A->m,
                         nullptr, exps.as<int>(), a16.as<uint16_t>());
        ops::gemm_rowsumsq_f16(c, A->n, X->n, A->m, a16.as<uint16_t>(), A->m, exps.as<int>(), X->ptr, X->dtype, X->ld,
                               (double*)O->ptr);
        c->sync();
        return BCUR_OK;
    }
    if (flags & BCUR_PRODUCT_GRAM) {
        if (x || !transpose || (flags & BCUR_PRODUCT_X_UPPER))
            fail(BCUR_E_INVALID_ARGUMENT, "sketch_product_ex: the Gram form takes x = NULL and transpose = 1");
        if (O->dtype != BCUR_F64 || O->m != A->n || O->n != A->n)
            fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product_ex: Gram output must be fp64 n × n");
        ops::gemm(c, ops::OP_T, ops::OP_N, A->n, A->n, A->m, 1.0, A->ptr, A->dtype, A->ld, A->ptr, A->dtype, A->ld, 0.0,
                  (double*)O->ptr, O->ld, ops::GEMM_SYM_UPPER);
    } else {
        DMat* X = M(x);
        if (X->dtype != BCUR_F64) fail(BCUR_E_INVALID_ARGUMENT, "sketch_product_ex: X must be fp64");
        const int64_t K = transpose ? A->m : A->n, rows = transpose ? A->n : A->m;
        if (X->m != K) fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product_ex: inner dimensions differ");
        if ((flags & BCUR_PRODUCT_X_UPPER) && X->m != X->n)
            fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product_ex: an upper-triangular X is square");
        if (O->dtype != BCUR_F64 || O->m != rows || O->n != X->n)
            fail(BCUR_E_DIMENSION_MISMATCH, "sketch_product_ex: output must be fp64 rows × N");
        ops::gemm(c, transpose ? ops::OP_T : ops::OP_N, ops::OP_N, rows, X->n, K, 1.0, A->ptr, A->dtype, A->ld, X->ptr,
                  BCUR_F64, X->ld, 0.0, (double*)O->ptr, O->ld, (flags & BCUR_PRODUCT_X_UPPER) ? ops::GEMM_B_UPPER : 0);
    }
    c->sync();
    API_END
}

bcur_status bcur_draw_blocks(bcur_ctx ctx, const double* probs, int64_t G, int64_t g, int mode, const double* uniforms,
                             uint64_t seed, bcur_block_draw* out, double* margins_out) {
    API_BEGIN
    Ctx* c = C(ctx);
    (void)seed;
    if (g < 1) fail(BCUR_E_INVALID_ARGUMENT, "draw_blocks: g must be >= 1");
    if (G < 1 || !probs) fail(BCUR_E_DISTRIBUTION_INVALID, "empty probability vector");
    if (mode != BCUR_WITH_REPLACEMENT && mode != BCUR_WITHOUT_REPLACEMENT) fail(BCUR_E_INVALID_ARGUMENT, "bad mode");
    DevBuf dp(c, G * sizeof(double)), du(c, g * sizeof(double)), dd(c, g * sizeof(bcur_block_draw)),
        dm(c, g * sizeof(double)), st(c, 16);
    CUDA_CHECK(cudaMemcpyAsync(dp.ptr, probs, G * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(du.ptr, uniforms, g * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    ops::distribution_draw(c, dp.as<double>(), G, 0, g, mode, du.as<double>(), dd.as<bcur_block_draw>(), dm.as<double>(),
                           st.as<int>());
    int status = 0;
    CUDA_CHECK(cudaMemcpyAsync(&status, st.ptr, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (status == BCUR_E_DISTRIBUTION_INVALID) fail(BCUR_E_DISTRIBUTION_INVALID, "draw_blocks: probabilities invalid or do not sum to 1");
    if (status == BCUR_E_NOT_ENOUGH_BLOCKS)
        fail(BCUR_E_NOT_ENOUGH_BLOCKS, "draw_blocks: asked for " + std::to_string(g) + " distinct blocks but too few have positive probability");
    if (status != BCUR_OK) fail((bcur_status)status, "draw_blocks failed");
    CUDA_CHECK(cudaMemcpyAsync(out, dd.ptr, g * sizeof(bcur_block_draw), cudaMemcpyDeviceToHost, c->stream));
    if (margins_out)
        CUDA_CHECK(cudaMemcpyAsync(margins_out, dm.ptr, g * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    API_END
}

static bcur_status materialize(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G,
                               const bcur_block_draw* draws, int64_t nd, int rows, bcur_dmat* out) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    const int64_t dim = rows ? d->m : d->n;
    check_partition(offsets, G, -1, "materialize");
    if (offsets[G] != dim)
        fail(BCUR_E_DIMENSION_MISMATCH, rows ? "materialize_rows: A rows do not match partition"
                                             : "materialize_columns: A columns do not match partition");
    if (nd < 1 || !draws) fail(BCUR_E_INVALID_ARGUMENT, "materialize: empty plan");
    int64_t total = 0;
    DevBuf dd, dst, doff;
    upload_draws(c, draws, nd, offsets, G, &total, &dd, &dst, &doff);
    bcur_dmat o = rows ? new_dmat(c, d->dtype, total, d->n) : new_dmat(c, d->dtype, d->m, total);
    ops::gather_blocks(c, d->ptr, d->dtype, d->m, d->n, d->ld, doff.as<int64_t>(), dd.as<bcur_block_draw>(),
                       dst.as<int64_t>(), nd, rows, 1, o->ptr, o->dtype, o->ld);
    c->sync();
    *out = o;
    API_END
}

bcur_status bcur_materialize_columns(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G,
                                     const bcur_block_draw* draws, int64_t nd, bcur_dmat* out) {
    return materialize(ctx, a, offsets, G, draws, nd, 0, out);
}
bcur_status bcur_materialize_row_blocks(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G,
                                        const bcur_block_draw* draws, int64_t nd, bcur_dmat* out) {
    return materialize(ctx, a, offsets, G, draws, nd, 1, out);
}

bcur_status bcur_error_report(bcur_ctx ctx, bcur_dmat a, bcur_dmat cm, bcur_dmat um, bcur_dmat rm, double* abs_err,
                              double* a_norm) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat *A = M(a), *Cm = M(cm), *U = M(um), *R = M(rm);
    if (Cm->m != A->m || R->n != A->n || U->m != Cm->n || U->n != R->m)
        fail(BCUR_E_DIMENSION_MISMATCH, "error_report: C U R shapes do not compose to the shape of A");
    // UR (c × n) then Σ (A − C·UR)²
    Mat64 UR(c, U->m, A->n), tot(c, 1, 1);
    ops::gemm(c, ops::OP_N, ops::OP_N, U->m, A->n, U->n, 1.0, U->ptr, U->dtype, U->ld, R->ptr, R->dtype, R->ld, 0.0,
              UR.p(), UR.ld);
    ops::gemm_resid_sumsq(c, ops::OP_N, ops::OP_N, A->m, A->n, Cm->n, Cm->ptr, Cm->dtype, Cm->ld, UR.p(), BCUR_F64,
                          UR.ld, A->ptr, A->dtype, A->ld, tot.p());
    double h = 0.0;
    CUDA_CHECK(cudaMemcpyAsync(&h, tot.p(), sizeof h, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (abs_err) *abs_err = std::sqrt(std::max(h, 0.0));
    if (a_norm) *a_norm = std::sqrt(sumsq(c, A));
    API_END
}

// --------------------------------------------------------------- pipelines
bcur_status bcur_block_css(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G, const bcur_options* opt,
                           const double* uniforms, double* scores_out, double* normalizer_out,
                           bcur_block_draw* draws_out, double* margins_out, bcur_report* rep) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    if (!opt || !uniforms) fail(BCUR_E_INVALID_ARGUMENT, "block_css: null options/uniforms");
    if (opt->mode != BCUR_WITH_REPLACEMENT && opt->mode != BCUR_WITHOUT_REPLACEMENT) fail(BCUR_E_INVALID_ARGUMENT, "bad mode");
    check_partition(offsets, G, -1, "block_css");
    CssOut o;
    block_css(c, d, offsets, G, *opt, uniforms, &o);
    if (scores_out) std::memcpy(scores_out, o.scores.data(), G * sizeof(double));
    if (normalizer_out) *normalizer_out = o.normalizer;
    if (draws_out) std::memcpy(draws_out, o.draws.data(), o.draws.size() * sizeof(bcur_block_draw));
    if (margins_out) std::memcpy(margins_out, o.margins.data(), o.margins.size() * sizeof(double));
    if (rep) *rep = o.rep;
    API_END
}

bcur_status bcur_greedy_select(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G, const bcur_options* opt,
                               bcur_greedy_step* steps_out, double* residuals_out, bcur_report* rep) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    if (!opt) fail(BCUR_E_INVALID_ARGUMENT, "greedy_select: null options");
    check_partition(offsets, G, -1, "greedy_select");
    GreedyOut o;
    greedy_select(c, d, offsets, G, *opt, &o);
    if (steps_out) std::memcpy(steps_out, o.steps.data(), o.steps.size() * sizeof(bcur_greedy_step));
    if (residuals_out) std::memcpy(residuals_out, o.residuals.data(), G * sizeof(double));
    if (rep) *rep = o.rep;
    API_END
}

bcur_status bcur_block_cur_alg1(bcur_ctx ctx, bcur_dmat a, const int64_t* offsets, int64_t G, int64_t k,
                                const bcur_row_draw* rows, int64_t r, int scaled_rows, int64_t g, int block_mode,
                                const double* uniforms, double* scores_out, double* normalizer_out,
                                bcur_block_draw* draws_out, double* margins_out, double* u_out,
                                bcur_alg1_report* report) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* A = M(a);
    if (!rows || !uniforms || !draws_out || !report) fail(BCUR_E_INVALID_ARGUMENT, "block_cur: null argument");
    if (block_mode != BCUR_WITH_REPLACEMENT && block_mode != BCUR_WITHOUT_REPLACEMENT)
        fail(BCUR_E_INVALID_ARGUMENT, "bad block sampling mode");
    check_partition(offsets, G, A->n, "block_cur");
    Alg1Out o;
    block_cur_alg1(c, A, offsets, G, k, rows, r, scaled_rows != 0, g, block_mode, uniforms, &o);
    if (scores_out) std::memcpy(scores_out, o.scores.data(), G * sizeof(double));
    if (normalizer_out) *normalizer_out = o.normalizer;
    std::memcpy(draws_out, o.draws.data(), g * sizeof(bcur_block_draw));
    if (margins_out) std::memcpy(margins_out, o.margins.data(), g * sizeof(double));
    if (u_out) {
        download_2d(c, u_out, (size_t)o.u.m * 8, o.u.p(), (size_t)o.u.ld * 8, (size_t)o.u.m * 8, o.u.n);
    }
    *report = o.rep;
    API_END
}

bcur_status bcur_block_cur(bcur_ctx ctx, bcur_dmat a, const int64_t* col_offsets, int64_t Gc,
                           const int64_t* row_offsets, int64_t Gr, const bcur_options* opt, const double* uniforms,
                           double* col_scores, double* row_scores, bcur_block_draw* col_draws,
                           bcur_block_draw* row_draws, double* u_out, int64_t ldu, bcur_report* rep) {
    API_BEGIN
    Ctx* c = C(ctx);
    DMat* d = M(a);
    if (!opt || !uniforms) fail(BCUR_E_INVALID_ARGUMENT, "block_cur: null options/uniforms");
    check_partition(col_offsets, Gc, -1, "block_cur columns");
    check_partition(row_offsets, Gr, d->m, "block_cur rows");
    CurOut o;
    block_cur(c, d, col_offsets, Gc, row_offsets, Gr, *opt, uniforms, u_out != nullptr, &o);
    if (col_scores) std::memcpy(col_scores, o.col_scores.data(), Gc * sizeof(double));
    if (row_scores) std::memcpy(row_scores, o.row_scores.data(), Gr * sizeof(double));
    if (col_draws) std::memcpy(col_draws, o.col_draws.data(), o.col_draws.size() * sizeof(bcur_block_draw));
    if (row_draws) std::memcpy(row_draws, o.row_draws.data(), o.row_draws.size() * sizeof(bcur_block_draw));
    if (u_out && o.u_valid) {
        if (ldu < o.u.m) fail(BCUR_E_INVALID_ARGUMENT, "block_cur: ldu < c");
        download_2d(c, u_out, ldu * 8, o.u.p(), o.u.ld * 8, o.u.m * 8, o.u.n);
    }
    if (rep) *rep = o.rep;
    API_END
}

}  // extern "C"
