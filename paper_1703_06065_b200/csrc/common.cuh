// common.cuh — runtime core shared by every translation unit of libbcur_b200.so:
// error model (errors.hpp:9-57 → bcur_status), device context (stream, pooled
// workspace, collective plumbing), device matrix handle (column-major + ld).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bcur_b200.h"

namespace bcur_b200 {

// ------------------------------------------------------------------ errors
struct Failure : std::runtime_error {
    bcur_status status;
    Failure(bcur_status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(bcur_status s, const std::string& msg) { throw Failure(s, msg); }

inline void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        fail(BCUR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" + std::to_string(line) + ")");
    }
}
#define CUDA_CHECK(x) ::bcur_b200::check_cuda((x), #x, __FILE__, __LINE__)
#define LAUNCH_CHECK(ctx) do { (ctx)->launches++; ::bcur_b200::check_cuda(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); } while (0)

inline size_t dtype_size(int dt) { return dt == BCUR_F32 ? 4 : 8; }

// ---------------------------------------------------------------- context
struct Ctx;

// Pooled device allocation (returned to the context's free list on release).
struct DevBuf {
    Ctx* ctx = nullptr;
    void* ptr = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(Ctx* c, size_t b);
    ~DevBuf();
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ctx(o.ctx), ptr(o.ptr), bytes(o.bytes) { o.ptr = nullptr; o.ctx = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept;
    template <class T> T* as() const { return static_cast<T*>(ptr); }
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sm_count = 148;
    int64_t launches = 0;
    bcur_comm comm{0, 1, nullptr, nullptr};
    // free blocks by size class, each tagged with the stream its last use was enqueued on and
    // a release sequence number
    struct FreeBlk {
        void* p;
        cudaStream_t s;
        uint64_t seq;
    };
    std::multimap<size_t, FreeBlk> free_list;
    uint64_t rel_seq = 0;
    // seen[{to, from}] = release sequence up to which `to` has waited for `from` (order())
    std::map<std::pair<cudaStream_t, cudaStream_t>, uint64_t> seen;
    bool safe_on(const FreeBlk& b, cudaStream_t s) const {
        if (b.s == s) return true;
        auto it = seen.find({s, b.s});
        return it != seen.end() && it->second > b.seq;
    }
    size_t pooled_bytes = 0;
    // pinned host staging for small device→host reads
    void* pinned = nullptr;
    size_t pinned_bytes = 0;

    // Workspace cache over cudaMalloc (large pages, TMA-friendly): blocks are kept in exact
    // size classes (≤ 12.5% rounding), so a repeated decomposition reuses every block and
    // never calls cudaMalloc in steady state.  Reuse is safe in stream order: a block carries
    // the stream that was current when it was released (its last use was enqueued there) and
    // a release sequence number; it is handed out again on that stream, or on another stream
    // that order() has since made wait for the releasing one.
    int64_t allocs = 0, allocs_mark = 0;
    void* acquire(size_t bytes) {
        const size_t want = round(bytes);
        for (auto it = free_list.lower_bound(want); it != free_list.end() && it->first == want; ++it) {
            if (!safe_on(it->second, stream)) continue;
            void* p = it->second.p;
            free_list.erase(it);
            pooled_bytes -= want;
            return p;
        }
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            trim();
            CUDA_CHECK(cudaMalloc(&p, want));
        }
        ++allocs;
        sizes[p] = want;
        return p;
    }
    void release(void* p) {
        if (!p) return;
        free_list.emplace(sizes[p], FreeBlk{p, stream, rel_seq++});
        pooled_bytes += sizes[p];
    }
    void trim() {
        CUDA_CHECK(cudaDeviceSynchronize());  // blocks may be tagged with any of the streams
        for (auto& kv : free_list) {
            cudaFree(kv.second.p);
            sizes.erase(kv.second.p);
        }
        free_list.clear();
        pooled_bytes = 0;
    }
    bool cached(size_t bytes) const {
        auto r = free_list.equal_range(round(bytes));
        for (auto it = r.first; it != r.second; ++it)
            if (safe_on(it->second, stream)) return true;
        return false;
    }
    static size_t round(size_t b) {
        if (b <= 256) return 256;
        size_t p = 256;
        while (p < b && p < (1u << 20)) p <<= 1;
        if (b <= (1u << 20)) return p;
        size_t top = 1;
        while ((top << 1) <= b) top <<= 1;
        const size_t g = std::max<size_t>(top >> 3, 2u << 20);
        return (b + g - 1) / g * g;
    }
    void* host_stage(size_t bytes) {
        if (bytes > pinned_bytes) {
            if (pinned) cudaFreeHost(pinned);
            pinned_bytes = bytes < (1u << 20) ? (1u << 20) : bytes;
            CUDA_CHECK(cudaMallocHost(&pinned, pinned_bytes));
        }
        return pinned;
    }
    void sync() { CUDA_CHECK(cudaStreamSynchronize(stream)); }
    std::map<void*, size_t> sizes;

    // Host → device uploads without a stream synchronization: the source is copied into a pinned
    // ring and the asynchronous copy reads it from there, so the caller's buffer (often on its
    // stack) may go away at once.  The ring is reused only after every stream that copied out
    // of it since its last wrap has been synchronized.  nullptr: too large for the ring.
    static constexpr size_t UP_RING = (size_t)4 << 20;
    char* up_ring = nullptr;
    size_t up_off = 0;
    std::vector<cudaStream_t> up_streams;
    const void* stage_upload(const void* host, size_t bytes) {
        if (bytes > UP_RING / 4) return nullptr;
        if (!up_ring) CUDA_CHECK(cudaMallocHost(&up_ring, UP_RING));
        const size_t b = (bytes + 255) & ~(size_t)255;
        if (up_off + b > UP_RING) {
            for (cudaStream_t s : up_streams) CUDA_CHECK(cudaStreamSynchronize(s));
            up_streams.clear();
            up_off = 0;
        }
        if (std::find(up_streams.begin(), up_streams.end(), stream) == up_streams.end()) up_streams.push_back(stream);
        char* p = up_ring + up_off;
        up_off += b;
        memcpy(p, host, bytes);
        return p;
    }
    // Device → host reads collected into a pinned area and delivered at the next read_all(): a
    // decomposition's small results (scores, statuses, norms) share one stream synchronization.
    static constexpr size_t RD_AREA = (size_t)4 << 20;
    char* rd_area = nullptr;
    size_t rd_off = 0;
    struct RdItem {
        void* host;
        size_t off, bytes;
    };
    std::vector<RdItem> rd_items;
    void read_later(void* host, const void* dev, size_t bytes) {
        if (!bytes) return;
        if (!rd_area) CUDA_CHECK(cudaMallocHost(&rd_area, RD_AREA));
        const size_t b = (bytes + 255) & ~(size_t)255;
        if (bytes > RD_AREA / 2) {  // large: read it directly (synchronizes)
            read_all();
            CUDA_CHECK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, stream));
            sync();
            return;
        }
        if (rd_off + b > RD_AREA) read_all();
        CUDA_CHECK(cudaMemcpyAsync(rd_area + rd_off, dev, bytes, cudaMemcpyDeviceToHost, stream));
        rd_items.push_back({host, rd_off, bytes});
        rd_off += b;
    }
    // one stream synchronization delivers every pending read
    void read_all() {
        try {
            sync();
        } catch (...) {  // the destinations may be gone once the failure unwinds: never deliver them
            rd_items.clear();
            rd_off = 0;
            throw;
        }
        for (const RdItem& it : rd_items) memcpy(it.host, rd_area + it.off, it.bytes);
        rd_items.clear();
        rd_off = 0;
    }

    // Second stream for overlapped work (the blocked Cholesky's look-ahead).  Work on it is
    // forked from `stream` and joined back into it before any buffer it touches is released,
    // so the workspace cache's stream-order reuse rule still holds.
    // A third stream (side2) carries work nothing on the chain waits for until the end (the
    // blocked inverse assembled alongside the factorization).
    // The serial chain itself runs on a high-priority stream (hp) so that the block scheduler
    // places its small kernels ahead of the side streams' wide DSYRK/DGEMM CTAs.
    cudaStream_t side = nullptr, side2 = nullptr, side3 = nullptr, hp = nullptr;
    cudaStream_t up = nullptr;  // host → device uploads (bcur_dmat_upload_async), created on first use
    cudaEvent_t side_ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaStream_t side_stream() {
        if (!side) {
            int lo = 0, hi = 0;
            CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CUDA_CHECK(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo));
            CUDA_CHECK(cudaStreamCreateWithPriority(&side2, cudaStreamNonBlocking, lo));
            CUDA_CHECK(cudaStreamCreateWithPriority(&side3, cudaStreamNonBlocking, lo));
            CUDA_CHECK(cudaStreamCreateWithPriority(&hp, cudaStreamNonBlocking, hi));
            for (auto& e : side_ev) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        return side;
    }
    cudaStream_t side_stream3() {
        side_stream();
        return side3;
    }
    cudaStream_t hp_stream() {
        side_stream();
        return hp;
    }
    cudaStream_t side_stream2() {
        side_stream();
        return side2;
    }
    // make `to` wait for everything enqueued so far on `from`
    void order(cudaStream_t from, cudaStream_t to, int slot) {
        CUDA_CHECK(cudaEventRecord(side_ev[slot], from));
        CUDA_CHECK(cudaStreamWaitEvent(to, side_ev[slot], 0));
        waited(from, to);
    }
    // `to` now waits for everything enqueued on `from` so far: blocks released there are safe on `to`
    void waited(cudaStream_t from, cudaStream_t to) { seen[{to, from}] = rel_seq; }
    // events for fork/join inside one operation (grown on demand, reused across calls)
    std::vector<cudaEvent_t> sync_events;
    cudaEvent_t sync_event(size_t i) {
        while (sync_events.size() <= i) {
            cudaEvent_t e;
            CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            sync_events.push_back(e);
        }
        return sync_events[i];
    }

    // --- per-kernel accounting (CUDA events on this stream; bench roofline) ---
    struct ProfRec {
        std::string tag;
        cudaEvent_t e0, e1;
        double flops, bytes;
    };
    bool prof = false;
    std::vector<ProfRec> prof_recs;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t event() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        CUDA_CHECK(cudaEventCreate(&e));
        return e;
    }
};

// RAII: records [start, stop) events around the kernels launched in its scope.
struct ProfScope {
    Ctx* c;
    size_t idx = (size_t)-1;
    ProfScope(Ctx* ctx, const char* tag, double flops, double bytes) : c(ctx) {
        if (!c->prof) return;
        Ctx::ProfRec r{tag, c->event(), c->event(), flops, bytes};
        CUDA_CHECK(cudaEventRecord(r.e0, c->stream));
        c->prof_recs.push_back(r);
        idx = c->prof_recs.size() - 1;
    }
    ~ProfScope() {
        if (idx != (size_t)-1) cudaEventRecord(c->prof_recs[idx].e1, c->stream);
    }
};

inline DevBuf::DevBuf(Ctx* c, size_t b) : ctx(c), bytes(b) { ptr = b ? c->acquire(b) : nullptr; }
inline DevBuf::~DevBuf() {
    if (ctx && ptr) ctx->release(ptr);
}
inline DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        if (ctx && ptr) ctx->release(ptr);
        ctx = o.ctx; ptr = o.ptr; bytes = o.bytes;
        o.ptr = nullptr; o.ctx = nullptr;
    }
    return *this;
}

// Device matrix: column-major, leading dimension ld (elements).
struct DMat {
    Ctx* ctx = nullptr;
    int dtype = BCUR_F64;
    int64_t m = 0, n = 0, ld = 0;
    void* ptr = nullptr;
    bool owned = false;
    int64_t col0 = 0, n_global = 0;  // column shard
    // bcur_dmat_upload_async: the copy's completion on the context's upload stream; every API
    // use of the matrix first makes the compute stream wait for it (capi.cu M())
    cudaEvent_t ready = nullptr;
    bool pending = false;
    size_t bytes() const { return (size_t)ld * (size_t)n * dtype_size(dtype); }
};

// Round an fp32 value to the nearest TF32 (10-bit mantissa), ties to even — the rounding
// of the X1 (1×TF32) tensor-core passes, shared by the kernels that pre-round A.
__device__ __forceinline__ float rn_tf32_dev(float x) {
    uint32_t u = __float_as_uint(x);
    u += 0xFFFu + ((u >> 13) & 1u);
    return __uint_as_float(u & 0xFFFFE000u);
}

// Lightweight non-owning view used by kernels wrappers.
template <class T>
struct View {
    T* p;
    int64_t m, n, ld;
    __host__ __device__ T& operator()(int64_t i, int64_t j) const { return p[i + j * ld]; }
};

}  // namespace bcur_b200

// Opaque handle types of the C ABI.
struct bcur_ctx_s : bcur_b200::Ctx {};
struct bcur_dmat_s : bcur_b200::DMat {};

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
