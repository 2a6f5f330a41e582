// blas.cu — cuBLAS DGEMM for the plain fp64 products of the small factorizations
// (the task rules allow a library for plain GEMMs; every fused hot-path product is a
// hand-written tcgen05 kernel in kernels_umma.cu).
#include <cublas_v2.h>

#include "ops.h"

namespace bcur_b200 {
namespace ops {

namespace {
struct Handle {
    cublasHandle_t h = nullptr;
    ~Handle() {
        if (h) cublasDestroy(h);
    }
};
// per device and stream, per host thread: the blocked Cholesky issues cuBLAS calls on three
// streams concurrently, and a handle's workspace must not be shared between them
thread_local std::map<std::pair<int, cudaStream_t>, Handle> g_handles;
cublasHandle_t handle(Ctx* c) {
    Handle& hd = g_handles[{c->device, c->stream}];
    if (!hd.h) {
        if (cublasCreate(&hd.h) != CUBLAS_STATUS_SUCCESS) fail(BCUR_E_CUDA, "cublasCreate failed");
        cublasSetPointerMode(hd.h, CUBLAS_POINTER_MODE_HOST);
        cublasSetStream(hd.h, c->stream);
    }
    return hd.h;
}
}  // namespace

void cublas_dgemm(Ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                  int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
    const cublasStatus_t st =
        cublasDgemm(handle(c), ta ? CUBLAS_OP_T : CUBLAS_OP_N, tb ? CUBLAS_OP_T : CUBLAS_OP_N, (int)M, (int)N, (int)K,
                    &alpha, A, (int)lda, B, (int)ldb, &beta, C, (int)ldc);
    if (st != CUBLAS_STATUS_SUCCESS) fail(BCUR_E_CUDA, "cublasDgemm failed (" + std::to_string((int)st) + ")");
    c->launches++;
}

// C(upper) = alpha·AᵀA + beta·C(upper), A k×n (ld lda): the symmetric GEMM of the blocked
// Cholesky's trailing update (half the flops of the full product; only the upper
// triangle is ever read)
void cublas_dsyrk_upper_t(Ctx* c, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, double beta,
                          double* C, int64_t ldc) {
    const cublasStatus_t st = cublasDsyrk(handle(c), CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, (int)n, (int)k, &alpha, A,
                                          (int)lda, &beta, C, (int)ldc);
    if (st != CUBLAS_STATUS_SUCCESS) fail(BCUR_E_CUDA, "cublasDsyrk failed (" + std::to_string((int)st) + ")");
    c->launches++;
}

}  // namespace ops
}  // namespace bcur_b200
