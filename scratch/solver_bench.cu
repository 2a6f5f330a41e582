// cuSOLVER potrf / trtri and cuBLAS trsm at the c3 factorization size, for comparison with chol_any/tri_inv_any.
#include <cstdio>
#include <vector>
#include <cusolverDn.h>
#include <cublas_v2.h>
#include <cuda_runtime.h>
__global__ void mk(double* g, int n) {  // SPD: diag-dominant
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n; e += gridDim.x * (long long)blockDim.x) {
        int i = e % n, j = e / n;
        g[e] = (i == j ? n : 0.0) + 1.0 / (1.0 + (i > j ? i - j : j - i));
    }
}
int main() {
    for (int n : {768, 4096}) {
        double *g, *a, *x, *work; int* info;
        cudaMalloc(&g, 8ll * n * n); cudaMalloc(&a, 8ll * n * n); cudaMalloc(&x, 8ll * n * n); cudaMalloc(&info, 4);
        mk<<<1024, 256>>>(g, n);
        cusolverDnHandle_t h; cusolverDnCreate(&h);
        cublasHandle_t b; cublasCreate(&b);
        int lw = 0; cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, n, a, n, &lw);
        cudaMalloc(&work, 8ll * lw);
        size_t dws = 0, hws = 0;
        cusolverDnXtrtri_bufferSize(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, x, n, &dws, &hws);
        void* dw; cudaMalloc(&dw, dws + 8); std::vector<char> hw(hws + 8);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        float ms; const double one = 1.0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemcpy(a, g, 8ll * n * n, cudaMemcpyDeviceToDevice);
            cudaEventRecord(e0);
            cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, n, a, n, work, lw, info);
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 2) printf("n=%d potrf %.3f ms\n", n, ms);
            cudaMemcpy(x, a, 8ll * n * n, cudaMemcpyDeviceToDevice);
            cudaEventRecord(e0);
            cusolverDnXtrtri(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, x, n, dw, dws, hw.data(), hws, info);
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 2) printf("n=%d trtri %.3f ms\n", n, ms);
            cudaMemset(x, 0, 8ll * n * n);
            cudaEventRecord(e0);
            // X = I·R⁻¹ would need I; time the RHS = n×n solve instead
            cublasDtrsm(b, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n, &one, a, n, x, n);
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 2) printf("n=%d trsm %.3f ms\n", n, ms);
        }
        int hi; cudaMemcpy(&hi, info, 4, cudaMemcpyDeviceToHost);
        printf("info %d %s\n", hi, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
