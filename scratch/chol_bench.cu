// Times the single-CTA factorization kernels in isolation (includes kernels_small.cu).
#include "../paper_1703_06065_b200/csrc/kernels_small.cu"
#include <cstdio>
#include <vector>
using namespace bcur_b200;
int main() {
    for (int w : {20, 60, 128}) {
        std::vector<double> h(w * w);
        for (int j = 0; j < w; ++j)
            for (int i = 0; i < w; ++i) h[i + j * w] = (i == j ? w + 1.0 : 0.0) + 1.0 / (1 + i + j);
        double *g, *r, *diag; int* info;
        cudaMalloc(&g, w * w * 8); cudaMalloc(&r, w * w * 8); cudaMalloc(&diag, 64); cudaMalloc(&info, 64);
        cudaMemcpy(g, h.data(), w * w * 8, cudaMemcpyHostToDevice);
        constexpr size_t smem_p = (size_t)CP_MAX * CP_LD * sizeof(double);
        cudaFuncSetAttribute(k_chol_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
        cudaFuncSetAttribute(k_cholesky, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            for (int it = 0; it < 20; ++it) k_chol_panel<<<1, CP_T, smem_p>>>(g, w, w, r, w, info, diag, 0, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            cudaEventRecord(e0);
            for (int it = 0; it < 20; ++it)
                k_cholesky<<<1, ST, (size_t)w * (w | 1) * 8>>>(g, w, w, r, w, nullptr, info, diag, 0, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms2; cudaEventElapsedTime(&ms2, e0, e1);
            if (rep == 2) printf("w=%d  chol_panel %.1f us  cholesky %.1f us  (%s)\n", w, ms * 1000 / 20, ms2 * 1000 / 20,
                                 cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
