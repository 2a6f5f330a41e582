// Times k_tri_inv_upper in isolation (includes kernels_small.cu).
#include "../paper_1703_06065_b200/csrc/kernels_small.cu"
#include <cstdio>
#include <vector>
using namespace bcur_b200;
int main() {
    for (int w : {1, 17, 60, 100, 128}) {
        std::vector<double> h(w * w, 0.0);
        for (int j = 0; j < w; ++j)
            for (int i = 0; i <= j; ++i) h[i + j * w] = (i == j ? 2.0 : 0.01 / (1 + j - i));
        double *r, *x;
        cudaMalloc(&r, w * w * 8); cudaMalloc(&x, w * w * 8);
        cudaMemcpy(r, h.data(), w * w * 8, cudaMemcpyHostToDevice);
        constexpr size_t smem = TRI_SMEM;
        cudaFuncSetAttribute(k_tri_inv_upper, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        {
            k_tri_inv_upper<<<1, ST, smem>>>(r, w, w, x, w);
            std::vector<double> hx(w * w);
            cudaMemcpy(hx.data(), x, w * w * 8, cudaMemcpyDeviceToHost);
            double err = 0;
            for (int i = 0; i < w; ++i) for (int j = 0; j < w; ++j) {
                double s = 0; for (int t = 0; t < w; ++t) s += h[i + t * w] * hx[t + j * w];
                err = fmax(err, fabs(s - (i == j)));
            }
            printf("w=%d max|RX-I| %.3e\n", w, err);
        }
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            for (int it = 0; it < 20; ++it) k_tri_inv_upper<<<1, ST, smem>>>(r, w, w, x, w);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 2) printf("w=%d tri_inv %.1f us (%s)\n", w, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
