#include "../paper_1703_06065_b200/csrc/kernels_small.cu"
#include <cstdio>
#include <vector>
using namespace bcur_b200;
namespace bcur_b200 {
#include "tri_prof.inc"
}
int main() {
    int w = 128;
    std::vector<double> h(w * w, 0.0);
    for (int j = 0; j < w; ++j) for (int i = 0; i <= j; ++i) h[i + j * w] = (i == j ? 2.0 : 0.01 / (1 + j - i));
    double *r, *x; long long* ts;
    cudaMalloc(&r, w * w * 8); cudaMalloc(&x, w * w * 8); cudaMalloc(&ts, 64 * 8); cudaMemset(ts, 0, 512);
    cudaMemcpy(r, h.data(), w * w * 8, cudaMemcpyHostToDevice);
    constexpr size_t smem = TRI_SMEM;
    cudaFuncSetAttribute(k_tri_prof, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 3; ++i) k_tri_prof<<<1, ST, smem>>>(r, w, w, x, w, ts);
    cudaDeviceSynchronize();
    long long t[64]; cudaMemcpy(t, ts, 512, cudaMemcpyDeviceToHost);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    long long prev = t[31];
    for (int i = 0; i < 31; ++i) if (t[i]) { printf("ts%d +%lld\n", i, t[i] - prev); prev = t[i]; }
    return 0;
}
