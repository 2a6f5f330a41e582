// fp64 FMA throughput of one SM: 1024 threads × 8 independent chains.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double s) {
    double a[8];
    for (int j = 0; j < 8; ++j) a[j] = s + threadIdx.x * 1e-3 + j;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < 512; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(a[j], 0.999999, 1e-7);
    __syncthreads();
    long long t1 = clock64();
    double r = 0;
    for (int j = 0; j < 8; ++j) r += a[j];
    out[threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void kf(float* out, long long* cyc, float s) {
    float a[8];
    for (int j = 0; j < 8; ++j) a[j] = s + threadIdx.x * 1e-3f + j;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < 512; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], 0.999999f, 1e-7f);
    __syncthreads();
    long long t1 = clock64();
    float r = 0;
    for (int j = 0; j < 8; ++j) r += a[j];
    out[threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o; float* of; long long* c; long long h;
    cudaMalloc(&o, 8192); cudaMalloc(&of, 8192); cudaMalloc(&c, 64);
    for (int rep = 0; rep < 2; ++rep) { k<<<1, 1024>>>(o, c, 1.0); }
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA: %lld cycles for %d FMAs -> %.1f FMA/clk/SM\n", h, 1024 * 512 * 8, 1024.0 * 512 * 8 / h);
    for (int rep = 0; rep < 2; ++rep) { kf<<<1, 1024>>>(of, c, 1.0f); }
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA: %lld cycles for %d FMAs -> %.1f FMA/clk/SM\n", h, 1024 * 512 * 8, 1024.0 * 512 * 8 / h);
    return 0;
}
