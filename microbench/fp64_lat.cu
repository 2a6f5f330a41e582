// Microbenchmark: latency of the fp64 building blocks of the small factorizations
// (dependent DFMA chain, fast_rsqrt, shuffle of a double, a 32-step warp Cholesky step).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double fast_rsqrt(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double hx = 0.5 * x;
    r = r * fma(-hx * r, r, 1.5);
    r = r * fma(-hx * r, r, 1.5);
    return r;
}

__global__ void k(double* out, long long* cyc, double seed) {
    const int lane = threadIdx.x & 31;
    double x = seed + lane * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < 1024; ++i) x = fma(x, 0.999999, 1e-7);  // dependent DFMA chain
    long long t1 = clock64();
    double y = x;
    for (int i = 0; i < 256; ++i) y = fast_rsqrt(y + 1.0);       // dependent rsqrt chain
    long long t2 = clock64();
    double z = y;
    for (int i = 0; i < 1024; ++i) z = __shfl_sync(0xffffffffu, z, (lane + 1) & 31) + 1e-9;  // dependent shuffle
    long long t3 = clock64();
    double w = z;
    for (int i = 0; i < 256; ++i) w = sqrt(w + 1.0);             // library sqrt
    long long t4 = clock64();
    double v = w;
    for (int i = 0; i < 256; ++i) v = 1.0 / (v + 1.0);           // IEEE division
    long long t5 = clock64();
    out[threadIdx.x] = x + y + z + w + v;
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / 1024;
        cyc[1] = (t2 - t1) / 256;
        cyc[2] = (t3 - t2) / 1024;
        cyc[3] = (t4 - t3) / 256;
        cyc[4] = (t5 - t4) / 256;
    }
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 1024 * 8);
    cudaMalloc(&c, 64);
    k<<<1, 32>>>(o, c, 1.0);
    k<<<1, 32>>>(o, c, 1.0);
    long long h[5];
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("cycles: DFMA %lld  fast_rsqrt %lld  shfl(double)+DADD %lld  sqrt %lld  div %lld (%s)\n", h[0], h[1], h[2],
           h[3], h[4], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
