// DMMA (mma.sync m8n8k4 .f64) and DFMA issue-rate microbenchmark: the fp64 roofline the
// DMMA GEMM (kernels_dmma.cu) is measured against.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_rate.cu -o /tmp/dmma_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void k_dmma(double* out, int iters, double a, double b) {
    double d[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-3;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma(d[i][0], d[i][1], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += d[i][0] + d[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// dependent chains: latency of one DMMA / DFMA / MUFU.RSQ64H-based rsqrt step (one warp)
__global__ void k_lat(double* out, long long* cyc, double a, double b) {
    double d0 = threadIdx.x * 1e-3, d1 = d0 + 1.0, x = d0 + 2.0, r = 1.0 + d0;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) dmma(d0, d1, a, b);
    long long t1 = clock64();
    for (int i = 0; i < 256; ++i) x = fma(x, a, b);
    long long t2 = clock64();
    for (int i = 0; i < 256; ++i) {
        double y;
        asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r));
        r = y + 1.0;
    }
    long long t3 = clock64();
    double z = x;
    for (int i = 0; i < 256; ++i) z = __shfl_sync(0xffffffffu, z, (threadIdx.x + 1) & 31) * a;
    long long t4 = clock64();
    out[threadIdx.x] = d0 + d1 + x + r + z;
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / 256; cyc[1] = (t2 - t1) / 256; cyc[2] = (t3 - t2) / 256; cyc[3] = (t4 - t3) / 256;
    }
}

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) d[i] = fma(d[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* o;
    cudaMalloc(&o, (size_t)sms * 8 * 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int wpc : {4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k_dmma<8><<<sms * 2, 32 * wpc / 2>>>(o, iters, 1.0000001, 0.9999999);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 256 * 8 * (double)iters * (sms * 2) * (wpc / 2);
        printf("DMMA m8n8k4: %2d warps/SM, 8 accumulators/warp: %.2f TF/s\n", wpc, flops / (ms * 1e-3) / 1e12);
    }
    for (int wpc : {8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k_dfma<<<sms * 2, 32 * wpc / 2>>>(o, iters, 1.0000001, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8 * (double)iters * (sms * 2) * (wpc / 2) * 32;
        printf("DFMA: %2d warps/SM: %.2f TF/s\n", wpc, flops / (ms * 1e-3) / 1e12);
    }
    long long* cyc;
    cudaMalloc(&cyc, 64);
    for (int rep = 0; rep < 2; ++rep) k_lat<<<1, 32>>>(o, cyc, 1.0000001, 1e-9);
    long long hc[4];
    cudaMemcpy(hc, cyc, sizeof hc, cudaMemcpyDeviceToHost);
    printf("latency (cycles, dependent chain): DMMA %lld  DFMA %lld  rsqrt.approx.f64+DADD %lld  SHFL(f64)+DMUL %lld\n",
           hc[0], hc[1], hc[2], hc[3]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
