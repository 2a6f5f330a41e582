// Cold instruction fetch of a long straight-line body executed once by one CTA (the shape of
// the factorization leaves): cycles per instruction, first launch vs repeated launches, and
// the same body as a 64-times executed loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 ifetch.cu -o /tmp/ifetch
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void k_straight(double* out, long long* cyc, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) {
        x0 = fma(x0, a, 1e-9); x1 = fma(x1, a, 1e-9); x2 = fma(x2, a, 1e-9); x3 = fma(x3, a, 1e-9);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x0 + x1 + x2 + x3;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int N>
__global__ void k_loop(double* out, long long* cyc, double a, int reps) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            x0 = fma(x0, a, 1e-9); x1 = fma(x1, a, 1e-9); x2 = fma(x2, a, 1e-9); x3 = fma(x3, a, 1e-9);
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x0 + x1 + x2 + x3;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 4096 * 8);
    cudaMalloc(&c, 64);
    long long h;
    for (int rep = 0; rep < 3; ++rep) {
        k_straight<2048><<<1, 256>>>(o, c, 0.999999);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("straight 8192 DFMA (~128 KB of SASS), 8 warps, launch %d: %lld cycles (%.2f cyc/instr/warp)\n", rep, h,
               (double)h / 8192);
    }
    for (int rep = 0; rep < 3; ++rep) {
        k_straight<2048><<<1, 32>>>(o, c, 0.999999);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("straight 8192 DFMA, 1 warp, launch %d: %lld cycles (%.2f cyc/instr)\n", rep, h, (double)h / 8192);
    }
    for (int rep = 0; rep < 2; ++rep) {
        k_loop<32><<<1, 256>>>(o, c, 0.999999, 64);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("loop 64 x 128 DFMA, 8 warps, launch %d: %lld cycles (%.2f cyc/instr/warp)\n", rep, h, (double)h / 8192);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
