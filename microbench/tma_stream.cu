// Microbenchmark: TMA streaming of a column-major fp32 matrix (m × n) through a
// shared-memory stage ring with no compute — what HBM bandwidth can the A-pass
// producer reach for a given box shape / stage count / CTA count?
//   mode 0: K-major box {bk rows, 128 cols} (AᵀX pattern: bk·4 bytes per column per stage)
//   mode 1: MN-major box {128 rows, bk cols} (A·X pattern: 512 B per column per stage)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1)
k_stream(const __grid_constant__ CUtensorMap tm, int mode, int tiles_m, int tiles_k, int stages, uint32_t stage_bytes,
         int bk, unsigned long long* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* full = (uint64_t*)(smem + stages * stage_bytes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned long long acc = 0;
    int gi = 0;
    for (int t = blockIdx.x; t < tiles_m; t += gridDim.x) {
        // prime the ring, then: wait stage, immediately refill (consumer = nothing)
        const int total = tiles_k;
        int issued = 0;
        auto issue = [&](int i) {
            const int s = (gi + i) % stages;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                         "r"(stage_bytes) : "memory");
            if (mode == 0)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                    ::"r"(smem_u32(smem + s * stage_bytes)), "l"(&tm), "r"(smem_u32(&full[s])), "r"(i * bk),
                    "r"(t * 128) : "memory");
            else
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                    ::"r"(smem_u32(smem + s * stage_bytes)), "l"(&tm), "r"(smem_u32(&full[s])), "r"(t * 128),
                    "r"(i * bk) : "memory");
        };
        for (; issued < stages && issued < total; ++issued) issue(issued);
        for (int i = 0; i < total; ++i) {
            const int s = (gi + i) % stages;
            const uint32_t ph = (uint32_t)((gi + i) / stages) & 1u;
            asm volatile(
                "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}"
                ::"r"(smem_u32(&full[s])), "r"(ph) : "memory");
            acc += *(volatile uint32_t*)(smem + s * stage_bytes);
            if (issued < total) issue(issued++);
        }
        gi += total;
    }
    if (acc == 0x12345) *sink = acc;
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    const int stages = argc > 2 ? atoi(argv[2]) : 4;
    const int bk = argc > 3 ? atoi(argv[3]) : 32;
    const int grid = argc > 4 ? atoi(argv[4]) : 148;
    const long m = 16384, n = 65536;
    float* a;
    cudaMalloc(&a, m * n * 4);
    cudaMemset(a, 0, m * n * 4);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n}, strides[1] = {(cuuint64_t)m * 4};
    cuuint32_t es[2] = {1, 1};
    uint32_t stage_bytes;
    int tiles_m, tiles_k;
    if (mode == 0) {  // AᵀX: box {bk rows, 128 columns}; tiles over columns, K = rows
        cuuint32_t box[2] = {(cuuint32_t)bk, 128};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            bk * 4 <= 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        stage_bytes = bk * 128 * 4;
        tiles_m = (int)(n / 128);
        tiles_k = (int)(m / bk);
    } else {  // A·X: box {128 rows, bk columns}; tiles over rows, K = columns
        cuuint32_t box[2] = {128, (cuuint32_t)bk};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        stage_bytes = 128 * bk * 4;
        tiles_m = (int)(m / 128);
        tiles_k = (int)(n / bk);
    }
    const size_t smem = stages * stage_bytes + 1024 + 256;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) {
        cudaEventRecord(e0);
        k_stream<<<grid, 64, smem>>>(tm, mode, tiles_m, tiles_k, stages, stage_bytes, bk, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it == 2)
            printf("mode %d stages %d bk %d grid %d stage %u B: %.3f ms  %.0f GB/s  (%s)\n", mode, stages, bk, grid,
                   stage_bytes, ms, m * n * 4 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
