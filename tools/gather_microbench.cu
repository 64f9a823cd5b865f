// tools/gather_microbench.cu -- random 32-byte row gathers (1M rows, L2-resident) into the SM:
// TMA tile::gather4 (4 rows per request, into shared memory, mbarrier) vs one LDG.256 per row.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o g4 tools/gather_microbench.cu
// Result (round 1, B200): LDG.256 275 G rows/s, gather4 90 G rows/s at 8-32 CTAs/SM -> the run
// kernel gathers candidate heads with LDG.256 (profiles/r1_tuning.md).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256) k_gather4(const __grid_constant__ CUtensorMap tm, const uint32_t* idx, uint64_t n, unsigned* sink) {
    __shared__ __align__(128) uint4 buf[2][256][2];  // 2 stages x 256 rows x 32B = 16KB
    __shared__ __align__(8) uint64_t bar[2];
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[b])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    uint32_t acc = 0;
    uint64_t it = 0;
    for (uint64_t base = (uint64_t)blockIdx.x * 256; base < n; base += (uint64_t)gridDim.x * 256, ++it) {
        const uint32_t s = it & 1;
        // warp 0 issues 64 gather4 (256 rows), lane l issues 2
        if (tid < 32) {
            if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(256u * 32u));
            __syncwarp();
            for (uint32_t g = tid; g < 64; g += 32) {
                const uint64_t k = base + g * 4;
                int r0 = idx[k], r1 = idx[k + 1], r2 = idx[k + 2], r3 = idx[k + 3];
                asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                    :: "r"(smem_u32(&buf[s][g * 4][0])), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&bar[s])) : "memory");
            }
        }
        // wait
        asm volatile("{ .reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=; }" :: "r"(smem_u32(&bar[s])), "r"((uint32_t)((it >> 1) & 1)) : "memory");
        const uint4 a = buf[s][tid][0], b = buf[s][tid][1];
        acc += a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
        __syncthreads();
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void __launch_bounds__(256) k_ldg(const uint32_t* rows, const uint32_t* idx, uint64_t n, unsigned* sink) {
    uint32_t acc = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * 256 + threadIdx.x; k < n; k += (uint64_t)gridDim.x * 256) {
        const uint32_t* p = rows + (size_t)idx[k] * 8;
        uint32_t t[8];
        asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(t[0]),"=r"(t[1]),"=r"(t[2]),"=r"(t[3]),"=r"(t[4]),"=r"(t[5]),"=r"(t[6]),"=r"(t[7]) : "l"(p));
        acc += t[0]^t[1]^t[2]^t[3]^t[4]^t[5]^t[6]^t[7];
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const uint64_t nrows = 1000000, n = 256ull << 20;
    uint32_t *rows, *idx; unsigned* sink;
    cudaMalloc(&rows, nrows * 32); cudaMalloc(&idx, n * 4); cudaMalloc(&sink, 4);
    std::vector<uint32_t> h(n); std::mt19937 g(1); 
    // candidates cluster: 70% from a window of 250K rows, like a probe window
    for (uint64_t k = 0; k < n; ++k) h[k] = g() % nrows;
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemset(rows, 1, nrows * 32);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (!fn) { printf("no encode fn\n"); return 1; }
    CUtensorMap tm;
    cuuint64_t dims[2] = {8, nrows}; cuuint64_t strides[1] = {32}; cuuint32_t box[2] = {8, 1}; cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, rows, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc %d\n", (int)r);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a); k_ldg<<<148 * 8, 256>>>(rows, idx, n, sink); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); printf("ldg256: %.3f ms %.1f G rows/s (%s)\n", ms, n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        for (int blocks : {8, 16, 32}) {
            cudaEventRecord(a); k_gather4<<<148 * blocks, 256>>>(tm, idx, n, sink); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b); printf("gather4 x%d: %.3f ms %.1f G rows/s (%s)\n", blocks, ms, n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
}
