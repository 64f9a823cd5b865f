// tools/tex_microbench.cu -- can the texture path add scattered-gather throughput beside the
// LSU path? Random 32-byte row gathers (1M rows = 32 MB, L2-resident) by
//   ldg : one LDG.256 per row                  tex : two TLD (uint4 texels) per row
//   mix : half the rows by LDG.256, half by TLD
// each alone and with 8 random byte lookups per row in an 8 KB shared map (the run kernel's
// first block). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tm tools/tex_microbench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

__device__ __forceinline__ void ldg8(const uint32_t* p, uint32_t* t) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7])
                 : "l"(p));
}

template <int kMode, int kLook>  // mode 0 ldg, 1 tex, 2 mix (odd k by tex)
__global__ void __launch_bounds__(256) k_gather(const uint32_t* rows, cudaTextureObject_t tex,
                                                const uint32_t* idx, uint64_t n, unsigned* sink) {
    __shared__ uint8_t map[8192 + 16];
    for (uint32_t i = threadIdx.x; i < 8192 + 16; i += 256) map[i] = (i * 2654435761u) >> 31;
    __syncthreads();
    uint32_t acc = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * 256 + threadIdx.x; k < n; k += (uint64_t)gridDim.x * 256) {
        const uint32_t r = __ldg(idx + k);
        uint32_t t[8];
        const bool use_tex = kMode == 1 || (kMode == 2 && ((k >> 5) & 1));
        if (use_tex) {
            const uint4 a = tex1Dfetch<uint4>(tex, 2 * r), b = tex1Dfetch<uint4>(tex, 2 * r + 1);
            t[0] = a.x; t[1] = a.y; t[2] = a.z; t[3] = a.w; t[4] = b.x; t[5] = b.y; t[6] = b.z; t[7] = b.w;
        } else {
            ldg8(rows + (size_t)r * 8, t);
        }
        if (kLook) {
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += map[min(t[q] & 0x3FFFu, 8192u)];
        } else {
            acc += t[0] ^ t[1] ^ t[2] ^ t[3] ^ t[4] ^ t[5] ^ t[6] ^ t[7];
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
    const uint64_t nrows = 1000000, n = 256ull << 20;
    uint32_t *rows, *idx; unsigned* sink;
    cudaMalloc(&rows, nrows * 32); cudaMalloc(&idx, n * 4); cudaMalloc(&sink, 4);
    std::vector<uint32_t> h(n), hr(nrows * 8);
    std::mt19937 g(1);
    for (uint64_t k = 0; k < n; ++k) h[k] = g() % nrows;
    for (auto& v : hr) v = g() % 7200;  // token-like row contents
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(rows, hr.data(), nrows * 32, cudaMemcpyHostToDevice);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = rows;
    rd.res.linear.desc = cudaCreateChannelDesc(32, 32, 32, 32, cudaChannelFormatKindUnsigned);
    rd.res.linear.sizeInBytes = nrows * 32;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    printf("tex create: %s\n", cudaGetErrorString(cudaCreateTextureObject(&tex, &rd, &td, nullptr)));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, auto kern, int blocks) {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a); kern<<<148 * blocks, 256>>>(rows, tex, idx, n, sink); cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("%-14s x%d: %.3f ms %.1f G rows/s (%s)\n", name, blocks, best, n / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int blocks : {4, 8}) {
        run("ldg", k_gather<0, 0>, blocks);
        run("tex", k_gather<1, 0>, blocks);
        run("mix", k_gather<2, 0>, blocks);
        run("ldg+lds8", k_gather<0, 1>, blocks);
        run("tex+lds8", k_gather<1, 1>, blocks);
        run("mix+lds8", k_gather<2, 1>, blocks);
    }
}
