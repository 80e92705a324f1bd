// Micro-benchmark: random-access L2 bandwidth on B200 -- the roofline denominator of the tuple-space
// probe (a6/a7), whose slot and rule tables stay L2-resident.  Every thread issues independent
// 16-byte loads (ld.global.cg: cached in L2 only, as the probe's L1-missing accesses behave) at
// random positions of a table; a 32-byte variant loads two adjacent uint4 (one 32-B sector).
// Reports sectors/s and GB/s of 32-byte sectors touched (what the L2 actually serves).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather scripts/l2_gather.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int kVec>   // 1: one uint4 (16 B) per access, 2: two adjacent uint4 (one 32-B sector)
__global__ void gather(const uint4* __restrict__ t, uint64_t mask16, int iters, uint4* sink) {
    uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll 1
    for (int i = 0; i < iters; i += 8) {
        uint4 v[8][kVec];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            const uint64_t idx = (x & mask16) & ~uint64_t(kVec - 1);
#pragma unroll
            for (int w = 0; w < kVec; ++w)
                asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u][w].x), "=r"(v[u][w].y), "=r"(v[u][w].z), "=r"(v[u][w].w) : "l"(t + idx + w));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int w = 0; w < kVec; ++w) { acc.x ^= v[u][w].x; acc.y += v[u][w].y; acc.z ^= v[u][w].z; acc.w += v[u][w].w; }
    }
    if (acc.x == 0x12345678u && acc.y == 7u) sink[0] = acc;     // keep the loads alive
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    printf("L2 %d MB, %d SMs\n", l2 >> 20, sms);
    uint4* sink;
    cudaMalloc(&sink, 64);
    for (size_t mb : {16, 32, 64, 1024}) {
        const size_t bytes = mb << 20;
        uint4* t;
        cudaMalloc(&t, bytes);
        cudaMemset(t, 1, bytes);
        const uint64_t mask16 = bytes / 16 - 1;               // power-of-two sizes only
        if (bytes & (bytes - 1)) { cudaFree(t); continue; }
        for (int vec : {1, 2})
            for (int tpb : {256}) {
                const int blocks = sms * 8, iters = 4096;
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a);
                    if (vec == 1) gather<1><<<blocks, tpb>>>(t, mask16, iters, sink);
                    else gather<2><<<blocks, tpb>>>(t, mask16, iters, sink);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                }
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                const double accesses = double(blocks) * tpb * iters;
                const double sectors = accesses * (vec == 2 ? 1.0 : 1.0);   // a 16-B or 32-B access touches one sector
                printf("table %4zu MB, %2d B per access: %7.1f G accesses/s, %7.1f GB/s of 32-B sectors, %7.1f GB/s useful\n",
                       mb, 16 * vec, accesses / ms / 1e6, sectors * 32 / ms / 1e6, accesses * 16 * vec / ms / 1e6);
            }
        cudaFree(t);
    }
    return 0;
}
