// Micro-benchmark (B200): issue rate of tcgen05.mma.cta_group::2.kind::f16 with A in TMEM (TS), M = 256,
// N = 128 or 256, warp-uniform issue, for the TMEM column placements the TS MLP kernel uses:
//   D at column 0 / 64 / 128, A steps contiguous from column 256 or at the kernel's packed-h columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ts_rate scripts/ts_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    uint64_t d = 0;
    d |= uint64_t((addr & 0x3FFFFu) >> 4);
    d |= uint64_t(1) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t hcol(int k16) {
    const int k = 16 * k16, half = k >> 8, kk = k & 255;
    return uint32_t(256 * half + (kk < 128 ? kk / 2 : 192 + (kk - 128) / 2));
}

struct Args { int dcol, apack, n, iters, ss, batch; long long* out; };

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) rate(Args a) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sB = sm;                 // 8 K-chunks x 128 rows x 128 B = 128 KB (B half, or A for SS)
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t slot;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int t = threadIdx.x, w = t >> 5;
    for (int i = t; i < 128 * 1024 / 16; i += 128) reinterpret_cast<uint4*>(sB)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    csync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (rank == 0 && w == 0) {
        const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t(a.n) >> 3) << 17) | ((256u >> 4) << 24);
        const uint64_t b0 = sdesc(s32(sB));
        long long t0 = clock64();
        for (int it = 0; it < a.iters; ++it) {
#pragma unroll 1
            for (int st = 0; st < 8; ++st)
              if (a.batch) {
                // four MMAs (one 64-wide K chunk) in one asm block under one elect.sync
                const uint64_t bd = b0 + uint64_t((st * 16384) >> 4);
                const uint32_t d = tmem + uint32_t(a.dcol);
                const uint32_t acc0 = (it | st) != 0;
                if (a.ss)
                    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b64 b1, b2, b3;\n\t"
                                 "add.s64 b1, %1, 2;\n\tadd.s64 b2, %1, 4;\n\tadd.s64 b3, %1, 6;\n\t"
                                 "setp.ne.b32 p, %3, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %1, %2, p;\n\t"
                                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], b1, b1, %2, 1;\n\t"
                                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], b2, b2, %2, 1;\n\t"
                                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], b3, b3, %2, 1;\n\t}"
                                 ::"r"(d), "l"(bd), "r"(id), "r"(acc0));
                else {
                    const uint32_t a0 = tmem + (a.apack ? hcol(st * 4) : 256u + 32u * uint32_t(st));
                    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b32 a1, a2, a3;\n\t"
                                 "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
                                 "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
                                 "setp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t"
                                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, 1;\n\t"
                                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a2], b2, %3, 1;\n\t"
                                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a3], b3, %3, 1;\n\t}"
                                 ::"r"(d), "r"(a0), "l"(bd), "r"(id), "r"(acc0));
                }
              } else
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int k16 = st * 4 + j;
                    const uint32_t acol = a.apack ? hcol(k16) : 256u + 8u * uint32_t(k16 & 31);
                    const uint64_t bd = b0 + uint64_t((st * 16384) >> 4) + uint64_t(2 * j);
                    if (a.ss)
                        asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                     ::"r"(tmem + uint32_t(a.dcol)), "l"(bd), "l"(bd), "r"(id), "r"(k16));
                    else
                        asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                                     ::"r"(tmem + uint32_t(a.dcol)), "r"(tmem + acol), "l"(bd), "r"(id), "r"(k16));
                }
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
                     ::"r"(s32(&bar)), "h"(uint16_t(3)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(ok) : "r"(s32(&bar)) : "memory");
        if (t == 0) a.out[blockIdx.x / 2] = clock64() - t0;
    } else if (rank == 1) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(ok) : "r"(s32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    csync();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 132 * 1024);
    struct C { int dcol, apack, n, ss, batch; const char* what; } cs[] = {
        {64, 1, 128, 0, 1, "BATCHED TS N=128 D@64 A packed-h (kernel)"},
        {0, 0, 128, 0, 1, "BATCHED TS N=128 D@0 A contiguous"},
        {0, 0, 256, 0, 1, "BATCHED TS N=256 D@0 A contiguous"},
        {0, 0, 256, 1, 1, "BATCHED SS N=256"},
        {0, 0, 128, 1, 1, "BATCHED SS N=128"},
        {0, 0, 128, 0, 0, "TS N=128 D@0   A contiguous@256"},
        {64, 0, 128, 0, 0, "TS N=128 D@64  A contiguous@256"},
        {128, 0, 128, 0, 0, "TS N=128 D@128 A contiguous@256"},
        {64, 1, 128, 0, 0, "TS N=128 D@64  A packed-h columns (kernel)"},
        {320, 1, 128, 0, 0, "TS N=128 D@320 A packed-h columns (kernel)"},
        {0, 0, 256, 0, 0, "TS N=256 D@0   A contiguous@256"},
        {0, 0, 256, 1, 0, "SS N=256 D@0"},
        {0, 0, 128, 1, 0, "SS N=128 D@0"},
    };
    for (auto& c : cs)
        for (int grid : {2, 148}) {
            Args a{c.dcol, c.apack, c.n, 200, c.ss, c.batch, d};
            rate<<<grid, 128, 132 * 1024>>>(a);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { std::printf("%s: %s\n", c.what, cudaGetErrorString(e)); return 1; }
            std::vector<long long> h(grid / 2);
            cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (auto x : h) mx = x > mx ? x : mx;
            std::printf("%-45s grid %3d: %.1f cycles per MMA (floor %d)\n", c.what, grid, double(mx) / (200.0 * 32),
                        c.n / 2);
        }
    return 0;
}
