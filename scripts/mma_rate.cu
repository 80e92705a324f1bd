// Micro-benchmark: back-to-back tcgen05.mma kind::f16 (bf16 x bf16 -> fp32) throughput on B200 with
// operands resident in shared memory (SWIZZLE_128B K-major, the MLP kernel's layouts):
//   cta_group::1, M = 128, N = 256 (the single kernel) and cta_group::2, M = 256, N = 256 (2SM),
// optionally with a TMA weight stream writing into shared memory at the same time (interference).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_rate scripts/mma_rate.cu -lcuda
#include <cuda.h>
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
__device__ __forceinline__ uint32_t idesc(uint32_t m, uint32_t n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(s32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }

struct Args { int two, n, iters, tma, ts, wu; long long* out; };

__global__ void __launch_bounds__(128, 1) mma_rate(const __grid_constant__ CUtensorMap map, const __grid_constant__ Args a) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = sm;                       // 128 rows x 64 K bf16 = 16 KB
    uint8_t* B = sm + 16384;               // up to 256 rows x 64 K = 32 KB
    uint8_t* T = sm + 16384 + 32768;       // TMA landing zone: 2 x 32 KB
    uint64_t* done = reinterpret_cast<uint64_t*>(T + 65536);
    uint64_t* tfull = done + 1;
    uint32_t* slot = reinterpret_cast<uint32_t*>(tfull + 2);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3F803F80u, 0, 0x3F803F80u, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        bar_init(done, 1);
        bar_init(&tfull[0], 1);
        bar_init(&tfull[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        if (a.two) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    csync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *slot;
    const uint32_t rank = crank();
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 32 && a.tma) {      // background weight stream (TMA into T, 2 x 32 KB ring)
        uint32_t ph[2] = {0, 0};
        const int loads = a.two ? a.iters / 2 : a.iters;   // the kernel's weight need: 32 / 64 B per cycle
        for (int i = 0; i < loads; ++i) {
            const int s = i & 1;
            if (i >= 2) { bar_wait(&tfull[s], ph[s]); ph[s] ^= 1; }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&tfull[s])), "r"(32768) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                         ::"r"(s32(T + s * 32768)), "l"(&map), "r"(s32(&tfull[s])), "r"((i % 8) * 64), "r"((i / 8 % 24) * 256)
                         : "memory");
        }
    }
    if (a.wu && warp == 0 && (!a.two || rank == 0)) {
        // warp-uniform issue: all 32 lanes run the loop, descriptors precomputed (+2 per 32 B of K),
        // one lane elected inside the asm -> no per-MMA ELECT / R2UR.BROADCAST loop in SASS
        const uint32_t id = idesc(a.two ? 256 : 128, a.n);
        const uint64_t a0 = sdesc(s32(A)), b0 = sdesc(s32(B));
        if (threadIdx.x == 0) t0 = clock64();
        for (int i = 0; i < a.iters; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t acc = (i | k) ? 1u : 0u;
                if (a.two)
                    asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem), "l"(a0 + 2 * k), "l"(b0 + 2 * k), "r"(id), "r"(acc));
                else
                    asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem), "l"(a0 + 2 * k), "l"(b0 + 2 * k), "r"(id), "r"(acc));
            }
        if (a.two)
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                         "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
                         ::"r"(s32(done)), "h"(uint16_t(3)) : "memory");
        else
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                         ::"r"(s32(done)) : "memory");
        bar_wait(done, 0);
        if (threadIdx.x == 0) a.out[blockIdx.x] = clock64() - t0;
    } else if (!a.wu && threadIdx.x == 0 && (!a.two || rank == 0)) {
        const uint32_t id = idesc(a.two ? 256 : 128, a.n);
        t0 = clock64();
        for (int i = 0; i < a.iters; ++i)
            for (int k = 0; k < 4; ++k) {
                const uint64_t ad = sdesc(s32(A) + k * 32), bd = sdesc(s32(B) + k * 32);
                const uint32_t acc = (i | k) ? 1u : 0u;
                const uint32_t at = tmem + 256u + uint32_t(k * 8);     // TS: A in TMEM columns 256..
                if (a.ts && a.two)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(tmem), "r"(at), "l"(bd), "r"(id), "r"(acc));
                else if (a.ts)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(tmem), "r"(at), "l"(bd), "r"(id), "r"(acc));
                else if (a.two)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(id), "r"(acc));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(id), "r"(acc));
            }
        if (a.two)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(s32(done)), "h"(uint16_t(3)) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(done)) : "memory");
        bar_wait(done, 0);
        t1 = clock64();
        a.out[blockIdx.x] = t1 - t0;
    }
    if (a.two && rank == 1 && threadIdx.x == 0) bar_wait(done, 0);
    (void)t1;
    __syncthreads();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    csync();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (a.two) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* out;
    cudaMalloc(&out, 1024 * 8);
    void* w;
    const int rows = 24 * 256;
    cudaMalloc(&w, size_t(rows) * 512 * 2);
    cudaMemset(w, 0, size_t(rows) * 512 * 2);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[2] = {512, cuuint64_t(rows)};
    cuuint64_t strides[1] = {1024};
    cuuint32_t box[2] = {64, 256};
    cuuint32_t es[2] = {1, 1};
    reinterpret_cast<EncodeFn>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t smem = 16384 + 32768 + 65536 + 1024 + 64;
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int wu : {0, 1})
    for (int ts : {0, 1})
    for (int two : {0, 1})
        for (int n : {128, 256})
            for (int tma : {0, 1}) {
                if (wu && ts) continue;
                Args a{two, n, 2000, tma, ts, wu, out};
                cudaLaunchConfig_t lc{};
                lc.gridDim = dim3((sms / 2) * 2);
                lc.blockDim = dim3(128);
                lc.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                cudaMemset(out, 0, 1024 * 8);
                cudaError_t e = cudaSuccess;
                for (int rep = 0; rep < 2 && e == cudaSuccess; ++rep) e = cudaLaunchKernelEx(&lc, mma_rate, map, a);
                if (e == cudaSuccess) e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
                std::vector<long long> h(lc.gridDim.x);
                cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
                long long mx = 0;
                for (long long v : h) mx = v > mx ? v : mx;
                const double per = double(mx) / (a.iters * 4);
                const double macs = double(two ? 256 : 128) * n * 16;
                printf("%s%s cta_group::%d M=%d N=%d tma=%d: %.1f cycles per MMA (K=16), %.0f MAC/cycle per %s\n",
                       ts ? "TS (A in TMEM)" : "SS (A in SMEM)", wu ? " warp-uniform issue" : "", two + 1,
                       two ? 256 : 128, n, tma, per, macs / per, two ? "SM pair" : "SM");
            }
    return 0;
}
