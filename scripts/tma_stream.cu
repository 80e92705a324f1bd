// Micro-benchmark: how fast can every SM stream the MLP's weight tensor from L2 into shared memory
// through an S-stage TMA/mbarrier ring?  (The bf16 MLP kernel's weight stream, without the MMAs.)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_stream scripts/tma_stream.cu -lcuda
//
// modes (per stage every CTA must end up with `rows` x 64 bf16 = rows*128 bytes):
//   uc   : cluster 1, one box {64, rows} per stage
//   mc2  : cluster 2, each CTA loads rows/2 and multicasts it to both
//   mc4  : cluster 4, each CTA loads rows/4 and multicasts it to all four
//   2sm  : cluster 2, each CTA loads its own rows-row box with the cta_group::2 form; both complete on the
//          leader's barrier (the bf16 kernel's 2SM weight path: each CTA holds half of an MMA's B)
// The consumer (one thread per CTA; the leader's in 2sm mode) waits `full`, spins `delay` cycles
// (the MMA time of a stage), then releases the stage in every CTA of the cluster.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(s32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ uint32_t rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ void arrive_remote(uint32_t a) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct Args { int mode, csize, stages, rows, delay, nrows_total, passes; long long* out; };

__global__ void stream(const __grid_constant__ CUtensorMap map, const __grid_constant__ Args a) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    const int S = a.stages;
    const uint32_t stage = uint32_t(a.rows) * 128;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * stage);
    uint64_t* empty = full + S;
    const uint32_t r = rank();
    const bool two = a.mode == 3;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], two ? 1 : a.csize); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    csync();
    const int KC = 8;                                          // 64-wide K chunks of a 512-wide row
    const int blocks = a.nrows_total / 256;                    // 256-row N blocks (one MMA's B)
    const long long t0 = clock64();
    if (threadIdx.x == 0) {                                    // producer
        uint32_t s = 0, ph = 0;
        for (int pass = 0; pass < a.passes; ++pass)
            for (int b = 0; b < blocks; ++b)
                for (int kc = 0; kc < KC; ++kc) {
                    if (a.delay < 0) {                         // self-paced: reuse a stage once it landed
                        if ((pass * blocks + b) * KC + kc >= S) bar_wait(&full[s], ph ^ 1);
                    } else {
                        bar_wait(&empty[s], ph ^ 1);
                    }
                    uint8_t* dst = sm + s * stage;
                    if (a.mode == 0) {
                        bar_expect(&full[s], stage);
                        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                                     ::"r"(s32(dst)), "l"(&map), "r"(s32(&full[s])), "r"(kc * 64), "r"(b * 256) : "memory");
                    } else if (!two) {
                        const int part = a.rows / a.csize;
                        const uint16_t mask = uint16_t((1u << a.csize) - 1);
                        bar_expect(&full[s], stage);
                        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;"
                                     ::"r"(s32(dst + r * part * 128)), "l"(&map), "r"(s32(&full[s])), "r"(kc * 64),
                                       "r"(b * 256 + int(r) * part), "h"(mask) : "memory");
                    } else {
                        if (r == 0) bar_expect(&full[s], 2 * stage);
                        asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                                     ::"r"(s32(dst)), "l"(&map), "r"(s32(&full[s]) & 0xFEFFFFFFu), "r"(kc * 64),
                                       "r"(b * 256 + int(r) * a.rows) : "memory");
                    }
                    if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                }
    } else if (threadIdx.x == 32 && (!two || r == 0) && a.delay >= 0) {   // consumer
        uint32_t s = 0, ph = 0;
        for (int pass = 0; pass < a.passes; ++pass)
            for (int b = 0; b < blocks; ++b)
                for (int kc = 0; kc < KC; ++kc) {
                    bar_wait(&full[s], ph);
                    const long long w = clock64();
                    while (clock64() - w < a.delay) {}
                    if (a.mode == 0) {
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[s])) : "memory");
                    } else {
                        for (int q = 0; q < a.csize; ++q) arrive_remote(mapa(s32(&empty[s]), q));
                    }
                    if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                }
    }
    __syncthreads();
    if (threadIdx.x == 0) a.out[blockIdx.x] = clock64() - t0;
    csync();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int nrows_total = 12 * 512 + 512;                   // 12 N=512 layers + output: ~6.3 MB of bf16
    void* w;
    cudaMalloc(&w, size_t(nrows_total) * 512 * 2);
    cudaMemset(w, 0, size_t(nrows_total) * 512 * 2);
    long long* out;
    cudaMalloc(&out, 1024 * sizeof(long long));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    const char* names[] = {"uc", "mc2", "mc4", "2sm"};
    struct Cfg { int mode, csize, rows; };
    const Cfg cfgs[] = {{0, 1, 256}, {0, 1, 128}, {1, 2, 256}, {2, 4, 256}, {3, 2, 128}, {1, 2, 128}, {2, 4, 128}};
    const int delays[] = {-1, 0, 512};
    for (const Cfg& c : cfgs)
        for (int delay : delays)
            for (int S : {2, 3, 4, 6, 8, 12}) {
                if (delay < 0 && c.mode != 0) continue;          // self-paced runs are unicast only
                const size_t smem = size_t(S) * c.rows * 128 + 1024 + 2 * S * 8 + 64;
                if (smem > 220 * 1024) continue;
                CUtensorMap map;
                const int box_rows = c.mode == 0 || c.mode == 3 ? c.rows : c.rows / c.csize;
                cuuint64_t dims[2] = {512, cuuint64_t(nrows_total)};
                cuuint64_t strides[1] = {1024};
                cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
                cuuint32_t es[2] = {1, 1};
                reinterpret_cast<EncodeFn>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es,
                                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                Args a{c.mode, c.csize, S, c.rows, delay, nrows_total, 4, out};
                cudaLaunchConfig_t lc{};
                const int cl = c.csize < 2 ? 2 : c.csize;         // uc: independent CTAs in 2-CTA clusters
                const int grid = (sms / cl) * cl;
                lc.gridDim = dim3(grid);
                lc.blockDim = dim3(64);
                lc.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                cudaError_t e = cudaSuccess;
                for (int rep = 0; rep < 2 && e == cudaSuccess; ++rep) e = cudaLaunchKernelEx(&lc, stream, map, a);
                if (e == cudaSuccess) e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("%s: %s\n", names[c.mode], cudaGetErrorString(e)); return 1; }
                std::vector<long long> h(grid);
                cudaMemcpy(h.data(), out, grid * sizeof(long long), cudaMemcpyDeviceToHost);
                double mx = 0, sum = 0;
                for (long long v : h) { mx = v > mx ? v : mx; sum += v; }
                // bytes every SM ends up holding per pass: the whole tensor in `rows`-row stages
                // (2sm: each CTA holds half of every 256-row block)
                const double per_sm = double(nrows_total) * 512 * 2 * (c.mode == 3 ? 0.5 : double(c.rows) / 256.0) * 4;
                const double stages_total = double(nrows_total / 256) * 8 * 4;
                printf("%-4s rows=%3d S=%2d delay=%3d : %6.1f B/cyc/SM received (max-CTA cycles), %5.0f cycles/stage\n",
                       names[c.mode], c.rows, S, delay, per_sm / mx, mx / stages_total);
            }
    return 0;
}
