// Micro-benchmark: TMEM <-> register bandwidth per SM on B200 (tcgen05.ld / tcgen05.st, 32x32b shapes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw scripts/tmem_bw.cu
// Each CTA (one per SM) allocates 512 columns; every warp streams over its lane quadrant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int X>
__device__ __forceinline__ void ld(uint32_t a, uint32_t* r);
template <>
__device__ __forceinline__ void ld<32>(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(a));
}
template <>
__device__ __forceinline__ void ld<16>(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(a));
}
__device__ __forceinline__ void st32(uint32_t a, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
                   "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
                   "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}

// mode 0: ld x32, wait every `depth` loads; mode 1: ld x16; mode 2: st x32 (wait::st at the end of a pass)
__global__ void bw(int mode, int depth, int reps, long long* cyc, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16);
    const int nw = blockDim.x / 32, per_quad = nw / 4, my = warp >> 2;     // column split among a quadrant's warps
    const int cols = 512 / per_quad, c0 = my * cols;
    uint32_t r[32], acc = 0;
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * i;
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        if (mode == 2) {
            for (int c = c0; c < c0 + cols; c += 32) st32(t + c, r);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        } else if (mode == 3) {          // the GEMM1 epilogue pattern: ld x32, wait, st x32 same columns
            for (int c = c0; c < c0 + cols; c += 32) {
                ld<32>(t + c, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                r[0] += 1;
                st32(t + c, r);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            acc += r[2];
        } else if (mode == 4) {          // same, but the next load is issued before the store
            ld<32>(t + c0, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int c = c0; c < c0 + cols; c += 32) {
                uint32_t r2[32];
                if (c + 32 < c0 + cols) ld<32>(t + c + 32, r2);
                r[0] += 1;
                st32(t + c, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                for (int q = 0; q < 32; ++q) r[q] = r2[q];
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            acc += r[2];
        } else {
            int inflight = 0;
            const int step = mode == 0 ? 32 : 16;
            for (int c = c0; c < c0 + cols; c += step) {
                if (mode == 0) ld<32>(t + c, r); else ld<16>(t + c, r);
                if (++inflight == depth) { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); inflight = 0; acc += r[0]; }
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += r[1];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    long long* cyc; uint32_t* sink;
    cudaMalloc(&cyc, 148 * sizeof(long long));
    cudaMalloc(&sink, 148 * 1024 * 4);
    const char* names[5] = {"ld.x32", "ld.x16", "st.x32", "ld-wait-st", "ld(next)-st-wait"};
    for (int mode = 0; mode < 5; ++mode)
        for (int warps : {4, 8, 16})
            for (int depth : {1, 2, 4, 8}) {
                if (mode >= 2 && depth > 1) continue;
                const int reps = 64;
                bw<<<148, warps * 32>>>(mode, depth, reps, cyc, sink);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                long long h[148];
                cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
                double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
                const double bytes = 128.0 * 512 * 4 * reps;      // whole TMEM, each rep
                printf("%s warps=%2d depth=%d : %.1f B/cycle/SM (%.0f cycles per 256 KB)\n", names[mode], warps, depth,
                       bytes / avg, avg / reps);
            }
    return 0;
}
