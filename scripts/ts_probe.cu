// Probe (run on the B200 box): pin the TMEM layout of a tcgen05.mma A operand held in tensor memory
// ("TS": A in TMEM, B in shared memory), as the bf16 MLP's TS kernel uses it, before writing the kernel.
//   cta_group::2, M = 256 (each CTA of the pair holds 128 rows of A and of D in its own TMEM lanes),
//   N = 128 (each CTA holds 64 rows of B, K-major SWIZZLE_128B), K = 64 as four K = 16 MMAs.
// Hypothesis: row r of A is TMEM lane r; a K = 16 step occupies 8 consecutive 32-bit columns at any
// column address; column c of a step holds bf16 elements k = 2c (bits 0-15) and 2c + 1 (bits 16-31).
// Mode 0 places the four steps contiguously, mode 1 at scattered columns (as the TS kernel's packed
// activations are).  Inputs are small integers, so every product and sum is exact in fp32: the
// check is bit-exact.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o ts_probe scripts/ts_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(const uint16_t* A, const uint8_t* Bsw, float* D, int mode) {
    __shared__ __align__(1024) uint8_t sB[64 * 128];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t slot;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int t = threadIdx.x, w = t >> 5;
    for (int i = t; i < 64 * 128 / 16; i += 128)
        reinterpret_cast<uint4*>(sB)[i] = reinterpret_cast<const uint4*>(Bsw + rank * 8192)[i];
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
    const uint32_t acol0[4] = {192, 200, 208, 216}, acol1[4] = {300, 8, 480, 200};
    const int row = 128 * int(rank) + t;
    for (int ks = 0; ks < 4; ++ks) {
        uint32_t v[8];
        for (int c = 0; c < 8; ++c)
            v[c] = uint32_t(A[row * 64 + 16 * ks + 2 * c]) | (uint32_t(A[row * 64 + 16 * ks + 2 * c + 1]) << 16);
        const uint32_t col = mode ? acol1[ks] : acol0[ks];
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                     ::"r"(tmem + (uint32_t(32 * w) << 16) + col), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),
                       "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    csync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (rank == 0 && w == 0) {
        // kind::f16, D f32, A/B bf16, K-major, N = 128, M = 256
        const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((256u >> 4) << 24);
        for (int ks = 0; ks < 4; ++ks) {
            const uint32_t col = mode ? acol1[ks] : acol0[ks];
            asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(tmem + 64u), "r"(tmem + col), "l"(sdesc(s32(sB) + 32 * ks)), "r"(id), "r"(ks));
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
                     ::"r"(s32(&bar)), "h"(uint16_t(3)) : "memory");
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(ok) : "r"(s32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < 128; c0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tmem + (uint32_t(32 * w) << 16) + 64u + uint32_t(c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 8; ++j) D[row * 128 + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    csync();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static uint16_t bf16_of_int(int v) {   // small integers are exact in bf16
    float f = float(v);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return uint16_t(u >> 16);
}

int main() {
    std::vector<int> a(256 * 64), b(128 * 64);
    srand(7);
    for (auto& x : a) x = rand() % 9 - 4;
    for (auto& x : b) x = rand() % 9 - 4;
    std::vector<uint16_t> ah(256 * 64);
    for (int i = 0; i < 256 * 64; ++i) ah[i] = bf16_of_int(a[i]);
    // B: CTA r holds rows n = 64r .. 64r + 63 (N index), K-major SWIZZLE_128B: byte n*128 + ((k/8) ^ (n%8))*16 + (k%8)*2
    std::vector<uint8_t> bs(2 * 8192);
    for (int n = 0; n < 128; ++n)
        for (int k = 0; k < 64; ++k) {
            const int r = n / 64, nl = n % 64;
            const size_t off = size_t(r) * 8192 + nl * 128 + ((k / 8) ^ (nl % 8)) * 16 + (k % 8) * 2;
            const uint16_t v = bf16_of_int(b[n * 64 + k]);
            std::memcpy(&bs[off], &v, 2);
        }
    uint16_t* dA;
    uint8_t* dB;
    float* dD;
    cudaMalloc(&dA, ah.size() * 2);
    cudaMalloc(&dB, bs.size());
    cudaMalloc(&dD, 256 * 128 * 4);
    cudaMemcpy(dA, ah.data(), ah.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, bs.data(), bs.size(), cudaMemcpyHostToDevice);
    int fails = 0;
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dD, 0, 256 * 128 * 4);
        probe<<<2, 128>>>(dA, dB, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { std::printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
        std::vector<float> d(256 * 128);
        cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < 256; ++m)
            for (int n = 0; n < 128; ++n) {
                long s = 0;
                for (int k = 0; k < 64; ++k) s += long(a[m * 64 + k]) * b[n * 64 + k];
                if (d[m * 128 + n] != float(s)) {
                    if (bad < 5) std::printf("mode %d: D[%d][%d] = %g, expected %ld\n", mode, m, n, d[m * 128 + n], s);
                    ++bad;
                }
            }
        std::printf("TS probe mode %d (%s A columns): %d of %d outputs differ from the exact product\n", mode,
                    mode ? "scattered" : "contiguous", bad, 256 * 128);
        fails += bad;
    }
    std::printf(fails ? "TS layout hypothesis REJECTED\n" : "TS layout hypothesis holds (bit-exact)\n");
    return fails != 0;
}
