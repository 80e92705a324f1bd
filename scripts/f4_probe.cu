// Probe of the NVFP4 block-scaled MMA on sm_100a (f2's NVFP4 stage, R24): one CTA runs
// D[128 x 256] = sum_k (a[m][k] sfa[m][k/16]) (b[n][k] sfb[n][k/16]) with
// tcgen05.mma.kind::mxf4nvf4.block_scale (M = 128, N = 256, K = 64 per instruction, 4 steps),
// A and B packed e2m1 in K-major SWIZZLE_128B shared memory, the ue4m3 scale factors copied
// shared -> TMEM by tcgen05.cp.32x128b.warpx4 from 512-byte blocks [row % 32][row / 32][4 k].
// Checks the operand layouts (nibble order, scale-factor placement) against a host reference and
// times the MMA issue rate.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f4_probe scripts/f4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 256, K = 256;

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t a) {
    return uint64_t((a & 0x3FFFFu) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
           (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// no swizzle, K-major core matrices of 8 rows x 16 B: rows 16 B apart, 8-row groups 128 B apart
__device__ __forceinline__ uint64_t sdesc_sf(uint32_t a) {
    return uint64_t((a & 0x3FFFFu) >> 4) | (uint64_t(128 >> 4) << 16) | (uint64_t(128 >> 4) << 32) |
           (uint64_t(1) << 46);
}
__device__ __forceinline__ uint32_t idesc_f4(uint32_t n) {
    // block-scaled layout: bits 4-5 are the B scale-factor id (D is always f32), A = B = E2M1
    // (MXF4 format 1) at bits 7 and 10, K-major, N >> 3 at 17,
    // scale format UE4M3 (bit 23 = 0), M >> 4 at 24, sf ids 0
    return (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

__global__ void probe(const uint8_t* ga, const uint8_t* gb, const uint8_t* gsfa, const uint8_t* gsfb, float* d,
                      int reps, long long* cycles, int skip, uint32_t idn) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a = sm;                     // 128 rows x 128 B
    uint8_t* b = a + M * 128;            // 256 rows x 128 B
    uint8_t* sfa = b + N * 128;          // 4 k-steps x 512 B
    uint8_t* sfb = sfa + 4 * 512;        // 4 k-steps x 2 x 512 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    // swizzle: 16-byte unit u of row r at r*128 + ((u ^ (r & 7)) << 4)
    for (int i = tid; i < M * 8; i += blockDim.x) {
        const int r = i / 8, u = i % 8;
        *reinterpret_cast<uint4*>(a + r * 128 + ((u ^ (r & 7)) << 4)) = reinterpret_cast<const uint4*>(ga)[i];
    }
    for (int i = tid; i < N * 8; i += blockDim.x) {
        const int r = i / 8, u = i % 8;
        *reinterpret_cast<uint4*>(b + r * 128 + ((u ^ (r & 7)) << 4)) = reinterpret_cast<const uint4*>(gb)[i];
    }
    for (int i = tid; i < 4 * 512 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sfa)[i] = reinterpret_cast<const uint4*>(gsfa)[i];
    for (int i = tid; i < 8 * 512 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sfb)[i] = reinterpret_cast<const uint4*>(gsfb)[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tslot;
    const uint32_t t_sfa = tm + 256, t_sfb = tm + 272;     // SFA: 4 cols per k-step; SFB: 8
    if (skip & 4) {       // SFA by tcgen05.st from the owning thread (diagonal only), no tcgen05.cp
        const int q = warp & 3, i = tid & 31, r = 32 * q + i;
        // clear all 16 SFA columns of this lane first (TMEM keeps stale data across launches), so
        // a read from any other column or lane quarter would see zero scales
        for (int c = 0; c < 16; ++c)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};"
                         ::"r"(t_sfa + (uint32_t(32 * q) << 16) + c), "r"(0u) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        for (int j = 0; j < 4; ++j) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(sfa + 512 * j + i * 16 + q * 4);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};"
                         ::"r"(t_sfa + (uint32_t(32 * q) << 16) + 4 * j + q), "r"(w) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        (void)r;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) {
        long long t0 = 0;
        for (int rep = 0; rep < reps; ++rep) {
            if (rep == 1) t0 = clock64();
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (skip & 1) break;
                if (!(skip & 4))
                asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                             "@e tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;\n\t}"
                             ::"r"(t_sfa + 4 * j), "l"(sdesc_sf(su32(sfa + 512 * j))));
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                                 "@e tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;\n\t}"
                                 ::"r"(t_sfb + 8 * j + 4 * h), "l"(sdesc_sf(su32(sfb + 1024 * j + 512 * h))));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (skip & 2) break;
                const uint64_t ad = sdesc_sw128(su32(a)) + 2 * j, bd = sdesc_sw128(su32(b)) + 2 * j;
                asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                             ::"r"(tm), "l"(ad), "l"(bd), "r"(idn), "r"(j > 0 ? 1u : 0u),
                               "r"(t_sfa + 4 * j), "r"(t_sfb + 8 * j));
            }
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                     ::"r"(su32(&bar)) : "memory");
        if (tid == 0) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
            if (reps > 1) cycles[0] = clock64() - t0;
        }
    }
    __syncthreads();
    if (tid != 0 || true) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = (warp & 3) * 32 + (tid & 31);
    for (int c = 0; c < N; c += 8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tm + (uint32_t((warp & 3) * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 8; ++j) d[row * N + c + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static float e2m1(int c) {
    const int s = c >> 3, e = (c >> 1) & 3, m = c & 1;
    const float v = e == 0 ? m * 0.5f : (1 + m / 2.0f) * std::ldexp(1.0f, e - 1);
    return s ? -v : v;
}
static float ue4m3(int c) {
    const int e = (c >> 3) & 15, m = c & 7;
    return e == 0 ? (m / 8.0f) * std::ldexp(1.0f, -6) : (1 + m / 8.0f) * std::ldexp(1.0f, e - 7);
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 3;       // bit 0: random A scales, bit 1: random B scales
    const int skip = argc > 2 ? atoi(argv[2]) : 0;      // bit 0: no scale copies, bit 1: no MMAs
    const int variant = argc > 3 ? atoi(argv[3]) : 0;
    const uint32_t id0 = (1u << 7) | (1u << 10) | ((uint32_t(N) >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t idv = variant == 1 ? ((id0 & ~((7u << 7) | (7u << 10))) | (5u << 7) | (5u << 10)) : id0;
    printf("idesc 0x%08x skip %d\n", idv, skip);
    srand(7);
    std::vector<int> ca(M * K), cb(N * K), sa(M * K / 16), sb(N * K / 16);
    for (auto& c : ca) c = rand() & 15;
    for (auto& c : cb) c = rand() & 15;
    const int scodes[4] = {0x30, 0x38, 0x40, 0x3C};       // 0.5, 1, 2, 1.5
    for (auto& s : sa) s = (mode & 1) ? scodes[rand() & 3] : 0x38;
    for (auto& s : sb) s = (mode & 2) ? scodes[rand() & 3] : 0x38;
    std::vector<uint8_t> pa(M * 128), pb(N * 128), psa(4 * 512), psb(8 * 512);
    for (int r = 0; r < M; ++r)
        for (int k = 0; k < K; k += 2) pa[r * 128 + k / 2] = uint8_t(ca[r * K + k] | (ca[r * K + k + 1] << 4));
    for (int r = 0; r < N; ++r)
        for (int k = 0; k < K; k += 2) pb[r * 128 + k / 2] = uint8_t(cb[r * K + k] | (cb[r * K + k + 1] << 4));
    // SF block of k-step j: byte (row % 32) * 16 + (row / 32) * 4 + (k-block within the step)
    for (int r = 0; r < M; ++r)
        for (int kb = 0; kb < K / 16; ++kb)
            psa[(kb / 4) * 512 + (r % 32) * 16 + (r / 32) * 4 + kb % 4] = uint8_t(sa[r * (K / 16) + kb]);
    for (int r = 0; r < N; ++r)
        for (int kb = 0; kb < K / 16; ++kb)
            psb[(kb / 4) * 1024 + (r / 128) * 512 + (r % 32) * 16 + ((r % 128) / 32) * 4 + kb % 4] =
                uint8_t(sb[r * (K / 16) + kb]);
    uint8_t *da, *db, *dsa, *dsb;
    float* dd;
    long long* dc;
    cudaMalloc(&da, pa.size()); cudaMalloc(&db, pb.size()); cudaMalloc(&dsa, psa.size()); cudaMalloc(&dsb, psb.size());
    cudaMalloc(&dd, M * N * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(da, pa.data(), pa.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, pb.data(), pb.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dsa, psa.data(), psa.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dsb, psb.data(), psb.size(), cudaMemcpyHostToDevice);
    const int smem = 1024 + M * 128 + N * 128 + 12 * 512;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 128, smem>>>(da, db, dsa, dsb, dd, 1, dc, skip, idv);
    cudaError_t e = cudaDeviceSynchronize();
    printf("launch: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<float> got(M * N);
    cudaMemcpy(got.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
    // references: nibble order lo-first (hypothesis) and hi-first
    for (int order = 0; order < 2; ++order) {
        double maxerr = 0, maxref = 0;
        int bad = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double s = 0;
                for (int k = 0; k < K; ++k) {
                    const int kk = order ? (k ^ 1) : k;
                    s += double(e2m1(ca[m * K + kk])) * ue4m3(sa[m * (K / 16) + k / 16]) *
                         double(e2m1(cb[n * K + kk])) * ue4m3(sb[n * (K / 16) + k / 16]);
                }
                const double err = std::fabs(s - got[m * N + n]);
                maxerr = std::max(maxerr, err);
                maxref = std::max(maxref, std::fabs(s));
                bad += err > 1e-3 * (1 + std::fabs(s));
            }
        printf("mode %d nibble order %s: max |err| %.4g (max |ref| %.4g), %d / %d mismatches\n", mode,
               order ? "hi-first" : "lo-first", maxerr, maxref, bad, M * N);
    }
    printf("D[0][0..3] = %g %g %g %g\n", got[0], got[1], got[2], got[3]);
    // issue rate: 4 MMAs + 12 scale copies per rep
    probe<<<1, 128, smem>>>(da, db, dsa, dsb, dd, 1001, dc, skip, idv);
    cudaDeviceSynchronize();
    long long cyc = 0;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("1000 reps of (12 tcgen05.cp + 4 MMA 128x256x64): %.1f cycles per MMA (nominal fp4 rate: 128)\n", cyc / 4000.0);
    return 0;
}
