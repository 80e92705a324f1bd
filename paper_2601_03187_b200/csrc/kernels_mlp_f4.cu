// N2-f4 (its "later NVFP4" stage): TaNG's residual MLP with NVFP4 GEMMs
// on the 5th-gen tensor cores (tcgen05.mma kind::mxf4nvf4 block_scale), one persistent kernel for
// sm_100a, hidden width N = 256.
//
// What it computes (§6.1, Eq. 1-2; "precision quantization" P:304 read as
// DESIGN.md R24): the fp8 chain of kernels_mlp_f8.cu (R23: per-tensor power-of-two weight scales,
// per-layer power-of-two activation scales, folded epilogue constants) with every e4m3 tensor
// replaced by NVFP4: e2m1 codes in blocks of 16 along K, each block with an unsigned e4m3 scale
// sf = e4m3(max / 6); the tensor core multiplies code * sf (scale vectors in TMEM).
//   h0  -> y = ReLU(fma(D0, 1/s_h0, b0/s_h0))                      (a3, exact bf16 split, R22)
//   u   -> y = ReLU(fma(D1, m1, b1/s_u))                            (a4 GEMM1)
//   h'  -> y = ReLU(fma(D2, m2, hdq r2 + b2/s_h'))                 (a4 GEMM2; hdq = code * sf of h,
//                                                                     r2 = s_h / s_h')
//   each y is quantised per block of 16: sf = e4m3(max(y) * (1/6)), codes = e2m1(y * rcp(sf))
//   logits = fma(D, mo, bo); pred = argmax / top-k (ties -> lower index)                    (a5)
//
// Design:
//   * TMEM (512 columns) holds the fp32 accumulator [0, Cp <= 320), the A scale factors (16
//     columns: 4 per K = 64 step) and the B scale factors (2 x 32 columns: 8 per K step, output
//     passes 0 / 1).  That is why the kernel is single-tile (one 128-packet tile in flight per
//     CTA, 1 CTA per SM) and why N is fixed at 256: a second accumulator (dual-tile) or N = 512
//     would leave no columns for the scale vectors.
//   * Epilogue: 16 warps, four per TMEM lane quadrant, each thread one packet row x 64 columns =
//     exactly one K = 64 step of the next GEMM, so its 4 block scales are one 32-bit word of the
//     512-byte scale block [row % 32][row / 32][4] that tcgen05.cp.32x128b.warpx4 copies to TMEM.
//   * A tile: 128 rows x 128 B (256 e2m1 values, K-major SWIZZLE_128B); layer 0 reuses it for the
//     bf16 split operand (K = 48).
//   * Weights: e2m1 [2BN + Cp][128 B] streamed by TMA, one 256-row box per GEMM pass, plus its
//     4 KB of pre-laid-out scale blocks by a bulk copy into the same stage; the MMA warp copies
//     them to TMEM (tcgen05.cp, ordered before the MMAs that read them).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/tang.h"
#include "tang_internal.h"
#include "tc_ptx.h"

namespace tang {

struct F4Plan {
    CUtensorMap tmap4;       // e2m1 weights [2BN + Cp][128] bytes, box {128, 256}
    CUtensorMap tmap0;       // layer-0 split operand [N][64] bf16, box {64, 256}
    WeightsF4 w;
    int stages;
    size_t smem;
    int grid;
};

namespace {

using namespace tc;
constexpr int kN = 256;
constexpr int kEpiThreads = 512, kThreads = 640, kProdWarp = 16, kMmaWarp = 17;   // warps 18, 19 idle
// setmaxnreg acts on warpgroups and only moves registers inside the CTA's launch allocation
// (20 warps launch at 96): (104 - 96) x 16 epilogue warps = (96 - 64) x 4 control warps.  At the
// former 112 / 32 split the producer / MMA warps spilled (ptxas -v)
constexpr uint32_t kEpiRegs = 104, kCtlRegs = 64;
constexpr uint32_t kLaunchRegs = (65536u / kThreads) & ~7u;
static_assert((kEpiRegs - kLaunchRegs) * 16 <= (kLaunchRegs - kCtlRegs) * 4, "setmaxnreg budget");
constexpr uint32_t kStageW = 256 * 128, kStageSF = 8 * 512, kStage = kStageW + kStageSF;
// TMEM columns: accumulator [0, 320), A scales [320, 336) (4 per K step), B scales 2 x 64 from 336
// (double-buffered by GEMM parity so the next GEMM's copies are issued early; 32 per output pass)
constexpr uint32_t kTmemCols = 512, kSfaCol = 320, kSfbCol = 336;
constexpr float kSixth = 1.0f / 6.0f;

struct F4Params {
    const void* hdr;
    size_t n;
    uint32_t k;
    uint32_t* pred;
    float* logits;
    const float* consts;     // [b0/s_h0 (N) | b1/s_u (B N) | b2/s_h' (B N) | bo (Cp)]
    const uint8_t* sf;       // [2B + 2 slots][8 blocks][512 B] weight scale blocks
    int B, C, Cp, stages;
    uint8_t* dbg;            // optional [(2B+1)][n][144]: 128 code bytes + 16 scale bytes per row
    long long* trace;        // optional clock64 stamps of block 0, first 4 tiles: [4][2B+2][8] (scripts/mlp_trace_f4.py)
    float inv_sh0, mo;
    float m1[kMaxBlocksF8], m2[kMaxBlocksF8];
    float r2[kMaxBlocksF8];       // s_h / s_h' of block b (power of two): skip = hdq * r2 in y units
    uint16_t r2h[kMaxBlocksF8];   // r2 as f16 bits ...
    int r2h_ok;                   // ... when sf * r2 is an exact f16 for every e4m3 sf (mixed-precision skip)
};

__device__ __forceinline__ uint32_t idesc_f4(uint32_t n) {
    // block-scaled layout: bits 4-5 = B scale-factor id (0), A = B = E2M1 (format 1) at bits 7 and
    // 10, K-major, N >> 3 at bit 17, scale format UE4M3 (bit 23 = 0), M >> 4 at bit 24
    return (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
// scale blocks: no swizzle, K-major core matrices of 8 rows x 16 B (rows 16 B apart, groups 128 B)
__device__ __forceinline__ uint64_t sdesc_sf(uint32_t a) {
    return uint64_t((a & 0x3FFFFu) >> 4) | (uint64_t(128 >> 4) << 16) | (uint64_t(128 >> 4) << 32) |
           (uint64_t(1) << 46);
}
// warp-uniform issue (tc_ptx.h): the whole issuer warp executes these, one lane is elected
__device__ __forceinline__ void mma_f4_w(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc, uint32_t sfa,
                                         uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
        ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void cp_sf_w(uint32_t taddr, uint64_t desc) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;\n\t}" ::"r"(taddr), "l"(desc));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ float4 lds4f(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
// (o0, o1) = (a0 b0 + c0, a1 b1 + c1): one packed FFMA2 (two IEEE fp32 fmas)
__device__ __forceinline__ void fma2(float& o0, float& o1, float a0, float a1, float b0, float b1, float c0, float c1) {
    asm("{\n\t.reg .b64 a, b, c, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
        "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(o0), "=f"(o1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ void mul2(float& o0, float& o1, float a0, float a1, float b) {
    asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %4};\n\t"
        "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(o0), "=f"(o1) : "f"(a0), "f"(a1), "f"(b));
}
// 8 values -> 8 e2m1 codes (ReLU, round to nearest even, saturating at 6); value 2i in the low
// nibble of byte i (the host packs the weights the same way)
__device__ __forceinline__ uint32_t e2m1x8(const float* x) {
    uint32_t r;
    asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
        "cvt.rn.satfinite.relu.e2m1x2.f32 b0, %2, %1;\n\t"
        "cvt.rn.satfinite.relu.e2m1x2.f32 b1, %4, %3;\n\t"
        "cvt.rn.satfinite.relu.e2m1x2.f32 b2, %6, %5;\n\t"
        "cvt.rn.satfinite.relu.e2m1x2.f32 b3, %8, %7;\n\t"
        "mov.b32 %0, {b0, b1, b2, b3};\n\t}"
        : "=r"(r) : "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]), "f"(x[7]));
    return r;
}
// NVFP4 quantisation of 32 consecutive values of one row (two blocks, R24): q = 16 code bytes,
// returns the two scale bytes (block 0 low)
__device__ __forceinline__ uint32_t quant32(float (&v)[32], uint32_t (&q)[4]) {
    float a0 = 0.0f, a1 = 0.0f;                 // max(0, ...) = the maximum after ReLU
#pragma unroll
    for (int j = 0; j < 16; j += 2) { a0 = fmax3(a0, v[j], v[j + 1]); a1 = fmax3(a1, v[16 + j], v[17 + j]); }
    uint16_t sc;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(sc) : "f"(a1 * kSixth), "f"(a0 * kSixth));
    uint32_t h;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"(sc));
    const __half2 hs = *reinterpret_cast<const __half2*>(&h);
    const float s0 = __low2float(hs), s1 = __high2float(hs);
    float r0, r1;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(s0));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(s1));
    r0 = s0 > 0.0f ? r0 : 0.0f;                 // sf = 0: every code 0
    r1 = s1 > 0.0f ? r1 : 0.0f;
#pragma unroll
    for (int j = 0; j < 32; j += 2) mul2(v[j], v[j + 1], v[j], v[j + 1], j < 16 ? r0 : r1);
#pragma unroll
    for (int w = 0; w < 4; ++w) q[w] = e2m1x8(v + 8 * w);
    return sc;
}
// skip terms of 8 codes (one word) of the block input h with block scale byte sb:
// o[j] = code_j * (sf * r2) + c[j]  (code * sf * r2 is exact; one fp32 rounding per add).
// Mixed path: sf * r2 as an exact f16, then fma.rn.f32.f16 (f16 x f16 exact product + f32 add);
// otherwise the codes go to fp32 first.
template <bool kMixed>
__device__ __forceinline__ void skip8(uint32_t w, uint32_t sb, uint16_t r2h, float r2, const float* c, float* o) {
    uint32_t sh;
    asm("{\n\t.reg .b16 s;\n\tcvt.u16.u32 s, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, s;\n\t}" : "=r"(sh) : "r"(sb));
    uint32_t h[4];
    asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\tmov.b32 {b0, b1, b2, b3}, %4;\n\t"
        "cvt.rn.f16x2.e2m1x2 %0, b0;\n\tcvt.rn.f16x2.e2m1x2 %1, b1;\n\t"
        "cvt.rn.f16x2.e2m1x2 %2, b2;\n\tcvt.rn.f16x2.e2m1x2 %3, b3;\n\t}"
        : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]) : "r"(w));
    if (kMixed) {
        uint16_t g;
        asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\tmul.rn.f16 %0, lo, %2;\n\t}" : "=h"(g) : "r"(sh), "h"(r2h));
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm("{\n\t.reg .b16 l, u;\n\tmov.b32 {l, u}, %2;\n\t"
                "fma.rn.f32.f16 %0, l, %3, %4;\n\tfma.rn.f32.f16 %1, u, %3, %5;\n\t}"
                : "=f"(o[2 * j]), "=f"(o[2 * j + 1]) : "r"(h[j]), "h"(g), "f"(c[2 * j]), "f"(c[2 * j + 1]));
    } else {
        const float g = __low2float(*reinterpret_cast<const __half2*>(&sh)) * r2;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const __half2 p = *reinterpret_cast<const __half2*>(&h[j]);
            fma2(o[2 * j], o[2 * j + 1], __low2float(p), __high2float(p), g, g, c[2 * j], c[2 * j + 1]);
        }
    }
}
__device__ __forceinline__ bool better(float z, int c, float bz, int bc) { return z > bz || (z == bz && c < bc); }

// kDbg: dump every GEMM input (tests); kMixed: the skip's f16 x f16 + f32 fma path (r2h_ok)
template <bool kDbg, bool kMixed>
__global__ void __launch_bounds__(kThreads, 1)
mlp_f4_kernel(const __grid_constant__ CUtensorMap tmap4, const __grid_constant__ CUtensorMap tmap0,
              const __grid_constant__ F4Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages, B = p.B;
    uint8_t* act = smem;                                     // 128 rows x 128 B
    const uint32_t act_s = smem_u32(act);
    uint8_t* wst = smem + kM * 128;                          // S x (32 KB weights + 4 KB scales)
    uint64_t* full = reinterpret_cast<uint64_t*>(wst + S * kStage);
    uint64_t* empty = full + S;
    uint64_t* acc_full = empty + S;
    uint64_t* act_ready = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(act_ready + 1);
    const int nv = kN + 2 * B * kN + p.Cp;
    const uint32_t sb0 = smem_u32(wst + S * kStage + 256);
    const uint32_t sb1 = sb0 + 4u * kN, sc2 = sb1 + 4u * B * kN, sbo = sc2 + 4u * B * kN;
    for (int v = threadIdx.x; v < nv / 4; v += blockDim.x)
        sts128(sb0 + 16u * v, __ldg(reinterpret_cast<const uint4*>(p.consts) + v));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = 2 * B + 1;
    const size_t ntiles = (p.n + kM - 1) / kM;
    const int nq_out = p.Cp > kN ? 2 : 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(acc_full, 1);
        mbar_init(act_ready, kEpiThreads / 32);   // warp_arrive
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap4)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap0)) : "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(tmem_slot)), "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kProdWarp) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs));
      if (warp == kProdWarp) {
        // ===== TMA producer: one 256-row box (+ its scale blocks) per GEMM pass =====
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(&empty[s], ph ^ 1);                    // layer 0: bf16 split operand
                mbar_expect_tx(&full[s], kStageW);
                tma_load_2d(wst + s * kStage, &tmap0, &full[s], 0, 0);
                if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                for (int g = 0; g < L; ++g) {
                    const bool is_out = g == L - 1;
                    const int row0 = is_out ? 2 * B * kN : ((g & 1) ? (B + g / 2) * kN : (g / 2) * kN);
                    const int slot0 = is_out ? 2 * B : ((g & 1) ? B + g / 2 : g / 2);
                    for (int q = 0; q < (is_out ? nq_out : 1); ++q) {
                        mbar_wait(&empty[s], ph ^ 1);
                        mbar_expect_tx(&full[s], kStage);
                        tma_load_2d(wst + s * kStage, &tmap4, &full[s], 0, row0 + q * kN);
                        bulk_load(wst + s * kStage + kStageW, p.sf + size_t(slot0 + q) * kStageSF, kStageSF, &full[s]);
                        if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                    }
                }
            }
        }
      } else if (warp == kMmaWarp) {
        // ===== MMA issuer (whole warp, one lane elected per instruction) =====
        // The B scale vectors of GEMM g + 1 are copied to TMEM right after GEMM g's MMAs are issued
        // (buffer (g + 1) & 1; its previous user, GEMM g - 1, completed before act_ready of g), so
        // only the MMAs wait for the epilogue.  The A scales are written by the epilogue itself.
        uint32_t s = 0, ph = 0, aph = 0;
        const uint64_t a_d0 = sdesc(act_s), w_d0 = sdesc(smem_u32(wst));
        const uint32_t t_sfa = tmem + kSfaCol;
        auto nq_of = [&](int g) { return g == L - 1 ? nq_out : 1; };
        auto sfb_prefetch = [&](int g) {         // GEMM g's stages start at the consumer position
            uint32_t ps = s, pph = ph;
            for (int q = 0; q < nq_of(g); ++q) {
                mbar_wait(&full[ps], pph);
                tc_fence_after();
                const uint32_t st = smem_u32(wst + ps * kStage) + kStageW;
                const uint32_t t_sfb = tmem + kSfbCol + 64 * (g & 1) + 32 * q;
#pragma unroll
                for (int j = 0; j < 8; ++j) cp_sf_w(t_sfb + 4 * j, sdesc_sf(st + 512 * j));
                if (++ps == uint32_t(S)) { ps = 0; pph ^= 1; }
            }
        };
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            // layer 0: bf16 split operands (R22), K = 48, kind::f16
            mbar_wait(act_ready, aph);
            aph ^= 1;
            tc_fence_after();
            long long* itr = (p.trace && blockIdx.x == 0 && t < 4 * gridDim.x && lane == 0)
                                 ? p.trace + (t / gridDim.x) * (L + 1) * 8 : nullptr;
            if (itr) itr[0] = clock64();
            mbar_wait(&full[s], ph);
            tc_fence_after();
            {
                const uint64_t b_d = w_d0 + uint64_t((s * kStage) >> 4);
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    mma_bf16_w(tmem, a_d0 + uint64_t(2 * j), b_d + uint64_t(2 * j), idesc(uint32_t(kN)), j);
            }
            mma_commit_w(&empty[s]);
            if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
            mma_commit_w(acc_full);
            sfb_prefetch(0);
            if (itr) itr[1] = clock64();
            for (int g = 0; g < L; ++g) {
                const bool is_out = g == L - 1;
                const int nq = nq_of(g);
                mbar_wait(act_ready, aph);                   // A codes + A scales written
                aph ^= 1;
                tc_fence_after();
                if (itr) itr[8 * (g + 1)] = clock64();
                for (int q = 0; q < nq; ++q) {
                    mbar_wait(&full[s], ph);                 // (already complete: sfb_prefetch waited)
                    tc_fence_after();
                    const uint32_t t_sfb = tmem + kSfbCol + 64 * (g & 1) + 32 * q;
                    const uint64_t b_d = w_d0 + uint64_t((s * kStage) >> 4);
                    const uint32_t nmma = uint32_t(min(kN, (is_out ? p.Cp : kN) - q * kN));
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        mma_f4_w(tmem + uint32_t(q * kN), a_d0 + uint64_t(2 * j), b_d + uint64_t(2 * j), idesc_f4(nmma),
                                 j > 0 ? 1u : 0u, t_sfa + 4 * j, t_sfb + 8 * j);
                    mma_commit_w(&empty[s]);
                    if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                }
                mma_commit_w(acc_full);
                if (g + 1 < L) sfb_prefetch(g + 1);
                if (itr) itr[8 * (g + 1) + 1] = clock64();
            }
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
        // ===== epilogue: thread = packet row r, columns [64 grp, 64 grp + 64) = one K step =====
        const int quad = warp & 3, grp = warp >> 2;
        const int r = quad * 32 + lane;
        const uint32_t t_row = tmem + (uint32_t(quad * 32) << 16);
        const int c00 = grp * 64;
        // this thread's A-scale word (K step grp, 4 blocks): TMEM lane r, column kSfaCol + 4 grp + quad --
        // the tensor core's datapath `quad` reads the scales of rows 32 quad .. 32 quad + 31 from its own
        // lane quarter, column (row / 32) of the K step's 4 (scripts/f4_probe.cu mode 4 pins this)
        const uint32_t t_sfa_me = t_row + kSfaCol + uint32_t(4 * grp + quad);
        const int ocw = ((p.Cp / 4 + 15) / 16) * 16;
        const int oc0 = min(grp * ocw, p.Cp), oc1 = min((grp + 1) * ocw, p.Cp);
        float* mv = reinterpret_cast<float*>(act);                 // [128][4 groups][4] (aliases the A tile
        int* mi = reinterpret_cast<int*>(act + kM * 16 * sizeof(float));   // after the output GEMM)
        uint32_t fph = 0;
        uint32_t hh[8], hs = 0;           // this thread's block input h: 64 codes, 4 block scales
        // quantise, store the A tile unit and the debug dump of one 32-column chunk cc (0 / 1)
        auto emit = [&](int l, size_t i, int cc, float (&y)[32], uint32_t (&q)[4]) -> uint32_t {
            const uint32_t sc = quant32(y, q);
            sts128(act_addr(act_s, r, grp * 2 + cc), make_uint4(q[0], q[1], q[2], q[3]));
            if (kDbg && i < p.n)
                *reinterpret_cast<uint4*>(p.dbg + (size_t(l) * p.n + i) * 144 + c00 / 2 + 16 * cc) =
                    make_uint4(q[0], q[1], q[2], q[3]);
            return sc;
        };
        auto finish = [&](int l, size_t i, uint32_t sw) {
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t_sfa_me), "r"(sw) : "memory");
            tmem_st_wait();
            if (kDbg && i < p.n) *reinterpret_cast<uint32_t*>(p.dbg + (size_t(l) * p.n + i) * 144 + 128 + grp * 4) = sw;
            fence_proxy_async();
            tc_fence_before();
            warp_arrive(act_ready);
        };
        uint4 hv_next = make_uint4(0, 0, 0, 0);       // grp 0: header of this row in the next tile
        if (grp == 0 && size_t(blockIdx.x) * kM + r < p.n)
            hv_next = __ldg(reinterpret_cast<const uint4*>(p.hdr) + size_t(blockIdx.x) * kM + r);
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const size_t i = t * kM + r;
            long long* etr = (p.trace && blockIdx.x == 0 && t < 4 * gridDim.x && (threadIdx.x == 0 || threadIdx.x == 511))
                                 ? p.trace + (t / gridDim.x) * (L + 1) * 8 + (threadIdx.x ? 3 : 0) : nullptr;
            // a2: A0 row (bf16, K = 48) = [xh | xl | xh | xl | xh | xl | 0..] (R22)
            if (grp == 0) {
                const uint4 hv = hv_next;
                const size_t in = i + size_t(gridDim.x) * kM;          // prefetch: hidden by this tile's layers
                if (t + gridDim.x < ntiles && in < p.n) hv_next = __ldg(reinterpret_cast<const uint4*>(p.hdr) + in);
                const uint32_t seg[7] = {hv.x >> 16, hv.x & 0xFFFFu, hv.y >> 16, hv.y & 0xFFFFu,
                                         hv.z & 0xFFFFu, hv.z >> 16, hv.w & 0xFFu};
                uint32_t e[24];
#pragma unroll
                for (int j = 0; j < 24; ++j) e[j] = 0;
#pragma unroll
                for (int f = 0; f < 7; ++f) {
                    const float x = float(seg[f]) * (1.0f / 65536.0f);
                    const __nv_bfloat16 xh = __float2bfloat16_rn(x);
                    const __nv_bfloat16 xl = __float2bfloat16_rn(x - __bfloat162float(xh));
                    const uint32_t hb = __bfloat16_as_ushort(xh), lb = __bfloat16_as_ushort(xl);
#pragma unroll
                    for (int c = 0; c < 6; ++c) {
                        const int k = 7 * c + f;
                        e[k >> 1] |= ((c & 1) ? lb : hb) << (16 * (k & 1));
                    }
                }
#pragma unroll
                for (int u = 0; u < 6; ++u)
                    sts128(act_addr(act_s, r, u), make_uint4(e[4 * u], e[4 * u + 1], e[4 * u + 2], e[4 * u + 3]));
            }
            fence_proxy_async();
            tc_fence_before();
            warp_arrive(act_ready);
            // a3: h0 -> NVFP4
            mbar_wait(acc_full, fph);
            fph ^= 1;
            tc_fence_after();
            if (etr) etr[2] = clock64();
            {
                uint32_t sw = 0;
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    uint32_t d[32];
                    tmem_ld32_async(t_row + uint32_t(c00 + 32 * cc), d);
                    float4 bq[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) bq[q] = lds4f(sb0 + 4u * (c00 + 32 * cc + 4 * q));
                    tmem_wait_ld();
                    float y[32];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        fma2(y[4 * q], y[4 * q + 1], __uint_as_float(d[4 * q]), __uint_as_float(d[4 * q + 1]),
                             p.inv_sh0, p.inv_sh0, bq[q].x, bq[q].y);
                        fma2(y[4 * q + 2], y[4 * q + 3], __uint_as_float(d[4 * q + 2]), __uint_as_float(d[4 * q + 3]),
                             p.inv_sh0, p.inv_sh0, bq[q].z, bq[q].w);
                    }
                    uint32_t q4[4];
                    sw |= emit(0, i, cc, y, q4) << (16 * cc);
#pragma unroll
                    for (int w = 0; w < 4; ++w) hh[4 * cc + w] = q4[w];
                }
                hs = sw;
                finish(0, i, sw);
                if (etr) etr[4] = clock64();
            }

            for (int g = 0; g < L; ++g) {
                mbar_wait(acc_full, fph);
                fph ^= 1;
                tc_fence_after();
                if (etr) etr[8 * (g + 1) + 2] = clock64();
                if (g == L - 1) {
                    // a5: logits = fma(D, mo, bo); top-k (ties -> lower index)
                    const int k = int(p.k);
                    float bv[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
                    int bc[4] = {0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF};
                    const bool fast = k == 1 && p.logits == nullptr;
                    float b0v = -FLT_MAX;                   // top-1 in scalars (the arrays live in local memory)
                    int b0c = 0x7FFFFFFF;
                    if (fast) {
                        // top-1 without logits: 16-column TMEM loads, the next one in flight;
                        // padding columns carry bias -3e38 and never win
                        uint32_t cur[16], nxt[16];
                        tmem_ld16_async(t_row + uint32_t(oc0), cur);
                        tmem_wait_ld();
                        for (int c0 = oc0; c0 < oc1; c0 += 16) {
                            if (c0 + 16 < oc1) tmem_ld16_async(t_row + uint32_t(c0 + 16), nxt);
                            float z[16];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float4 f4 = lds4f(sbo + 4u * (c0 + 4 * q));
                                fma2(z[4 * q], z[4 * q + 1], __uint_as_float(cur[4 * q]), __uint_as_float(cur[4 * q + 1]),
                                     p.mo, p.mo, f4.x, f4.y);
                                fma2(z[4 * q + 2], z[4 * q + 3], __uint_as_float(cur[4 * q + 2]), __uint_as_float(cur[4 * q + 3]),
                                     p.mo, p.mo, f4.z, f4.w);
                            }
#pragma unroll
                            for (int q = 0; q < 16; ++q)
                                if (z[q] > b0v) { b0v = z[q]; b0c = c0 + q; }
                            tmem_wait_ld();
#pragma unroll
                            for (int q = 0; q < 16; ++q) cur[q] = nxt[q];
                        }
                    }
                    for (int c0 = oc0; c0 < oc1 && !fast; c0 += 16) {
                        uint32_t v[16];
                        tmem_ld16_async(t_row + uint32_t(c0), v);
                        float bq[16];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float4 f4 = lds4f(sbo + 4u * (c0 + 4 * q));
                            bq[4 * q] = f4.x; bq[4 * q + 1] = f4.y; bq[4 * q + 2] = f4.z; bq[4 * q + 3] = f4.w;
                        }
                        tmem_wait_ld();
                        for (int j = 0; j < 16; ++j) {
                            const int c = c0 + j;
                            if (c >= p.C) break;
                            const float z = fmaf(__uint_as_float(v[j]), p.mo, bq[j]);
                            if (p.logits && i < p.n) p.logits[i * p.C + c] = z;
                            if (z > bv[k - 1]) {
                                int pos = k - 1;
                                while (pos > 0 && z > bv[pos - 1]) { bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos; }
                                bv[pos] = z;
                                bc[pos] = c;
                            }
                        }
                    }
                    if (etr) etr[8 * (g + 1) + 3] = clock64();     // argmax of this thread's columns done
                    tc_fence_before();
                    if (fast) { mv[(r * 4 + grp) * 4] = b0v; mi[(r * 4 + grp) * 4] = b0c; }
                    else
                        for (int q = 0; q < k; ++q) { mv[(r * 4 + grp) * 4 + q] = bv[q]; mi[(r * 4 + grp) * 4 + q] = bc[q]; }
                    epi_bar(1, kEpiThreads);
                    if (grp == 0 && fast) {
                        // groups hold increasing column ranges: strict > keeps the lower index on ties
                        float z = mv[r * 16];
                        int c = mi[r * 16];
#pragma unroll
                        for (int gg = 1; gg < 4; ++gg)
                            if (mv[r * 16 + 4 * gg] > z) { z = mv[r * 16 + 4 * gg]; c = mi[r * 16 + 4 * gg]; }
                        if (i < p.n) p.pred[i] = uint32_t(c);
                    } else if (grp == 0) {
                        // merge the 4 column groups' lists (ties on the value -> lower index)
                        float mvv[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
                        int mcc[4] = {0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF};
                        for (int gg = 0; gg < 4; ++gg)
                            for (int q = 0; q < k; ++q) {
                                const float z = mv[(r * 4 + gg) * 4 + q];
                                const int c = mi[(r * 4 + gg) * 4 + q];
                                if (!better(z, c, mvv[k - 1], mcc[k - 1])) continue;
                                int pos = k - 1;
                                while (pos > 0 && better(z, c, mvv[pos - 1], mcc[pos - 1])) {
                                    mvv[pos] = mvv[pos - 1]; mcc[pos] = mcc[pos - 1]; --pos;
                                }
                                mvv[pos] = z;
                                mcc[pos] = c;
                            }
                        if (i < p.n)
                            for (int q = 0; q < k; ++q) p.pred[i * k + q] = uint32_t(mcc[q]);
                    }
                    epi_bar(2, kEpiThreads);
                    if (etr) etr[8 * (g + 1) + 4] = clock64();
                } else if ((g & 1) == 0) {
                    // GEMM1 of block b: u -> NVFP4; the block input h stays in hh / hs
                    const int b = g / 2;
                    const float m1 = p.m1[b];
                    const uint32_t b1s = sb1 + 4u * b * kN;
                    uint32_t sw = 0;
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        const int c0 = c00 + 32 * cc;
                        uint32_t d[32];
                        tmem_ld32_async(t_row + uint32_t(c0), d);
                        float4 bb[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) bb[q] = lds4f(b1s + 4u * (c0 + 4 * q));
                        tmem_wait_ld();
                        float y[32];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            fma2(y[4 * q], y[4 * q + 1], __uint_as_float(d[4 * q]), __uint_as_float(d[4 * q + 1]),
                                 m1, m1, bb[q].x, bb[q].y);
                            fma2(y[4 * q + 2], y[4 * q + 3], __uint_as_float(d[4 * q + 2]), __uint_as_float(d[4 * q + 3]),
                                 m1, m1, bb[q].z, bb[q].w);
                        }
                        uint32_t q4[4];
                        sw |= emit(g + 1, i, cc, y, q4) << (16 * cc);
                    }
                    finish(g + 1, i, sw);
                    if (etr) etr[8 * (g + 1) + 4] = clock64();
                } else {
                    // GEMM2 of block b: y = ReLU(fma(D2, m2, hdq r2 + b2 / s_h')) -> NVFP4 (new hh / hs)
                    const int b = g / 2;
                    const float m2 = p.m2[b], r2 = p.r2[b];
                    const uint16_t r2h = p.r2h[b];
                    const uint32_t c2 = sc2 + 4u * b * kN;
                    uint32_t sw = 0, nh[8];
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        const int c0 = c00 + 32 * cc;
                        uint32_t d[32];
                        tmem_ld32_async(t_row + uint32_t(c0), d);
                        float sv[32];                  // skip + bias, computed while the load flies
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const float4 ca = lds4f(c2 + 4u * (c0 + 8 * w)), cb = lds4f(c2 + 4u * (c0 + 8 * w + 4));
                            const float cv[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
                            skip8<kMixed>(hh[4 * cc + w], (hs >> (8 * (2 * cc + w / 2))) & 0xFFu, r2h, r2, cv, sv + 8 * w);
                        }
                        tmem_wait_ld();
                        float y[32];
#pragma unroll
                        for (int j = 0; j < 32; j += 2)
                            fma2(y[j], y[j + 1], __uint_as_float(d[j]), __uint_as_float(d[j + 1]), m2, m2, sv[j], sv[j + 1]);
                        uint32_t q4[4];
                        sw |= emit(g + 1, i, cc, y, q4) << (16 * cc);
#pragma unroll
                        for (int w = 0; w < 4; ++w) nh[4 * cc + w] = q4[w];
                    }
                    for (int w = 0; w < 8; ++w) hh[w] = nh[w];
                    hs = sw;
                    finish(g + 1, i, sw);
                    if (etr) etr[8 * (g + 1) + 4] = clock64();
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool encode(EncodeTiledFn fn, CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t rows,
            uint64_t row_bytes, uint32_t box_inner, uint32_t box_rows) {
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) std::fprintf(stderr, "libtang: cuTensorMapEncodeTiled failed (%d)\n", int(r));
    return r == CUDA_SUCCESS;
}

}  // namespace

F4Plan* f4_plan_create(const WeightsF4& w, int device, int* err) {
    *err = TANG_OK;
    if (w.s.N != kN || w.s.Cp > 320 || w.s.B > kMaxBlocksF8) { *err = TANG_EMODEL; return nullptr; }
    F4Plan* p = new F4Plan();
    p->w = w;
    const size_t act = size_t(kM) * 128;
    const size_t budget = 227 * 1024 - 1024 - 256;
    const size_t cbytes = size_t(kN + 2 * w.s.B * kN + w.s.Cp) * 4;   // epilogue constants (smem)
    if (budget < act + cbytes + 2 * kStage) { delete p; *err = TANG_EMODEL; return nullptr; }
    p->stages = int((budget - act - cbytes) / kStage);
    if (p->stages > 8) p->stages = 8;
    p->smem = 1024 + act + p->stages * kStage + 256 + cbytes;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    p->grid = sms;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    const uint64_t rows4 = uint64_t(2) * w.s.B * kN + w.s.Cp;
    if (!encode(reinterpret_cast<EncodeTiledFn>(fn), &p->tmap4, CU_TENSOR_MAP_DATA_TYPE_UINT8, w.Wq, 128, rows4, 128, 128,
                uint32_t(kN)) ||
        !encode(reinterpret_cast<EncodeTiledFn>(fn), &p->tmap0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, w.s.B0, 64,
                uint64_t(kN), 128, 64, uint32_t(kN))) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    if (cudaFuncSetAttribute(mlp_f4_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) ||
        cudaFuncSetAttribute(mlp_f4_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) ||
        cudaFuncSetAttribute(mlp_f4_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) ||
        cudaFuncSetAttribute(mlp_f4_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem))) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    return p;
}

void f4_plan_set_scales(F4Plan* p, const WeightsF4& w) { if (p) p->w = w; }

void f4_plan_destroy(F4Plan* p) { delete p; }

int launch_mlp_f4(const F4Plan* pl, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                  cudaStream_t s, uint8_t* dbg, long long* trace) {
    if (!pl) return TANG_EMODEL;
    if (n == 0) return TANG_OK;
    F4Params p{};
    const WeightsF8& w = pl->w.s;
    p.hdr = hdr; p.n = n; p.k = k; p.pred = pred; p.logits = logits;
    p.sf = pl->w.SF;
    p.B = w.B; p.C = w.C; p.Cp = w.Cp; p.stages = pl->stages;
    p.dbg = dbg;
    p.trace = trace;
    p.inv_sh0 = w.inv_sh0;
    p.mo = w.mo;
    p.consts = pl->w.consts;
    p.r2h_ok = 1;
    for (int b = 0; b < w.B; ++b) {
        p.m1[b] = w.m1[b]; p.m2[b] = w.m2[b]; p.r2[b] = pl->w.r2[b];
        // sf * r2 must be an exact f16 for every e4m3 sf in [2^-9, 448]: r2 in [2^-12, 2^7]
        const float r = pl->w.r2[b];
        if (!(r >= 0x1p-12f && r <= 0x1p7f)) p.r2h_ok = 0;
        p.r2h[b] = __half_as_ushort(__float2half_rn(r));
    }
    const size_t tiles = (n + kM - 1) / kM;
    const int grid = int(tiles < size_t(pl->grid) ? tiles : size_t(pl->grid));
    auto kern = dbg ? (p.r2h_ok ? mlp_f4_kernel<true, true> : mlp_f4_kernel<true, false>)
                    : (p.r2h_ok ? mlp_f4_kernel<false, true> : mlp_f4_kernel<false, false>);
    kern<<<grid, kThreads, pl->smem, s>>>(pl->tmap4, pl->tmap0, p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::fprintf(stderr, "libtang: mlp_f4_kernel launch failed: %s (smem %zu)\n", cudaGetErrorString(e), pl->smem);
        return TANG_ECUDA;
    }
    return TANG_OK;
}

}  // namespace tang
