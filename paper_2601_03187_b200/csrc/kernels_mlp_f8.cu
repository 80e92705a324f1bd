// N2-f8: TaNG's residual MLP with FP8 E4M3 GEMMs on the 5th-gen tensor
// cores (tcgen05.mma kind::f8f6f4), one persistent kernel for sm_100a.
//
// What it computes (§6.1, Eq. 1-2; "precision quantization" P:304 read as
// DESIGN.md R23): per-tensor power-of-two scales s_w for W1, W2, Wo and static per-layer
// power-of-two activation scales (model blob); every quantisation is e4m3 round-to-nearest-even
// with saturation; bias, skip and ReLU act on the dequantised values before each quantisation.
//   x  = 7 header segments / 65536                                  (a2)
//   h0 = ReLU(x.W0 + b0)  -> e4m3(h0 / s_h0)      (a3: exact bf16 split on the tensor core, R22)
//   B times: u = ReLU(s_h s_w1 (hq.W1q) + b1)          -> uq = e4m3(u / s_u)
//            h = ReLU(s_u s_w2 (uq.W2q) + b2 + s_h hq)  -> hq = e4m3(h / s_h')          (a4)
//   logits = s_h s_wo (hq.Woq) + bo;  pred = argmax / top-k (ties -> lower index)        (a5)
// Because every scale is a power of two, the folded epilogue forms below scale exactly, so the
// kernel differs from the exact result only by fp32 accumulation order and one rounding per
// bias add (R23):
//   uq   = e4m3(ReLU(fma(D1, m1, b1 / s_u)))           m1 = s_h s_w1 / s_u
//   TMEM <- fma(hq, k2, b2 / (s_u s_w2))               k2 = s_h / (s_u s_w2)    (skip fold)
//   hq'  = e4m3(ReLU(D2 * m2))                          m2 = s_u s_w2 / s_h'
//   h0q  = e4m3(ReLU(fma(D0, 1 / s_h0, b0 / s_h0)))
//   logit = fma(D, mo, bo)                              mo = s_h s_wo
//
// Design: the bf16 kernel's structure (kernels_mlp_tc.cu) with e4m3 tiles:
//   * A tile [128 x N] e4m3 in shared memory (K-major SWIZZLE_128B, 128 K per 128-byte row):
//     64 KB at N = 512, which leaves room for 5 weight stages of 32 KB (256 rows x 128 K).
//   * weights e4m3 K-major [out][in] stream by TMA; layer 0's split bf16 operand has its own map.
//   * tcgen05.mma kind::f8f6f4 M=128 N=256 K=32, fp32 accumulators in TMEM (N <= 512 columns).
//   * epilogue overlap as in the bf16 kernel: N-half 0 of every hidden GEMM is processed under
//     acc_half (outputs held in registers: 32 per thread) and released with half_ready.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/tang.h"
#include "tang_internal.h"
#include "tc_ptx.h"

namespace tang {

struct F8Plan {
    CUtensorMap tmap8;       // e4m3 weights [2BN + Cp][N] bytes, box {128, R}
    CUtensorMap tmap0;       // layer-0 split operand [N][64] bf16, box {64, R}
    WeightsF8 w;
    int R, stages;
    size_t smem;
    bool dual;               // N <= 256: mlp_f8x2_kernel (two tiles in flight)
    int stages2;
    size_t smem2;
    int grid;
    uint32_t tmem_cols;
};

namespace {

using namespace tc;
constexpr int kEpiThreads = 256, kThreads = 384, kProdWarp = 8, kMmaWarp = 9;
// setmaxnreg: launch 168; (224 - 168) * 8 warps <= (168 - 56) * 4 warps
constexpr uint32_t kEpiRegs = 224, kCtlRegs = 56;
constexpr int CW = 32;                    // epilogue column chunk (tcgen05.ld 32x32b.x32)

struct F8Params {
    const void* hdr;
    size_t n;
    uint32_t k;
    uint32_t* pred;
    float* logits;
    const float* b0s;        // [N]     b0 / s_h0
    const float* b1s;        // [B][N]  b1 / s_u
    const float* c2;         // [B][N]  b2 / (s_u s_w2)
    const float* bo;         // [Cp]
    int N, B, C, Cp, R, stages;
    uint32_t tmem_cols;
    uint8_t* dbg;            // optional [(2B+1)][n][N] e4m3 dump of every GEMM input (tests)
    long long* trace;        // optional phase timestamps of block 0: [4 tiles][2B+1][8]
    float inv_sh0, mo;
    float m1[kMaxBlocksF8], k2[kMaxBlocksF8], m2[kMaxBlocksF8];
    uint16_t k2h[kMaxBlocksF8];   // k2 as an f16 bit pattern (every k2 is a power of two) ...
    int k2h_ok;                   // ... when all of them are representable in f16
};

__device__ __forceinline__ uint32_t idesc_f8(uint32_t n) {
    // D = f32 (bit 4), A = B = E4M3 (format 0), both K-major, N >> 3 at bit 17, M >> 4 at bit 24
    return (1u << 4) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
// warp-uniform issue (tc_ptx.h): the whole issuer warp executes it, one lane is elected
__device__ __forceinline__ void mma_f8_w(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
// ReLU + e4m3 RNE satfinite of 4 values; byte j (lowest first) = value j
__device__ __forceinline__ uint32_t q8x4(float a, float b, float c, float d) {
    uint16_t lo, hi;
    asm("cvt.rn.satfinite.relu.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(b), "f"(a));
    asm("cvt.rn.satfinite.relu.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(d), "f"(c));
    return uint32_t(lo) | (uint32_t(hi) << 16);
}
// exact e4m3 -> fp32 of the 4 bytes of w (via f16x2: every e4m3 value is an f16 value)
__device__ __forceinline__ void dq8x4(uint32_t w, float (&f)[4]) {
    uint32_t h01, h23;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h01) : "h"(uint16_t(w & 0xFFFFu)));
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h23) : "h"(uint16_t(w >> 16)));
    const __half2 a = *reinterpret_cast<const __half2*>(&h01), b = *reinterpret_cast<const __half2*>(&h23);
    f[0] = __low2float(a); f[1] = __high2float(a); f[2] = __low2float(b); f[3] = __high2float(b);
}
__device__ __forceinline__ float4 lds4f(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
// 16-byte unit u (16 e4m3 columns) of row r of the A tile (chunk = 128 columns)
__device__ __forceinline__ uint32_t act8_addr(uint32_t act_s, int r, int u) { return act_addr(act_s, r, u); }
__device__ __forceinline__ void dbg8(const F8Params& p, int l, size_t i, int col, uint4 v) {
    if (p.dbg && i < p.n) *reinterpret_cast<uint4*>(p.dbg + (size_t(l) * p.n + i) * p.N + col) = v;
}

__global__ void __launch_bounds__(kThreads, 1)
mlp_f8_kernel(const __grid_constant__ CUtensorMap tmap8, const __grid_constant__ CUtensorMap tmap0,
              const __grid_constant__ F8Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int N = p.N, R = p.R, S = p.stages;
    const int KC = N / 128;                                 // 128-wide e4m3 K chunks
    const int actc = KC > 0 ? KC : 1;
    const uint32_t stage_bytes = uint32_t(R) * 128;
    uint8_t* act = smem;                                     // actc x 16 KB
    const uint32_t act_s = smem_u32(act);
    uint8_t* wst = smem + actc * (kM * 128);
    uint64_t* full = reinterpret_cast<uint64_t*>(wst + S * stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* acc_full = empty + S;
    uint64_t* act_ready = acc_full + 1;
    uint64_t* half_ready = act_ready + 1;
    uint64_t* acc_half = half_ready + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_half + 1);
    // epilogue constants [b0/s_h0 (N) | b1/s_u (B N) | c2 (B N) | bo (Cp)] (contiguous from p.b0s)
    // copied to shared memory once per CTA: broadcast LDS on the epilogue chains
    const int nv = N + 2 * p.B * N + p.Cp;
    const uint32_t sb0 = smem_u32(wst + S * stage_bytes + 256);
    const uint32_t sb1 = sb0 + 4u * N, sc2 = sb1 + 4u * p.B * N, sbo = sc2 + 4u * p.B * N;
    for (int v = threadIdx.x; v < nv / 4; v += blockDim.x)
        sts128(sb0 + 16u * v, __ldg(reinterpret_cast<const uint4*>(p.b0s) + v));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = 2 * p.B + 1;
    const size_t ntiles = (p.n + kM - 1) / kM;
    const int Hs = N > R ? R : N;          // epilogue part 0 = the first MMA N-half
    const bool split = N > R;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(acc_full, 1);
        mbar_init(act_ready, kEpiThreads / 32);   // warp_arrive
        mbar_init(half_ready, kEpiThreads / 32);
        mbar_init(acc_half, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap8)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap0)) : "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(tmem_slot)), "r"(p.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kProdWarp) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs));
      if (warp == kProdWarp) {
        // ===== TMA producer =====
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            auto load = [&](const CUtensorMap* map, int c0, int row) {
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], stage_bytes);
                tma_load_2d(wst + s * stage_bytes, map, &full[s], c0, row);
                if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
            };
            for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int q = 0; q < (N + R - 1) / R; ++q) load(&tmap0, 0, q * R);      // layer 0
                for (int g = 0; g < L; ++g) {
                    const int nout = (g == L - 1) ? p.Cp : N;
                    const int row0 = (g == L - 1) ? 2 * p.B * N : ((g & 1) ? (p.B + g / 2) * N : (g / 2) * N);
                    for (int q = 0; q < (nout + R - 1) / R; ++q)
                        for (int kc = 0; kc < KC; ++kc) load(&tmap8, kc * 128, row0 + q * R);
                }
            }
        }
      } else if (warp == kMmaWarp) {
        // ===== MMA issuer (whole warp, one lane elected per instruction; descriptors base + offset >> 4) =====
        {
            uint32_t s = 0, ph = 0, aph = 0, hph = 0;
            const uint64_t a_d0 = sdesc(smem_u32(act)), w_d0 = sdesc(smem_u32(wst));
            for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                // layer 0: bf16 split operands (R22), K = 48
                mbar_wait(act_ready, aph);
                aph ^= 1;
                tc_fence_after();
                for (int q = 0; q < (N + R - 1) / R; ++q) {
                    const int nmma = min(R, N - q * R);
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint64_t b_d = w_d0 + uint64_t((s * stage_bytes) >> 4);
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        mma_bf16_w(tmem + uint32_t(q * R), a_d0 + uint64_t(2 * j), b_d + uint64_t(2 * j),
                                   idesc(uint32_t(nmma)), j);
                    mma_commit_w(&empty[s]);
                    if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                }
                mma_commit_w(acc_full);
                for (int g = 0; g < L; ++g) {
                    const bool is_out = g == L - 1;
                    const bool skip_init = false;          // the skip is added in the GEMM2 epilogue
                    const int nout = is_out ? p.Cp : N;
                    const int nq = (nout + R - 1) / R;
                    int lvl = 0;
                    auto reach = [&](int need) {
                        while (lvl < need) {
                            if (lvl == 0) { mbar_wait(half_ready, hph); hph ^= 1; }
                            else { mbar_wait(act_ready, aph); aph ^= 1; }
                            ++lvl;
                        }
                        tc_fence_after();
                    };
                    reach(1);
                    long long* tr = (p.trace && lane == 0 && blockIdx.x == 0 && t < 4 * gridDim.x)
                                        ? p.trace + ((t / gridDim.x) * L + g) * 8 : nullptr;
                    long long wfull = 0;
                    if (tr) tr[0] = clock64();
                    for (int q = 0; q < nq; ++q)
                        for (int kc = 0; kc < KC; ++kc) {
                            const int need = (q > 0 || kc * 128 >= Hs) ? 2 : 1;
                            if (lvl < need) reach(need);
                            const int nmma = min(R, nout - q * R);
                            long long w0 = tr ? clock64() : 0;
                            mbar_wait(&full[s], ph);
                            if (tr) wfull += clock64() - w0;
                            tc_fence_after();
                            const uint64_t a_k = a_d0 + uint64_t((kc * (kM * 128)) >> 4);
                            const uint64_t b_d = w_d0 + uint64_t((s * stage_bytes) >> 4);
                            mma4_f8_1(tmem + uint32_t(q * R), a_k, b_d, idesc_f8(uint32_t(nmma)),
                                      (skip_init || kc > 0) ? 1u : 0u);   // one K chunk under one elect
                            mma_commit_w(&empty[s]);
                            if (split && !is_out && q == 0 && kc == KC - 1) mma_commit_w(acc_half);
                            if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                        }
                    if (lvl < 2) reach(2);
                    mma_commit_w(acc_full);
                    if (tr) { tr[1] = clock64(); tr[2] = wfull; }
                }
            }
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
        // ===== epilogue: thread = packet row; group grp owns one slice of each N-half =====
        const int quad = warp & 3, grp = warp >> 2;
        const int r = quad * 32 + lane;
        const uint32_t t_row = tmem + (uint32_t(quad * 32) << 16);
        const int wd0 = Hs / 2, wd1 = (N - Hs) / 2;
        const int lo0 = grp * wd0, lo1 = Hs + grp * wd1;
        const int nch0 = wd0 / CW, nch = (wd0 + wd1) / CW;
        auto col_of = [&](int k) { return k < nch0 ? lo0 + k * CW : lo1 + (k - nch0) * CW; };
        const int ocw = ((p.Cp / 2 + 15) / 16) * 16;
        const int oc0 = min(grp * ocw, p.Cp), oc1 = min((grp + 1) * ocw, p.Cp);
        float* mv = reinterpret_cast<float*>(act);
        int* mi = reinterpret_cast<int*>(act + kM * 4 * sizeof(float));
        uint32_t fph = 0, hfph = 0;
        auto arrive_part = [&](int h) {
            fence_proxy_async();
            tc_fence_before();
            warp_arrive(h ? act_ready : half_ready);
        };
        // store one 32-column chunk (8 packed words) of the A tile and the debug dump
        auto put32 = [&](int l, size_t i, int c0, const uint32_t (&o)[8]) {
            const uint4 v0 = make_uint4(o[0], o[1], o[2], o[3]), v1 = make_uint4(o[4], o[5], o[6], o[7]);
            sts128(act8_addr(act_s, r, c0 / 16), v0);
            sts128(act8_addr(act_s, r, c0 / 16 + 1), v1);
            dbg8(p, l, i, c0, v0);
            dbg8(p, l, i, c0 + 16, v1);
        };
        uint32_t hh[8][8];        // e4m3 block input h of this thread's columns (<= 8 chunks): the skip
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const size_t i = t * kM + r;
            long long* ltr = (p.trace && blockIdx.x == 0 && t < 4 * gridDim.x && threadIdx.x == 0) ? p.trace + ((t / gridDim.x) * L) * 8 : nullptr;
            if (ltr) ltr[5] = clock64();
            // a2: A0 row (bf16, K = 48) = [xh | xl | xh | xl | xh | xl | 0..] (R22)
            if (grp == 0) {
                uint4 hv = make_uint4(0, 0, 0, 0);
                if (i < p.n) hv = __ldg(reinterpret_cast<const uint4*>(p.hdr) + i);
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
            // a3: h0q = e4m3(ReLU(fma(D0, 1/s_h0, b0/s_h0)))
            mbar_wait(acc_full, fph);
            fph ^= 1;
            tc_fence_after();
            {
                uint32_t d[CW];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    if (kk >= nch) break;
                    const int c0 = col_of(kk);
                    tmem_ld32_async(t_row + uint32_t(c0), d);
                    float4 bq[CW / 4];
#pragma unroll
                    for (int q = 0; q < CW / 4; ++q) bq[q] = lds4f(sb0 + 4u * (c0 + 4 * q));
                    tmem_wait_ld();
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float* f = reinterpret_cast<const float*>(d) + 4 * q;
                        hh[kk][q] = q8x4(fmaf(f[0], p.inv_sh0, bq[q].x), fmaf(f[1], p.inv_sh0, bq[q].y),
                                         fmaf(f[2], p.inv_sh0, bq[q].z), fmaf(f[3], p.inv_sh0, bq[q].w));
                    }
                    put32(0, i, c0, hh[kk]);
                    if (kk == nch0 - 1) arrive_part(0);
                }
                arrive_part(1);
            }
            if (ltr) ltr[6] = clock64();

            for (int g = 0; g < L; ++g) {
                const int b = g / 2;
                const bool sp = split && g < L - 1;
                if (sp) { mbar_wait(acc_half, hfph); hfph ^= 1; }
                else { mbar_wait(acc_full, fph); fph ^= 1; }
                tc_fence_after();
                long long* etr = (p.trace && blockIdx.x == 0 && t < 4 * gridDim.x && threadIdx.x == 0) ? p.trace + ((t / gridDim.x) * L + g) * 8 : nullptr;
                if (etr) etr[3] = clock64();
                if (g == L - 1) {
                    // a5: logits = fma(D, mo, bo); top-k (ties -> lower index)
                    const int k = int(p.k);
                    float bv[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
                    int bc[4] = {0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF};
                    float b0v = -FLT_MAX;
                    int b0c = 0x7FFFFFFF;
                    const bool fast = k == 1 && p.logits == nullptr;
                    __syncwarp();
                    int cs = oc0;                          // first column left for the 16-wide loop
                    if (fast && oc1 - oc0 >= 32) {
                        // top-1 without logits: 32-column TMEM loads, the next one in flight
                        const int cend = oc0 + (oc1 - oc0) / 32 * 32;
                        uint32_t cur[32], nxt[32];
                        tmem_ld32_async(t_row + uint32_t(oc0), cur);
                        tmem_wait_ld();
                        for (int c0 = oc0; c0 < cend; c0 += 32) {
                            if (c0 + 32 < cend) tmem_ld32_async(t_row + uint32_t(c0 + 32), nxt);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 f4 = lds4f(sbo + 4u * (c0 + 4 * q));
                                const float bq[4] = {f4.x, f4.y, f4.z, f4.w};
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    const float z = fmaf(__uint_as_float(cur[4 * q + j]), p.mo, bq[j]);
                                    if (c0 + 4 * q + j < p.C && z > b0v) { b0v = z; b0c = c0 + 4 * q + j; }
                                }
                            }
                            tmem_wait_ld();
#pragma unroll
                            for (int j = 0; j < 32; ++j) cur[j] = nxt[j];
                        }
                        cs = cend;
                    }
                    for (int c0 = cs; c0 < oc1; c0 += 16) {
                        uint32_t v[16];
                        tmem_ld16_async(t_row + uint32_t(c0), v);
                        float bq[16];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float4 f4 = lds4f(sbo + 4u * (c0 + 4 * q));
                            bq[4 * q] = f4.x; bq[4 * q + 1] = f4.y; bq[4 * q + 2] = f4.z; bq[4 * q + 3] = f4.w;
                        }
                        tmem_wait_ld();
                        if (fast) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const float z = fmaf(__uint_as_float(v[j]), p.mo, bq[j]);
                                if (c0 + j < p.C && z > b0v) { b0v = z; b0c = c0 + j; }
                            }
                            continue;
                        }
                        for (int j = 0; j < 16; ++j) {
                            const int c = c0 + j;
                            if (c >= p.C) break;
                            const float z = fmaf(__uint_as_float(v[j]), p.mo, bq[j]);
                            if (p.logits && i < p.n) p.logits[i * p.C + c] = z;
                            if (k == 1) {
                                if (z > b0v) { b0v = z; b0c = c; }
                            } else if (z > bv[k - 1]) {
                                int pos = k - 1;
                                while (pos > 0 && z > bv[pos - 1]) { bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos; }
                                bv[pos] = z;
                                bc[pos] = c;
                            }
                        }
                    }
                    if (k == 1) { bv[0] = b0v; bc[0] = b0c; }
                    tc_fence_before();
                    if (grp > 0)
                        for (int q = 0; q < k; ++q) { mv[r * 4 + q] = bv[q]; mi[r * 4 + q] = bc[q]; }
                    epi_bar(1, kEpiThreads);
                    if (grp == 0) {
                        const float* gv = mv + r * 4;
                        const int* gi = mi + r * 4;
                        if (k == 1) {
                            if (gv[0] > bv[0]) { bv[0] = gv[0]; bc[0] = gi[0]; }
                        } else {
                            for (int q2 = 0; q2 < k; ++q2) {
                                const float z = gv[q2];
                                const int c = gi[q2];
                                if (z > bv[k - 1]) {
                                    int pos = k - 1;
                                    while (pos > 0 && z > bv[pos - 1]) { bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos; }
                                    bv[pos] = z;
                                    bc[pos] = c;
                                }
                            }
                        }
                        if (i < p.n)
                            for (int q = 0; q < k; ++q) p.pred[i * k + q] = uint32_t(bc[q]);
                    }
                    epi_bar(2, kEpiThreads);
                    if (etr) etr[4] = clock64();
                } else if ((g & 1) == 0) {
                    // GEMM1 of block b: uq = e4m3(ReLU(fma(D1, m1, b1/s_u))); the block input h stays in hh
                    const float m1 = p.m1[b];
                    const uint32_t b1s = sb1 + 4u * b * N;
                    auto chunk = [&](int c0, uint32_t (&o)[8]) {
                        uint32_t d[CW];
                        tmem_ld32_async(t_row + uint32_t(c0), d);
                        float4 bb[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) bb[q] = lds4f(b1s + 4u * (c0 + 4 * q));
                        tmem_wait_ld();
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float* f = reinterpret_cast<const float*>(d) + 4 * q;
                            o[q] = q8x4(fmaf(f[0], m1, bb[q].x), fmaf(f[1], m1, bb[q].y), fmaf(f[2], m1, bb[q].z),
                                        fmaf(f[3], m1, bb[q].w));
                        }
                    };
                    int kk0 = 0;
                    if (sp) {
                        uint32_t held[4][8];
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) chunk(lo0 + kk * CW, held[kk]);
                        mbar_wait(acc_full, fph);             // the MMAs no longer read hq: store uq
                        fph ^= 1;
                        tc_fence_after();
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) put32(g + 1, i, lo0 + kk * CW, held[kk]);
                        arrive_part(0);
                        kk0 = nch0;
                    }
                    for (int kk = kk0; kk < nch; ++kk) {
                        uint32_t o[8];
                        const int c0 = col_of(kk);
                        chunk(c0, o);
                        put32(g + 1, i, c0, o);
                        if (kk == nch0 - 1) arrive_part(0);
                    }
                    arrive_part(1);
                    if (etr) etr[4] = clock64();
                } else {
                    // GEMM2 of block b: hq' = e4m3(ReLU((D2 + fma(hq, k2, c2)) * m2)), hq from hh
                    const float m2 = p.m2[b], k2 = p.k2[b];
                    const uint32_t c2 = sc2 + 4u * b * N;
                    auto chunk = [&](int c0, uint32_t (&h)[8]) {    // h: old hq in, new hq out
                        uint32_t d[CW];
                        tmem_ld32_async(t_row + uint32_t(c0), d);
                        float sv[CW];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            float hq[4];
                            dq8x4(h[q], hq);
                            const float4 cc = lds4f(c2 + 4u * (c0 + 4 * q));
                            sv[4 * q] = fmaf(hq[0], k2, cc.x); sv[4 * q + 1] = fmaf(hq[1], k2, cc.y);
                            sv[4 * q + 2] = fmaf(hq[2], k2, cc.z); sv[4 * q + 3] = fmaf(hq[3], k2, cc.w);
                        }
                        tmem_wait_ld();
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float* f = reinterpret_cast<const float*>(d) + 4 * q;
                            h[q] = q8x4((f[0] + sv[4 * q]) * m2, (f[1] + sv[4 * q + 1]) * m2,
                                        (f[2] + sv[4 * q + 2]) * m2, (f[3] + sv[4 * q + 3]) * m2);
                        }
                    };
                    if (sp) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) chunk(lo0 + kk * CW, hh[kk]);
                        mbar_wait(acc_full, fph);
                        fph ^= 1;
                        tc_fence_after();
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) put32(g + 1, i, lo0 + kk * CW, hh[kk]);
                        arrive_part(0);
                    }
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        if (kk >= nch) break;
                        if (sp && kk < nch0) continue;
                        const int c0 = col_of(kk);
                        chunk(c0, hh[kk]);
                        put32(g + 1, i, c0, hh[kk]);
                        if (kk == nch0 - 1) arrive_part(0);
                    }
                    arrive_part(1);
                    if (etr) etr[4] = clock64();
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols));
    }
}

// ---- dual-tile variant (N <= 256): two 128-packet tiles in flight per CTA ---------------------
// Slot s in {0, 1} owns TMEM columns [256 s, 256 s + 256), its own A tile and its own 8 epilogue
// warps (warps 8 s .. 8 s + 7: two per TMEM lane quadrant, each taking half the columns), so the
// two slots' epilogues run concurrently (4 epilogue warps per SM sub-partition hide the TMEM-load
// and shared-memory latencies of each other) while the tensor core works on the other slot.
// Jobs: layer 0, each hidden GEMM, and each <= N-column pass of the output layer (one weight box).
// The MMA issuer runs job j for slot 0, then for slot 1, on the SAME weight stages: each weight
// box is fetched from L2 once per tile pair (half the L2 -> shared traffic of one fetch per tile).
// act_ready[s] doubles as "the slot's TMEM region has been read" between output passes.
// (ties in the top-k merge are broken on the index explicitly: the two column groups' index
// ranges interleave across passes)
constexpr int kThreads2 = 640, kProdWarp2 = 16, kMmaWarp2 = 17;   // warps 18, 19 idle
// setmaxnreg acts on whole warpgroups, so the control warpgroup is warps 16-19 (producer, MMA
// issuer, two idle). 20 warps launch at 96 registers (5 warps per SM sub-partition: 5 x 96 <= 512
// per lane). An increase is served only from registers other warps of the CTA released: the
// control warpgroup drops to 64, freeing (96 - 64) x 4 = 128 = (104 - 96) x 16 for the epilogue.
// (At the former 112 / 32 split the MMA issuer spilled its descriptors and phase bits inside the
// issue loop, ptxas -v; profiles/r02_ctlregs_ab.txt.)
constexpr uint32_t kEpiRegs2 = 104, kCtlRegs2 = 64;
static_assert((kEpiRegs2 - 96) * 16 <= (96 - kCtlRegs2) * 4 && (65536 / kThreads2) / 8 * 8 == 96, "setmaxnreg budget");

__device__ __forceinline__ bool better(float z, int c, float bz, int bc) { return z > bz || (z == bz && c < bc); }
// (o0, o1) = (a0 b0 + c0, a1 b1 + c1): one packed FFMA2 (sm_100a fma.rn.f32x2, two IEEE fp32 fmas,
// bit-identical to two fmaf)
__device__ __forceinline__ void fma2(float& o0, float& o1, float a0, float a1, float b0, float b1, float c0, float c1) {
    asm("{\n\t.reg .b64 a, b, c, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
        "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(o0), "=f"(o1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void mul2(float& o0, float& o1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
        "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(o0), "=f"(o1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void add2(float& o0, float& o1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
        "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(o0), "=f"(o1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ float4 ldsf4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
// e4m3 bytes of ReLU(v * m + b) for 4 consecutive columns (two FFMA2, two cvt)
// skip values hq * k2 + c of the 4 e4m3 bytes of w: e4m3 -> f16x2 (exact), then the mixed
// f16 x f16 + f32 fma (sm_100a FHFMA: exact product, one fp32 rounding = fmaf(float(hq), k2, c))
__device__ __forceinline__ void skip4(uint32_t w, uint16_t k2h, float4 c, float* o) {
    uint32_t h01, h23;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h01) : "h"(uint16_t(w & 0xFFFFu)));
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h23) : "h"(uint16_t(w >> 16)));
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
        "fma.rn.f32.f16 %0, l, %3, %4;\n\tfma.rn.f32.f16 %1, h, %3, %5;\n\t}"
        : "=f"(o[0]), "=f"(o[1]) : "r"(h01), "h"(k2h), "f"(c.x), "f"(c.y));
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
        "fma.rn.f32.f16 %0, l, %3, %4;\n\tfma.rn.f32.f16 %1, h, %3, %5;\n\t}"
        : "=f"(o[2]), "=f"(o[3]) : "r"(h23), "h"(k2h), "f"(c.z), "f"(c.w));
}
__device__ __forceinline__ uint32_t q8fma4(const float* v, float m, float4 b) {
    float y0, y1, y2, y3;
    fma2(y0, y1, v[0], v[1], m, m, b.x, b.y);
    fma2(y2, y3, v[2], v[3], m, m, b.z, b.w);
    return q8x4(y0, y1, y2, y3);
}

// kMode bit 0: phase trace (block 0), bit 1: e4m3 activation dump (tests); 0 in production
template <int kMode>
__global__ void __launch_bounds__(kThreads2, 1)
mlp_f8x2_kernel(const __grid_constant__ CUtensorMap tmap8, const __grid_constant__ CUtensorMap tmap0,
                const __grid_constant__ F8Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int N = p.N, S = p.stages;                        // N <= 256: one MMA N-pass per hidden layer
    const int KC = N / 128;
    const int actc = KC > 0 ? KC : 1;
    const uint32_t stage_bytes = uint32_t(N) * 128;         // R = N
    const uint32_t act_bytes = uint32_t(actc) * (kM * 128);
    uint8_t* wst = smem + 2 * act_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(wst + S * stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* acc_full = empty + S;                         // [2]
    uint64_t* act_ready = acc_full + 2;                     // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(act_ready + 2);
    const uint32_t act_s0 = smem_u32(smem);
    // all epilogue constants in shared memory, [b0/s_h0 (N) | b1/s_u (B N) | c2 (B N) | bo (Cp)]
    // (contiguous in global memory from p.b0s): broadcast LDS instead of L1-missing LDGs
    const int nv = N + 2 * p.B * N + p.Cp;
    const uint32_t sb0 = smem_u32(wst + S * stage_bytes + 256);
    const uint32_t sb1 = sb0 + 4u * N, sc2 = sb1 + 4u * p.B * N, sbo = sc2 + 4u * p.B * N;
    for (int v = threadIdx.x; v < nv / 4; v += blockDim.x)
        sts128(sb0 + 16u * v, __ldg(reinterpret_cast<const uint4*>(p.b0s) + v));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int npass = (p.Cp + N - 1) / N;                  // output passes of <= N columns (one box each)
    const int J = 1 + 2 * p.B + npass;                      // jobs per tile
    const size_t ntiles = (p.n + kM - 1) / kM;
    const size_t mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const size_t npairs = (mine + 1) / 2;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(&acc_full[s], 1); mbar_init(&act_ready[s], kEpiThreads / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap8)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap0)) : "memory");
    }
    if (warp == kMmaWarp2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(tmem_slot)), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // job j of a tile: 0 = layer 0, 1..2B = hidden GEMM g = j - 1, then output pass q = j - 1 - 2B
    if (warp >= kProdWarp2) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs2));
      if (warp == kProdWarp2) {
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            auto load = [&](const CUtensorMap* map, int c0, int row) {
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], stage_bytes);
                tma_load_2d(wst + s * stage_bytes, map, &full[s], c0, row);
                if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
            };
            for (size_t k = 0; k < npairs; ++k)
                for (int j = 0; j < J; ++j) {              // one fetch per job, shared by both slots
                    if (j == 0) { load(&tmap0, 0, 0); continue; }
                    const int g = j - 1;
                    const int row0 = g < 2 * p.B ? ((g & 1) ? (p.B + g / 2) * N : (g / 2) * N)
                                                 : 2 * p.B * N + N * (g - 2 * p.B);
                    for (int kc = 0; kc < KC; ++kc) load(&tmap8, kc * 128, row0);
                }
        }
      } else if (warp == kMmaWarp2) {
        {                                          // whole warp, one lane elected per instruction
            uint32_t s = 0, ph = 0, aph[2] = {0, 0};
            const uint64_t w_d0 = sdesc(smem_u32(wst));
            for (size_t k = 0; k < npairs; ++k)
                for (int j = 0; j < J; ++j) {
                    const int ns = j == 0 ? 1 : KC;        // weight stages of this job
                    const int g = j - 1;
                    const bool hidden = j > 0 && g < 2 * p.B;
                    const int nmma = j == 0 || hidden ? N : min(N, p.Cp - N * (g - 2 * p.B));
                    const bool skip_init = false;          // the skip is added in the GEMM2 epilogue
#pragma unroll
                    for (int sl = 0; sl < 2; ++sl) {
                        mbar_wait(&act_ready[sl], aph[sl]);
                        aph[sl] ^= 1;
                        tc_fence_after();
                        long long* tr = (kMode & 1) && lane == 0 && blockIdx.x == 0 && k < 2
                                            ? p.trace + ((k * J + j) * 2 + sl) * 4 : nullptr;
                        if (tr) tr[0] = clock64();
                        const uint32_t d = tmem + uint32_t(256 * sl);
                        const uint64_t a_d = sdesc(act_s0 + uint32_t(sl) * act_bytes);
                        uint32_t ss = s, sp = ph;
                        for (int kc = 0; kc < ns; ++kc) {
                            if (sl == 0) { mbar_wait(&full[ss], sp); tc_fence_after(); }
                            const uint64_t b_d = w_d0 + uint64_t((ss * stage_bytes) >> 4);
                            if (j == 0) {
#pragma unroll
                                for (int jj = 0; jj < 3; ++jj)
                                    mma_bf16_w(d, a_d + uint64_t(2 * jj), b_d + uint64_t(2 * jj), idesc(uint32_t(N)), jj);
                            } else {
                                const uint64_t a_k = a_d + uint64_t((kc * (kM * 128)) >> 4);
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj)    // (batched issue measured 5 % slower here, r02f8b)
                                    mma_f8_w(d, a_k + uint64_t(2 * jj), b_d + uint64_t(2 * jj), idesc_f8(uint32_t(nmma)),
                                             (skip_init || kc > 0 || jj > 0) ? 1u : 0u);
                            }
                            if (sl == 1) mma_commit_w(&empty[ss]);   // both slots have read the stage
                            if (++ss == uint32_t(S)) { ss = 0; sp ^= 1; }
                        }
                        mma_commit_w(&acc_full[sl]);
                        if (tr) tr[1] = clock64();
                        if (sl == 1) { s = ss; ph = sp; }
                    }
                }
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs2));
        const int sl = warp >> 3, quad = warp & 3, grp = (warp >> 2) & 1;
        const int r = quad * 32 + lane;
        const int wd = N / 2, lo = grp * wd, nch = wd / CW;  // this group's hidden columns
        const uint32_t act_s = act_s0 + uint32_t(sl) * act_bytes;
        const uint32_t t_row = tmem + (uint32_t(quad * 32) << 16) + uint32_t(256 * sl);
        const int bar_a = 1 + 2 * sl, bar_b = 2 + 2 * sl;  // named barriers of this slot's 256 threads
        uint32_t fph = 0;
        float bv[4];                                         // top-k state, carried across output passes
        int bc[4];
        // header of packet i (zero past the end): loaded one output pass ahead of write_a0 so the
        // HBM latency of the next tile's headers is off the slot's critical path
        auto load_hdr = [&](size_t i) {
            uint4 hv = make_uint4(0, 0, 0, 0);
            if (grp == 0 && i < p.n) hv = __ldg(reinterpret_cast<const uint4*>(p.hdr) + i);
            return hv;
        };
        auto write_a0 = [&](uint4 hv) {                      // layer-0 A operand (R22), group 0 only
            if (grp == 0) {
                const uint32_t seg[7] = {hv.x >> 16, hv.x & 0xFFFFu, hv.y >> 16, hv.y & 0xFFFFu,
                                         hv.z & 0xFFFFu, hv.z >> 16, hv.w & 0xFFu};
                uint32_t e[24];
#pragma unroll
                for (int jx = 0; jx < 24; ++jx) e[jx] = 0;
#pragma unroll
                for (int f = 0; f < 7; ++f) {
                    const float x = float(seg[f]) * (1.0f / 65536.0f);
                    const __nv_bfloat16 xh = __float2bfloat16_rn(x);
                    const __nv_bfloat16 xl = __float2bfloat16_rn(x - __bfloat162float(xh));
                    const uint32_t hb = __bfloat16_as_ushort(xh), lb = __bfloat16_as_ushort(xl);
#pragma unroll
                    for (int c = 0; c < 6; ++c) {
                        const int kx = 7 * c + f;
                        e[kx >> 1] |= ((c & 1) ? lb : hb) << (16 * (kx & 1));
                    }
                }
#pragma unroll
                for (int u = 0; u < 6; ++u)
                    sts128(act_addr(act_s, r, u), make_uint4(e[4 * u], e[4 * u + 1], e[4 * u + 2], e[4 * u + 3]));
            }
            fence_proxy_async();
            tc_fence_before();
            warp_arrive(&act_ready[sl]);
        };
        auto put32 = [&](int l, size_t i, int c0, const uint32_t (&o)[8]) {
            const uint4 v0 = make_uint4(o[0], o[1], o[2], o[3]), v1 = make_uint4(o[4], o[5], o[6], o[7]);
            sts128(act8_addr(act_s, r, c0 / 16), v0);
            sts128(act8_addr(act_s, r, c0 / 16 + 1), v1);
            if (kMode & 2) {
                dbg8(p, l, i, c0, v0);
                dbg8(p, l, i, c0 + 16, v1);
            }
        };
        if (npairs > 0) write_a0(load_hdr((size_t(blockIdx.x) + size_t(sl) * gridDim.x) * kM + r));
        uint4 next_hv = make_uint4(0, 0, 0, 0);
        uint32_t hh[4][8];                                  // e4m3 block input h of this thread's columns
        for (size_t k = 0; k < npairs; ++k)
            for (int j = 0; j < J; ++j) {
                const size_t t = blockIdx.x + (2 * k + sl) * size_t(gridDim.x);
                const size_t i = t * kM + r;
                mbar_wait(&acc_full[sl], fph);
                fph ^= 1;
                tc_fence_after();
                // phase stamps of block 0's first two pairs (tests/scripts: tang_debug_trace)
                long long* etr = (kMode & 1) && blockIdx.x == 0 && k < 2 && (warp & 7) == 0 && lane == 0
                                     ? p.trace + ((k * J + j) * 2 + sl) * 4 : nullptr;
                if (etr) etr[2] = clock64();
                const int g = j - 1;
                if (j == 0) {
                    // h0q = e4m3(ReLU(fma(D0, 1/s_h0, b0/s_h0))); also held in registers (skip)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        if (kk >= nch) break;
                        const int c0 = lo + kk * CW;
                        uint32_t d[CW];
                        tmem_ld32_async(t_row + uint32_t(c0), d);
                        float4 bq[CW / 4];
#pragma unroll
                        for (int q = 0; q < CW / 4; ++q) bq[q] = ldsf4(sb0 + 4u * (c0 + 4 * q));
                        tmem_wait_ld();
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            hh[kk][q] = q8fma4(reinterpret_cast<const float*>(d) + 4 * q, p.inv_sh0, bq[q]);
                        put32(0, i, c0, hh[kk]);
                    }
                    fence_proxy_async();
                    tc_fence_before();
                    warp_arrive(&act_ready[sl]);
                } else if (g < 2 * p.B && (g & 1) == 0) {
                    // GEMM1: uq = e4m3(ReLU(fma(D1, m1, b1/s_u))) (the block input h stays in hh)
                    const int b = g / 2;
                    const float m1 = p.m1[b];
                    const uint32_t b1s = sb1 + 4u * b * N;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        if (kk >= nch) break;
                        const int c0 = lo + kk * CW;
                        uint32_t d[CW];
                        tmem_ld32_async(t_row + uint32_t(c0), d);
                        float4 bq[CW / 4];
#pragma unroll
                        for (int q = 0; q < CW / 4; ++q) bq[q] = ldsf4(b1s + 4u * (c0 + 4 * q));
                        tmem_wait_ld();
                        uint32_t o[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            o[q] = q8fma4(reinterpret_cast<const float*>(d) + 4 * q, m1, bq[q]);
                        put32(g + 1, i, c0, o);
                    }
                    fence_proxy_async();
                    tc_fence_before();
                    warp_arrive(&act_ready[sl]);
                } else if (g < 2 * p.B) {
                    // GEMM2: hq' = e4m3(ReLU((D2 + fma(hq, k2, c2)) * m2)), hq from registers
                    const int b = g / 2;
                    const float m2 = p.m2[b], k2 = p.k2[b];
                    const uint16_t k2h = p.k2h[b];
                    const uint32_t c2 = sc2 + 4u * b * N;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        if (kk >= nch) break;
                        const int c0 = lo + kk * CW;
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf) {   // 16-column halves (register budget)
                            uint32_t d[16];
                            tmem_ld16_async(t_row + uint32_t(c0 + 16 * hf), d);
                            float sv[16];                  // skip values while the TMEM load is in flight
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float4 cc = ldsf4(c2 + 4u * (c0 + 16 * hf + 4 * q));
                                const uint32_t hw = hh[kk][4 * hf + q];
                                if (p.k2h_ok) {            // f16 x f16 + f32 (exact product, one rounding)
                                    skip4(hw, k2h, cc, &sv[4 * q]);
                                } else {
                                    float hq[4];
                                    dq8x4(hw, hq);
                                    fma2(sv[4 * q], sv[4 * q + 1], hq[0], hq[1], k2, k2, cc.x, cc.y);
                                    fma2(sv[4 * q + 2], sv[4 * q + 3], hq[2], hq[3], k2, k2, cc.z, cc.w);
                                }
                            }
                            tmem_wait_ld();
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float* f = reinterpret_cast<const float*>(d) + 4 * q;
                                float y0, y1, y2, y3;
                                add2(y0, y1, f[0], f[1], sv[4 * q], sv[4 * q + 1]);
                                add2(y2, y3, f[2], f[3], sv[4 * q + 2], sv[4 * q + 3]);
                                mul2(y0, y1, y0, y1, m2, m2);
                                mul2(y2, y3, y2, y3, m2, m2);
                                hh[kk][4 * hf + q] = q8x4(y0, y1, y2, y3);
                            }
                        }
                        put32(g + 1, i, c0, hh[kk]);
                    }
                    fence_proxy_async();
                    tc_fence_before();
                    warp_arrive(&act_ready[sl]);
                } else {
                    // output pass q: logits = fma(D, mo, bo) over C columns [N q, N q + nq)
                    const int q = g - 2 * p.B;
                    const int nq = min(N, p.Cp - N * q);
                    const int ocw = ((nq / 2 + 15) / 16) * 16;
                    const int oc0 = min(grp * ocw, nq), oc1 = min((grp + 1) * ocw, nq);
                    const int kk_ = int(p.k);
                    if (q == 0) {
#pragma unroll
                        for (int x = 0; x < 4; ++x) { bv[x] = -FLT_MAX; bc[x] = 0x7FFFFFFF; }
                        if (k + 1 < npairs) next_hv = load_hdr((blockIdx.x + (2 * (k + 1) + sl) * size_t(gridDim.x)) * kM + r);
                    }
                    __syncwarp();
                    if (kk_ == 1 && p.logits == nullptr) {
                        // top-1 fast path: 32-column TMEM loads, pairwise tree argmax per chunk (the
                        // left operand wins ties, so the chunk result is its first maximum), then one
                        // strict merge (chunks ascend); padded columns c >= C carry bo = -3e38
                        int c0 = oc0;
                        for (; c0 + 32 <= oc1; c0 += 32) {
                            uint32_t v[32];
                            tmem_ld32_async(t_row + uint32_t(c0), v);
                            const int cb = N * q + c0;
                            float bq[32];
#pragma unroll
                            for (int x = 0; x < 8; ++x) {
                                const float4 f4 = ldsf4(sbo + 4u * (cb + 4 * x));
                                bq[4 * x] = f4.x; bq[4 * x + 1] = f4.y; bq[4 * x + 2] = f4.z; bq[4 * x + 3] = f4.w;
                            }
                            tmem_wait_ld();
                            float z[32];
                            int zi[32];
#pragma unroll
                            for (int x = 0; x < 32; x += 2)
                                fma2(z[x], z[x + 1], __uint_as_float(v[x]), __uint_as_float(v[x + 1]), p.mo, p.mo,
                                     bq[x], bq[x + 1]);
#pragma unroll
                            for (int x = 0; x < 32; ++x) zi[x] = x;
#pragma unroll
                            for (int st = 1; st < 32; st *= 2)
#pragma unroll
                                for (int x = 0; x < 32; x += 2 * st)
                                    if (z[x + st] > z[x]) { z[x] = z[x + st]; zi[x] = zi[x + st]; }
                            if (z[0] > bv[0]) { bv[0] = z[0]; bc[0] = cb + zi[0]; }
                        }
                        for (; c0 < oc1; c0 += 16) {
                            uint32_t v[16];
                            tmem_ld16_async(t_row + uint32_t(c0), v);
                            const int cb = N * q + c0;
                            float bq[16];
#pragma unroll
                            for (int x = 0; x < 4; ++x) {
                                const float4 f4 = ldsf4(sbo + 4u * (cb + 4 * x));
                                bq[4 * x] = f4.x; bq[4 * x + 1] = f4.y; bq[4 * x + 2] = f4.z; bq[4 * x + 3] = f4.w;
                            }
                            tmem_wait_ld();
                            float z[16];
                            int zi[16];
#pragma unroll
                            for (int x = 0; x < 16; x += 2)
                                fma2(z[x], z[x + 1], __uint_as_float(v[x]), __uint_as_float(v[x + 1]), p.mo, p.mo,
                                     bq[x], bq[x + 1]);
#pragma unroll
                            for (int x = 0; x < 16; ++x) zi[x] = x;
#pragma unroll
                            for (int st = 1; st < 16; st *= 2)
#pragma unroll
                                for (int x = 0; x < 16; x += 2 * st)
                                    if (z[x + st] > z[x]) { z[x] = z[x + st]; zi[x] = zi[x + st]; }
                            if (z[0] > bv[0]) { bv[0] = z[0]; bc[0] = cb + zi[0]; }
                        }
                    } else
                    for (int c0 = oc0; c0 < oc1; c0 += 16) {
                        uint32_t v[16];
                        tmem_ld16_async(t_row + uint32_t(c0), v);
                        const int cb = N * q + c0;               // C index of column c0
                        float bq[16];
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            const float4 f4 = ldsf4(sbo + 4u * (cb + 4 * x));
                            bq[4 * x] = f4.x; bq[4 * x + 1] = f4.y; bq[4 * x + 2] = f4.z; bq[4 * x + 3] = f4.w;
                        }
                        tmem_wait_ld();
                        float z[16];
#pragma unroll
                        for (int x = 0; x < 16; x += 2)
                            fma2(z[x], z[x + 1], __uint_as_float(v[x]), __uint_as_float(v[x + 1]), p.mo, p.mo,
                                 bq[x], bq[x + 1]);
                        for (int x = 0; x < 16; ++x) {
                            const int c = cb + x;
                            if (c >= p.C) break;
                            if (p.logits && i < p.n) p.logits[i * p.C + c] = z[x];
                            if (z[x] > bv[kk_ - 1]) {            // columns ascend within a group
                                int pos = kk_ - 1;
                                while (pos > 0 && z[x] > bv[pos - 1]) {
                                    bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos;
                                }
                                bv[pos] = z[x];
                                bc[pos] = c;
                            }
                        }
                    }
                    tc_fence_before();
                    if (q < npass - 1) {
                        warp_arrive(&act_ready[sl]);               // TMEM region read: next pass may start
                    } else {
                        // merge the two groups' candidates through shared memory (the slot's A
                        // tile is free: no MMA reads it any more), index-aware tie-break
                        float* mv = reinterpret_cast<float*>(smem + sl * act_bytes);
                        int* mi = reinterpret_cast<int*>(smem + sl * act_bytes + kM * 4 * sizeof(float));
                        if (grp > 0)
                            for (int x = 0; x < kk_; ++x) { mv[r * 4 + x] = bv[x]; mi[r * 4 + x] = bc[x]; }
                        epi_bar(bar_a, kEpiThreads);
                        if (grp == 0) {
                            for (int x2 = 0; x2 < kk_; ++x2) {
                                const float zz = mv[r * 4 + x2];
                                const int c = mi[r * 4 + x2];
                                if (better(zz, c, bv[kk_ - 1], bc[kk_ - 1])) {
                                    int pos = kk_ - 1;
                                    while (pos > 0 && better(zz, c, bv[pos - 1], bc[pos - 1])) {
                                        bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos;
                                    }
                                    bv[pos] = zz;
                                    bc[pos] = c;
                                }
                            }
                            if (i < p.n)
                                for (int x = 0; x < kk_; ++x) p.pred[i * kk_ + x] = uint32_t(bc[x]);
                        }
                        epi_bar(bar_b, kEpiThreads);
                        if (k + 1 < npairs) write_a0(next_hv);    // next tile of this slot
                    }
                }
                if (etr) etr[3] = clock64();
            }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
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

F8Plan* f8_plan_create(const WeightsF8& w, int device, bool allow_dual, int* err) {
    *err = TANG_OK;
    if (w.N % 128 || w.N > 512 || w.Cp > 512 || w.B > kMaxBlocksF8) { *err = TANG_EMODEL; return nullptr; }
    F8Plan* p = new F8Plan();
    p->w = w;
    p->R = w.N < 256 ? w.N : 256;
    const size_t act = size_t(w.N / 128) * kM * 128;
    const size_t stage = size_t(p->R) * 128;
    const size_t budget = 227 * 1024 - 1024 - 256;
    const size_t cbytes = size_t(w.N + 2 * w.B * w.N + w.Cp) * 4;   // epilogue constants (smem)
    p->stages = int((budget - act - cbytes) / stage);
    if (p->stages > 8) p->stages = 8;
    if (p->stages < 2) { delete p; *err = TANG_EMODEL; return nullptr; }
    p->smem = 1024 + act + p->stages * stage + 256 + cbytes;
    uint32_t cols = 32;
    const int need = w.N > w.Cp ? w.N : w.Cp;
    while (cols < uint32_t(need)) cols <<= 1;
    p->tmem_cols = cols;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    p->grid = sms;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    const uint64_t rows8 = uint64_t(2) * w.B * w.N + w.Cp;
    if (!encode(reinterpret_cast<EncodeTiledFn>(fn), &p->tmap8, CU_TENSOR_MAP_DATA_TYPE_UINT8, w.Wq, uint64_t(w.N), rows8,
                uint64_t(w.N), 128, uint32_t(p->R)) ||
        !encode(reinterpret_cast<EncodeTiledFn>(fn), &p->tmap0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, w.B0, 64,
                uint64_t(w.N), 128, 64, uint32_t(p->R))) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    if (cudaFuncSetAttribute(mlp_f8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) != cudaSuccess) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    // dual-tile variant: two A tiles + stages (N <= 256); tang_config.mlp_kernel = SINGLE forces the
    // single-tile kernel
    p->dual = w.N <= 256 && allow_dual;
    if (p->dual) {
        const size_t bias = size_t(w.N + 2 * w.B * w.N + w.Cp) * 4;   // epilogue constants (smem)
        p->stages2 = int((budget - 2 * act - bias) / stage);
        if (p->stages2 > 8) p->stages2 = 8;
        p->smem2 = 1024 + 2 * act + p->stages2 * stage + 256 + bias;
        if (p->stages2 < 2 ||
            cudaFuncSetAttribute(mlp_f8x2_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem2)) != cudaSuccess ||
            cudaFuncSetAttribute(mlp_f8x2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem2)) != cudaSuccess ||
            cudaFuncSetAttribute(mlp_f8x2_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem2)) != cudaSuccess)
            p->dual = false;
    }
    return p;
}

void f8_plan_set_scales(F8Plan* p, const WeightsF8& w) { if (p) p->w = w; }

void f8_plan_destroy(F8Plan* p) { delete p; }

int launch_mlp_f8(const F8Plan* pl, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                  cudaStream_t s, uint8_t* dbg, long long* trace) {
    if (!pl) return TANG_EMODEL;
    if (n == 0) return TANG_OK;
    F8Params p{};
    const WeightsF8& w = pl->w;
    p.hdr = hdr; p.n = n; p.k = k; p.pred = pred; p.logits = logits;
    p.b0s = w.b0s; p.b1s = w.b1s; p.c2 = w.c2; p.bo = w.bo;
    p.N = w.N; p.B = w.B; p.C = w.C; p.Cp = w.Cp; p.R = pl->R; p.stages = pl->dual ? pl->stages2 : pl->stages;
    p.tmem_cols = pl->tmem_cols;
    p.dbg = dbg;
    p.trace = trace;
    p.inv_sh0 = w.inv_sh0;
    p.mo = w.mo;
    p.k2h_ok = 1;
    for (int b = 0; b < w.B; ++b) {
        p.m1[b] = w.m1[b]; p.k2[b] = w.k2[b]; p.m2[b] = w.m2[b];
        const __half h = __float2half_rn(w.k2[b]);
        if (__half2float(h) != w.k2[b]) p.k2h_ok = 0;
        p.k2h[b] = __half_as_ushort(h);
    }
    const size_t tiles = (n + kM - 1) / kM;
    if (pl->dual) {           // two tiles in flight per CTA
        const size_t pairs = (tiles + 1) / 2;
        const int grid = int(pairs < size_t(pl->grid) ? pairs : size_t(pl->grid));
        if (dbg)
            mlp_f8x2_kernel<2><<<grid, kThreads2, pl->smem2, s>>>(pl->tmap8, pl->tmap0, p);
        else if (trace)
            mlp_f8x2_kernel<1><<<grid, kThreads2, pl->smem2, s>>>(pl->tmap8, pl->tmap0, p);
        else
            mlp_f8x2_kernel<0><<<grid, kThreads2, pl->smem2, s>>>(pl->tmap8, pl->tmap0, p);
    } else {
        const int grid = int(tiles < size_t(pl->grid) ? tiles : size_t(pl->grid));
        mlp_f8_kernel<<<grid, kThreads, pl->smem, s>>>(pl->tmap8, pl->tmap0, p);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::fprintf(stderr, "libtang: mlp_f8_kernel launch failed: %s (smem %zu)\n", cudaGetErrorString(e), pl->smem);
        return TANG_ECUDA;
    }
    return TANG_OK;
}

}  // namespace tang
