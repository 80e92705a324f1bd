// a2-a5, bf16, N <= 256 (the reduced models): TaNG's residual MLP (§6.1, Eq. 1-2 P:377-381,
// P:383, §6.2) with TWO 128-packet tiles in flight per CTA.
//
// Same arithmetic and quantisation points as mlp_tc_kernel (kernels_mlp_tc.cu; R5, R22): x split
// exactly into bf16 hi + lo for layer 0 on the tensor core, h and u rounded RNE to bf16 as GEMM
// inputs, bias / skip / ReLU in fp32, the GEMM2 skip folded into its accumulator (h + b2 stored into
// the drained TMEM columns before GEMM2 accumulates onto them).
//
// Why: at N <= 256 a hidden layer is one MMA N-pass, so in the one-tile kernel the
// tensor core waits for every epilogue (MMA -> drain -> MMA ...).  Here each CTA owns two slots,
// each with its own [128 x N] A tile in shared memory, its own 256-column TMEM region and its own 8
// epilogue warps; the MMA issuer runs job j (layer 0, each hidden GEMM, each <= N-column output
// pass) for slot 0 and then for slot 1 on the SAME weight stages (each weight box is fetched once
// per tile pair), so one slot's epilogue overlaps the other slot's MMAs.  The structure follows the
// FP8 dual-tile kernel (kernels_mlp_f8.cu, mlp_f8x2_kernel) with bf16 operands.
//
// Warps: 0-15 epilogue (slot = warp / 8; within a slot quad = warp % 4, column group (warp / 4) % 2;
// thread = packet row), 16 TMA producer, 17 MMA issuer + TMEM owner, 18-19 idle.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdio>

#include "../../include/tang.h"
#include "tang_internal.h"
#include "tc_ptx.h"

namespace tang {

struct Tc2Plan {
    CUtensorMap tmap;        // weights [rows][N] bf16, box {64, N}
    CUtensorMap tmap_tail;   // box {64, tail}: the output layer's partial last pass
    int tail;
    WeightsBF16 w;
    int stages;
    size_t smem;
    int grid;
};

namespace {

using namespace tc;
constexpr int kThreads = 640, kProdWarp = 16, kMmaWarp = 17;
constexpr int kSlotThreads = 256;
// 20 warps launch at 96 registers; setmaxnreg only moves registers inside the CTA's launch
// allocation: (104 - 96) x 16 epilogue warps = (96 - 64) x 4 control warps.  The control warps
// spilled descriptors inside the MMA loop at 32 (ptxas -v); at 104 the epilogue does not spill either
constexpr uint32_t kEpiRegs = 104, kCtlRegs = 64;
constexpr uint32_t kLaunchRegs = (65536u / kThreads) & ~7u;
static_assert((kEpiRegs - kLaunchRegs) * 16 <= (kLaunchRegs - kCtlRegs) * 4, "setmaxnreg budget");
constexpr int CW = 32;                    // epilogue chunk (TMEM columns per load)

struct P2 {
    const void* hdr;
    size_t n;
    uint32_t k;
    uint32_t* pred;
    float* logits;
    const float* bias;        // [b0 | b1 x B | b2 x B | bo] contiguous
    int N, B, C, Cp, stages;
    int row_l0;
    uint16_t* dbg;            // optional [(2B+1)][n][N] bf16 dump of every GEMM input (tests)
    int tail;                 // rows of the output layer's partial last pass (0: none)
};

__device__ __forceinline__ float4 bias4s(uint32_t sb, int off) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(sb + 4u * uint32_t(off)));
    return v;
}
template <bool kDbg>
__device__ __forceinline__ void dbg_put(const P2& p, int l, size_t i, int col, uint4 v) {
    if (!kDbg) return;
    if (p.dbg && i < p.n) *reinterpret_cast<uint4*>(p.dbg + (size_t(l) * p.n + i) * p.N + col) = v;
}
__device__ __forceinline__ bool better(float z, int c, float bz, int bc) { return z > bz || (z == bz && c < bc); }

template <bool kDbg>
__global__ void __launch_bounds__(kThreads, 1)
mlp_tc2_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_tail,
               const __grid_constant__ P2 p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int N = p.N, S = p.stages, B = p.B;
    const int KC = N / 64;
    const uint32_t stage_bytes = uint32_t(N) * 128;        // N rows x 64 K bf16
    const uint32_t act_bytes = uint32_t(KC) * (kM * 128);   // one slot's [128 x N] A tile
    uint8_t* wst = smem + 2 * act_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(wst + S * stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* acc_full = empty + S;                         // [2] MMA -> epilogue of slot s
    uint64_t* act_ready = acc_full + 2;                     // [2] slot s: A tile written, TMEM region read
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(act_ready + 2);
    const uint32_t act_s0 = smem_u32(smem);
    const uint32_t sb = smem_u32(wst + S * stage_bytes + 256);
    {
        const int nv = N + 2 * B * N + p.Cp;
        for (int v = threadIdx.x; v < nv / 4; v += blockDim.x)
            sts128(sb + 16u * v, __ldg(reinterpret_cast<const uint4*>(p.bias) + v));
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int npass = (p.Cp + N - 1) / N;                   // output passes of <= N columns
    const int J = 1 + 2 * B + npass;                         // jobs per tile
    const size_t ntiles = (p.n + kM - 1) / kM;
    const size_t mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const size_t npairs = (mine + 1) / 2;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(&acc_full[s], 1); mbar_init(&act_ready[s], kSlotThreads / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_tail)) : "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kProdWarp) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs));
      if (warp == kProdWarp) {
        // ===== TMA producer: one fetch per job, shared by both slots =====
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            auto load = [&](int c0, int row, bool tl) {
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], tl ? uint32_t(p.tail) * 128u : stage_bytes);
                tma_load_2d(wst + s * stage_bytes, tl ? &tmap_tail : &tmap, &full[s], c0, row);
                if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
            };
            for (size_t k = 0; k < npairs; ++k)
                for (int j = 0; j < J; ++j) {
                    if (j == 0) { load(0, p.row_l0, false); continue; }   // layer 0: K chunk 0 of B0
                    const int g = j - 1;
                    const int row0 = g < 2 * B ? ((g & 1) ? (B + g / 2) * N : (g / 2) * N) : 2 * B * N + N * (g - 2 * B);
                    const bool tl = p.tail && g == 2 * B + npass - 1;      // partial last output pass
                    for (int kc = 0; kc < KC; ++kc) load(kc * 64, row0, tl);
                }
        }
      } else if (warp == kMmaWarp) {
        // ===== MMA issuer (whole warp; one lane elected per instruction) =====
        uint32_t s = 0, ph = 0, aph = 0;
        const uint64_t w_d0 = sdesc(smem_u32(wst));
        for (size_t k = 0; k < npairs; ++k)
            for (int j = 0; j < J; ++j) {
                const int g = j - 1;
                const bool hidden = j > 0 && g < 2 * B;
                const int nmma = j == 0 || hidden ? N : min(N, p.Cp - N * (g - 2 * B));
                const bool skip_init = hidden && (g & 1);       // GEMM2: TMEM holds h + b2
                const int ns = j == 0 ? 1 : KC;
                const uint32_t id = idesc(uint32_t(nmma));
                // the two slots alternate per weight stage: slot 0 runs K chunk kc, then slot 1 on the
                // same stage, which it then frees (a whole job per slot would need more stages than fit
                // beside the two A tiles; per stage measured 2.5 % faster than per 2-stage group,
                // profiles/r02_bf16_dual_micro.txt)
                uint32_t ss = s, sp = ph;
                for (int g0 = 0; g0 < ns; ++g0) {
                    const int gn = 1;
                    const uint32_t s0 = ss, p0 = sp;
                    for (int sl = 0; sl < 2; ++sl) {
                        if (g0 == 0) {
                            mbar_wait(&act_ready[sl], (aph >> sl) & 1u);    // A tile written, TMEM region drained
                            aph ^= 1u << sl;
                            tc_fence_after();
                        }
                        const uint32_t d = tmem + uint32_t(256 * sl);
                        const uint64_t a_d = sdesc(act_s0 + uint32_t(sl) * act_bytes);
                        ss = s0;
                        sp = p0;
                        for (int kc = g0; kc < g0 + gn; ++kc) {
                            if (sl == 0) { mbar_wait(&full[ss], sp); tc_fence_after(); }
                            const uint64_t b_d = w_d0 + uint64_t((ss * stage_bytes) >> 4);
                            if (j == 0) {
#pragma unroll
                                for (int jj = 0; jj < 3; ++jj)     // K = 48: the exact split of layer 0 (R22)
                                    mma_bf16_w(d, a_d + uint64_t(2 * jj), b_d + uint64_t(2 * jj), id, jj);
                            } else {
                                // one elect per MMA: measured 4 % faster here than one per K chunk
                                // (mma4_ss_1), profiles/r02_bf16_dual_micro.txt
                                const uint64_t a_k = a_d + uint64_t((kc * (kM * 128)) >> 4);
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj)
                                    mma_bf16_w(d, a_k + uint64_t(2 * jj), b_d + uint64_t(2 * jj), id,
                                               (skip_init || kc > 0 || jj > 0) ? 1u : 0u);
                            }
                            if (sl == 1) mma_commit_w(&empty[ss]);   // both slots have read the stage
                            if (++ss == uint32_t(S)) { ss = 0; sp ^= 1; }
                        }
                        if (g0 + gn == ns) mma_commit_w(&acc_full[sl]);
                    }
                }
                s = ss;
                ph = sp;
            }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
        // ===== epilogue of slot sl: thread = packet row r, column group grp =====
        const int sl = warp >> 3, quad = warp & 3, grp = (warp >> 2) & 1;
        const int r = quad * 32 + lane;
        const int wd = N / 2, lo = grp * wd, nch = wd / CW;   // this group's hidden columns
        const uint32_t act_s = act_s0 + uint32_t(sl) * act_bytes;
        const uint32_t t_row = tmem + (uint32_t(quad * 32) << 16) + uint32_t(256 * sl);
        const int bar_a = 1 + 2 * sl, bar_b = 2 + 2 * sl;    // named barriers of this slot's 256 threads
        const int ob = N + 2 * B * N;                         // offset of bo in the bias vectors
        uint32_t fph = 0;
        float bv[4];
        int bc[4];
        float b0v = -FLT_MAX;                                 // top-1 fast path state (registers)
        int b0c = 0x7FFFFFFF;
        auto write_a0 = [&](size_t i) {                       // a2: A0 row (R22), group 0
            if (grp == 0) {
                uint4 hv = make_uint4(0, 0, 0, 0);
                if (i < p.n) hv = __ldg(reinterpret_cast<const uint4*>(p.hdr) + i);
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
        auto done = [&]() {                                   // A tile written / TMEM region read
            fence_proxy_async();
            tc_fence_before();
            warp_arrive(&act_ready[sl]);
        };
        // h = ReLU(D [+ b0]) -> A tile (layer 0, every GEMM2)
        auto drain_relu = [&](bool add_b0, int dl, size_t i) {
            for (int kk = 0; kk < nch; ++kk) {
                const int c0 = lo + kk * CW;
                uint32_t d[CW];
                tmem_ld32_async(t_row + uint32_t(c0), d);
                tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < CW / 8; ++q) {
                    float* f = reinterpret_cast<float*>(d) + 8 * q;
                    if (add_b0) {
                        const float4 ba = bias4s(sb, c0 + 8 * q), bb = bias4s(sb, c0 + 8 * q + 4);
                        add2(f[0], f[1], f[0], f[1], ba.x, ba.y);
                        add2(f[2], f[3], f[2], f[3], ba.z, ba.w);
                        add2(f[4], f[5], f[4], f[5], bb.x, bb.y);
                        add2(f[6], f[7], f[6], f[7], bb.z, bb.w);
                    }
                    const uint4 o = make_uint4(relu_pack_bf16(f[0], f[1]), relu_pack_bf16(f[2], f[3]),
                                               relu_pack_bf16(f[4], f[5]), relu_pack_bf16(f[6], f[7]));
                    sts128(act_addr(act_s, r, c0 / 8 + q), o);
                    dbg_put<kDbg>(p, dl, i, c0 + 8 * q, o);
                }
            }
            done();
        };
        if (npairs > 0) write_a0((size_t(blockIdx.x) + size_t(sl) * gridDim.x) * kM + r);
        for (size_t k = 0; k < npairs; ++k)
            for (int j = 0; j < J; ++j) {
                const size_t t = blockIdx.x + (2 * k + sl) * size_t(gridDim.x);
                const size_t i = t * kM + r;
                mbar_wait(&acc_full[sl], fph);
                fph ^= 1;
                tc_fence_after();
                __syncwarp();
                const int g = j - 1;
                if (j == 0) {
                    drain_relu(true, 0, i);                   // a3: h0 = ReLU(x.W0 + b0)
                } else if (g < 2 * B && (g & 1) == 0) {
                    // a4 GEMM1: u = ReLU(D + b1) over h in smem; TMEM <- h + b2 (skip fold)
                    const int b = g / 2;
                    const int o1 = N + b * N, o2 = N + B * N + b * N;
                    for (int kk = 0; kk < nch; ++kk) {
                        const int c0 = lo + kk * CW;
                        uint32_t d[CW];
                        tmem_ld32_async(t_row + uint32_t(c0), d);
                        uint4 hh[CW / 8];
#pragma unroll
                        for (int q = 0; q < CW / 8; ++q) hh[q] = lds128(act_addr(act_s, r, c0 / 8 + q));
                        tmem_wait_ld();
#pragma unroll
                        for (int q = 0; q < CW / 8; ++q) {          // u over h
                            const float4 ba = bias4s(sb, o1 + c0 + 8 * q), bb = bias4s(sb, o1 + c0 + 8 * q + 4);
                            const float* f = reinterpret_cast<const float*>(d) + 8 * q;
                            float z[8];
                            add2(z[0], z[1], f[0], f[1], ba.x, ba.y);
                            add2(z[2], z[3], f[2], f[3], ba.z, ba.w);
                            add2(z[4], z[5], f[4], f[5], bb.x, bb.y);
                            add2(z[6], z[7], f[6], f[7], bb.z, bb.w);
                            const uint4 o = make_uint4(relu_pack_bf16(z[0], z[1]), relu_pack_bf16(z[2], z[3]),
                                                       relu_pack_bf16(z[4], z[5]), relu_pack_bf16(z[6], z[7]));
                            sts128(act_addr(act_s, r, c0 / 8 + q), o);
                            dbg_put<kDbg>(p, g + 1, i, c0 + 8 * q, o);
                        }
#pragma unroll
                        for (int hf = 0; hf < CW / 16; ++hf) {      // h + b2 -> the drained TMEM columns
                            float sv[16];
#pragma unroll
                            for (int q2 = 0; q2 < 2; ++q2) {
                                const int q = 2 * hf + q2;
                                const float4 ba = bias4s(sb, o2 + c0 + 8 * q), bb = bias4s(sb, o2 + c0 + 8 * q + 4);
                                float* o = sv + 8 * q2;
                                add2(o[0], o[1], bf16_lo(hh[q].x), bf16_hi(hh[q].x), ba.x, ba.y);
                                add2(o[2], o[3], bf16_lo(hh[q].y), bf16_hi(hh[q].y), ba.z, ba.w);
                                add2(o[4], o[5], bf16_lo(hh[q].z), bf16_hi(hh[q].z), bb.x, bb.y);
                                add2(o[6], o[7], bf16_lo(hh[q].w), bf16_hi(hh[q].w), bb.z, bb.w);
                            }
                            tmem_st16(t_row + uint32_t(c0 + 16 * hf), sv);
                        }
                    }
                    tmem_st_wait();
                    done();
                } else if (g < 2 * B) {
                    drain_relu(false, g + 1, i);              // a4 GEMM2: h = ReLU(D) (D = u.W2 + b2 + h)
                } else {
                    // a5: output pass q: logits = D + bo over classes [N q, N q + nq); top-k carried
                    const int q = g - 2 * B;
                    const int nq = min(N, p.Cp - N * q);
                    const int ocw = ((nq / 2 + 15) / 16) * 16;
                    const int oc0 = min(grp * ocw, nq), oc1 = min((grp + 1) * ocw, nq);
                    const int kk_ = int(p.k);
                    if (q == 0) {
#pragma unroll
                        for (int x = 0; x < 4; ++x) { bv[x] = -FLT_MAX; bc[x] = 0x7FFFFFFF; }
                        b0v = -FLT_MAX;
                        b0c = 0x7FFFFFFF;
                    }
                    const bool top1 = kk_ == 1 && p.logits == nullptr;
                    int cs = oc0;                                    // first column of the general loop
                    if (top1) {
                        // top-1 without logits: 32-column TMEM loads, pairwise tree argmax per chunk
                        // (the left operand wins ties, so the chunk result is its first maximum), then
                        // one strict merge (chunks ascend); padded columns c >= C carry bo = -3e38
                        for (; cs + 32 <= oc1; cs += 32) {
                            uint32_t v[32];
                            tmem_ld32_async(t_row + uint32_t(cs), v);
                            const int cb = N * q + cs;
                            float z[32];
#pragma unroll
                            for (int x = 0; x < 8; ++x) {
                                const float4 f4 = bias4s(sb, ob + cb + 4 * x);
                                z[4 * x] = f4.x; z[4 * x + 1] = f4.y; z[4 * x + 2] = f4.z; z[4 * x + 3] = f4.w;
                            }
                            tmem_wait_ld();
                            int zi[32];
#pragma unroll
                            for (int x = 0; x < 32; x += 2) {
                                add2(z[x], z[x + 1], __uint_as_float(v[x]), __uint_as_float(v[x + 1]), z[x], z[x + 1]);
                                zi[x] = x;
                                zi[x + 1] = x + 1;
                            }
#pragma unroll
                            for (int st = 1; st < 32; st *= 2)
#pragma unroll
                                for (int x = 0; x < 32; x += 2 * st)
                                    if (z[x + st] > z[x]) { z[x] = z[x + st]; zi[x] = zi[x + st]; }
                            if (z[0] > b0v) { b0v = z[0]; b0c = cb + zi[0]; }
                        }
                    }
                    for (int c0 = cs; c0 < oc1; c0 += 16) {
                        uint32_t v[16];
                        tmem_ld16_async(t_row + uint32_t(c0), v);
                        const int cb = N * q + c0;                   // class index of column c0
                        float bq[16];
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            const float4 f4 = bias4s(sb, ob + cb + 4 * x);
                            bq[4 * x] = f4.x; bq[4 * x + 1] = f4.y; bq[4 * x + 2] = f4.z; bq[4 * x + 3] = f4.w;
                        }
                        tmem_wait_ld();
                        if (top1) {                                  // the < 32-column remainder
#pragma unroll
                            for (int x = 0; x < 16; ++x) {
                                const float z = __uint_as_float(v[x]) + bq[x];
                                if (z > b0v) { b0v = z; b0c = cb + x; }
                            }
                            continue;
                        }
                        for (int x = 0; x < 16; ++x) {
                            const int c = cb + x;
                            if (c >= p.C) break;
                            const float z = __uint_as_float(v[x]) + bq[x];
                            if (p.logits && i < p.n) p.logits[i * p.C + c] = z;
                            if (z > bv[kk_ - 1]) {                   // columns ascend within a group
                                int pos = kk_ - 1;
                                while (pos > 0 && z > bv[pos - 1]) { bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos; }
                                bv[pos] = z;
                                bc[pos] = c;
                            }
                        }
                    }
                    if (q < npass - 1) {
                        tc_fence_before();
                        warp_arrive(&act_ready[sl]);                 // TMEM region read: next pass may start
                    } else {
                        // merge the two groups' candidates (index-aware: their class ranges interleave
                        // across passes) through the slot's A tile, which no MMA reads any more
                        tc_fence_before();
                        float* mv = reinterpret_cast<float*>(smem + sl * act_bytes);
                        int* mi = reinterpret_cast<int*>(smem + sl * act_bytes + kM * 4 * sizeof(float));
                        if (top1) { bv[0] = b0v; bc[0] = b0c; }
                        if (grp > 0)
                            for (int x = 0; x < kk_; ++x) { mv[r * 4 + x] = bv[x]; mi[r * 4 + x] = bc[x]; }
                        epi_bar(bar_a, kSlotThreads);
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
                        epi_bar(bar_b, kSlotThreads);              // scratch consumed before A0 overwrites it
                        if (k + 1 < npairs) write_a0((blockIdx.x + (2 * (k + 1) + sl) * size_t(gridDim.x)) * kM + r);
                    }
                }
            }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

Tc2Plan* tc2_plan_create(const WeightsBF16& w, int device, int* err) {
    *err = TANG_OK;
    if (w.N > 256 || w.N < 64 || w.N % 64 || w.Cp > 512 || w.Cp % 16) { *err = TANG_EMODEL; return nullptr; }
    Tc2Plan* p = new Tc2Plan();
    p->w = w;
    const size_t act = size_t(w.N / 64) * kM * 128;
    const size_t stage = size_t(w.N) * 128;
    const size_t budget = 227 * 1024 - 1024 - 256;
    const size_t cbytes = size_t(w.N + 2 * w.B * w.N + w.Cp) * 4;
    if (budget < 2 * act + cbytes + 2 * stage) { delete p; *err = TANG_EMODEL; return nullptr; }
    p->stages = int((budget - 2 * act - cbytes) / stage);
    if (p->stages > 8) p->stages = 8;
    p->smem = 1024 + 2 * act + p->stages * stage + 256 + cbytes;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    p->grid = sms;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    const uint64_t rows = uint64_t(2) * w.B * w.N + w.Cp + w.N;
    cuuint64_t dims[2] = {cuuint64_t(w.N), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(w.N) * 2};
    cuuint32_t box[2] = {64, cuuint32_t(w.N)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(
        &p->tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(w.W1t), dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::fprintf(stderr, "libtang: cuTensorMapEncodeTiled failed (%d)\n", int(r));
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    const int np = (w.Cp + w.N - 1) / w.N;
    const int tail = w.Cp - w.N * (np - 1);
    p->tail = tail < w.N ? tail : 0;
    cuuint32_t box_t[2] = {64, cuuint32_t(p->tail ? p->tail : w.N)};
    r = reinterpret_cast<EncodeTiledFn>(fn)(
        &p->tmap_tail, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(w.W1t), dims, strides, box_t, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::fprintf(stderr, "libtang: cuTensorMapEncodeTiled (tail) failed (%d)\n", int(r));
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    if (cudaFuncSetAttribute(mlp_tc2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) !=
            cudaSuccess ||
        cudaFuncSetAttribute(mlp_tc2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) !=
            cudaSuccess) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    return p;
}

void tc2_plan_destroy(Tc2Plan* p) { delete p; }

int launch_mlp_tc2(const Tc2Plan* pl, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                   cudaStream_t s, uint16_t* dbg) {
    if (!pl) return TANG_EMODEL;
    if (n == 0) return TANG_OK;
    P2 p{};
    p.hdr = hdr; p.n = n; p.k = k; p.pred = pred; p.logits = logits;
    p.bias = pl->w.b0;
    p.N = pl->w.N; p.B = pl->w.B; p.C = pl->w.C; p.Cp = pl->w.Cp; p.stages = pl->stages;
    p.row_l0 = 2 * pl->w.B * pl->w.N + pl->w.Cp;
    p.dbg = dbg;
    p.tail = pl->tail;
    const size_t tiles = (n + kM - 1) / kM;
    const int grid = int(tiles < size_t(pl->grid) ? tiles : size_t(pl->grid));
    if (dbg) mlp_tc2_kernel<true><<<grid, kThreads, pl->smem, s>>>(pl->tmap, pl->tmap_tail, p);
    else mlp_tc2_kernel<false><<<grid, kThreads, pl->smem, s>>>(pl->tmap, pl->tmap_tail, p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::fprintf(stderr, "libtang: mlp_tc2_kernel launch failed: %s (smem %zu)\n", cudaGetErrorString(e), pl->smem);
        return TANG_ECUDA;
    }
    return TANG_OK;
}

}  // namespace tang
