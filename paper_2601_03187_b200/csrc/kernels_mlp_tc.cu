// N1+N2: TaNG's residual MLP as one persistent tcgen05/TMEM kernel for sm_100a.
//
// What it computes (§6.1, Eq. 1-2, §6.2):
//   x  = 7 header segments / 65536                      (encode, fused: a2)
//   h  = ReLU(x.W0 + b0)      (a3: tensor core, x and W0 split into bf16 hi/lo: ~fp32 accurate, R22)
//   B times:  u = ReLU(h.W1 + b1);  h = ReLU(u.W2 + b2 + h)   (bf16 x bf16 -> fp32, tensor: a4)
//   logits = h.Wo + bo;  pred = argmax / top-k (ties -> lower index)            (a5)
// Quantisation points: h and u are rounded to bf16 (RNE) as GEMM inputs; bias, skip and ReLU
// are applied in fp32 before rounding (SURVEY.md §8(c) reading 5; the oracle's bf16 mode).
//
// Design:
//   * one CTA per SM, persistent over 128-packet tiles; M = 128 rows = 128 TMEM lanes.
//   * activations stay on chip for the whole chain: a [128 x N] bf16 tile in shared memory in
//     the UMMA K-major SWIZZLE_128B layout (the A operand), accumulators in TMEM (<= 512 cols).
//   * weights (K-major = [out][in] bf16) stream from L2 by TMA (SWIZZLE_128B boxes of 64 K x R
//     rows) through a STAGES-deep mbarrier ring; one elected thread issues tcgen05.mma.
//   * the residual skip is folded into the accumulator: after GEMM1 of a block completes, the
//     epilogue reads D1 chunk by chunk, writes u over h in shared memory (h is no longer an
//     operand) and stores (h + b2) into the just-drained TMEM columns; GEMM2 then accumulates
//     onto it, so h never needs a second buffer.
//   * warp roles: warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer,
//     warps 2..9 = epilogue (thread = packet row; warp w reads TMEM lanes 32*(w%4).. and
//     column half (w-2)/4 of every layer; the two halves' top-k merge through shared memory).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/tang.h"
#include "tang_internal.h"
#include "tc_ptx.h"

namespace tang {

struct TcPlan {
    CUtensorMap tmap;        // weights viewed as [rows_total][N] bf16, box {64, R}
    WeightsBF16 w;
    int R;                   // box rows (MMA N per instruction) = min(256, N)
    int stages;
    size_t smem;
    int grid;
    uint32_t tmem_cols;
    bool two_sm;             // cta_group::2 pairs (box {64, R/2}: each CTA loads half of B)
    int groups;              // epilogue warps per TMEM lane quadrant (2 or 4)
};

namespace {

using namespace tc;
// kG epilogue warps per TMEM lane quadrant (2 or 4); derived role constants per variant:
// warps 0..7 epilogue (warpgroups 0-1), warp 8 TMA producer, warp 9 MMA issuer + TMEM owner,
// warps 10-11 idle; warpgroup 2 gives registers to the epilogue warpgroups with setmaxnreg
template <int kG> struct Roles {
    static constexpr int kEpiThreads = 128 * kG;
    static constexpr int kThreads = kEpiThreads + 128;
    static constexpr int kProdWarp = 4 * kG, kMmaWarp = 4 * kG + 1;
    // setmaxnreg budgets: inc must fit in what dec frees (per warp: 32 lanes x regs)
    //   kG = 2: launch 168; (224-168)*8 warps <= (168-56)*4 warps.   kG = 4: launch 96; (104-96)*16 <= (96-56)*4
    static constexpr uint32_t kEpiRegs = kG == 2 ? 224 : 104, kCtlRegs = kG == 2 ? 56 : 56;
    static constexpr int kCW = kG == 2 ? 32 : 16;   // epilogue column chunk (TMEM load width)
};
constexpr int kTraceSlots = 64;           // clock64 stamps per (tile, layer) of the profiling trace

struct Params {
    const void* hdr;
    size_t n;
    uint32_t k;
    uint32_t* pred;
    float* logits;
    const float* W0; const float* b0;
    const float* b1; const float* b2;
    const float* bo;
    int N, B, C, Cp, R, stages;
    uint32_t tmem_cols;
    uint16_t* dbg;            // optional [(2B+1)][n][N] bf16 dump of every GEMM input (tests)
    int row_l0;               // first row of the split-bf16 layer-0 operand B0 in the weight tensor
    long long* trace;         // optional phase timestamps of block 0 (profiling): [4 tiles][layer][kTraceSlots]
};

// copy one 16-byte chunk (8 bf16 columns starting at col) of row i of layer l to the debug dump
template <bool kDbg>
__device__ __forceinline__ void dbg_put(const Params& p, int l, size_t i, int col, uint4 v) {
    if (!kDbg) return;
    if (p.dbg && i < p.n)
        *reinterpret_cast<uint4*>(p.dbg + (size_t(l) * p.n + i) * p.N + col) = v;
}

// cta_group::2 helpers (cta_rank, mapa_u32, cluster_sync_all, tma_load_2d_2sm, tma_load_2d_mc,
// mma_commit_mc, mma_bf16_2sm, mma_commit_2sm): tc_ptx.h

// bias vector element `off` of [b0 | b1 x B | b2 x B | bo] from its shared-memory copy at sb
__device__ __forceinline__ float4 bias4s(uint32_t sb, int off) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(sb + 4u * uint32_t(off)));
    return v;
}
// k2SM: a 2-CTA cluster runs M = 256 MMAs (tcgen05 cta_group::2): each CTA keeps its own 128-packet
// tile and epilogue, the leader issues the MMAs, and each CTA streams only HALF of every weight tile
// (B is split across the pair), which halves the shared-memory and L2 traffic per SM.
template <int W> __device__ __forceinline__ void tmem_ldw(uint32_t a, uint32_t (&r)[W]);
template <> __device__ __forceinline__ void tmem_ldw<16>(uint32_t a, uint32_t (&r)[16]) { tmem_ld16_async(a, r); }
template <> __device__ __forceinline__ void tmem_ldw<32>(uint32_t a, uint32_t (&r)[32]) { tmem_ld32_async(a, r); }

template <bool kDbg, int kG, bool k2SM>
__global__ void __launch_bounds__(Roles<kG>::kThreads, 1)
mlp_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ Params p) {
    constexpr int kEpiThreads = Roles<kG>::kEpiThreads;
    constexpr int kProdWarp = Roles<kG>::kProdWarp, kMmaWarp = Roles<kG>::kMmaWarp;
    constexpr uint32_t kEpiRegs = Roles<kG>::kEpiRegs, kCtlRegs = Roles<kG>::kCtlRegs;
    constexpr int CW = Roles<kG>::kCW;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int N = p.N, R = p.R, S = p.stages;
    const int KC = N / 64;                                  // 64-wide K chunks
    const uint32_t rank = cta_rank();                      // both modes run 2-CTA clusters
    const bool leader = rank == 0;
    const uint32_t stage_bytes = uint32_t(k2SM ? R / 2 : R) * 128;   // 2SM: this CTA's half of B
    uint8_t* act = smem;                                     // KC x 16 KB
    const uint32_t act_s = smem_u32(act);
    uint8_t* wst = smem + KC * (kM * 128);                  // S x stage_bytes
    uint64_t* full = reinterpret_cast<uint64_t*>(wst + S * stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* acc_full = empty + S;
    uint64_t* act_ready = acc_full + 1;
    uint64_t* half_ready = act_ready + 1;                   // first N-half of the A tile written
    uint64_t* acc_half = half_ready + 1;                    // accumulator N-half 0 complete
    uint64_t* a_lo_free = acc_half + 1;                     // A chunks [0, Hs / 64) no longer read
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_lo_free + 1);
    // bias vectors [b0 | b1 x B | b2 x B | bo] (contiguous from p.b0) in shared memory, copied once
    // per CTA: broadcast LDS on the epilogue chains instead of L1-prefetched global loads
    const uint32_t sb = smem_u32(wst + S * stage_bytes + 256);
    {
        const int nv = N + 2 * p.B * N + p.Cp;
        for (int v = threadIdx.x; v < nv / 4; v += blockDim.x)
            sts128(sb + 16u * v, __ldg(reinterpret_cast<const uint4*>(p.b0) + v));
    }

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = 2 * p.B + 1;                              // GEMMs per tile
    // split point of every epilogue: columns [0, Hs) (the first MMA N-half) are drained and
    // signalled first, so the next GEMM's (q = 0, kc < Hs / 64) MMAs overlap the rest
    const int Hs = N > R ? R : N;
    // N > R: two accumulator N-halves; the epilogue of a hidden GEMM processes half 0 (holding its
    // A-tile output in registers) while the MMAs of half 1 still run
    const bool split = N > R;
    size_t ntiles = (p.n + kM - 1) / kM;
    ntiles = (ntiles + 1) & ~size_t(1);                     // both CTAs of a pair run the same tile count
    // profiling trace record of (tile t, layer g): block 0, its first 4 tiles
    auto trace_rec = [&](size_t t, int g) -> long long* {
        return (p.trace && blockIdx.x == 0 && t < 4 * size_t(gridDim.x))
                   ? p.trace + ((t / gridDim.x) * L + g) * kTraceSlots : nullptr;
    };

    if (threadIdx.x == 0) {
        // single mode: a stage is free once BOTH CTAs' MMAs have read it (the peer multicasts into it)
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], k2SM ? 1 : 2); }
        mbar_init(acc_full, 1);
        // one arrival per epilogue warp (lane 0 after __syncwarp) of this CTA; in 2SM mode the leader's
        // barriers also count the peer's forwarder (its warp kMmaWarp), which collects the peer's warps on
        // the peer's own copy and passes one arrival on: per-warp remote release-arrives from the peer
        // measured ~0.5 us each, which made the peer CTA trail the leader at every epilogue barrier
        const uint32_t ne = kEpiThreads / 32 + ((k2SM && leader) ? 1 : 0);
        mbar_init(act_ready, ne);
        mbar_init(half_ready, ne);
        mbar_init(acc_half, 1);
        mbar_init(a_lo_free, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    if (warp == kMmaWarp) {
        if (k2SM) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                         ::"r"(smem_u32(tmem_slot)), "r"(p.tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                         ::"r"(smem_u32(tmem_slot)), "r"(p.tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    cluster_sync_all();                                     // peers' barriers initialised
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kProdWarp) {
      // control warpgroup: hand registers to the epilogue warpgroups, then split into roles
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs));
      if (warp == kProdWarp) {
        // ===== TMA producer: the weight tiles of every GEMM of every tile, in MMA order =====
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            long long* ptr = nullptr;                   // trace record of the layer being loaded
            auto load = [&](int kc, int row0, int nout, int q) {
                mbar_wait(&empty[s], ph ^ 1);
                const int si = q * KC + kc;
                if (ptr && si < 8) ptr[48 + 8 * blockIdx.x + si] = clock64();
                if (k2SM) {
                    // B of an N = nmma MMA is split: rows [0, nmma/2) from the leader, the rest
                    // from the peer; the leader's barrier expects both halves
                    const int nmma = min(R, nout - q * R);
                    if (leader) mbar_expect_tx(&full[s], 2 * stage_bytes);
                    tma_load_2d_2sm(wst + s * stage_bytes, &tmap, &full[s], kc * 64,
                                    row0 + q * R + int(rank) * (nmma / 2));
                } else {
                    // each CTA of the pair fetches half of the box's rows and multicasts them to both
                    const int nmma = min(R, nout - q * R);
                    mbar_expect_tx(&full[s], stage_bytes);
                    tma_load_2d_mc(wst + s * stage_bytes + uint32_t(rank) * uint32_t(nmma / 2) * 128u, &tmap, &full[s],
                                   kc * 64, row0 + q * R + int(rank) * (nmma / 2));
                }
                if (ptr && si < 8) ptr[16 + 8 * blockIdx.x + si] = clock64();
                if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
            };
            for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                ptr = nullptr;
                for (int q = 0; q < (N + R - 1) / R; ++q) load(0, p.row_l0, N, q);   // layer 0: K chunk 0 of B0
                for (int g = 0; g < L; ++g) {
                    // blocks 0 and 1 (the first pair) stamp their stage acquisitions and TMA issues
                    ptr = (p.trace && blockIdx.x < 2 && t < 4 * size_t(gridDim.x))
                              ? p.trace + ((t / gridDim.x) * L + g) * kTraceSlots : nullptr;
                    const int nout = (g == L - 1) ? p.Cp : N;
                    const int row0 = (g == L - 1) ? 2 * p.B * N : ((g & 1) ? (p.B + g / 2) * N : (g / 2) * N);
                    const int nq = (nout + R - 1) / R;
                    for (int q = 0; q < nq; ++q)
                        for (int kc = 0; kc < KC; ++kc) load(kc, row0, nout, q);
                }
            }
        }
      } else if (warp == kMmaWarp) {
        // ===== MMA issuer (the whole warp, one lane elected per instruction; the pair leader's warp
        //       in 2SM mode).  Descriptors are base + offset >> 4 (the start-address field). =====
        if (k2SM && !leader) {
            // forwarder: lane 0 relays act_ready, lane 1 half_ready, phase by phase, to the leader.
            // Per tile the epilogue arrives 2B + 2 times on act_ready (A0, layer 0, every hidden GEMM)
            // and 2B + 1 times on half_ready (layer 0, every hidden GEMM)
            if (lane < 2) {
                uint64_t* bar = lane == 0 ? act_ready : half_ready;
                const size_t per_tile = size_t(2 * p.B + (lane == 0 ? 2 : 1));
                const size_t my_tiles = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
                const uint32_t remote = mapa_u32(smem_u32(bar), 0);
                for (size_t k = 0; k < per_tile * my_tiles; ++k) {
                    mbar_wait(bar, uint32_t(k & 1));
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
                }
            }
        } else {
            uint32_t s = 0, ph = 0, aph = 0, hph = 0;
            // epilogue barriers: in 2SM mode they also receive the peer forwarder's release.cluster arrivals
            auto wait_epi = [&](uint64_t* bar, uint32_t parity) {
                if (k2SM) mbar_wait_cluster(bar, parity);
                else mbar_wait(bar, parity);
            };
            const uint64_t a_d0 = sdesc(smem_u32(act));
            const uint64_t w_d0 = sdesc(smem_u32(wst));
            for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                // layer 0 on the tensor core: D = A0.B0 over K = 48 (x and W0 split into exact bf16 pieces)
                wait_epi(act_ready, aph);
                aph ^= 1;
                tc_fence_after();
                for (int q = 0; q < (N + R - 1) / R; ++q) {
                    const int nmma = min(R, N - q * R);
                    const uint32_t id_r = k2SM ? (idesc(uint32_t(nmma)) & ~(0x1Fu << 24)) | ((256u >> 4) << 24)
                                               : idesc(uint32_t(nmma));
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint64_t b_d = w_d0 + uint64_t((s * stage_bytes) >> 4);
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        const uint64_t a = a_d0 + uint64_t(j * 2), b = b_d + uint64_t(j * 2);
                        if (k2SM) mma_bf16_2sm(tmem + uint32_t(q * R), a, b, id_r, j);
                        else mma_bf16_w(tmem + uint32_t(q * R), a, b, id_r, j);
                    }
                    if (k2SM) mma_commit_2sm(&empty[s]);
                    else mma_commit_mc(&empty[s]);
                    if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                }
                if (k2SM) mma_commit_2sm(acc_full);
                else mma_commit_w(acc_full);
                for (int g = 0; g < L; ++g) {
                    const bool is_out = g == L - 1;
                    const bool skip_init = !is_out && (g & 1);       // GEMM2: TMEM holds h + b2
                    const int nout = is_out ? p.Cp : N;
                    const int nq = (nout + R - 1) / R;
                    wait_epi(half_ready, hph);             // A chunks [0, Hs / 64) and TMEM [0, Hs) ready
                    hph ^= 1;
                    tc_fence_after();
                    bool whole = false;
                    long long* tr = lane == 0 ? trace_rec(t, g) : nullptr;
                    long long wfull = 0;
                    if (tr) tr[0] = clock64();
                    for (int q = 0; q < nq; ++q)
                        for (int kc = 0; kc < KC; ++kc) {
                            if (!whole && (q > 0 || kc * 64 >= Hs)) {
                                wait_epi(act_ready, aph);      // the whole A tile (and TMEM init) ready
                                aph ^= 1;
                                tc_fence_after();
                                whole = true;
                                if (tr) tr[3] = clock64();
                            }
                            const int nmma = min(R, nout - q * R);
                            const uint32_t id = k2SM ? (idesc(uint32_t(nmma)) & ~(0x1Fu << 24)) | ((256u >> 4) << 24)
                                                     : idesc(uint32_t(nmma));
                            long long w0 = tr ? clock64() : 0;
                            mbar_wait(&full[s], ph);
                            if (tr) {
                                const long long w1 = clock64();
                                wfull += w1 - w0;
                                if (q * KC + kc < 8) tr[32 + q * KC + kc] = w1;
                            }
                            tc_fence_after();
                            const uint64_t a_k = a_d0 + uint64_t((kc * (kM * 128)) >> 4);
                            const uint64_t b_d = w_d0 + uint64_t((s * stage_bytes) >> 4);
                            // one K chunk = four K = 16 MMAs under one elect (tc_ptx.h mma4_*)
                            const uint32_t acc = (skip_init || kc > 0) ? 1u : 0u;
                            if (k2SM) mma4_ss_2sm(tmem + uint32_t(q * R), a_k, b_d, id, acc);
                            else mma4_ss_1(tmem + uint32_t(q * R), a_k, b_d, id, acc);
                            if (k2SM) mma_commit_2sm(&empty[s]);     // frees the stage in both CTAs
                            else mma_commit_mc(&empty[s]);           // frees the stage (both CTAs read it)
                            if (split && !is_out && q == 0 && kc == KC - 1) {   // N-half 0 accumulated
                                if (k2SM) mma_commit_2sm(acc_half);
                                else mma_commit_w(acc_half);
                            }
                            // the last MMA reading A chunks [0, Hs / 64): the epilogue may overwrite
                            // them with this layer's N-half 0 output while N-half 1 still accumulates
                            if (split && !is_out && q == nq - 1 && kc == Hs / 64 - 1) {
                                if (k2SM) mma_commit_2sm(a_lo_free);
                                else mma_commit_w(a_lo_free);
                            }
                            if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                        }
                    if (!whole) {                               // keep the barrier phases in step
                        wait_epi(act_ready, aph);
                        aph ^= 1;
                    }
                    if (k2SM) mma_commit_2sm(acc_full);              // both CTAs' accumulators complete
                    else mma_commit_w(acc_full);                     // accumulator complete
                    if (tr) { tr[1] = clock64(); tr[2] = wfull; }
                }
            }
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
        // ===== epilogue: kEpiGroups warps per TMEM lane quadrant; thread = packet row,
        //       group g handles column half g of every layer =====
        const int quad = warp & 3;                          // TMEM lane quadrant of this warp
        const int grp = warp >> 2;                          // column group
        const int r = quad * 32 + lane;                     // row within the tile
        const uint32_t t_row = tmem + (uint32_t(quad * 32) << 16);
        // hidden columns of this group: one slice of each N-half, [lo[h], lo[h] + wd[h]) for h = 0, 1
        const int wd0 = Hs / kG, wd1 = (N - Hs) / kG;
        const int lo0 = grp * wd0, lo1 = Hs + grp * wd1;
        const int nch0 = wd0 / CW, nch = (wd0 + wd1) / CW;    // chunks in part 0, in total
        auto col_of = [&](int k) { return k < nch0 ? lo0 + k * CW : lo1 + (k - nch0) * CW; };
        const int ocw = ((p.Cp / kG + 15) / 16) * 16;        // output columns per group (multiple of 16)
        const int oc0 = min(grp * ocw, p.Cp), oc1 = min((grp + 1) * ocw, p.Cp);
        // top-k merge scratch for groups 1..kG-1 (the A tile is free while the output epilogue runs)
        float* mv = reinterpret_cast<float*>(act);
        int* mi = reinterpret_cast<int*>(act + (kG - 1) * kM * 4 * sizeof(float));
        uint32_t fph = 0, hfph = 0, lph = 0;
        long long* etr = nullptr;                           // trace record of the current layer
        const int eo = threadIdx.x == 128 ? 4 : 0;          // stamps of threads 0 and 128 (column groups 0, 1)
        // every lane has fenced its own writes; __syncwarp orders them before lane 0's release-arrive
        // (one arrival per warp: 256 per-thread remote arrivals of the peer CTA per barrier phase
        // measured ~1-2k cycles of skew at the pair's barriers)
        auto arrive_act = [&]() {
            __syncwarp();
            if (lane == 0) mbar_arrive(act_ready);      // 2SM peer: its own copy, relayed by its forwarder
        };
        // A tile (and TMEM init) of N-half h written: h = 0 -> half_ready, h = 1 -> act_ready
        auto arrive_part = [&](int h) {
            if (etr) etr[(h ? 7 : 6) + eo] = clock64();
            fence_proxy_async();
            tc_fence_before();
            if (h) { arrive_act(); return; }
            __syncwarp();
            if (lane == 0) mbar_arrive(half_ready);
        };
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const size_t i = t * kM + r;
            long long* ltr = threadIdx.x == 0 ? trace_rec(t, 0) : nullptr;
            if (ltr) ltr[12] = clock64();
            etr = nullptr;
            // h = ReLU(D [+ b0]) over this group's columns -> bf16 A tile (layer 0 and every GEMM2)
            // sp: entered on acc_half; part 0 (4 chunks) is packed into registers while the MMAs of
            // N-half 1 still read the A tile, stored after acc_full
            auto drain_relu = [&](bool add_b0, int dl, bool sp) {
                uint32_t cur[CW], nxt[CW];
                int kk0 = 0;
                __syncwarp();
                if (sp) {
                    uint32_t held[4][CW / 2];
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {          // off the critical path: no prefetch
                        tmem_ldw<CW>(t_row + uint32_t(lo0 + kk * CW), cur);
                        tmem_wait_ld();
#pragma unroll
                        for (int j = 0; j < CW / 2; ++j)
                            held[kk][j] = relu_pack_bf16(__uint_as_float(cur[2 * j]), __uint_as_float(cur[2 * j + 1]));
                    }
                    // A chunks [0, Hs / 64) are no longer read once a_lo_free fires (N-half 1 may
                    // still accumulate): store N-half 0 and let the next GEMM start on it
                    mbar_wait(a_lo_free, lph);
                    lph ^= 1;
                    tc_fence_after();
                    if (etr) etr[5 + eo] = clock64();
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                        for (int q = 0; q < CW / 8; ++q) {
                            const uint4 o = make_uint4(held[kk][4 * q], held[kk][4 * q + 1], held[kk][4 * q + 2],
                                                       held[kk][4 * q + 3]);
                            sts128(act_addr(act_s, r, (lo0 + kk * CW) / 8 + q), o);
                            dbg_put<kDbg>(p, dl, i, lo0 + kk * CW + 8 * q, o);
                        }
                    arrive_part(0);
                    mbar_wait(acc_full, fph);                 // N-half 1 accumulated
                    fph ^= 1;
                    tc_fence_after();
                    if (etr) etr[14 + (eo ? 1 : 0)] = clock64();
                    kk0 = nch0;
                    tmem_ldw<CW>(t_row + uint32_t(lo1), cur);
                } else {
                    tmem_ldw<CW>(t_row + uint32_t(lo0), cur);
                }
                tmem_wait_ld();
                for (int kk = kk0; kk < nch; ++kk) {
                    const int c0 = col_of(kk);
                    if (kk + 1 < nch) tmem_ldw<CW>(t_row + uint32_t(col_of(kk + 1)), nxt);
#pragma unroll
                    for (int q = 0; q < CW / 8; ++q) {
                        float* f = reinterpret_cast<float*>(cur) + 8 * q;
                        if (add_b0) {
                            const float4 ba = bias4s(sb, c0 + 8 * q), bb = bias4s(sb, c0 + 8 * q + 4);
                            f[0] += ba.x; f[1] += ba.y; f[2] += ba.z; f[3] += ba.w;
                            f[4] += bb.x; f[5] += bb.y; f[6] += bb.z; f[7] += bb.w;
                        }
                        const uint4 o = make_uint4(relu_pack_bf16(f[0], f[1]), relu_pack_bf16(f[2], f[3]),
                                                   relu_pack_bf16(f[4], f[5]), relu_pack_bf16(f[6], f[7]));
                        sts128(act_addr(act_s, r, c0 / 8 + q), o);
                        dbg_put<kDbg>(p, dl, i, c0 + 8 * q, o);
                    }
                    if (kk == nch0 - 1) arrive_part(0);       // N-half 0 done: the next GEMM may start
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < CW; ++j) cur[j] = nxt[j];
                }
                arrive_part(1);
            };
            // a2: features x = segment / 65536 split exactly into bf16 hi + lo; A0 row (K = 48, chunk 0)
            // = [xh | xl | xh | xl | xh | xl | 0..] against B0 = [W0h | W0h | W0m | W0m | W0l | W0l | 0..]
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
            arrive_act();
            // a3: layer 0, h0 = ReLU(x.W0 + b0) -> bf16 A tile
            mbar_wait(acc_full, fph);
            fph ^= 1;
            tc_fence_after();
            drain_relu(true, 0, false);
            if (ltr) ltr[13] = clock64();

            for (int g = 0; g < L; ++g) {
                const bool sp = split && g < L - 1;      // hidden GEMM with two N-halves
                if (sp) { mbar_wait(acc_half, hfph); hfph ^= 1; }
                else { mbar_wait(acc_full, fph); fph ^= 1; }
                tc_fence_after();
                etr = (threadIdx.x == 0 || threadIdx.x == 128) ? trace_rec(t, g) : nullptr;
                if (etr) etr[4 + eo] = clock64();
                if (g == L - 1) {
                    // a5: logits = D + bo; top-k (ties -> lower index), optional logits out
                    const int k = int(p.k);
                    float bv[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
                    int bc[4] = {0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF};
                    float b0v = -FLT_MAX;                // top-1 running max stays in registers
                    int b0c = 0x7FFFFFFF;
                    const bool fast = k == 1 && p.logits == nullptr;
                    __syncwarp();
                    int cs = oc0;                          // first column left for the 16-wide loop
                    if (fast) {
                        // top-1 without logits: 32-column TMEM loads, pairwise tree argmax per
                        // chunk (left operand wins ties = first maximum; padded columns c >= C
                        // enter as -inf), one strict merge per chunk
                        for (; cs + 32 <= oc1; cs += 32) {
                            uint32_t v[32];
                            tmem_ld32_async(t_row + uint32_t(cs), v);
                            float z[32];
                            int zi[32];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 f4 = bias4s(sb, N + 2 * p.B * N + cs + 4 * q);
                                z[4 * q] = f4.x; z[4 * q + 1] = f4.y; z[4 * q + 2] = f4.z; z[4 * q + 3] = f4.w;
                            }
                            tmem_wait_ld();
#pragma unroll
                            for (int x = 0; x < 32; ++x) {
                                z[x] = cs + x < p.C ? __uint_as_float(v[x]) + z[x] : -INFINITY;
                                zi[x] = x;
                            }
#pragma unroll
                            for (int st = 1; st < 32; st *= 2)
#pragma unroll
                                for (int x = 0; x < 32; x += 2 * st)
                                    if (z[x + st] > z[x]) { z[x] = z[x + st]; zi[x] = zi[x + st]; }
                            if (z[0] > b0v) { b0v = z[0]; b0c = cs + zi[0]; }
                        }
                    }
                    for (int c0 = cs; c0 < oc1; c0 += 16) {
                        uint32_t v[16];
                        tmem_ld16_async(t_row + uint32_t(c0), v);
                        float bq[16];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float4 f4 = bias4s(sb, N + 2 * p.B * N + c0 + 4 * q);
                            bq[4 * q] = f4.x; bq[4 * q + 1] = f4.y; bq[4 * q + 2] = f4.z; bq[4 * q + 3] = f4.w;
                        }
                        tmem_wait_ld();
                        if (fast) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const float z = __uint_as_float(v[j]) + bq[j];
                                if (c0 + j < p.C && z > b0v) { b0v = z; b0c = c0 + j; }
                            }
                            continue;
                        }
                        for (int j = 0; j < 16; ++j) {
                            const int c = c0 + j;
                            if (c >= p.C) break;
                            const float z = __uint_as_float(v[j]) + bq[j];
                            if (p.logits && i < p.n) p.logits[i * p.C + c] = z;
                            if (k == 1) {
                                if (z > b0v) { b0v = z; b0c = c; }
                            } else if (z > bv[k - 1]) {   // insertion, strict > keeps the lower index
                                int pos = k - 1;
                                while (pos > 0 && z > bv[pos - 1]) { bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos; }
                                bv[pos] = z;
                                bc[pos] = c;
                            }
                        }
                    }
                    if (k == 1) { bv[0] = b0v; bc[0] = b0c; }
                    tc_fence_before();   // TMEM reads done before the next tile's GEMMs
                    // merge the column groups' candidates (group 1's indices are all larger,
                    // so strict > keeps ties on the lower index)
                    if (grp > 0)
                        for (int q = 0; q < k; ++q) {
                            mv[((grp - 1) * kM + r) * 4 + q] = bv[q];
                            mi[((grp - 1) * kM + r) * 4 + q] = bc[q];
                        }
                    epi_bar(1, kEpiThreads);
                    if (grp == 0) {
                        // groups in column order: strict > keeps ties on the lower index
                        for (int g2 = 1; g2 < kG; ++g2) {
                            const float* gv = mv + ((g2 - 1) * kM + r) * 4;
                            const int* gi = mi + ((g2 - 1) * kM + r) * 4;
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
                        }
                        if (i < p.n)
                            for (int q = 0; q < k; ++q) p.pred[i * k + q] = uint32_t(bc[q]);
                    }
                    epi_bar(2, kEpiThreads);          // scratch consumed before the next tile's layer 0
                    if (etr) etr[7 + eo] = clock64();
                } else if ((g & 1) == 0) {
                    // GEMM1 of block b: u = ReLU(D + b1) over h in smem; TMEM <- h + b2 (skip fold).
                    // 32-column chunks; the next chunk's accumulator load is in flight while this
                    // one is processed (D[c] is read before h + b2 overwrites the same columns).
                    const int b = g / 2;
                    const int o1 = N + b * N, o2 = N + p.B * N + b * N;    // offsets of b1, b2 of block b
                    uint32_t bufA[CW], bufB[CW];
                    __syncwarp();
                    auto chunk = [&](int kk, uint32_t (&cur)[CW], uint32_t (&nxt)[CW]) {
                        const int c0 = col_of(kk);
                        uint32_t aa[CW / 8];
                        uint4 hh[CW / 8];
#pragma unroll
                        for (int q = 0; q < CW / 8; ++q) { aa[q] = act_addr(act_s, r, c0 / 8 + q); hh[q] = lds128(aa[q]); }
                        if (kk + 1 < nch) tmem_ldw<CW>(t_row + uint32_t(col_of(kk + 1)), nxt);   // next chunk in flight
#pragma unroll
                        for (int hf = 0; hf < CW / 16; ++hf) {    // h + b2 -> TMEM in 16-column pieces
                            float sv[16];
#pragma unroll
                            for (int q2 = 0; q2 < 2; ++q2) {
                                const int q = 2 * hf + q2;
                                const float4 ba = bias4s(sb, o2 + c0 + 8 * q);
                                const float4 bb = bias4s(sb, o2 + c0 + 8 * q + 4);
                                float* o = sv + 8 * q2;
                                add2(o[0], o[1], bf16_lo(hh[q].x), bf16_hi(hh[q].x), ba.x, ba.y);
                                add2(o[2], o[3], bf16_lo(hh[q].y), bf16_hi(hh[q].y), ba.z, ba.w);
                                add2(o[4], o[5], bf16_lo(hh[q].z), bf16_hi(hh[q].z), bb.x, bb.y);
                                add2(o[6], o[7], bf16_lo(hh[q].w), bf16_hi(hh[q].w), bb.z, bb.w);
                            }
                            tmem_st16(t_row + uint32_t(c0 + 16 * hf), sv);
                        }
#pragma unroll
                        for (int q = 0; q < CW / 8; ++q) {
                            const float4 ba = bias4s(sb, o1 + c0 + 8 * q);
                            const float4 bb = bias4s(sb, o1 + c0 + 8 * q + 4);
                            const float* f = reinterpret_cast<const float*>(cur) + 8 * q;
                            float z[8];
                            add2(z[0], z[1], f[0], f[1], ba.x, ba.y);
                            add2(z[2], z[3], f[2], f[3], ba.z, ba.w);
                            add2(z[4], z[5], f[4], f[5], bb.x, bb.y);
                            add2(z[6], z[7], f[6], f[7], bb.z, bb.w);
                            const uint4 o = make_uint4(relu_pack_bf16(z[0], z[1]), relu_pack_bf16(z[2], z[3]),
                                                       relu_pack_bf16(z[4], z[5]), relu_pack_bf16(z[6], z[7]));
                            sts128(aa[q], o);
                            dbg_put<kDbg>(p, g + 1, i, c0 + 8 * q, o);
                        }
                        if (kk == nch0 - 1) {                 // N-half 0 (u and h + b2) done
                            tmem_st_wait();
                            arrive_part(0);
                        }
                        tmem_wait_ld();
                    };
                    int kk0 = 0;
                    if (sp) {                                 // part 0 = 4 chunks while N-half 1 accumulates
                        uint32_t held[4][CW / 2];
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const int c0 = lo0 + kk * CW;
                            uint32_t d[CW];
                            tmem_ldw<CW>(t_row + uint32_t(c0), d);
#pragma unroll
                            for (int hf = 0; hf < CW / 16; ++hf) {    // h + b2 -> TMEM (16 columns)
                                float sv[16];
#pragma unroll
                                for (int q2 = 0; q2 < 2; ++q2) {
                                    const int q = 2 * hf + q2;
                                    const uint4 hq = lds128(act_addr(act_s, r, c0 / 8 + q));
                                    const float4 ba = bias4s(sb, o2 + c0 + 8 * q);
                                    const float4 bb = bias4s(sb, o2 + c0 + 8 * q + 4);
                                    float* o = sv + 8 * q2;
                                    add2(o[0], o[1], bf16_lo(hq.x), bf16_hi(hq.x), ba.x, ba.y);
                                    add2(o[2], o[3], bf16_lo(hq.y), bf16_hi(hq.y), ba.z, ba.w);
                                    add2(o[4], o[5], bf16_lo(hq.z), bf16_hi(hq.z), bb.x, bb.y);
                                    add2(o[6], o[7], bf16_lo(hq.w), bf16_hi(hq.w), bb.z, bb.w);
                                }
                                tmem_wait_ld();                       // D read before h + b2 overwrites it
                                tmem_st16(t_row + uint32_t(c0 + 16 * hf), sv);
                            }
#pragma unroll
                            for (int q = 0; q < CW / 8; ++q) {        // u = ReLU(D + b1) -> registers
                                const float4 ba = bias4s(sb, o1 + c0 + 8 * q);
                                const float4 bb = bias4s(sb, o1 + c0 + 8 * q + 4);
                                const float* f = reinterpret_cast<const float*>(d) + 8 * q;
                                float z[8];
                                add2(z[0], z[1], f[0], f[1], ba.x, ba.y);
                                add2(z[2], z[3], f[2], f[3], ba.z, ba.w);
                                add2(z[4], z[5], f[4], f[5], bb.x, bb.y);
                                add2(z[6], z[7], f[6], f[7], bb.z, bb.w);
                                held[kk][4 * q] = relu_pack_bf16(z[0], z[1]);
                                held[kk][4 * q + 1] = relu_pack_bf16(z[2], z[3]);
                                held[kk][4 * q + 2] = relu_pack_bf16(z[4], z[5]);
                                held[kk][4 * q + 3] = relu_pack_bf16(z[6], z[7]);
                            }
                        }
                        tmem_st_wait();
                        mbar_wait(a_lo_free, lph);            // the MMAs no longer read h chunks 0..: store u
                        lph ^= 1;
                        tc_fence_after();
                        if (etr) etr[5 + eo] = clock64();
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                            for (int q = 0; q < CW / 8; ++q) {
                                const uint4 o = make_uint4(held[kk][4 * q], held[kk][4 * q + 1], held[kk][4 * q + 2],
                                                           held[kk][4 * q + 3]);
                                sts128(act_addr(act_s, r, (lo0 + kk * CW) / 8 + q), o);
                                dbg_put<kDbg>(p, g + 1, i, lo0 + kk * CW + 8 * q, o);
                            }
                        arrive_part(0);
                        mbar_wait(acc_full, fph);             // N-half 1 accumulated
                        fph ^= 1;
                        tc_fence_after();
                        if (etr) etr[14 + (eo ? 1 : 0)] = clock64();
                        kk0 = nch0;
                    }
                    tmem_ldw<CW>(t_row + uint32_t(col_of(kk0)), bufA);
                    tmem_wait_ld();
                    for (int kk = kk0; kk < nch; kk += 2) {   // ping-pong: no register copy between chunks
                        chunk(kk, bufA, bufB);
                        if (kk + 1 < nch) chunk(kk + 1, bufB, bufA);
                    }
                    tmem_st_wait();
                    arrive_part(1);
                } else {
                    // GEMM2 of block b: h = ReLU(D) (D already holds u.W2 + b2 + h)
                    drain_relu(false, g + 1, sp);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();                // 2SM: the leader's MMAs also wrote the peer's TMEM; single: the
                                       // peer's multicast commits target this CTA's barriers
    if (warp == kMmaWarp) {
        tc_fence_after();
        if (k2SM) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols));
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

template <bool kDbg, int kG, bool k2SM>
static bool set_smem(size_t smem) {
    return cudaFuncSetAttribute(mlp_tc_kernel<kDbg, kG, k2SM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(smem)) == cudaSuccess;
}

TcPlan* tc_plan_create(const WeightsBF16& w, const float* h_bias, int device, int two_sm, int groups, int* err) {
    *err = TANG_OK;
    if (w.Cp > 512 || w.N % 64 || w.N > 512) { *err = TANG_EMODEL; return nullptr; }
    TcPlan* p = new TcPlan();
    p->w = w;
    p->two_sm = two_sm != 0 && w.N >= 256;
    p->groups = (groups == 4 && !p->two_sm && w.N >= 64) ? 4 : 2;
    p->R = w.N < 256 ? w.N : 256;            // N = 256 per MMA: A is re-read once per 256 outputs
    const int KC = w.N / 64;
    const size_t act = size_t(KC) * kM * 128;
    const size_t stage = size_t(p->two_sm ? p->R / 2 : p->R) * 128;
    const size_t budget = 227 * 1024 - 1024 - 256;
    const size_t cbytes = size_t(w.N + 2 * w.B * w.N + w.Cp) * 4;   // bias vectors (smem)
    p->stages = int((budget - act - cbytes) / stage);
    if (p->stages > 12) p->stages = 12;
    if (p->stages < 2) { delete p; *err = TANG_EMODEL; return nullptr; }
    p->smem = 1024 + act + p->stages * stage + 256 + cbytes;
    uint32_t cols = 32;
    const int need = w.N > w.Cp ? w.N : w.Cp;
    while (cols < uint32_t(need)) cols <<= 1;
    p->tmem_cols = cols;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    // every variant runs as 2-CTA clusters (2SM pairs, or the single kernel's weight-sharing pairs):
    // an even grid, also on parts / partitions with an odd SM count
    p->grid = (sms / 2) * 2;

    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    const uint64_t rows = uint64_t(2) * w.B * w.N + w.Cp + w.N;   // + the split-bf16 layer-0 block B0
    cuuint64_t dims[2] = {cuuint64_t(w.N), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(w.N) * 2};
    cuuint32_t box[2] = {64, cuuint32_t(p->R / 2)};    // half boxes: 2SM split / single multicast
    cuuint32_t estr[2] = {1, 1};
    CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(
        &p->tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(w.W1t), dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::fprintf(stderr, "libtang: cuTensorMapEncodeTiled failed (%d)\n", int(r));
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    const bool ok = set_smem<false, 2, false>(p->smem) && set_smem<true, 2, false>(p->smem) &&
                    set_smem<false, 4, false>(p->smem) && set_smem<true, 4, false>(p->smem) &&
                    set_smem<false, 2, true>(p->smem) && set_smem<true, 2, true>(p->smem);
    if (!ok) { delete p; *err = TANG_ECUDA; return nullptr; }
    return p;
}

void tc_plan_destroy(TcPlan* p) { delete p; }

template <bool kDbg, int kG, bool k2SM>
static cudaError_t launch_variant(const TcPlan* pl, int grid, const Params& p, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(Roles<kG>::kThreads);
    cfg.dynamicSmemBytes = pl->smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, mlp_tc_kernel<kDbg, kG, k2SM>, pl->tmap, p);
}

int launch_mlp_tc(const TcPlan* pl, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                  cudaStream_t s, uint16_t* dbg, long long* trace) {
    if (!pl) return TANG_EMODEL;
    if (n == 0) return TANG_OK;
    Params p{};
    p.hdr = hdr; p.n = n; p.k = k; p.pred = pred; p.logits = logits;
    p.W0 = pl->w.W0; p.b0 = pl->w.b0; p.b1 = pl->w.b1; p.b2 = pl->w.b2; p.bo = pl->w.bo;
    p.N = pl->w.N; p.B = pl->w.B; p.C = pl->w.C; p.Cp = pl->w.Cp; p.R = pl->R; p.stages = pl->stages;
    p.tmem_cols = pl->tmem_cols;
    p.row_l0 = 2 * pl->w.B * pl->w.N + pl->w.Cp;
    p.dbg = dbg;
    p.trace = trace;
    size_t tiles = (n + kM - 1) / kM;
    tiles = (tiles + 1) & ~size_t(1);                 // 2-CTA clusters: an even grid
    const int grid = int(tiles < size_t(pl->grid) ? tiles : size_t(pl->grid));
    const bool db = dbg != nullptr;
    cudaError_t e;
    if (pl->two_sm)
        e = db ? launch_variant<true, 2, true>(pl, grid, p, s) : launch_variant<false, 2, true>(pl, grid, p, s);
    else if (pl->groups == 4)
        e = db ? launch_variant<true, 4, false>(pl, grid, p, s) : launch_variant<false, 4, false>(pl, grid, p, s);
    else
        e = db ? launch_variant<true, 2, false>(pl, grid, p, s) : launch_variant<false, 2, false>(pl, grid, p, s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, mlp_tc_kernel<false, 2, false>);
        std::fprintf(stderr, "libtang: mlp_tc_kernel launch failed: %s (smem %zu, regs %d, maxThreads %d)\n",
                     cudaGetErrorString(e), pl->smem, fa.numRegs, fa.maxThreadsPerBlock);
        return TANG_ECUDA;
    }
    return TANG_OK;
}

}  // namespace tang
