// a2-a5, bf16: TaNG's residual MLP (§6.1, Eq. 1-2, §6.2) as one persistent
// tcgen05 kernel for sm_100a in which half of the GEMMs read their A operand from TENSOR memory.
//
// Same arithmetic and quantisation points as mlp_tc_kernel (kernels_mlp_tc.cu):
//   x = 7 segments / 65536 (split exactly into bf16 hi + lo), h0 = ReLU(x.W0 + b0) on the tensor core
//   from exact bf16 pieces; B blocks u = ReLU(h.W1 + b1), h = ReLU(u.W2 + b2 + h); logits = h.Wo + bo;
//   h and u rounded RNE to bf16 as GEMM inputs, bias / skip / ReLU in fp32 before rounding.
//
// Why (profiles/r02_ab_bf16_cluster4_multicast.txt): in mlp_tc_kernel every GEMM reads
// its [128 x 512] A tile from shared memory twice (once per 256-column MMA N-half) while the weight TMA
// writes and the epilogue's loads/stores share the same shared-memory port; that port, not the tensor
// core, sets the layer time.  Here the chain alternates two GEMM kinds over a 2-CTA cta_group::2 pair
// (M = 256, each CTA owns 128 packets = 128 TMEM lanes):
//   S (A in smem): layer 0 (A0 = split features, K = 48) and every GEMM2 (A = u).  N = 512 as two
//     256-column MMA halves; the fp32 accumulator fills TMEM [0, 512).
//   T (A in TMEM, "TS"): every GEMM1 (A = h) and the output layer (A = h).  A = h is kept in TMEM as
//     packed bf16 pairs (256 columns); the output runs as N = 128 sub-passes into two 128-column
//     accumulators P0 = [64, 192), P1 = [320, 448) that the epilogue drains in turn.
// So GEMM1 and the output layer read no A from shared memory, GEMM1's u goes to shared memory (the A
// of GEMM2) and GEMM2's h never touches shared memory: it is packed into TMEM in place.
//
// TMEM map (columns, per CTA; TS operand layout pinned by scripts/ts_probe.cu, profiles/r02_ts_probe.txt):
//   S accumulator half q:          [256q, 256q + 256)
//   packed h of half q (bf16 x 2): group 0 (columns 256q + [0, 128) of h) at [256q, 256q + 64),
//                                  group 1 (columns 256q + [128, 256))   at [256q + 192, 256q + 256)
//   T accumulators:                P0 = [64, 192), P1 = [320, 448)
// The epilogue packs in place: group 0 drains its 128 columns upwards and writes chunk c at c / 2,
// group 1 drains downwards and writes chunk c at 192 + (c - 128) / 2, so a thread only ever writes
// columns it has already read, and the T accumulators are the two contiguous holes that remain.
// The GEMM2 skip is folded into its accumulator: before GEMM2 half q starts, the epilogue reads the
// packed h of half q and stores h + b2 over [256q, 256q + 256) (TMEM loads/stores, not shared memory).
//
// Warp roles: warps 0-7 epilogue (thread = packet row; warp w reads lane quadrant w % 4, column
// group w / 4), warp 8 TMA producer, warp 9 MMA issuer + TMEM owner (the pair leader's), 10-11 idle.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdio>

#include "../../include/tang.h"
#include "tang_internal.h"
#include "tc_ptx.h"

namespace tang {

struct TsPlan {
    CUtensorMap tmap;        // weights as [rows][N] bf16, box {64, 64}
    WeightsBF16 w;
    int stages;
    size_t smem;
    int grid;
};

namespace {

using namespace tc;
constexpr int kEpi = 256;                 // epilogue threads (2 column groups x 4 lane quadrants x 32)
constexpr int kThreads = kEpi + 128;
constexpr int kProdWarp = 8, kMmaWarp = 9;
constexpr uint32_t kStage = 16384;        // weight bytes per CTA per stage (two 64 x 64 boxes)
constexpr uint32_t kBox = 8192;
constexpr int kTraceSlots = 192;

struct TsParams {
    const void* hdr;
    size_t n;
    uint32_t k;
    uint32_t* pred;
    float* logits;
    const float* bias;        // [b0 | b1 x B | b2 x B | bo] contiguous
    int B, C, Cp, stages;
    int row_l0;               // first row of the split-bf16 layer-0 block B0
    uint16_t* dbg;            // optional [(2B+1)][n][512] bf16 dump of every GEMM input (tests)
    long long* trace;         // optional phase stamps of block 0: [4 tiles][2B+2 GEMMs][kTraceSlots]
};

constexpr int N = 512;        // hidden width this kernel is built for (the paper's model)

__device__ __forceinline__ uint32_t idesc2(uint32_t n) {   // kind::f16, M = 256 (cta_group::2), N = n
    return (idesc(n) & ~(0x1Fu << 24)) | ((256u >> 4) << 24);
}
__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ float4 bias4s(uint32_t sb, int off) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(sb + 4u * uint32_t(off)));
    return v;
}
// TMEM column of the packed h holding K step k16 (h columns 16 k16 .. 16 k16 + 15)
__device__ __forceinline__ uint32_t hcol(int k16) {
    const int k = 16 * k16, half = k >> 8, kk = k & 255;
    return uint32_t(256 * half + (kk < 128 ? kk / 2 : 192 + (kk - 128) / 2));
}
template <bool kDbg>
__device__ __forceinline__ void dbg_put(const TsParams& p, int l, size_t i, int col, uint4 v) {
    if (!kDbg) return;
    if (p.dbg && i < p.n) *reinterpret_cast<uint4*>(p.dbg + (size_t(l) * p.n + i) * N + col) = v;
}
// "better" for the top-k merge across column groups: larger logit, ties to the lower class index
__device__ __forceinline__ bool better(float z, int c, float bz, int bc) { return z > bz || (z == bz && c < bc); }

template <bool kDbg>
__global__ void __launch_bounds__(kThreads, 1)
mlp_ts_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TsParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages, B = p.B;
    uint8_t* act = smem;                                     // [128 x 512] bf16, 8 K-chunks of 16 KB
    const uint32_t act_s = smem_u32(act);
    uint8_t* wst = smem + 8 * (kM * 128);
    uint64_t* full = reinterpret_cast<uint64_t*>(wst + S * kStage);
    uint64_t* empty = full + S;
    uint64_t* accb = empty + S;                              // [2] MMA -> epilogue (S halves / T sub-passes)
    uint64_t* a0_ready = accb + 2;                           // A0 written, TMEM free (tile start)
    uint64_t* h_half = a0_ready + 1;                         // [2] packed h of half q in TMEM
    uint64_t* fold = h_half + 2;                             // [2] GEMM2 accumulator half q = h + b2
    uint64_t* p_free = fold + 2;                             // [2] T accumulator P_x drained
    uint64_t* h0_read = p_free + 2;                          // GEMM1's last MMA reading h half 0 done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h0_read + 1);
    const uint32_t sb = smem_u32(wst + S * kStage + 256);   // bias vectors in shared memory
    {
        const int nv = N + 2 * B * N + p.Cp;
        for (int v = threadIdx.x; v < nv / 4; v += blockDim.x)
            sts128(sb + 16u * v, __ldg(reinterpret_cast<const uint4*>(p.bias) + v));
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    const bool leader = rank == 0;
    const int nj = (p.Cp + 127) / 128;                       // output sub-passes
    size_t ntiles = (p.n + kM - 1) / kM;
    ntiles = (ntiles + 1) & ~size_t(1);                      // both CTAs of the pair run the same tiles
    const int L = 2 * B + 2;                                 // GEMMs per tile (with layer 0)
    auto trace_rec = [&](size_t t, int g) -> long long* {
        return (p.trace && blockIdx.x == 0 && t < 4 * size_t(gridDim.x))
                   ? p.trace + ((t / gridDim.x) * L + g) * kTraceSlots : nullptr;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        // epilogue -> MMA barriers: one arrival per epilogue warp of this CTA; the leader's also count the
        // peer's forwarder (its warp 9), which collects the peer's warps on the peer's own copy of the
        // barrier and passes one arrival on (a per-warp remote release-arrive measured ~0.5 us each)
        const uint32_t ne = kEpi / 32 + (cta_rank() == 0 ? 1 : 0);
        for (int x = 0; x < 2; ++x) {
            mbar_init(&accb[x], 1);
            mbar_init(&h_half[x], ne);
            mbar_init(&fold[x], ne);
            mbar_init(&p_free[x], ne);
        }
        mbar_init(a0_ready, ne);
        mbar_init(h0_read, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kProdWarp) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");   // (224 - 216) budget: 8 x 216 + 4 x 72 <= 12 x 168
      if (warp == kProdWarp) {
        // ===== TMA producer: every weight stage of every GEMM in MMA order =====
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            // one stage = two 64 x 64 boxes: (k0, row0) at +0 and (k1, row1) at +8 KB
            long long* ptr = nullptr;               // profiling: GEMM record of block 0 / its stage counter
            int pi = 0;
            auto load = [&](int k0, int row0, int k1, int row1) {
                mbar_wait(&empty[s], ph ^ 1);
                if (ptr && pi >= 4 && pi < 8) ptr[40 + pi - 4] = clock64();   // stage acquired, TMA issued
                ++pi;
                if (leader) mbar_expect_tx(&full[s], 2 * kStage);
                tma_load_2d_2sm(wst + s * kStage, &tmap, &full[s], k0, row0);
                tma_load_2d_2sm(wst + s * kStage + kBox, &tmap, &full[s], k1, row1);
                if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
            };
            // S GEMM half q: this CTA's 128 rows of the 256-row block, one 64-wide K chunk per stage
            auto load_s = [&](int rowblk, int nk) {
                for (int q = 0; q < 2; ++q) {
                    const int r0 = rowblk + 256 * q + 128 * int(rank);
                    for (int kc = 0; kc < nk; ++kc) load(64 * kc, r0, 64 * kc, r0 + 64);
                }
            };
            // T GEMM sub-pass j: this CTA's half of the nmma rows, two K chunks per stage
            auto load_t = [&](int rowblk, int nout) {
                for (int j = 0; j < (nout + 127) / 128; ++j) {
                    const int nmma = min(128, nout - 128 * j);
                    const int r0 = rowblk + 128 * j + int(rank) * (nmma / 2);
                    // K chunks (0, 2), (1, 3), (4, 6), (5, 7): the two boxes of a stage lie 256 B apart in
                    // each row, so they land in different L2 slices (adjacent 128-B lines share one)
                    for (int st = 0; st < 4; ++st) {
                        const int kc = (st >> 1) * 4 + (st & 1);
                        load(64 * kc, r0, 64 * (kc + 2), r0);
                    }
                }
            };
            for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                auto rec = [&](int g) { ptr = trace_rec(t, g); pi = 0; };
                rec(0);
                load_s(p.row_l0, 1);                                  // layer 0: K chunk 0 of B0
                for (int b = 0; b < B; ++b) {
                    rec(2 * b + 1);
                    load_t(b * N, N);                                 // GEMM1 of block b
                    rec(2 * b + 2);
                    load_s((B + b) * N, 8);                           // GEMM2 of block b
                }
                rec(L - 1);
                load_t(2 * B * N, p.Cp);                              // output layer
            }
        }
      } else if (warp == kMmaWarp && !leader) {
        // ===== forwarder (peer CTA): lane i relays epilogue barrier i to the leader, phase by phase =====
        if (lane < 7) {
            uint64_t* bars[7] = {a0_ready, &h_half[0], &h_half[1], &fold[0], &fold[1], &p_free[0], &p_free[1]};
            const int nj = (p.Cp + 127) / 128;
            const int per_tile[7] = {1, 1 + B, 1 + B, B, B, 2 * B + (nj + 1) / 2, 2 * B + nj / 2};
            const size_t my_tiles = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
            uint64_t* bar = bars[0];
            int cnt = per_tile[0];
#pragma unroll
            for (int x = 1; x < 7; ++x)
                if (lane == x) { bar = bars[x]; cnt = per_tile[x]; }
            const uint32_t remote = mapa_u32(smem_u32(bar), 0);
            const size_t total = size_t(cnt) * my_tiles;
            for (size_t k = 0; k < total; ++k) {
                mbar_wait(bar, uint32_t(k & 1));
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
            }
        }
      } else if (warp == kMmaWarp && leader) {
        // ===== MMA issuer (warp-uniform, one lane elected per instruction) =====
        uint32_t s = 0, ph = 0;
        // barrier phase parities as bits of one register (a0_ready: bit 0, h_half: 1-2, fold: 3-4, p_free: 5-6)
        uint32_t par = 0;
        const uint64_t a_d0 = sdesc(act_s);
        const uint64_t w_d0 = sdesc(smem_u32(wst));
        const uint32_t id256 = idesc2(256), id128 = idesc2(128);
        long long* ctr = nullptr;                 // trace record of the GEMM being issued (profiling)
        auto wait_bar = [&](uint64_t* bar, int bit) {
            const long long t0 = ctr ? clock64() : 0;
            mbar_wait(bar, (par >> bit) & 1u);
            par ^= 1u << bit;
            tc_fence_after();
            if (ctr) ctr[5] += clock64() - t0;    // cycles waiting on the epilogue
        };
        int isc = 0;                              // stage counter within the GEMM (profiling)
        auto next_stage = [&]() -> uint64_t {
            const long long t0 = ctr ? clock64() : 0;
            mbar_wait(&full[s], ph);
            tc_fence_after();
            if (ctr) {
                const long long t1 = clock64();
                ctr[4] += t1 - t0;                // cycles waiting on weights
                if (isc >= 4 && isc < 8) ctr[24 + isc - 4] = t1;
                ++isc;
            }
            return w_d0 + uint64_t((s * kStage) >> 4);
        };
        auto release_stage = [&]() {
            mma_commit_2sm(&empty[s]);
            if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
        };
        // T GEMM: A = packed h in TMEM, sub-passes of N <= 128 into P0 / P1
        auto gemm_t = [&](int nout, long long* tr, bool gemm1) {
            wait_bar(&h_half[0], 1);
            const int nsp = (nout + 127) / 128;
            for (int j = 0; j < nsp; ++j) {
                const int nmma = min(128, nout - 128 * j);
                const uint32_t id = nmma == 128 ? id128 : idesc2(uint32_t(nmma));
                const uint32_t d = tmem + (j & 1 ? 320u : 64u);
                if (j >= 2) wait_bar(&p_free[j & 1], 5 + (j & 1));   // drain j - 2 freed this accumulator
                if (tr && j < 4) tr[8 + j] = clock64();
#pragma unroll 1
                for (int st = 0; st < 4; ++st) {
                    if (j == 0 && st == 2) wait_bar(&h_half[1], 2);   // K >= 256: half 1 of h
                    const uint64_t b_d = next_stage();
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int kc = (st >> 1) * 4 + (st & 1) + 2 * c;           // 64-wide K chunk
                        mma4_ts_2sm(d, tmem + hcol(4 * kc), b_d + uint64_t((c * kBox) >> 4), id, (st | c) != 0 ? 1u : 0u);
                    }
                    release_stage();
                    // GEMM1: after the last sub-pass's K < 256 steps nothing reads h half 0 any more, so
                    // the epilogue may fold h + b2 over it while the rest of the sub-pass runs
                    if (gemm1 && j == nsp - 1 && st == 1) mma_commit_2sm(h0_read);
                }
                mma_commit_2sm(&accb[j & 1]);
            }
            return nsp;
        };
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            // layer 0 (S, K = 48): A0 in act chunk 0
            long long* tr = lane == 0 ? trace_rec(t, 0) : nullptr;
            ctr = tr;
            isc = 0;
            if (tr) tr[0] = clock64();
            wait_bar(a0_ready, 0);
            for (int q = 0; q < 2; ++q) {
                const uint64_t b_d = next_stage();
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    mma_bf16_2sm(tmem + uint32_t(256 * q), a_d0 + uint64_t(2 * j), b_d + uint64_t(2 * j), id256, j);
                release_stage();
                mma_commit_2sm(&accb[q]);
            }
            for (int b = 0; b < B; ++b) {
                if (tr) tr[1] = clock64();
                tr = lane == 0 ? trace_rec(t, 2 * b + 1) : nullptr;
                ctr = tr;
                isc = 0;
            isc = 0;
                if (tr) tr[0] = clock64();
                gemm_t(N, tr, true);                                  // GEMM1: u = h.W1
                if (tr) tr[1] = clock64();
                tr = lane == 0 ? trace_rec(t, 2 * b + 2) : nullptr;
                ctr = tr;
                isc = 0;
            isc = 0;
                if (tr) tr[0] = clock64();
                // GEMM2 (S): A = u in shared memory; accumulator half q pre-set to h + b2 (fold)
                for (int q = 0; q < 2; ++q) {
                    wait_bar(&fold[q], 3 + q);
                    if (tr) tr[2 + q] = clock64();
#pragma unroll 1
                    for (int kc = 0; kc < 8; ++kc) {
                        // u chunks 4-5 come from T drain 2 (P0), 6-7 from drain 3 (P1)
                        if (q == 0 && kc == 4) wait_bar(&p_free[0], 5);
                        if (q == 0 && kc == 6) wait_bar(&p_free[1], 6);
                        const uint64_t b_d = next_stage();
                        const uint64_t a_k = a_d0 + uint64_t((kc * (kM * 128)) >> 4);
                        mma4_ss_2sm(tmem + uint32_t(256 * q), a_k, b_d, id256, 1u);
                        release_stage();
                    }
                    mma_commit_2sm(&accb[q]);
                }
                if (tr) tr[1] = clock64();
            }
            tr = lane == 0 ? trace_rec(t, L - 1) : nullptr;
            ctr = tr;
            isc = 0;
            if (tr) tr[0] = clock64();
            const int nsp = gemm_t(p.Cp, tr, false);                   // output layer
            if (tr) tr[1] = clock64();
            ctr = nullptr;
            // consume the output drains not waited for above (keeps every barrier's phase in step)
            for (int j = nsp >= 2 ? nsp - 2 : 0; j < nsp; ++j) wait_bar(&p_free[j & 1], 5 + (j & 1));
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
        // ===== epilogue: thread = packet row r; column group grp =====
        const int quad = warp & 3, grp = warp >> 2;
        const int r = quad * 32 + lane;
        const uint32_t t_row = tmem + (uint32_t(quad * 32) << 16);
        int eg = 0, eu = 0;                           // profiling: GEMM record / unit / tile
        size_t et = 0;
        uint32_t aph = 0;                             // accb[x] phase parity in bit x
        uint32_t h0ph = 0;
        // on the pair leader's barrier, once per warp: every lane has fenced its own writes, __syncwarp
        // orders them before lane 0's release-arrive
        auto arrive = [&](uint64_t* bar) {
            __syncwarp();
            if (lane != 0) return;
            if (p.trace && blockIdx.x < 2 && eu < 4 && et < 4 * size_t(gridDim.x)) {   // before the arrive
                long long* rec = p.trace + ((et / gridDim.x) * L + eg) * kTraceSlots;
                long long g;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                rec[64 + 16 * eu + 8 * int(blockIdx.x) + warp] = g;
            }
            mbar_arrive(bar);                          // the peer's warp 9 forwards (see the init)
        };
        // profiling: epilogue threads 0 / 128 stamp, in the record of GEMM eg, when each unit ends
        // (slots 16 + u / 32 + u) and when thread 0 woke for it (48 + u)
        auto estamp = [&](int slot) {
            if (p.trace && (threadIdx.x == 0 || threadIdx.x == 128)) {
                long long* rec = trace_rec(et, eg);
                if (rec) rec[slot] = clock64();
            }
        };
        // slots 64 + 16 * (unit & 3) + 8 * rank + warp: lane 0 of every epilogue warp of blocks 0 and 1
        // stamps the end of units 0-3 (per-warp / per-CTA skew at the barriers)
        auto unit_end = [&]() {
            estamp((grp ? 32 : 16) + eu);

            ++eu;
        };
        auto wait_acc = [&](int x) {
            mbar_wait(&accb[x], (aph >> x) & 1u);
            aph ^= 1u << x;
            tc_fence_after();
            if (grp == 0) estamp(48 + eu);
            if (p.trace && lane == 0 && blockIdx.x < 2 && eu < 4 && et < 4 * size_t(gridDim.x)) {
                long long* rec = p.trace + ((et / gridDim.x) * L + eg) * kTraceSlots;
                long long g;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                rec[128 + 16 * eu + 8 * int(blockIdx.x) + warp] = g;   // woke for unit eu (ns)
            }
        };
        float* mv = reinterpret_cast<float*>(act);    // top-k merge scratch (act is free during the output)
        int* mi = reinterpret_cast<int*>(act + kM * 4 * sizeof(float));
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const size_t i = t * kM + r;
            // ---- a2: A0 row = [xh | xl | xh | xl | xh | xl | 0..] (K = 48 of chunk 0, R22) ----
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
            arrive(a0_ready);

            // ---- S drain of half q: h = ReLU(D [+ b0]) packed in place into TMEM ----
            auto drain_s = [&](int q, bool add_b0, int dl) {
                wait_acc(q);
                uint32_t cur[32], nxt[32];
                const int base = 256 * q;
                // group 0: chunks 0, 32, 64, 96 upwards -> c / 2; group 1: 224 .. 128 downwards -> 192 + (c - 128) / 2
                auto chunk_col = [&](int m) { return grp == 0 ? 32 * m : 224 - 32 * m; };
                __syncwarp();
                tmem_ld32_async(t_row + uint32_t(base + chunk_col(0)), cur);
                tmem_wait_ld();
#pragma unroll 1
                for (int m = 0; m < 4; ++m) {
                    const int c = chunk_col(m);
                    if (m < 3) tmem_ld32_async(t_row + uint32_t(base + chunk_col(m + 1)), nxt);
                    uint32_t o[16];
#pragma unroll
                    for (int q8 = 0; q8 < 4; ++q8) {
                        float* f = reinterpret_cast<float*>(cur) + 8 * q8;
                        if (add_b0) {
                            const float4 ba = bias4s(sb, base + c + 8 * q8), bb = bias4s(sb, base + c + 8 * q8 + 4);
                            add2(f[0], f[1], f[0], f[1], ba.x, ba.y);
                            add2(f[2], f[3], f[2], f[3], ba.z, ba.w);
                            add2(f[4], f[5], f[4], f[5], bb.x, bb.y);
                            add2(f[6], f[7], f[6], f[7], bb.z, bb.w);
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) o[4 * q8 + u] = relu_pack_bf16(f[2 * u], f[2 * u + 1]);
                        dbg_put<kDbg>(p, dl, i, base + c + 8 * q8,
                                      make_uint4(o[4 * q8], o[4 * q8 + 1], o[4 * q8 + 2], o[4 * q8 + 3]));
                    }
                    tmem_st16u(t_row + uint32_t(base + (grp == 0 ? c / 2 : 192 + (c - 128) / 2)), o);
                    if (m < 3) {
                        tmem_wait_ld();
#pragma unroll
                        for (int j = 0; j < 32; ++j) cur[j] = nxt[j];
                    }
                }
                tmem_st_wait();
                tc_fence_before();
                arrive(&h_half[q]);
                unit_end();
            };
            // ---- fold for GEMM2 half q: accumulator [256q, 256q + 256) = h + b2 of block b ----
            auto fold_half = [&](int q, int b) {
                const int base = 256 * q;
                uint32_t hp[64];
                uint32_t (&h0)[32] = *reinterpret_cast<uint32_t(*)[32]>(hp);
                uint32_t (&h1)[32] = *reinterpret_cast<uint32_t(*)[32]>(hp + 32);
                const uint32_t src = t_row + uint32_t(base + (grp == 0 ? 0 : 192));
                __syncwarp();
                tmem_ld32_async(src, h0);
                tmem_ld32_async(src + 32u, h1);
                tmem_wait_ld();
                const int o2 = N + B * N + b * N + base + 128 * grp;   // b2 of block b, this group's columns
#pragma unroll
                for (int piece = 0; piece < 8; ++piece) {            // 16 h columns per TMEM store
                    float sv[16];
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 bv = bias4s(sb, o2 + 16 * piece + 4 * q4);
                        const uint32_t w0 = hp[8 * piece + 2 * q4], w1 = hp[8 * piece + 2 * q4 + 1];
                        add2(sv[4 * q4], sv[4 * q4 + 1], bf16_lo(w0), bf16_hi(w0), bv.x, bv.y);
                        add2(sv[4 * q4 + 2], sv[4 * q4 + 3], bf16_lo(w1), bf16_hi(w1), bv.z, bv.w);
                    }
                    tmem_st16(t_row + uint32_t(base + 128 * grp + 16 * piece), sv);
                }
                tmem_st_wait();
                tc_fence_before();
                arrive(&fold[q]);
                unit_end();
            };
            // ---- T drain of GEMM1 sub-pass j: u = ReLU(D + b1) -> shared memory (A of GEMM2) ----
            auto drain_u = [&](int j, int b, int dl) {
                wait_acc(j & 1);
                const uint32_t pc = (j & 1 ? 320u : 64u) + 64u * grp;
                const int c0 = 128 * j + 64 * grp;                  // output columns of this group
                const int o1 = N + b * N + c0;
                uint32_t v0[32], v1[32];
                __syncwarp();
                tmem_ld32_async(t_row + pc, v0);
                tmem_ld32_async(t_row + pc + 32u, v1);
                tmem_wait_ld();
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const uint32_t* v = hf ? v1 : v0;
#pragma unroll
                    for (int q8 = 0; q8 < 4; ++q8) {
                        const float4 ba = bias4s(sb, o1 + 32 * hf + 8 * q8), bb = bias4s(sb, o1 + 32 * hf + 8 * q8 + 4);
                        const float* f = reinterpret_cast<const float*>(v) + 8 * q8;
                        float z[8];
                        add2(z[0], z[1], f[0], f[1], ba.x, ba.y);
                        add2(z[2], z[3], f[2], f[3], ba.z, ba.w);
                        add2(z[4], z[5], f[4], f[5], bb.x, bb.y);
                        add2(z[6], z[7], f[6], f[7], bb.z, bb.w);
                        const uint4 o = make_uint4(relu_pack_bf16(z[0], z[1]), relu_pack_bf16(z[2], z[3]),
                                                   relu_pack_bf16(z[4], z[5]), relu_pack_bf16(z[6], z[7]));
                        sts128(act_addr(act_s, r, (c0 + 32 * hf) / 8 + q8), o);
                        dbg_put<kDbg>(p, dl, i, c0 + 32 * hf + 8 * q8, o);
                    }
                }
                fence_proxy_async();
                tc_fence_before();
                arrive(&p_free[j & 1]);
                unit_end();
            };

            // a3: layer 0 -> packed h0
            et = t; eg = 0; eu = 0;
            drain_s(0, true, 0);
            drain_s(1, true, 0);
            for (int b = 0; b < B; ++b) {
                // a4 GEMM1: four T sub-passes; the fold of half 0 needs every GEMM1 MMA done (h is its A)
                eg = 2 * b + 1; eu = 0;
                drain_u(0, b, 2 * b + 1);
                drain_u(1, b, 2 * b + 1);
                drain_u(2, b, 2 * b + 1);
                mbar_wait(h0_read, h0ph);                       // GEMM1 no longer reads h half 0
                h0ph ^= 1;
                tc_fence_after();
                fold_half(0, b);
                drain_u(3, b, 2 * b + 1);
                fold_half(1, b);
                // a4 GEMM2: h = ReLU(D) (D already holds u.W2 + b2 + h), packed into TMEM
                eg = 2 * b + 2; eu = 0;
                drain_s(0, false, 2 * b + 2);
                drain_s(1, false, 2 * b + 2);
            }
            // ---- a5: logits = D + bo over the output sub-passes; top-k (ties -> lower index) ----
            {
                const int k = int(p.k);
                float bv[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
                int bc[4] = {0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF};
                eg = 2 * B + 1; eu = 0;
                float b1v = -FLT_MAX;                   // top-1 (k = 1) stays in registers
                int b1c = 0x7FFFFFFF;
                const int ob = N + 2 * B * N;
                for (int j = 0; j < nj; ++j) {
                    wait_acc(j & 1);
                    const uint32_t pc = (j & 1 ? 320u : 64u) + 64u * grp;
                    const int c0 = 128 * j + 64 * grp;
                    const int cw = max(0, min(64, p.Cp - c0));
                    __syncwarp();
                    for (int x = 0; x < cw; x += 16) {
                        uint32_t v[16];
                        tmem_ld16_async(t_row + pc + uint32_t(x), v);
                        float bq[16];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            const float4 f4 = bias4s(sb, ob + c0 + x + 4 * q4);
                            bq[4 * q4] = f4.x; bq[4 * q4 + 1] = f4.y; bq[4 * q4 + 2] = f4.z; bq[4 * q4 + 3] = f4.w;
                        }
                        tmem_wait_ld();
                        if (k == 1 && !p.logits) {        // top-1: running max in registers
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) {
                                const float z = __uint_as_float(v[jj]) + bq[jj];
                                if (c0 + x + jj < p.C && z > b1v) { b1v = z; b1c = c0 + x + jj; }
                            }
                            continue;
                        }
                        for (int jj = 0; jj < 16; ++jj) {
                            const int c = c0 + x + jj;
                            if (c >= p.C) break;
                            const float z = __uint_as_float(v[jj]) + bq[jj];
                            if (p.logits && i < p.n) p.logits[i * p.C + c] = z;
                            if (k == 1) {
                                if (z > b1v) { b1v = z; b1c = c; }
                            } else if (z > bv[k - 1]) {   // insertion; columns ascend within a thread
                                int pos = k - 1;
                                while (pos > 0 && z > bv[pos - 1]) { bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos; }
                                bv[pos] = z;
                                bc[pos] = c;
                            }
                        }
                    }
                    tc_fence_before();
                    arrive(&p_free[j & 1]);
                    unit_end();
                }
                // merge group 1's candidates into group 0's (value desc, index asc)
                if (k == 1) {
                    if (grp == 1) { mv[r * 4] = b1v; mi[r * 4] = b1c; }
                    epi_bar(1, kEpi);
                    if (grp == 0) {
                        if (better(mv[r * 4], mi[r * 4], b1v, b1c)) { b1v = mv[r * 4]; b1c = mi[r * 4]; }
                        if (i < p.n) p.pred[i] = uint32_t(b1c);
                    }
                    epi_bar(2, kEpi);
                    continue;
                }
                if (grp == 1)
                    for (int q = 0; q < k; ++q) { mv[r * 4 + q] = bv[q]; mi[r * 4 + q] = bc[q]; }
                epi_bar(1, kEpi);
                if (grp == 0) {
                    for (int q2 = 0; q2 < k; ++q2) {
                        const float z = mv[r * 4 + q2];
                        const int c = mi[r * 4 + q2];
                        if (better(z, c, bv[k - 1], bc[k - 1])) {
                            int pos = k - 1;
                            while (pos > 0 && better(z, c, bv[pos - 1], bc[pos - 1])) {
                                bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos;
                            }
                            bv[pos] = z;
                            bc[pos] = c;
                        }
                    }
                    if (i < p.n)
                        for (int q = 0; q < k; ++q) p.pred[i * k + q] = uint32_t(bc[q]);
                }
                epi_bar(2, kEpi);                       // scratch consumed before the next tile's A0
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

TsPlan* ts_plan_create(const WeightsBF16& w, int device, int* err) {
    *err = TANG_OK;
    if (w.N != N || w.Cp > 512 || w.Cp % 16) { *err = TANG_EMODEL; return nullptr; }
    TsPlan* p = new TsPlan();
    p->w = w;
    const size_t act = 8 * size_t(kM) * 128;
    const size_t budget = 227 * 1024 - 1024 - 256;
    const size_t cbytes = size_t(N + 2 * w.B * N + w.Cp) * 4;
    if (budget < act + cbytes + 2 * kStage) { delete p; *err = TANG_EMODEL; return nullptr; }
    p->stages = int((budget - act - cbytes) / kStage);
    if (p->stages > 8) p->stages = 8;
    p->smem = 1024 + act + p->stages * kStage + 256 + cbytes;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    p->grid = (sms / 2) * 2;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    const uint64_t rows = uint64_t(2) * w.B * N + w.Cp + N;   // W1 x B, W2 x B, Wo, B0 (layer 0)
    cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(N) * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(
        &p->tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(w.W1t), dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::fprintf(stderr, "libtang: cuTensorMapEncodeTiled failed (%d)\n", int(r));
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    if (cudaFuncSetAttribute(mlp_ts_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) !=
            cudaSuccess ||
        cudaFuncSetAttribute(mlp_ts_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) !=
            cudaSuccess) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    return p;
}

void ts_plan_destroy(TsPlan* p) { delete p; }

int launch_mlp_ts(const TsPlan* pl, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                  cudaStream_t s, uint16_t* dbg, long long* trace) {
    if (!pl) return TANG_EMODEL;
    if (n == 0) return TANG_OK;
    TsParams p{};
    p.hdr = hdr; p.n = n; p.k = k; p.pred = pred; p.logits = logits;
    p.bias = pl->w.b0;
    p.B = pl->w.B; p.C = pl->w.C; p.Cp = pl->w.Cp; p.stages = pl->stages;
    p.row_l0 = 2 * pl->w.B * N + pl->w.Cp;
    p.dbg = dbg;
    p.trace = trace;
    size_t tiles = (n + kM - 1) / kM;
    tiles = (tiles + 1) & ~size_t(1);
    const int grid = int(tiles < size_t(pl->grid) ? tiles : size_t(pl->grid));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = pl->smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = dbg ? cudaLaunchKernelEx(&cfg, mlp_ts_kernel<true>, pl->tmap, p)
                        : cudaLaunchKernelEx(&cfg, mlp_ts_kernel<false>, pl->tmap, p);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::fprintf(stderr, "libtang: mlp_ts_kernel launch failed: %s (smem %zu)\n", cudaGetErrorString(e), pl->smem);
        return TANG_ECUDA;
    }
    return TANG_OK;
}

}  // namespace tang
