// N2 v3: TaNG's residual MLP on a 2-CTA cluster that splits every layer's output columns.
//
// Same computation and quantisation points as kernels_mlp_tc.cu (§6.1, Eq. 1-2
// P:377-381; SURVEY.md §8(c) reading 5).  Why a pair: at N = 512 one layer's
// fp32 accumulator (128 x 512) fills all of TMEM, so on one SM the epilogue of layer g and the
// MMAs of layer g+1 cannot overlap.  Here the two CTAs of a cluster (two SMs) share a 128-packet
// tile and CTA x computes output columns [x N/2, (x+1) N/2) of every layer:
//   * each CTA keeps the FULL [128 x N] bf16 activation tile (the A operand) in shared memory,
//     in the UMMA K-major SWIZZLE_128B layout, K chunks of 64 columns = 16 KB each;
//   * TMEM holds two 256-column fp32 accumulators: MMA(g+1) writes one while the epilogue of g
//     drains the other;
//   * the epilogue writes its half of A(g+1) into its own shared memory, chunk by chunk, and the
//     MMA thread forwards every finished 16 KB chunk to the peer with one cp.async.bulk
//     shared::cta -> shared::cluster copy that completes on the peer's chunk mbarrier;
//   * MMA(g+1) consumes K chunks in arrival order (own chunks first), so it starts while the
//     epilogue of g is still producing the rest: MMA and epilogue overlap across layers;
//   * the residual skip is folded into the accumulator (h + b2 is tcgen05.st'd into the GEMM2
//     accumulator before GEMM2 starts), as in v2;
//   * a CTA writes into its peer's A tile only after both CTAs' MMAs of the previous layer are
//     done (tcgen05.commit multicast to a 2-arrival mbarrier in each CTA).
// Weights: CTA x streams only its output rows of each K-major weight matrix (TMA, 3-stage ring).
// Warp roles per CTA: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer + chunk forwarder,
// warps 2..9 epilogue (thread = packet row; 2 column groups per TMEM lane quadrant).
#include <cuda.h>

#include <cfloat>

#include "../../include/tang.h"
#include "tang_internal.h"
#include "tc_ptx.h"

namespace tang {

namespace {

using namespace tc;

constexpr int kGroups = 2;
constexpr int kEpiThreads = 128 * kGroups;
// warps 0..7 epilogue (warpgroups 0-1), warp 8 TMA producer, warp 9 MMA issuer + chunk forwarder,
// warps 10-11 idle; the control warpgroup hands registers to the epilogue with setmaxnreg
constexpr int kThreads = kEpiThreads + 128;
constexpr int kProdWarp = kEpiThreads / 32, kMmaWarp = kProdWarp + 1;
constexpr uint32_t kEpiRegs = 216, kCtlRegs = 72;
constexpr uint32_t kDCols = 256;                  // columns of one TMEM accumulator buffer
constexpr int kMaxKC = 8;                          // K chunks at N = 512

struct PairParams {
    const void* hdr;
    size_t n;
    uint32_t k;
    uint32_t* pred;
    float* logits;
    const float* W0; const float* b0;
    const float* b1; const float* b2;
    const float* bo;
    int N, B, C, Cp;
    int osplit;          // output columns [0, osplit) on CTA 0, [osplit, Cp) on CTA 1
    int stages;
    uint16_t* dbg;
    long long* trace;    // optional phase timestamps of cluster 0: [cta][tile<4][layer][8]
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ bool mbar_try_cluster(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    return ok != 0;
}
// wait with cluster-scope acquire (data written by the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
    const uint32_t a = smem_u32(b);
    uint32_t spins = 0;
    while (!mbar_try_cluster(a, parity)) {
        if (++spins == (1u << 26)) {
            printf("libtang: mlp_pair_kernel cluster mbarrier timeout (block %d thread %d)\n", blockIdx.x, threadIdx.x);
            __trap();
        }
    }
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                                  uint32_t bar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst_cluster), "r"(src_cta), "r"(bytes), "r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(bar)), "h"(uint16_t(3)) : "memory");
}

__device__ __forceinline__ void dbg_put2(const PairParams& p, int l, size_t i, int col, uint4 v) {
    if (p.dbg && i < p.n) *reinterpret_cast<uint4*>(p.dbg + (size_t(l) * p.n + i) * p.N + col) = v;
}

// K-chunk visiting order of CTA x: its own chunks first, then the peer's; within a CTA's half
// the two epilogue column groups finish their first chunk together, so interleave the groups
// (N = 512: x4+0, x4+2, x4+1, x4+3)
__device__ __forceinline__ int chunk_at(int q, int KC, uint32_t x) {
    const int half = KC / 2;
    const uint32_t owner = q < half ? x : (x ^ 1u);
    const int r = q < half ? q : q - half;
    return int(owner) * half + (r & 1) * (half / 2) + (r >> 1);
}

// top-k insertion, strict > keeps the lower index on ties (candidates arrive in index order)
__device__ __forceinline__ void topk_insert(float (&bv)[4], int (&bc)[4], int k, float z, int c) {
    if (z > bv[k - 1]) {
        int pos = k - 1;
        while (pos > 0 && z > bv[pos - 1]) { bv[pos] = bv[pos - 1]; bc[pos] = bc[pos - 1]; --pos; }
        bv[pos] = z;
        bc[pos] = c;
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
mlp_pair_kernel(const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_o,
                PairParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t x = cluster_rank();                    // which output half this CTA computes
    const uint32_t peer = x ^ 1u;
    const int N = p.N, S = p.stages;
    const int KC = N / 64, HALF = KC / 2;                 // K chunks; chunks owned per CTA
    const int NH = N / 2;                                 // own hidden columns
    const uint32_t stage_bytes = 256 * 128;               // largest box (output layer)
    uint8_t* act = smem;                                  // KC x 16 KB
    const uint32_t act_s = smem_u32(act);
    uint8_t* wst = smem + KC * (kM * 128);                // S x 32 KB
    uint64_t* full = reinterpret_cast<uint64_t*>(wst + S * stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* chunk = empty + S;                          // [KC] A-chunk ready (own: 128 thread arrivals; peer: bulk tx)
    uint64_t* acc_full = chunk + kMaxKC;                  // local MMA of the layer done -> local epilogue
    uint64_t* pair_done = acc_full + 1;                   // both CTAs' MMAs of the layer done (2 arrivals)
    uint64_t* init_done = pair_done + 1;                  // GEMM2 accumulator init written (256 arrivals)
    uint64_t* xmerge = init_done + 1;                     // CTA 1's top-k candidates landed in CTA 0 (128 arrivals)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xmerge + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = 2 * p.B + 1;
    const size_t ntiles = (p.n + kM - 1) / kM;
    const size_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    // output-layer columns of this CTA
    const int oc_lo = x == 0 ? 0 : p.osplit, oc_hi = x == 0 ? p.osplit : p.Cp;
    const int own_out = oc_hi - oc_lo;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int c = 0; c < KC; ++c) mbar_init(&chunk[c], (c / HALF) == int(x) ? 128 : 1);
        mbar_init(acc_full, 1);
        mbar_init(pair_done, 2);
        mbar_init(init_done, kEpiThreads);
        mbar_init(xmerge, 128);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_h)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_o)) : "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(tmem_slot)), "r"(2 * kDCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();                                         // peer barriers initialised before any remote op
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kProdWarp) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs));
      if (warp == kProdWarp) {
        // ===== TMA producer: this CTA's output rows of every weight matrix, in MMA chunk order =====
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            for (size_t t = cl; t < ntiles; t += ncl) {
                for (int g = 0; g < L; ++g) {
                    const bool is_out = g == L - 1;
                    const int row0 = is_out ? 2 * p.B * N + oc_lo
                                            : ((g & 1) ? (p.B + g / 2) * N : (g / 2) * N) + int(x) * NH;
                    const uint32_t bytes = uint32_t(is_out ? 256 : NH) * 128;
                    for (int q = 0; q < KC; ++q) {
                        const int kc = chunk_at(q, KC, x);
                        mbar_wait(&empty[s], ph ^ 1);
                        mbar_expect_tx(&full[s], bytes);
                        tma_load_2d(wst + s * stage_bytes, is_out ? &tmap_o : &tmap_h, &full[s], kc * 64, row0);
                        if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                    }
                }
            }
        }
      } else if (warp == kMmaWarp) {
        // ===== MMA issuer + chunk forwarder (one thread) =====
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            uint32_t cph = 0;          // chunk barriers flip once per layer
            uint32_t iph = 0;          // init_done phase
            const uint32_t a_base = smem_u32(act), w_base = smem_u32(wst);
            const uint32_t act_peer = mapa(a_base, peer);
            const uint32_t chunk_peer = mapa(smem_u32(chunk), peer);
            uint32_t G = 0;            // global layer counter -> TMEM buffer G & 1
            bool first = true;
            for (size_t t = cl; t < ntiles; t += ncl) {
                for (int g = 0; g < L; ++g, ++G) {
                    const bool is_out = g == L - 1;
                    const bool skip_init = !is_out && (g & 1);
                    const int nmma = is_out ? own_out : NH;
                    const uint32_t id = idesc(uint32_t(nmma));
                    const uint32_t d_tmem = tmem + (G & 1u) * kDCols;
                    // arm the peer-owned chunks of this layer's A (filled by the peer's bulk copies)
                    for (int q = HALF; q < KC; ++q) mbar_expect_tx(&chunk[chunk_at(q, KC, x)], kM * 128);
                    // we may overwrite the peer's copy of our chunks only after both CTAs' MMAs of
                    // the previous layer (global index G - 1) are done
                    long long* tr = (p.trace && cl == 0 && t < 4) ? p.trace + ((x * 4 + t) * L + g) * 8 : nullptr;
                    long long w_own = 0, w_peer = 0, w_full = 0, t0 = 0;
                    if (tr) tr[0] = clock64();
                    if (!first) mbar_wait_cluster(pair_done, (G - 1) & 1u);
                    first = false;
                    if (skip_init) { mbar_wait(init_done, iph); iph ^= 1; }
                    if (tr) tr[1] = clock64();
                    for (int q = 0; q < KC; ++q) {
                        const int kc = chunk_at(q, KC, x);
                        if (tr) t0 = clock64();
                        if (q < HALF) {
                            mbar_wait(&chunk[kc], cph);                 // our epilogue wrote it
                            if (tr) w_own += clock64() - t0;
                            bulk_copy_to_peer(act_peer + kc * (kM * 128), a_base + kc * (kM * 128), kM * 128,
                                              chunk_peer + kc * 8);
                        } else {
                            mbar_wait_cluster(&chunk[kc], cph);         // the peer's copy landed
                            if (tr) w_peer += clock64() - t0;
                        }
                        if (tr) t0 = clock64();
                        mbar_wait(&full[s], ph);
                        if (tr) w_full += clock64() - t0;
                        tc_fence_after();
                        const uint32_t b_stage = w_base + s * stage_bytes;
                        if (nmma > 0) {          // CTA 1 owns no output column when Cp == 16
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const uint64_t a = sdesc(a_base + kc * (kM * 128) + j * 32);
                                const uint64_t b = sdesc(b_stage + j * 32);
                                mma_bf16(d_tmem, a, b, id, (skip_init || q > 0 || j > 0) ? 1u : 0u);
                            }
                        }
                        mma_commit(&empty[s]);
                        if (++s == uint32_t(S)) { s = 0; ph ^= 1; }
                    }
                    cph ^= 1;
                    mma_commit(acc_full);
                    mma_commit_pair(pair_done);
                    if (tr) { tr[2] = clock64(); tr[3] = w_own; tr[4] = w_peer; tr[5] = w_full; }
                }
            }
            // drain: the last layer's pair_done, so no copy into a finished peer is pending
            if (!first) mbar_wait_cluster(pair_done, (G - 1) & 1u);
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
        // ===== epilogue =====
        const int quad = warp & 3;
        const int grp = warp >> 2;
        const int r = quad * 32 + lane;
        const uint32_t lane_off = uint32_t(quad * 32) << 16;
        // own hidden columns of this group: [hc0, hc1) in global column index
        const int hc0 = int(x) * NH + grp * (NH / kGroups), hc1 = hc0 + NH / kGroups;
        // output columns of this group
        const int osub = oc_lo + (((own_out / 2) + 15) / 16) * 16;
        const int og0 = grp == 0 ? oc_lo : min(osub, oc_hi), og1 = grp == 0 ? min(osub, oc_hi) : oc_hi;
        // merge scratch inside an A chunk owned by this CTA (only our epilogue writes it)
        float* mv = reinterpret_cast<float*>(act + (int(x) * HALF) * (kM * 128));
        int* mi = reinterpret_cast<int*>(act + (int(x) * HALF) * (kM * 128) + 2048);
        // cross-CTA candidates live in CTA 0's chunk 0 (a CTA-0-owned chunk: only CTA 0's
        // epilogue writes it, never a bulk copy); CTA 1 addresses it through mapa
        float* xv = reinterpret_cast<float*>(act + 8192);
        int* xi = reinterpret_cast<int*>(act + 10240);
        const uint32_t xv_peer = mapa(smem_u32(xv), peer), xi_peer = mapa(smem_u32(xi), peer);
        const uint32_t xmerge_peer = mapa(smem_u32(xmerge), peer);
        uint32_t fph = 0, xph = 0;
        uint32_t G = 0;

        // signal "chunk kc of the next A is written" after this warp's rows of it are stored
        auto chunk_done = [&](int kc) {
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&chunk[kc]);        // 128 arrivals: the 4 warps of this column group
        };

        for (size_t t = cl; t < ntiles; t += ncl) {
            const size_t i = t * kM + r;
            // a2 + a3: features and layer 0 (fp32 FFMA) for our columns
            for (int s7 = 0; s7 < 7; ++s7) prefetch_l1(p.W0 + s7 * N + hc0, hc1 - hc0, lane);
            prefetch_l1(p.b0 + hc0, hc1 - hc0, lane);
            uint4 hv = make_uint4(0, 0, 0, 0);
            if (i < p.n) hv = __ldg(reinterpret_cast<const uint4*>(p.hdr) + i);
            const float sc = 1.0f / 65536.0f;
            float xf[7];
            xf[0] = float(hv.x >> 16) * sc;
            xf[1] = float(hv.x & 0xFFFFu) * sc;
            xf[2] = float(hv.y >> 16) * sc;
            xf[3] = float(hv.y & 0xFFFFu) * sc;
            xf[4] = float(hv.z & 0xFFFFu) * sc;
            xf[5] = float(hv.z >> 16) * sc;
            xf[6] = float(hv.w & 0xFFu) * sc;
            for (int q = hc0 / 8; q < hc1 / 8; ++q) {
                const float4 ba = __ldg(reinterpret_cast<const float4*>(p.b0 + q * 8));
                const float4 bb = __ldg(reinterpret_cast<const float4*>(p.b0 + q * 8 + 4));
                float h[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                for (int s7 = 0; s7 < 7; ++s7) {
                    const float4 w0 = __ldg(reinterpret_cast<const float4*>(p.W0 + s7 * N + q * 8));
                    const float4 w1 = __ldg(reinterpret_cast<const float4*>(p.W0 + s7 * N + q * 8 + 4));
                    h[0] = fmaf(xf[s7], w0.x, h[0]); h[1] = fmaf(xf[s7], w0.y, h[1]);
                    h[2] = fmaf(xf[s7], w0.z, h[2]); h[3] = fmaf(xf[s7], w0.w, h[3]);
                    h[4] = fmaf(xf[s7], w1.x, h[4]); h[5] = fmaf(xf[s7], w1.y, h[5]);
                    h[6] = fmaf(xf[s7], w1.z, h[6]); h[7] = fmaf(xf[s7], w1.w, h[7]);
                }
                uint4 o;
                o.x = relu_pack_bf16(h[0], h[1]);
                o.y = relu_pack_bf16(h[2], h[3]);
                o.z = relu_pack_bf16(h[4], h[5]);
                o.w = relu_pack_bf16(h[6], h[7]);
                sts128(act_addr(act_s, r, q), o);
                dbg_put2(p, 0, i, q * 8, o);
                if ((q & 7) == 7) chunk_done(q >> 3);
            }

            for (int g = 0; g < L; ++g, ++G) {
                if (g == L - 1) prefetch_l1(p.bo + og0, og1 - og0, lane);
                else if ((g & 1) == 0) {
                    prefetch_l1(p.b1 + (g / 2) * N + hc0, hc1 - hc0, lane);
                    prefetch_l1(p.b2 + (g / 2) * N + hc0, hc1 - hc0, lane);
                }
                mbar_wait(acc_full, fph);
                fph ^= 1;
                tc_fence_after();
                long long* etr = (p.trace && cl == 0 && t < 4 && threadIdx.x == 0) ? p.trace + ((x * 4 + t) * L + g) * 8 : nullptr;
                if (etr) etr[6] = clock64();
                const uint32_t t_cur = tmem + lane_off + (G & 1u) * kDCols;        // this layer's accumulator
                const uint32_t t_nxt = tmem + lane_off + ((G + 1) & 1u) * kDCols;  // next layer's accumulator
                if (g == L - 1) {
                    // a5: logits + top-k over our output columns (top-1 stays in registers)
                    float bv[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
                    int bc[4] = {0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF};
                    const int k = int(p.k);
                    const bool fast = k == 1 && p.logits == nullptr;
                    float b0v = -FLT_MAX;
                    int b0c = 0x7FFFFFFF;
                    __syncwarp();
                    for (int c0 = og0; c0 < og1; c0 += 16) {
                        uint32_t v[16];
                        tmem_ld16_async(t_cur + uint32_t(c0 - oc_lo), v);
                        float bq[16];
                        ld_f16x(p.bo + c0, bq);
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
                            topk_insert(bv, bc, k, z, c);
                        }
                    }
                    if (fast) { bv[0] = b0v; bc[0] = b0c; }
                    tc_fence_before();
                    // merge the two column groups of this CTA
                    if (grp == 1) for (int q = 0; q < k; ++q) { mv[r * 4 + q] = bv[q]; mi[r * 4 + q] = bc[q]; }
                    epi_bar(1, kEpiThreads);
                    if (grp == 0) {
                        for (int q = 0; q < k; ++q) topk_insert(bv, bc, k, mv[r * 4 + q], mi[r * 4 + q]);
                        if (x == 1) {
                            // hand our candidates to CTA 0 once its MMAs of this layer are done
                            mbar_wait_cluster(pair_done, G & 1u);   // parity of this (output) layer
                            for (int q = 0; q < k; ++q) {
                                asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(xv_peer + uint32_t(r * 4 + q) * 4),
                                             "f"(bv[q]) : "memory");
                                asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(xi_peer + uint32_t(r * 4 + q) * 4),
                                             "r"(uint32_t(bc[q])) : "memory");
                            }
                            mbar_arrive_remote(xmerge_peer);
                        } else {
                            mbar_wait_cluster(xmerge, xph);
                            for (int q = 0; q < k; ++q) topk_insert(bv, bc, k, xv[r * 4 + q], xi[r * 4 + q]);
                            if (i < p.n)
                                for (int q = 0; q < k; ++q) p.pred[i * k + q] = uint32_t(bc[q]);
                        }
                    }
                    xph ^= 1;
                    epi_bar(2, kEpiThreads);     // scratch consumed before the next tile's layer 0
                    if (etr) etr[7] = clock64();
                } else {
                    const bool gemm1 = (g & 1) == 0;
                    const int b = g / 2;
                    const float* bias = gemm1 ? p.b1 + b * N : nullptr;
                    if (gemm1) {
                        // fold the skip: next accumulator <- h + b2 on our columns, before GEMM2 runs
                        // (its MMAs wait for this pass, so it goes first and touches no TMEM reads)
                        const float* b2 = p.b2 + b * N;
                        __syncwarp();
                        for (int c0 = hc0; c0 < hc1; c0 += 32) {
                            uint4 hh[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) hh[q] = lds128(act_addr(act_s, r, c0 / 8 + q));
                            float sv[32];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float4 ba = __ldg(reinterpret_cast<const float4*>(b2 + c0 + 8 * q));
                                const float4 bb = __ldg(reinterpret_cast<const float4*>(b2 + c0 + 8 * q + 4));
                                sv[8 * q + 0] = bf16_lo(hh[q].x) + ba.x; sv[8 * q + 1] = bf16_hi(hh[q].x) + ba.y;
                                sv[8 * q + 2] = bf16_lo(hh[q].y) + ba.z; sv[8 * q + 3] = bf16_hi(hh[q].y) + ba.w;
                                sv[8 * q + 4] = bf16_lo(hh[q].z) + bb.x; sv[8 * q + 5] = bf16_hi(hh[q].z) + bb.y;
                                sv[8 * q + 6] = bf16_lo(hh[q].w) + bb.z; sv[8 * q + 7] = bf16_hi(hh[q].w) + bb.w;
                            }
                            tmem_st32(t_nxt + uint32_t(c0 - int(x) * NH), sv);
                        }
                        tmem_st_wait();
                        tc_fence_before();
                        mbar_arrive(init_done);
                    }
                    // drain this layer's accumulator into our half of the next A, 32 columns at a time
                    // (next chunk's accumulator and biases in flight), signalling each finished 64-col chunk
                    uint32_t cur[32], nxt[32];
                    __syncwarp();
                    tmem_ld32_async(t_cur + uint32_t(hc0 - int(x) * NH), cur);
                    tmem_wait_ld();
                    for (int c0 = hc0; c0 < hc1; c0 += 32) {
                        if (c0 + 32 < hc1) tmem_ld32_async(t_cur + uint32_t(c0 + 32 - int(x) * NH), nxt);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float* f = reinterpret_cast<const float*>(cur) + 8 * q;
                            float4 ba = make_float4(0.f, 0.f, 0.f, 0.f), bb = ba;
                            if (gemm1) {
                                ba = __ldg(reinterpret_cast<const float4*>(bias + c0 + 8 * q));
                                bb = __ldg(reinterpret_cast<const float4*>(bias + c0 + 8 * q + 4));
                            }
                            const uint4 o = make_uint4(relu_pack_bf16(f[0] + ba.x, f[1] + ba.y),
                                                       relu_pack_bf16(f[2] + ba.z, f[3] + ba.w),
                                                       relu_pack_bf16(f[4] + bb.x, f[5] + bb.y),
                                                       relu_pack_bf16(f[6] + bb.z, f[7] + bb.w));
                            sts128(act_addr(act_s, r, c0 / 8 + q), o);
                            dbg_put2(p, g + 1, i, c0 + 8 * q, o);
                        }
                        tmem_wait_ld();
#pragma unroll
                        for (int j = 0; j < 32; ++j) cur[j] = nxt[j];
                        if (((c0 + 32) & 63) == 0) chunk_done((c0 + 32) / 64 - 1);
                    }
                    if (etr) etr[7] = clock64();
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();                     // no CTA leaves while its peer may still touch its smem
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kDCols));
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

struct PairPlan {
    CUtensorMap tmap_h, tmap_o;
    WeightsBF16 w;
    int stages;
    size_t smem;
    int grid;
    int osplit;
};

PairPlan* pair_plan_create(const WeightsBF16& w, int device, int* err) {
    *err = TANG_OK;
    if (!(w.N == 256 || w.N == 512) || w.Cp > 512) { *err = TANG_EMODEL; return nullptr; }
    PairPlan* p = new PairPlan();
    p->w = w;
    const int KC = w.N / 64;
    const size_t act = size_t(KC) * kM * 128;
    const size_t stage = 256 * 128;
    const size_t budget = 227 * 1024 - 1024 - 512;
    p->stages = int((budget - act) / stage);
    if (p->stages > 6) p->stages = 6;
    if (p->stages < 2) { delete p; *err = TANG_EMODEL; return nullptr; }
    p->smem = 1024 + act + p->stages * stage + 512;
    // output columns: CTA 0 takes the first half (multiple of 16), CTA 1 the rest (<= 256 each)
    p->osplit = ((w.Cp / 2 + 15) / 16) * 16;
    if (p->osplit > 256 || w.Cp - p->osplit > 256) { delete p; *err = TANG_EMODEL; return nullptr; }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    p->grid = (sms / 2) * 2;

    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    const uint64_t rows = uint64_t(2) * w.B * w.N + w.Cp;
    cuuint64_t dims[2] = {cuuint64_t(w.N), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(w.N) * 2};
    cuuint32_t estr[2] = {1, 1};
    cuuint32_t box_h[2] = {64, cuuint32_t(w.N / 2)};
    cuuint32_t box_o[2] = {64, 256};
    auto enc = reinterpret_cast<EncodeTiledFn>(fn);
    CUresult r1 = enc(&p->tmap_h, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(w.W1t), dims, strides,
                      box_h, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(&p->tmap_o, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(w.W1t), dims, strides,
                      box_o, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) {
        std::fprintf(stderr, "libtang: cuTensorMapEncodeTiled failed (%d, %d)\n", int(r1), int(r2));
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    if (cudaFuncSetAttribute(mlp_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) != cudaSuccess) {
        delete p; *err = TANG_ECUDA; return nullptr;
    }
    return p;
}

void pair_plan_destroy(PairPlan* p) { delete p; }

int launch_mlp_pair(const PairPlan* pl, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                    cudaStream_t s, uint16_t* dbg, long long* trace) {
    if (!pl) return TANG_EMODEL;
    if (n == 0) return TANG_OK;
    PairParams p;
    p.hdr = hdr; p.n = n; p.k = k; p.pred = pred; p.logits = logits;
    p.W0 = pl->w.W0; p.b0 = pl->w.b0; p.b1 = pl->w.b1; p.b2 = pl->w.b2; p.bo = pl->w.bo;
    p.N = pl->w.N; p.B = pl->w.B; p.C = pl->w.C; p.Cp = pl->w.Cp;
    p.osplit = pl->osplit; p.stages = pl->stages; p.dbg = dbg; p.trace = trace;
    const size_t tiles = (n + kM - 1) / kM;
    size_t grid = 2 * tiles;
    if (grid > size_t(pl->grid)) grid = size_t(pl->grid);
    mlp_pair_kernel<<<unsigned(grid), kThreads, pl->smem, s>>>(pl->tmap_h, pl->tmap_o, p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::fprintf(stderr, "libtang: mlp_pair_kernel launch failed: %s\n", cudaGetErrorString(e));
        return TANG_ECUDA;
    }
    return TANG_OK;
}

}  // namespace tang
