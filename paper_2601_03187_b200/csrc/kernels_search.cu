// Stage-2 kernels of libtang for sm_100a: feature encode (a2), tuple probe (a6),
// post-verification fallback (a7), priority reduction (a8) and in-place update apply (a10).
//
// P:274 (§5.1.1): "Using the tuple's prefix signature, the engine truncates the relevant
// field value of P and computes a hash value from the truncated values ... the rules are
// compared one by one to return the action associated with the highest-priority matching rule."
// "If none exists, an ordered search is performed across the remaining tuples until
// the highest-priority rule is located."
#include "tang_internal.h"

namespace tang {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t TANG_MAX_TOPK_DEV = 4;
constexpr uint32_t kRecBatch = 1;     // bucket records whose loads are in flight together (pass 1)

struct Hdr { uint32_t sip, dip, sp, dp, proto; };

__device__ __forceinline__ Hdr load_hdr(const void* base, size_t i) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(base) + i);
    Hdr h;
    h.sip = v.x;
    h.dip = v.y;
    h.sp = v.z & 0xFFFFu;
    h.dp = v.z >> 16;
    h.proto = v.w & 0xFFu;
    return h;
}

__device__ __forceinline__ uint32_t mask_of(uint32_t len) {
    return len ? (0xFFFFFFFFu << (32u - len)) : 0u;
}

// every field condition of P:77 (§2.1): prefixes, inclusive port ranges, masked protocol
__device__ __forceinline__ bool rule_match(const uint4& a, const uint4& b, const Hdr& h) {
    const uint32_t lens = b.x;
    const uint32_t sl = lens & 0xFFu, dl = (lens >> 8) & 0xFFu;
    const uint32_t pv = (lens >> 16) & 0xFFu, pm = lens >> 24;
    return (((h.sip ^ a.x) & mask_of(sl)) == 0u) & (((h.dip ^ a.y) & mask_of(dl)) == 0u) &
           (h.sp >= (a.z & 0xFFFFu)) & (h.sp <= (a.z >> 16)) &
           (h.dp >= (a.w & 0xFFFFu)) & (h.dp <= (a.w >> 16)) &
           ((h.proto & pm) == (pv & pm));
}

__device__ __forceinline__ bool key_less(uint32_t p0, uint32_t i0, uint32_t p1, uint32_t i1) {
    return p0 < p1 || (p0 == p1 && i0 < i1);
}

// Probe tuple j for packet h; on a match better than (bp, bi), lower (bp, bi).
// Returns the number of memory accesses (1 per slot probe + 1 per rule compared).
__device__ __forceinline__ void probe_tuple(const Tables& t, uint32_t slot_mask, uint32_t j, const Hdr& h,
                                            uint32_t& bp, uint32_t& bi) {
    const uint4 tv = __ldg(reinterpret_cast<const uint4*>(t.tuples) + j);
    const uint32_t ms = h.sip & tv.x, md = h.dip & tv.y;
    uint32_t s = slot_hash(j, ms, md) & slot_mask;
    const uint4* slots = reinterpret_cast<const uint4*>(t.slots);
    while (true) {
        const uint4 sv = __ldg(slots + s);
        if (sv.z == kSlotEmpty) return;                         // key absent
        if ((sv.z & kTupleMask) == j && sv.x == ms && sv.y == md) {
            const uint32_t cnt = sv.z >> kTupleBits;
            const uint4* rp = reinterpret_cast<const uint4*>(t.rules) + 2ull * sv.w;
            for (uint32_t r = 0; r < cnt; ++r) {                 // bucket sorted by (prio, id)
                const uint4 a = __ldg(rp + 2 * r);
                const uint4 b = __ldg(rp + 2 * r + 1);
                if (!key_less(b.y, b.z, bp, bi)) return;        // nothing later can win
                if (rule_match(a, b, h)) { bp = b.y; bi = b.z; return; }
            }
            return;
        }
        s = (s + 1) & slot_mask;
    }
}

// ---- a2: encode ---------------------------------------------------------------------
// [SIP_hi, SIP_lo, DIP_hi, DIP_lo, SP, DP, PRO] / 65536.  16-byte loads, the block's
// 7 x 256 floats staged in shared memory and written back as coalesced float4 stores.
__global__ void __launch_bounds__(256) encode_kernel(const void* __restrict__ hdr, size_t n,
                                                     float* __restrict__ feat) {
    __shared__ __align__(16) float tile[256 * kS];
    const size_t base = size_t(blockIdx.x) * 256;
    const size_t i = base + threadIdx.x;
    if (i < n) {
        const Hdr h = load_hdr(hdr, i);
        const float sc = 1.0f / 65536.0f;
        float* o = tile + threadIdx.x * kS;
        o[0] = float(h.sip >> 16) * sc;
        o[1] = float(h.sip & 0xFFFFu) * sc;
        o[2] = float(h.dip >> 16) * sc;
        o[3] = float(h.dip & 0xFFFFu) * sc;
        o[4] = float(h.sp) * sc;
        o[5] = float(h.dp) * sc;
        o[6] = float(h.proto) * sc;
    }
    __syncthreads();
    const size_t cnt = (n - base < 256) ? (n - base) : 256;
    float* out = feat + base * kS;
    if (cnt == 256) {
        const float4* src = reinterpret_cast<const float4*>(tile);
        float4* dst = reinterpret_cast<float4*>(out);
        for (int q = threadIdx.x; q < 256 * kS / 4; q += 256) dst[q] = src[q];
    } else {
        for (size_t q = threadIdx.x; q < cnt * kS; q += 256) out[q] = tile[q];
    }
}

// ---- a6: probe the predicted tuple(s) ----------------------------------------------------
// Pass 1, thread per packet: mask -> hash -> linear probe of the 16-byte slots; the first
// kShortBucket records of the bucket are scanned in-thread (first full match in (priority, id)
// order, kRecBatch records' loads in flight); only the undecided tail of a longer bucket is deferred to
// pass 2, so no lane walks a thousand-record bucket alone and packets that match early in a
// heavy wildcard bucket never leave the thread.
__global__ void __launch_bounds__(256) probe_kernel(Tables t, const void* __restrict__ hdr, size_t n,
                                                    const uint32_t* __restrict__ pred, uint32_t k, Scratch sc) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t slot_mask = t.meta->slot_mask;
    uint32_t bp = 0xFFFFFFFFu, bi = 0xFFFFFFFFu;
    uint32_t nlong = 0;
    uint4 ent[TANG_MAX_TOPK_DEV];
    if (i < n) {
        const Hdr h = load_hdr(hdr, i);
        const uint4* slots = reinterpret_cast<const uint4*>(t.slots);
        for (uint32_t q = 0; q < k; ++q) {
            const uint32_t j = __ldg(pred + i * k + q);
            if (j >= t.C) continue;
            const uint4 tv = __ldg(reinterpret_cast<const uint4*>(t.tuples) + j);
            const uint32_t ms = h.sip & tv.x, md = h.dip & tv.y;
            uint32_t s = slot_hash(j, ms, md) & slot_mask;
            while (true) {
                const uint4 sv = __ldg(slots + s);
                if (sv.z == kSlotEmpty) break;
                if ((sv.z & kTupleMask) == j && sv.x == ms && sv.y == md) {
                    const uint32_t cnt = sv.z >> kTupleBits;
                    // the first kShortBucket records in-thread, kRecBatch records' loads in flight at a time
                    // (the bucket is sorted by (priority, id): stop at the first match or at the
                    // first record that cannot beat the best so far)
                    const uint32_t head = cnt < kShortBucket ? cnt : kShortBucket;
                    const uint4* rp = reinterpret_cast<const uint4*>(t.rules) + 2ull * sv.w;
                    bool done = false;
                    for (uint32_t r0 = 0; r0 < head && !done; r0 += kRecBatch) {
                        uint4 a[kRecBatch], b[kRecBatch];
#pragma unroll
                        for (uint32_t u = 0; u < kRecBatch; ++u)
                            if (r0 + u < head) { a[u] = __ldg(rp + 2 * (r0 + u)); b[u] = __ldg(rp + 2 * (r0 + u) + 1); }
#pragma unroll
                        for (uint32_t u = 0; u < kRecBatch; ++u) {
                            if (done || r0 + u >= head) break;
                            if (!key_less(b[u].y, b[u].z, bp, bi)) { done = true; break; }
                            if (rule_match(a[u], b[u], h)) { bp = b[u].y; bi = b[u].z; done = true; break; }
                        }
                    }
                    // a long bucket still undecided: its tail goes to the warp-per-bucket pass
                    if (!done && cnt > head) ent[nlong++] = make_uint4(uint32_t(i), sv.w + head, cnt - head, 0);
                    break;
                }
                s = (s + 1) & slot_mask;
            }
        }
        sc.best_key[i] = (static_cast<unsigned long long>(bp) << 32) | bi;
    }
    // warp-aggregated append of the deferred long buckets
    for (uint32_t q = 0; q < TANG_MAX_TOPK_DEV; ++q) {
        const bool has = q < nlong;
        const uint32_t m = __ballot_sync(kFull, has);
        if (!m) break;
        const int leader = __ffs(m) - 1;
        uint32_t pos0 = 0;
        if (lane == uint32_t(leader)) pos0 = atomicAdd(sc.long_count, uint32_t(__popc(m)));
        pos0 = __shfl_sync(kFull, pos0, leader);
        if (has) sc.long_ent[pos0 + __popc(m & ((1u << lane) - 1u))] = ent[q];
    }
}

// Pass 2, warp per deferred bucket: lanes test 32 consecutive records (sorted by priority) at
// once; the first matching lane of the ballot is the bucket's winner; stop at the first window
// whose head cannot beat the packet's current best.  Result merged with a 64-bit atomicMin.
__global__ void __launch_bounds__(256) probe_long_kernel(Tables t, const void* __restrict__ hdr, Scratch sc) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nlong = *sc.long_count;
    for (uint32_t w = warp; w < nlong; w += nwarps) {
        const uint4 e = sc.long_ent[w];
        const Hdr h = load_hdr(hdr, e.x);
        const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(sc.best_key + e.x);
        const uint32_t cp = uint32_t(cur >> 32), ci = uint32_t(cur);
        const uint4* rp = reinterpret_cast<const uint4*>(t.rules) + 2ull * e.y;
        for (uint32_t base = 0; base < e.z; base += 32) {
            const uint32_t r = base + lane;
            uint32_t kp = 0xFFFFFFFFu, ki = 0xFFFFFFFFu;
            bool m = false;
            if (r < e.z) {
                const uint4 a = __ldg(rp + 2 * r);
                const uint4 b = __ldg(rp + 2 * r + 1);
                kp = b.y;
                ki = b.z;
                m = key_less(kp, ki, cp, ci) && rule_match(a, b, h);
            }
            const uint32_t hp = __shfl_sync(kFull, kp, 0), hi = __shfl_sync(kFull, ki, 0);
            if (!key_less(hp, hi, cp, ci)) break;                 // sorted: nothing here can win
            const uint32_t bal = __ballot_sync(kFull, m);
            if (bal) {
                const int wl = __ffs(bal) - 1;                     // lowest record = best key
                if (lane == uint32_t(wl))
                    atomicMin(sc.best_key + e.x, (static_cast<unsigned long long>(kp) << 32) | ki);
                break;
            }
        }
    }
}

// Pass 3, thread per packet: rule id, fallback decision, compacted miss list (post-verification
// input).  Strict mode also sends packets whose match could be beaten by another tuple.
__global__ void __launch_bounds__(256) probe_finalize_kernel(Tables t, size_t n, uint32_t strict,
                                                             uint32_t* __restrict__ rule_id,
                                                             uint8_t* __restrict__ fellback, Scratch sc) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31u;
    bool miss = false;
    uint32_t bp = 0xFFFFFFFFu, bi = 0xFFFFFFFFu;
    if (i < n) {
        const unsigned long long key = sc.best_key[i];
        bp = uint32_t(key >> 32);
        bi = uint32_t(key);
        if (bi == 0xFFFFFFFFu) {
            miss = true;                                          // post-verification
        } else if (strict) {
            miss = key_less(t.meta->best_prio, t.meta->best_id, bp, bi);   // some tuple could still win
        }
        rule_id[i] = bi;
        if (fellback) fellback[i] = miss ? 1 : 0;
    }
    const uint32_t m = __ballot_sync(kFull, miss);
    if (m) {
        const int leader = __ffs(m) - 1;
        uint32_t pos0 = 0;
        if (lane == uint32_t(leader)) pos0 = atomicAdd(sc.miss_count, uint32_t(__popc(m)));
        pos0 = __shfl_sync(kFull, pos0, leader);
        if (miss) {
            const uint32_t pos = pos0 + __popc(m & ((1u << lane) - 1u));
            sc.miss_idx[pos] = uint32_t(i);
            sc.miss_bound[2 * pos] = bp;
            sc.miss_bound[2 * pos + 1] = bi;
        }
    }
}

// ---- a7 + a8: post-verification search, one thread per missed packet -------------------
// The result is the minimum (priority, id) match over the remaining tuples (its visit order
// only affects cost, reading R13).  Instead of walking all C tuples in precedence order, each
// thread reads its packet's two candidate-tuple rows (kRegCand: tuple j can hold a match only if
// bit j is set for both the packet's top 16 SIP bits and its top 16 DIP bits -- ~6.5 of 300 tuples
// on the 512k ACL trace) and probes only those candidates whose best key can still win.  With a
// handful of candidates per packet, a thread per packet keeps ~64 K probe chains in flight where a
// warp per packet (round 1) left most lanes idle.
__global__ void __launch_bounds__(256) fallback_kernel(Tables t, const void* __restrict__ hdr,
                                                       uint32_t* __restrict__ rule_id, Scratch sc) {
    const uint32_t n_miss = *sc.miss_count;
    const uint32_t slot_mask = t.meta->slot_mask;
    const uint32_t W4 = t.meta->cand_words / 4;             // row length in uint4 (padded to 4 words)
    const uint4* tuples = reinterpret_cast<const uint4*>(t.tuples);
    const uint4* cand = reinterpret_cast<const uint4*>(t.cand);
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < n_miss; w += gridDim.x * blockDim.x) {
        const uint32_t i = sc.miss_idx[w];
        const Hdr h = load_hdr(hdr, i);
        const uint4* cs = cand + size_t(h.sip >> 16) * W4;
        const uint4* cd = cand + (size_t(65536) + (h.dip >> 16)) * W4;
        uint32_t bp = sc.miss_bound[2 * w], bi = sc.miss_bound[2 * w + 1];
        for (uint32_t q = 0; q < W4; ++q) {
            const uint4 a = __ldg(cs + q), b = __ldg(cd + q);
            const uint32_t m[4] = {a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint32_t bits = m[u];
                while (bits) {
                    const uint32_t j = 32 * (4 * q + u) + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const uint4 tv = __ldg(tuples + j);
                    if (key_less(tv.z, tv.w, bp, bi)) probe_tuple(t, slot_mask, j, h, bp, bi);
                }
            }
        }
        rule_id[i] = bi;
    }
}

struct RegionBases { void* p[kNumRegions]; uint32_t words[kNumRegions]; };

// a10: the planner's word writes, in place.  d[0] is the header; a delta planned for
// another table layout (different rule_capacity) writes nothing.
__global__ void apply_delta_kernel(const DeltaWord* __restrict__ d, size_t nwords, RegionBases rb, uint32_t layout,
                                   uint32_t* rejected) {
    const DeltaWord h = d[0];
    const bool ok = h.region == kDeltaHeader && h.word == layout && size_t(h.value) + 1 == nwords;
    uint32_t bad = 0;
    for (size_t w = size_t(blockIdx.x) * blockDim.x + threadIdx.x + 1; w < nwords; w += size_t(gridDim.x) * blockDim.x) {
        const DeltaWord x = d[w];
        if (ok && x.region < kNumRegions && x.word < rb.words[x.region])
            reinterpret_cast<uint32_t*>(rb.p[x.region])[x.word] = x.value;
        else
            ++bad;
    }
    if (bad) atomicAdd(rejected, bad);
}

// table digest (digest_word summed over every word of every region), one atomic per warp
__global__ void table_digest_kernel(RegionBases rb, unsigned long long* out) {
    unsigned long long acc = 0;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (uint32_t r = 0; r < kNumRegions; ++r) {
        const uint32_t* p = static_cast<const uint32_t*>(rb.p[r]);
        for (size_t w = size_t(blockIdx.x) * blockDim.x + threadIdx.x; w < rb.words[r]; w += stride)
            acc += digest_word(r, uint32_t(w), __ldg(p + w));
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

}  // namespace

void launch_table_digest(void* const* region_base, const uint32_t* region_words, unsigned long long* d_out,
                         cudaStream_t s) {
    RegionBases rb;
    for (int r = 0; r < kNumRegions; ++r) { rb.p[r] = region_base[r]; rb.words[r] = region_words[r]; }
    cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), s);
    table_digest_kernel<<<148 * 4, 256, 0, s>>>(rb, d_out);
}

void launch_encode(const void* hdr, size_t n, float* feat, cudaStream_t s) {
    if (n == 0) return;
    encode_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(hdr, n, feat);
}

void launch_probe(const Tables& t, const void* hdr, size_t n, const uint32_t* pred, uint32_t k, uint32_t mode,
                  uint32_t* rule_id, uint8_t* fellback, const Scratch& sc, cudaStream_t s) {
    cudaMemsetAsync(sc.miss_count, 0, 2 * sizeof(uint32_t), s);          // miss_count, long_count
    if (n == 0) return;
    const unsigned blocks = unsigned((n + 255) / 256);
    probe_kernel<<<blocks, 256, 0, s>>>(t, hdr, n, pred, k, sc);
    // enough warps for the deferred buckets without a host round trip on their count
    const size_t warps = n * k < 148 * 64 ? n * k : 148 * 64;
    if (warps) probe_long_kernel<<<unsigned((warps * 32 + 255) / 256), 256, 0, s>>>(t, hdr, sc);
    probe_finalize_kernel<<<blocks, 256, 0, s>>>(t, n, mode, rule_id, fellback, sc);
}

void launch_fallback(const Tables& t, const void* hdr, size_t n, uint32_t* rule_id, uint8_t* /*fellback*/,
                     const Scratch& sc, cudaStream_t s) {
    if (n == 0) return;
    // enough warps for the worst case without a host round trip on the miss count;
    // a thread per missed packet (the miss count stays on the device): 148 SMs x 8 blocks x 256
    size_t threads = n < 148 * 2048 ? n : 148 * 2048;
    unsigned blocks = unsigned((threads + 255) / 256);
    fallback_kernel<<<blocks, 256, 0, s>>>(t, hdr, rule_id, sc);
}

void launch_apply_delta(const DeltaWord* d, size_t nwords, void* const* region_base, const uint32_t* region_words,
                        uint32_t layout, uint32_t* rejected, cudaStream_t s) {
    if (nwords == 0) return;
    RegionBases rb;
    for (int r = 0; r < kNumRegions; ++r) { rb.p[r] = region_base[r]; rb.words[r] = region_words[r]; }
    unsigned blocks = unsigned((nwords + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    apply_delta_kernel<<<blocks, 256, 0, s>>>(d, nwords, rb, layout, rejected);
}

}  // namespace tang
