// Internal layouts and kernel launchers of libtang (not part of the C ABI).
//
// HBM / L2 layout:
//   TupleDev  tuples[C]     16 B  signature masks + best (priority, id) of the tuple
//   uint32    order[C]            non-empty tuples by ascending best key (fallback visit order)
//   SlotDev   slots[2^s]    16 B  open-addressing hash table keyed by (tuple, masked SIP, masked DIP)
//   RuleDev   rules[cap]    32 B  rule records, each bucket contiguous and sorted by (priority, id)
//   MetaDev   meta          64 B  scalars that updates change (order length, global best, epoch)
//   uint32    cand[2][65536][W]   candidate-tuple bitmaps by the top 16 bits of SIP and of DIP (W = C/32
//                                 rounded up to a multiple of 4): bit j of row r is set when tuple j has a key whose prefix
//                                 agrees with r -- a packet can match in tuple j only if both its rows
//                                 have bit j (a superset: deletes leave bits set)
// All tables of a 512k-rule set total ~30 MB and stay resident in the 126 MB L2.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace tang {

constexpr uint32_t kSlotEmpty = 0xFFFFFFFFu;
constexpr uint32_t kTupleBits = 11;                   // tuple index < 2048 (C <= 1089)
constexpr uint32_t kTupleMask = (1u << kTupleBits) - 1;
constexpr uint32_t kMaxBucket = (1u << (32 - kTupleBits)) - 1;
constexpr int kS = 7;                                 // input segments

struct __align__(16) TupleDev {
    uint32_t sip_mask, dip_mask;   // mask(l_sip^T), mask(l_dip^T)
    uint32_t best_prio, best_id;   // smallest (priority, id) in the tuple; 0xFFFFFFFF x2 if empty
};

struct __align__(16) SlotDev {
    uint32_t msip, mdip;           // truncated key
    uint32_t tup_cnt;              // tuple | count << kTupleBits; kSlotEmpty = never used
    uint32_t first;                // index of the bucket's first rule record
};

struct __align__(16) RuleDev {
    uint32_t sip, dip;             // canonical prefixes
    uint32_t sp, dp;               // lo | hi << 16
    uint32_t lens;                 // sip_len | dip_len << 8 | proto << 16 | proto_mask << 24
    uint32_t prio, id, action;
};

struct __align__(16) MetaDev {
    uint32_t n_order;              // entries of order[] in use
    uint32_t slot_mask;            // slots - 1
    uint32_t best_prio, best_id;   // global best key over all tuples (strict-mode gate)
    uint32_t epoch;
    uint32_t n_tuples;
    uint32_t cand_words;           // W, 32-bit words per candidate-bitmap row
    uint32_t pad[9];
};

// Delta = sequence of word writes (region, word offset, value); regions below.
enum Region : uint32_t { kRegTuples = 0, kRegOrder = 1, kRegSlots = 2, kRegRules = 3, kRegMeta = 4, kRegCand = 5,
                         kNumRegions = 6 };
struct DeltaWord { uint32_t region, word, value; };
// first word of every delta: {kDeltaHeader, layout hash of the planner's tables, words that follow}
constexpr uint32_t kDeltaHeader = 0xDE17A000u;

__host__ __device__ inline uint32_t prefix_mask(uint32_t len) {
    return len == 0 ? 0u : (0xFFFFFFFFu << (32u - len));
}

__host__ __device__ inline uint32_t slot_hash(uint32_t tuple, uint32_t msip, uint32_t mdip) {
    uint32_t h = msip * 0x9E3779B1u ^ (mdip * 0x85EBCA77u + 0x165667B1u) ^ (tuple * 0xC2B2AE3Du);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    return h;
}

// Device pointers of one ctx's tables (passed by value to kernels).
struct Tables {
    const TupleDev* tuples;
    const uint32_t* order;
    const SlotDev* slots;
    const RuleDev* rules;
    const MetaDev* meta;
    const uint32_t* cand;          // [2][65536][W]
    uint32_t C;
};

// Weights in device memory.
struct WeightsF32 {   // [in][out] fp32, as in the blob
    const float* W0; const float* b0;
    const float* W1; const float* b1;   // B x [N][N], B x [N]
    const float* W2; const float* b2;
    const float* Wo; const float* bo;   // [N][C], [C]
    int N, B, C;
};

struct WeightsBF16 {  // tensor-core operands: K-major (= [out][in]) bf16
    const float* W0; const float* b0;     // fp32 layer 0, [7][N]
    const uint16_t* W1t; const float* b1; // B x [N][N] (out-major), B x [N]
    const uint16_t* W2t; const float* b2;
    const uint16_t* Wot; const float* bo; // [Cp][N], [Cp] (padding rows zero, bias -inf)
    int N, B, C, Cp;
};

constexpr int kMaxBlocksF8 = 32;
struct WeightsF8 {    // e4m3 tensor-core operands (R23): per-tensor / per-layer power-of-two scales
    const uint8_t* Wq;    // [2BN + Cp][N] e4m3 K-major: W1t(b) rows bN.., W2t(b) rows (B+b)N.., Wot rows 2BN..
    const uint16_t* B0;   // [N][64] bf16 split layer-0 operand (R22)
    const float* b0s;     // [N]    b0 / s_h0
    const float* b1s;     // [B][N] b1 / s_u(b)
    const float* c2;      // [B][N] b2 / (s_u(b) s_w2(b))
    const float* bo;      // [Cp]   (padding -inf)
    int N, B, C, Cp;
    float inv_sh0, mo;                                   // 1 / s_h0;  s_h(B) s_wo
    float m1[kMaxBlocksF8], k2[kMaxBlocksF8], m2[kMaxBlocksF8];   // s_h s_w1 / s_u;  s_h / (s_u s_w2);  s_u s_w2 / s_h'
};

struct WeightsF4 {    // NVFP4 tensor-core operands (R24), N = 256
    WeightsF8 s;          // per-tensor / per-layer scales, epilogue constants, layer-0 operand (shared with R23)
    const uint8_t* Wq;    // [2BN + Cp][N / 2] e2m1 codes, K-major, value 2i in the low nibble of byte i
    const uint8_t* SF;    // [2B + 2 pass slots][8][512] ue4m3 block scales in tcgen05.cp block layout
    const float* consts;  // [b0/s_h0 (N) | b1/s_u (B N) | b2/s_h' (B N) | bo (Cp)] (GEMM2 folds m2 into the skip)
    float r2[kMaxBlocksF8];   // s_h / s_h' of block b
};

struct Scratch {       // per-stream classify scratch, sized for max_batch packets
    uint32_t* pred;        // [max_batch * topk]
    uint32_t* miss_idx;    // [max_batch]
    uint32_t* miss_bound;  // [max_batch * 2] (prio, id) of the in-tuple match (strict mode)
    uint32_t* miss_count;  // [1]
    unsigned long long* best_key;   // [max_batch] (priority << 32 | id) of the best in-tuple match so far
    uint4* long_ent;       // [max_batch * topk] deferred long buckets: (packet, first record, count, -)
    uint32_t* long_count;  // [1]
};
constexpr uint32_t kShortBucket = 16;   // buckets longer than this are scanned by a whole warp

// ---- launchers (kernels_search.cu) ---------------------------------------------------
void launch_encode(const void* hdr, size_t n, float* feat, cudaStream_t s);
void launch_probe(const Tables& t, const void* hdr, size_t n, const uint32_t* pred, uint32_t k,
                  uint32_t mode, uint32_t* rule_id, uint8_t* fellback, const Scratch& sc, cudaStream_t s);
void launch_fallback(const Tables& t, const void* hdr, size_t n, uint32_t* rule_id, uint8_t* fellback,
                     const Scratch& sc, cudaStream_t s);
// Order-independent 64-bit digest of the tables: sum over every word of splitmix64(region << 61 |
// word << 32 | value) mod 2^64 -- the same function on the host mirror and on the device tables,
// so ranks compare 8 bytes after each update window instead of copying the tables back.
__host__ __device__ inline uint64_t digest_word(uint32_t region, uint32_t word, uint32_t value) {
    uint64_t z = (uint64_t(region) << 61) ^ (uint64_t(word) << 32) ^ uint64_t(value);
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
void launch_table_digest(void* const* region_base, const uint32_t* region_words, unsigned long long* d_out,
                         cudaStream_t s);

// d[0] must be the header with `layout`; words beyond region_words[region] are dropped; every
// refused word is counted in *rejected (device)
void launch_apply_delta(const DeltaWord* d, size_t nwords, void* const* region_base, const uint32_t* region_words,
                        uint32_t layout, uint32_t* rejected, cudaStream_t s);

// ---- launchers (kernels_mlp_ffma.cu) ---------------------------------------------------
void launch_mlp_ffma(const WeightsF32& w, const void* hdr, size_t n, uint32_t k, uint32_t* pred,
                     float* logits, cudaStream_t s);

// ---- launchers (kernels_mlp_tc.cu) -----------------------------------------------------
struct TcPlan;   // TMA descriptors + launch geometry, built once per ctx
TcPlan* tc_plan_create(const WeightsBF16& w, const float* h_bias, int device, int two_sm, int groups, int* err);
void tc_plan_destroy(TcPlan* p);
int launch_mlp_tc(const TcPlan* p, const void* hdr, size_t n, uint32_t k, uint32_t* pred,
                  float* logits, cudaStream_t s, uint16_t* dbg = nullptr, long long* trace = nullptr);

// ---- launchers (kernels_mlp_tc2.cu): bf16 chain, two tiles in flight per CTA (N <= 256) ---------
struct Tc2Plan;
Tc2Plan* tc2_plan_create(const WeightsBF16& w, int device, int* err);
void tc2_plan_destroy(Tc2Plan* p);
int launch_mlp_tc2(const Tc2Plan* p, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                   cudaStream_t s, uint16_t* dbg = nullptr);

// ---- launchers (kernels_mlp_f8.cu): e4m3 chain, tcgen05 kind::f8f6f4 (§8(f) f2) ------------
struct F8Plan;
F8Plan* f8_plan_create(const WeightsF8& w, int device, bool allow_dual, int* err);
void f8_plan_set_scales(F8Plan* p, const WeightsF8& w);
void f8_plan_destroy(F8Plan* p);
int launch_mlp_f8(const F8Plan* p, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                  cudaStream_t s, uint8_t* dbg = nullptr, long long* trace = nullptr);
// ---- launchers (kernels_mlp_f4.cu): NVFP4 chain, tcgen05 kind::mxf4nvf4 (§8(f) f2, R24) ------
struct F4Plan;
F4Plan* f4_plan_create(const WeightsF4& w, int device, int* err);
void f4_plan_set_scales(F4Plan* p, const WeightsF4& w);
void f4_plan_destroy(F4Plan* p);
int launch_mlp_f4(const F4Plan* p, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                  cudaStream_t s, uint8_t* dbg = nullptr, long long* trace = nullptr);

}  // namespace tang
