// libtang host runtime: the C ABI of include/tang.h.
//
//  * model blob parsing (class j = tuple j, signatures carried in the blob)
//  * TSS table builder: tuples fixed by the blob, rules placed by exact signature or by the
//    restricted choice of P:330 (§5.2.1), buckets keyed by truncated (SIP, DIP)
//    laid out as an open-addressing slot table + contiguous sorted rule records
//  * immediate-update planner that edits a host mirror of the device tables and
//    emits the word-level delta the device applies in place (and that ranks broadcast)
//  * classify drivers: device-pointer async path and the pinned-ring streaming path that
//    overlaps H2D, kernels and D2H over several CUDA streams (Fig. 6)
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tang.h"
#include "tang_internal.h"

using namespace tang;

namespace {

struct KeyHash {
    size_t operator()(const std::tuple<uint32_t, uint32_t, uint32_t>& k) const {
        return slot_hash(std::get<0>(k), std::get<1>(k), std::get<2>(k));
    }
};

inline uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < n; ++i) { h ^= b[i]; h *= 1099511628211ull; }
    return h;
}

uint32_t next_pow2(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return uint32_t(p);
}

inline uint16_t f32_to_bf16_rne(float f) {
    uint32_t b;
    std::memcpy(&b, &f, 4);
    b += 0x7FFFu + ((b >> 16) & 1u);
    return uint16_t(b >> 16);
}

// e4m3 (OCP fn: bias 7, max 448, subnormals m * 2^-9) code of v, round to nearest even, saturating
uint8_t to_e4m3_code(double v) {
    const uint8_t sign = std::signbit(v) ? 0x80u : 0u;
    const double a = std::fabs(v);
    if (!(a > 0)) return sign;
    int ex;
    std::frexp(a, &ex);
    const int e = std::max(ex - 1, -6);
    const double sp = std::ldexp(1.0, e - 3);
    double q = std::nearbyint(a / sp) * sp;          // a / sp exact; nearbyint: ties to even
    if (q > 448.0) q = 448.0;
    if (q == 0) return sign;
    std::frexp(q, &ex);
    const int eq = ex - 1;
    if (eq < -6) return uint8_t(sign | uint8_t(q / std::ldexp(1.0, -9)));        // subnormal
    return uint8_t(sign | uint8_t(((eq + 7) << 3) | int((q / std::ldexp(1.0, eq) - 1.0) * 8.0)));
}
// value of an e4m3 code (sign bit ignored: used for the unsigned block scales of R24)
double e4m3_value(uint8_t c) {
    const int e = (c >> 3) & 15, m = c & 7;
    return e == 0 ? std::ldexp(m / 8.0, -6) : std::ldexp(1.0 + m / 8.0, e - 7);
}
// e2m1 code (s.ee.m: 0, 0.5, 1, 1.5, 2, 3, 4, 6 = magnitude codes 0..7) of v, round to nearest
// even code, saturating at 6 (R24)
uint8_t to_e2m1_code(double v) {
    static const double mag[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
    const uint8_t sign = std::signbit(v) ? 0x8u : 0u;
    const double a = std::fabs(v);
    int best = 0;
    for (int i = 1; i < 8; ++i) {
        const double d = std::fabs(a - mag[i]), db = std::fabs(a - mag[best]);
        if (d < db || (d == db && (i & 1) == 0)) best = i;
    }
    return best ? uint8_t(sign | best) : 0u;
}
// smallest e with amax <= 448 * 2^e (exact comparisons), 0 for amax <= 0 (R23)
int pow2_exp(double amax) {
    if (!(amax > 0)) return 0;
    int ex;
    std::frexp(amax, &ex);
    int e = ex - 9;
    for (int i = 0; i < 3; ++i) {
        if (amax > std::ldexp(448.0, e)) ++e;
        if (amax <= std::ldexp(448.0, e - 1)) --e;
    }
    return e;
}

struct ProfEntry { const char* name; cudaEvent_t a, b; };

}  // namespace

struct tang_ctx {
    tang_config cfg{};
    bool host_only = false, follower = false;
    // model
    uint32_t S = 0, N = 0, B = 0, C = 0, Cp = 0;
    std::vector<std::pair<uint8_t, uint8_t>> sigs;
    std::vector<float> wblob;      // fp32 weights in blob order
    std::vector<int32_t> act_exp;  // fp8 activation-scale exponents (blob trailer), empty if absent
    // host mirror of the device tables
    std::vector<TupleDev> tuples;
    std::vector<uint32_t> order;
    std::vector<SlotDev> slots;
    std::vector<RuleDev> rules;
    MetaDev meta{};
    std::vector<uint32_t> cand;    // [2][65536][W] candidate-tuple bitmaps (kRegCand)
    // planner indexes
    struct Loc { uint32_t slot, prio; };
    std::unordered_map<uint32_t, Loc> where;
    std::vector<uint32_t> slot_cap;
    std::vector<std::set<std::pair<uint32_t, uint32_t>>> tuple_keys;
    std::map<std::pair<uint32_t, uint32_t>, uint32_t> exact;
    uint32_t pool_top = 0, keys = 0, mismatch = 0;
    uint32_t live_keys = 0;                        // slots whose bucket holds >= 1 rule (keys - tombstones)
    std::multimap<uint32_t, uint32_t> free_recs;   // released record blocks: capacity -> first record
    std::vector<uint32_t> touched[kNumRegions];
    std::vector<DeltaWord> delta;
    // device
    int device = -1;
    void* d_tab[kNumRegions] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    size_t tab_bytes[kNumRegions] = {0, 0, 0, 0, 0, 0};
    uint32_t* d_rejected = nullptr;          // delta words the device refused (tang_stats)
    uint32_t host_rejected = 0;
    float* d_wf32 = nullptr;
    void* d_wbf = nullptr;
    WeightsF32 wf{};
    WeightsBF16 wb{};
    std::vector<float> h_bias;      // [b0 | b1 x B | b2 x B | bo (Cp, pad -inf)] host copy
    TcPlan* tc = nullptr;
    Tc2Plan* tc2 = nullptr;  // bf16, N <= 256, AUTO: two tiles in flight per CTA
    void* d_wf8 = nullptr;
    WeightsF8 w8{};
    F8Plan* f8 = nullptr;
    void* d_wf4 = nullptr;
    WeightsF4 w4{};
    F4Plan* f4 = nullptr;
    std::vector<cudaStream_t> streams;
    std::vector<Scratch> scratch;            // [streams] internal + [1] for *_async callers
    std::vector<void*> scratch_mem;
    DeltaWord* d_delta = nullptr;
    size_t d_delta_cap = 0;
    DeltaWord* h_delta_pinned = nullptr;
    size_t h_delta_cap = 0;
    // streaming rings
    std::vector<uint8_t*> ring_hdr;          // pinned [ring][batch*16]
    std::vector<uint32_t*> ring_out;         // pinned [ring][batch]
    std::vector<cudaEvent_t> ring_done;
    std::vector<void*> dev_hdr;              // [streams]
    std::vector<uint32_t*> dev_out;
    std::vector<std::array<cudaEvent_t, 4>> lat_ev;   // per ring chunk: H2D start, H2D end, compute end, D2H end
    std::vector<float> last_lat;
    std::vector<float> last_timeline;        // [chunk][4] ms since chunk 0's H2D start
    // profiling
    bool prof = false;
    std::vector<ProfEntry> prof_pending;
    std::vector<cudaEvent_t> ev_pool;
    std::map<std::string, std::pair<double, uint64_t>> prof_acc;
    uint64_t device_bytes = 0;

    Tables tables() const {
        Tables t;
        t.tuples = static_cast<const TupleDev*>(d_tab[kRegTuples]);
        t.order = static_cast<const uint32_t*>(d_tab[kRegOrder]);
        t.slots = static_cast<const SlotDev*>(d_tab[kRegSlots]);
        t.rules = static_cast<const RuleDev*>(d_tab[kRegRules]);
        t.meta = static_cast<const MetaDev*>(d_tab[kRegMeta]);
        t.cand = static_cast<const uint32_t*>(d_tab[kRegCand]);
        t.C = C;
        return t;
    }
    void* region_host(uint32_t r) {
        switch (r) {
            case kRegTuples: return tuples.data();
            case kRegOrder: return order.data();
            case kRegSlots: return slots.data();
            case kRegRules: return rules.data();
            case kRegCand: return cand.data();
            default: return &meta;
        }
    }
    size_t region_bytes(uint32_t r) const {
        switch (r) {
            case kRegTuples: return tuples.size() * sizeof(TupleDev);
            case kRegOrder: return order.size() * sizeof(uint32_t);
            case kRegSlots: return slots.size() * sizeof(SlotDev);
            case kRegRules: return rules.size() * sizeof(RuleDev);
            case kRegCand: return cand.size() * sizeof(uint32_t);
            default: return sizeof(MetaDev);
        }
    }
    cudaEvent_t ev() {
        if (!ev_pool.empty()) { cudaEvent_t e = ev_pool.back(); ev_pool.pop_back(); return e; }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};

#define CK(x)                                                                             \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) {                                                          \
            std::fprintf(stderr, "libtang: %s failed: %s (%s:%d)\n", #x, cudaGetErrorString(e_), \
                         __FILE__, __LINE__);                                             \
            return TANG_ECUDA;                                                            \
        }                                                                                 \
    } while (0)

namespace {

// ---------------------------------------------------------------------------------------
// rule records
// ---------------------------------------------------------------------------------------
RuleDev to_dev(const tang_rule& r) {
    RuleDev d;
    d.sip = r.sip & prefix_mask(r.sip_len);
    d.dip = r.dip & prefix_mask(r.dip_len);
    d.sp = uint32_t(r.sp_lo) | (uint32_t(r.sp_hi) << 16);
    d.dp = uint32_t(r.dp_lo) | (uint32_t(r.dp_hi) << 16);
    d.lens = uint32_t(r.sip_len) | (uint32_t(r.dip_len) << 8) | (uint32_t(r.proto) << 16) |
             (uint32_t(r.proto_mask) << 24);
    d.prio = r.priority;
    d.id = r.id;
    d.action = r.action;
    return d;
}

int check_rule(const tang_rule& r) {
    if (r.sip_len > 32 || r.dip_len > 32 || r.sp_lo > r.sp_hi || r.dp_lo > r.dp_hi || r.id == TANG_NO_MATCH)
        return TANG_EINVAL;
    return TANG_OK;
}

inline bool key_less(uint32_t p0, uint32_t i0, uint32_t p1, uint32_t i1) {
    return p0 < p1 || (p0 == p1 && i0 < i1);
}

// ---------------------------------------------------------------------------------------
// model blob (include/tang.h)
// ---------------------------------------------------------------------------------------
int parse_blob(tang_ctx* c, const void* blob, size_t len) {
    const uint8_t* p = static_cast<const uint8_t*>(blob);
    if (!blob || len < 24) return TANG_EMODEL;
    uint32_t hdr[6];
    std::memcpy(hdr, p, 24);
    if (hdr[0] != TANG_BLOB_MAGIC || hdr[1] != TANG_BLOB_VERSION) return TANG_EMODEL;
    c->S = hdr[2]; c->N = hdr[3]; c->B = hdr[4]; c->C = hdr[5];
    if (c->S != uint32_t(kS) || c->N < 64 || c->N > 512 || c->N % 64 || c->B > 64 || c->C < 1 || c->C > 1089)
        return TANG_EMODEL;
    size_t off = 24;
    const size_t sig_bytes = (size_t(c->C) * 2 + 3) & ~size_t(3);
    if (len < off + sig_bytes) return TANG_EMODEL;
    c->sigs.resize(c->C);
    for (uint32_t j = 0; j < c->C; ++j) {
        c->sigs[j] = {p[off + 2 * j], p[off + 2 * j + 1]};
        if (c->sigs[j].first > 32 || c->sigs[j].second > 32) return TANG_EMODEL;
    }
    off += sig_bytes;
    const size_t S = c->S, N = c->N, B = c->B, C = c->C;
    const size_t nw = S * N + N + B * (2 * N * N + 2 * N) + N * C + C;
    const size_t ntr = 8 + 4 * (2 * B + 1);
    if (len != off + nw * 4 && len != off + nw * 4 + ntr) return TANG_EMODEL;
    c->act_exp.clear();
    if (len == off + nw * 4 + ntr) {                   // fp8 activation-scale trailer
        uint32_t th[2];
        std::memcpy(th, p + off + nw * 4, 8);
        if (th[0] != TANG_BLOB_F8_MAGIC || th[1] != 2 * B + 1) return TANG_EMODEL;
        c->act_exp.resize(2 * B + 1);
        std::memcpy(c->act_exp.data(), p + off + nw * 4 + 8, 4 * (2 * B + 1));
        for (int32_t e : c->act_exp)
            if (e < -100 || e > 100) return TANG_EMODEL;
    }
    c->wblob.resize(nw);
    std::memcpy(c->wblob.data(), p + off, nw * 4);
    for (float v : c->wblob)
        if (!(v == v) || v > 3.0e38f || v < -3.0e38f) return TANG_EMODEL;   // finite weights only
    c->Cp = (c->C + 15) / 16 * 16;
    return TANG_OK;
}

// ---------------------------------------------------------------------------------------
// table builder + planner
// ---------------------------------------------------------------------------------------
void touch(tang_ctx* c, uint32_t region, size_t byte_off, size_t nbytes) {
    for (size_t w = byte_off / 4; w < (byte_off + nbytes + 3) / 4; ++w) c->touched[region].push_back(uint32_t(w));
}
void touch_rule(tang_ctx* c, uint32_t idx) { touch(c, kRegRules, size_t(idx) * sizeof(RuleDev), sizeof(RuleDev)); }
void touch_slot(tang_ctx* c, uint32_t s) { touch(c, kRegSlots, size_t(s) * sizeof(SlotDev), sizeof(SlotDev)); }

int choose_tuple(const tang_ctx* c, uint32_t ls, uint32_t ld, uint32_t* out) {
    auto it = c->exact.find({ls, ld});
    if (it != c->exact.end()) { *out = it->second; return TANG_OK; }
    int best = -1, best_sum = -1;
    for (uint32_t j = 0; j < c->C; ++j) {
        const uint32_t a = c->sigs[j].first, b = c->sigs[j].second;
        if (a <= ls && b <= ld && int(a + b) > best_sum) { best = int(j); best_sum = int(a + b); }
    }
    if (best < 0) return TANG_ENOTUPLE;
    *out = uint32_t(best);
    return TANG_OK;
}

// find the slot of key (j, ms, md); returns index, or the first empty slot on its probe path
uint32_t find_slot(const tang_ctx* c, uint32_t j, uint32_t ms, uint32_t md, bool* found) {
    const uint32_t mask = c->meta.slot_mask;
    uint32_t s = slot_hash(j, ms, md) & mask;
    while (true) {
        const SlotDev& sv = c->slots[s];
        if (sv.tup_cnt == kSlotEmpty) { *found = false; return s; }
        if ((sv.tup_cnt & kTupleMask) == j && sv.msip == ms && sv.mdip == md) { *found = true; return s; }
        s = (s + 1) & mask;
    }
}

// as find_slot, also reporting the first tombstone (a key whose bucket is empty) on the probe path
uint32_t find_slot_tomb(const tang_ctx* c, uint32_t j, uint32_t ms, uint32_t md, bool* found, uint32_t* tomb) {
    const uint32_t mask = c->meta.slot_mask;
    uint32_t s = slot_hash(j, ms, md) & mask;
    *tomb = kSlotEmpty;
    while (true) {
        const SlotDev& sv = c->slots[s];
        if (sv.tup_cnt == kSlotEmpty) { *found = false; return s; }
        if ((sv.tup_cnt & kTupleMask) == j && sv.msip == ms && sv.mdip == md) { *found = true; return s; }
        if (*tomb == kSlotEmpty && (sv.tup_cnt >> kTupleBits) == 0) *tomb = s;
        s = (s + 1) & mask;
    }
}

// Candidate-tuple bitmaps (kRegCand): set tuple j's bit in every row whose top 16 bits agree with the
// key's prefix (one row for prefixes >= 16 bits, a range of 2^(16 - len) rows otherwise).
void cand_add_field(tang_ctx* c, uint32_t j, int f, uint32_t key, bool track) {
    const uint32_t W = c->meta.cand_words, word = j >> 5, bit = 1u << (j & 31);
    const uint32_t len = f ? c->sigs[j].second : c->sigs[j].first;
    const uint32_t lo = key >> 16, hi = len >= 16 ? lo : ((key | ~prefix_mask(len)) >> 16);
    uint32_t* base = c->cand.data() + size_t(f) * 65536 * W;
    for (uint32_t r = lo; r <= hi; ++r) {
        uint32_t& w = base[size_t(r) * W + word];
        if (!(w & bit)) {
            w |= bit;
            if (track) touch(c, kRegCand, (size_t(f) * 65536 * W + size_t(r) * W + word) * 4, 4);
        }
    }
}

void cand_add_key(tang_ctx* c, uint32_t j, uint32_t ms, uint32_t md, bool track) {
    cand_add_field(c, j, 0, ms, track);
    cand_add_field(c, j, 1, md, track);
}

void refresh_tuple(tang_ctx* c, uint32_t j, bool* order_dirty) {
    TupleDev& t = c->tuples[j];
    uint32_t bp = 0xFFFFFFFFu, bi = 0xFFFFFFFFu;
    if (!c->tuple_keys[j].empty()) { bp = c->tuple_keys[j].begin()->first; bi = c->tuple_keys[j].begin()->second; }
    if (t.best_prio != bp || t.best_id != bi) {
        t.best_prio = bp;
        t.best_id = bi;
        touch(c, kRegTuples, size_t(j) * sizeof(TupleDev), sizeof(TupleDev));
        *order_dirty = true;
    }
}

void rebuild_order(tang_ctx* c) {
    std::vector<uint32_t> ne;
    for (uint32_t j = 0; j < c->C; ++j)
        if (!c->tuple_keys[j].empty()) ne.push_back(j);
    std::sort(ne.begin(), ne.end(), [&](uint32_t a, uint32_t b) {
        const TupleDev &x = c->tuples[a], &y = c->tuples[b];
        return key_less(x.best_prio, x.best_id, y.best_prio, y.best_id);
    });
    std::fill(c->order.begin(), c->order.end(), 0u);
    std::copy(ne.begin(), ne.end(), c->order.begin());
    c->meta.n_order = uint32_t(ne.size());
    if (!ne.empty()) {
        c->meta.best_prio = c->tuples[ne[0]].best_prio;
        c->meta.best_id = c->tuples[ne[0]].best_id;
    } else {
        c->meta.best_prio = c->meta.best_id = 0xFFFFFFFFu;
    }
    touch(c, kRegOrder, 0, c->order.size() * 4);
    touch(c, kRegMeta, 0, sizeof(MetaDev));
}

// Record storage for in-place updates: a bump pointer over the slack the build reserved, plus reuse of
// blocks released by relocated or emptied buckets (best fit, at most 2x the request; any size once the
// bump region is exhausted).  Deltas are applied between batches, so a block released and reused
// inside one update window is never read half-written.
void release_records(tang_ctx* c, uint32_t first, uint32_t cap) {
    if (cap) c->free_recs.emplace(cap, first);
}

int alloc_records(tang_ctx* c, uint32_t n, uint32_t* first, uint32_t* got) {
    auto it = c->free_recs.lower_bound(n);
    if (it != c->free_recs.end() && it->first <= 2 * n) {
        *first = it->second; *got = it->first;
        c->free_recs.erase(it);
        return TANG_OK;
    }
    if (uint64_t(c->pool_top) + n <= c->rules.size()) {
        *first = c->pool_top; *got = n;
        c->pool_top += n;
        return TANG_OK;
    }
    if (it != c->free_recs.end()) {
        *first = it->second; *got = it->first;
        c->free_recs.erase(it);
        return TANG_OK;
    }
    return TANG_ENOMEM;
}

// Last resort when no block fits: pack every live bucket again (capacity cnt + cnt/4 + 1, as the
// build does), drop the free lists, and touch only the words that changed.  The build reserved
// that much for its rules plus twice the headroom, so the live rules always fit.
void compact_records(tang_ctx* c) {
    std::vector<RuleDev> nr(c->rules.size(), RuleDev{});
    uint32_t top = 0;
    for (uint32_t s = 0; s < c->slots.size(); ++s) {
        SlotDev& sv = c->slots[s];
        if (sv.tup_cnt == kSlotEmpty) continue;
        const uint32_t cnt = sv.tup_cnt >> kTupleBits;
        const uint32_t old_first = sv.first;
        if (cnt == 0) {
            c->slot_cap[s] = 0;
            sv.first = 0;
        } else {
            uint32_t cap = cnt + cnt / 4 + 1;
            if (uint64_t(top) + cap > nr.size()) cap = cnt;              // (cannot overflow: see above)
            for (uint32_t q = 0; q < cnt; ++q) nr[top + q] = c->rules[sv.first + q];
            sv.first = top;
            c->slot_cap[s] = cap;
            top += cap;
        }
        if (sv.first != old_first) touch_slot(c, s);
    }
    for (uint32_t i = 0; i < nr.size(); ++i)
        if (std::memcmp(&nr[i], &c->rules[i], sizeof(RuleDev)) != 0) touch_rule(c, i);
    c->rules.swap(nr);
    c->pool_top = top;
    c->free_recs.clear();
}

int alloc_records_or_compact(tang_ctx* c, uint32_t n, uint32_t* first, uint32_t* got) {
    if (alloc_records(c, n, first, got) == TANG_OK) return TANG_OK;
    compact_records(c);
    return alloc_records(c, n, first, got);
}

// Rehash the slot table from the live keys only (drops tombstones: keys whose bucket emptied).
void rehash_slots(tang_ctx* c) {
    std::vector<SlotDev> old = c->slots;
    std::vector<uint32_t> old_cap = c->slot_cap;
    std::fill(c->slots.begin(), c->slots.end(), SlotDev{0, 0, kSlotEmpty, 0});
    std::fill(c->slot_cap.begin(), c->slot_cap.end(), 0u);
    c->keys = 0;
    for (uint32_t s = 0; s < old.size(); ++s) {
        const SlotDev& o = old[s];
        if (o.tup_cnt == kSlotEmpty) continue;
        const uint32_t cnt = o.tup_cnt >> kTupleBits;
        if (cnt == 0) { release_records(c, o.first, old_cap[s]); continue; }
        bool found;
        const uint32_t t = find_slot(c, o.tup_cnt & kTupleMask, o.msip, o.mdip, &found);
        c->slots[t] = o;
        c->slot_cap[t] = old_cap[s];
        c->keys++;
        for (uint32_t q = 0; q < cnt; ++q) c->where[c->rules[o.first + q].id].slot = t;
    }
    for (uint32_t s = 0; s < old.size(); ++s)
        if (std::memcmp(&old[s], &c->slots[s], sizeof(SlotDev)) != 0) touch_slot(c, s);
    c->live_keys = c->keys;
}

int plan_insert(tang_ctx* c, const tang_rule& r, int32_t* status, bool counting, bool* order_dirty) {
    int e = check_rule(r);
    if (e) return e;
    if (c->where.count(r.id)) return TANG_EINVAL;
    uint32_t j;
    e = choose_tuple(c, r.sip_len, r.dip_len, &j);
    if (e) return e;
    const RuleDev rd = to_dev(r);
    const uint32_t ms = rd.sip & c->tuples[j].sip_mask, md = rd.dip & c->tuples[j].dip_mask;
    bool found;
    uint32_t tomb;
    uint32_t s = find_slot_tomb(c, j, ms, md, &found, &tomb);
    if (!found && tomb == kSlotEmpty && uint64_t(c->keys + 1) * 4 > uint64_t(c->slots.size()) * 3) {
        if (c->live_keys == c->keys) return TANG_ENOMEM;          // load <= 0.75 of live keys
        rehash_slots(c);                                          // reclaim the tombstones
        s = find_slot_tomb(c, j, ms, md, &found, &tomb);
    }
    if (!found) {
        if (tomb != kSlotEmpty) {                      // reuse an emptied key's slot on the probe path
            s = tomb;
            release_records(c, c->slots[s].first, c->slot_cap[s]);
            c->slot_cap[s] = 0;
        } else {
            c->keys++;
        }
        c->slots[s] = SlotDev{ms, md, j, 0};
        touch_slot(c, s);
    }
    SlotDev& sv = c->slots[s];
    uint32_t cnt = sv.tup_cnt >> kTupleBits;
    if (cnt + 1 > kMaxBucket) return TANG_ENOMEM;
    if (cnt == c->slot_cap[s]) {                       // (re)allocate the bucket with doubled capacity
        uint32_t first, got;
        if ((e = alloc_records_or_compact(c, std::max(4u, 2 * c->slot_cap[s]), &first, &got))) return e;
        SlotDev& sv2 = c->slots[s];                    // compaction may have moved the bucket
        for (uint32_t q = 0; q < cnt; ++q) {
            c->rules[first + q] = c->rules[sv2.first + q];
            touch_rule(c, first + q);
        }
        release_records(c, sv2.first, c->slot_cap[s]);
        sv2.first = first;
        c->slot_cap[s] = got;
        touch_slot(c, s);
    }
    if (cnt == 0) {
        c->live_keys++;
        cand_add_key(c, j, ms, md, true);               // the tuple may now match these packets
    }
    // position by (priority, id), shift the tail up by one
    uint32_t pos = 0;
    while (pos < cnt && key_less(c->rules[sv.first + pos].prio, c->rules[sv.first + pos].id, rd.prio, rd.id)) ++pos;
    for (uint32_t q = cnt; q > pos; --q) {
        c->rules[sv.first + q] = c->rules[sv.first + q - 1];
        touch_rule(c, sv.first + q);
    }
    c->rules[sv.first + pos] = rd;
    touch_rule(c, sv.first + pos);
    sv.tup_cnt = j | ((cnt + 1) << kTupleBits);
    touch_slot(c, s);
    c->where[r.id] = {s, r.priority};
    c->tuple_keys[j].insert({r.priority, r.id});
    if (counting && (c->sigs[j].first != r.sip_len || c->sigs[j].second != r.dip_len)) c->mismatch++;
    refresh_tuple(c, j, order_dirty);
    if (status) *status = int32_t(j);
    return TANG_OK;
}

int plan_delete(tang_ctx* c, uint32_t id, bool* order_dirty) {
    auto it = c->where.find(id);
    if (it == c->where.end()) return TANG_ENOENT;
    const uint32_t s = it->second.slot, prio = it->second.prio;
    SlotDev& sv = c->slots[s];
    const uint32_t j = sv.tup_cnt & kTupleMask;
    const uint32_t cnt = sv.tup_cnt >> kTupleBits;
    uint32_t pos = 0;
    while (pos < cnt && c->rules[sv.first + pos].id != id) ++pos;
    if (pos == cnt) return TANG_ENOENT;
    for (uint32_t q = pos; q + 1 < cnt; ++q) {
        c->rules[sv.first + q] = c->rules[sv.first + q + 1];
        touch_rule(c, sv.first + q);
    }
    c->rules[sv.first + cnt - 1] = RuleDev{};
    touch_rule(c, sv.first + cnt - 1);
    sv.tup_cnt = j | ((cnt - 1) << kTupleBits);    // tuples are never removed
    if (cnt == 1) {                                // the bucket emptied: its key becomes a tombstone
        release_records(c, sv.first, c->slot_cap[s]);
        c->slot_cap[s] = 0;
        sv.first = 0;
        c->live_keys--;
    }
    touch_slot(c, s);
    c->where.erase(it);
    c->tuple_keys[j].erase({prio, id});
    refresh_tuple(c, j, order_dirty);
    return TANG_OK;
}

// hash of the table layout (region sizes): a delta only applies to tables of the same shape
uint32_t layout_hash(const tang_ctx* c) {
    uint64_t h = 1469598103934665603ull;
    for (uint32_t r = 0; r < kNumRegions; ++r) {
        const uint64_t b = c->region_bytes(r);
        h = fnv1a(h, &b, sizeof(b));
    }
    return uint32_t(h ^ (h >> 32));
}

void emit_delta(tang_ctx* c) {
    c->delta.clear();
    c->delta.push_back(DeltaWord{kDeltaHeader, layout_hash(c), 0});
    for (uint32_t r = 0; r < kNumRegions; ++r) {
        auto& v = c->touched[r];
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        const uint32_t* base = static_cast<const uint32_t*>(c->region_host(r));
        for (uint32_t w : v) c->delta.push_back(DeltaWord{r, w, base[w]});
        v.clear();
    }
    c->delta[0].value = uint32_t(c->delta.size() - 1);
}

int build_tables(tang_ctx* c, const tang_rule* rules, size_t n) {
    c->tuples.assign(c->C, TupleDev{0, 0, 0xFFFFFFFFu, 0xFFFFFFFFu});
    c->order.assign(c->C, 0u);
    c->tuple_keys.assign(c->C, {});
    for (uint32_t j = 0; j < c->C; ++j) {
        c->tuples[j].sip_mask = prefix_mask(c->sigs[j].first);
        c->tuples[j].dip_mask = prefix_mask(c->sigs[j].second);
        if (!c->exact.emplace(std::make_pair(uint32_t(c->sigs[j].first), uint32_t(c->sigs[j].second)), j).second)
            return TANG_EMODEL;                           // duplicate signature in the blob
    }
    // place every rule (exact signature, else restricted choice: P:330)
    std::unordered_map<std::tuple<uint32_t, uint32_t, uint32_t>, std::vector<uint32_t>, KeyHash> buckets;
    std::vector<RuleDev> rd(n);
    std::unordered_map<uint32_t, uint32_t> ids;
    ids.reserve(n * 2);
    for (size_t i = 0; i < n; ++i) {
        int e = check_rule(rules[i]);
        if (e) return e;
        if (!ids.emplace(rules[i].id, uint32_t(i)).second) return TANG_EINVAL;
        uint32_t j;
        if ((e = choose_tuple(c, rules[i].sip_len, rules[i].dip_len, &j))) return e;
        rd[i] = to_dev(rules[i]);
        buckets[{j, rd[i].sip & c->tuples[j].sip_mask, rd[i].dip & c->tuples[j].dip_mask}].push_back(uint32_t(i));
    }
    const uint64_t headroom = c->cfg.rule_capacity;
    c->slots.assign(next_pow2(std::max<uint64_t>(1024, 2 * (buckets.size() + headroom))),
                    SlotDev{0, 0, kSlotEmpty, 0});
    c->slot_cap.assign(c->slots.size(), 0);
    c->meta = MetaDev{};
    c->meta.slot_mask = uint32_t(c->slots.size() - 1);
    c->meta.n_tuples = c->C;
    uint64_t pool = 0;
    for (auto& kv : buckets) {
        const uint64_t cnt = kv.second.size();
        if (cnt > kMaxBucket) return TANG_ENOMEM;
        pool += cnt + cnt / 4 + 1;
    }
    pool += 2 * headroom + 64;
    if (pool > 0x7FFFFFFFull) return TANG_ENOMEM;
    c->rules.assign(pool, RuleDev{});
    c->pool_top = 0;
    // deterministic layout: buckets in key order
    std::vector<std::tuple<uint32_t, uint32_t, uint32_t>> order_keys;
    order_keys.reserve(buckets.size());
    for (auto& kv : buckets) order_keys.push_back(kv.first);
    std::sort(order_keys.begin(), order_keys.end());
    for (auto& k : order_keys) {
        auto& lst = buckets[k];
        std::sort(lst.begin(), lst.end(), [&](uint32_t a, uint32_t b) {
            return key_less(rd[a].prio, rd[a].id, rd[b].prio, rd[b].id);
        });
        const uint32_t j = std::get<0>(k), ms = std::get<1>(k), md = std::get<2>(k);
        const uint32_t cnt = uint32_t(lst.size()), cap = cnt + cnt / 4 + 1;
        uint32_t first, got;
        alloc_records(c, cap, &first, &got);
        for (uint32_t q = 0; q < cnt; ++q) {
            c->rules[first + q] = rd[lst[q]];
            c->where[rd[lst[q]].id] = {0, rd[lst[q]].prio};
            c->tuple_keys[j].insert({rd[lst[q]].prio, rd[lst[q]].id});
        }
        bool found;
        const uint32_t s = find_slot(c, j, ms, md, &found);
        c->slots[s] = SlotDev{ms, md, j | (cnt << kTupleBits), first};
        c->slot_cap[s] = cap;
        for (uint32_t q = 0; q < cnt; ++q) c->where[rd[lst[q]].id].slot = s;
        c->keys++;
        c->live_keys++;
    }
    // candidate-tuple bitmaps; tuples with short prefixes set long row ranges, so each distinct
    // (tuple, masked prefix) is expanded once per field
    c->meta.cand_words = ((c->C + 31) / 32 + 3) / 4 * 4;   // rows padded to whole uint4s
    c->cand.assign(size_t(2) * 65536 * c->meta.cand_words, 0u);
    {
        std::vector<std::set<std::pair<uint32_t, uint32_t>>> seen(2);
        for (uint32_t s = 0; s < c->slots.size(); ++s) {
            const SlotDev& sv = c->slots[s];
            if (sv.tup_cnt == kSlotEmpty || !(sv.tup_cnt >> kTupleBits)) continue;
            const uint32_t j = sv.tup_cnt & kTupleMask;
            if (c->sigs[j].first >= 16 || seen[0].insert({j, sv.msip}).second) cand_add_field(c, j, 0, sv.msip, false);
            if (c->sigs[j].second >= 16 || seen[1].insert({j, sv.mdip}).second) cand_add_field(c, j, 1, sv.mdip, false);
        }
    }
    bool dirty = false;
    for (uint32_t j = 0; j < c->C; ++j) refresh_tuple(c, j, &dirty);
    rebuild_order(c);
    for (auto& v : c->touched) v.clear();
    return TANG_OK;
}

uint64_t mirror_checksum(tang_ctx* c) {
    uint64_t h = 1469598103934665603ull;
    for (uint32_t r = 0; r < kNumRegions; ++r) h = fnv1a(h, c->region_host(r), c->region_bytes(r));
    return h;
}

// ---------------------------------------------------------------------------------------
// device side
// ---------------------------------------------------------------------------------------
// (Re)write both weight formats into the ctx's device buffers (allocated on first use).
int upload_weights(tang_ctx* c) {
    // fp32 weights ([in][out], blob order)
    const size_t S = c->S, N = c->N, B = c->B, C = c->C, Cp = c->Cp;
    const bool first = c->d_wf32 == nullptr;
    if (first) {
        CK(cudaMalloc(&c->d_wf32, c->wblob.size() * 4));
        c->device_bytes += c->wblob.size() * 4;
    }
    const float* base = c->d_wf32;
    c->wf.W0 = base; base += S * N;
    c->wf.b0 = base; base += N;
    // blocks are interleaved in the blob: W1, b1, W2, b2 per block -> keep per-block pointers
    // by re-packing into [B][N][N] arrays below for both weight formats
    std::vector<float> W1(B * N * N), b1(B * N), W2(B * N * N), b2(B * N);
    const float* hp = c->wblob.data() + S * N + N;
    for (size_t b = 0; b < B; ++b) {
        std::memcpy(&W1[b * N * N], hp, N * N * 4); hp += N * N;
        std::memcpy(&b1[b * N], hp, N * 4); hp += N;
        std::memcpy(&W2[b * N * N], hp, N * N * 4); hp += N * N;
        std::memcpy(&b2[b * N], hp, N * 4); hp += N;
    }
    const float* Wo = hp; hp += N * C;
    const float* bo = hp;
    // fp32 path: repack into the device buffer layout W0 b0 | W1[B] | b1[B] | W2[B] | b2[B] | Wo | bo
    {
        std::vector<float> pk;
        pk.reserve(c->wblob.size());
        pk.insert(pk.end(), c->wblob.begin(), c->wblob.begin() + S * N + N);
        pk.insert(pk.end(), W1.begin(), W1.end());
        pk.insert(pk.end(), b1.begin(), b1.end());
        pk.insert(pk.end(), W2.begin(), W2.end());
        pk.insert(pk.end(), b2.begin(), b2.end());
        pk.insert(pk.end(), Wo, Wo + N * C);
        pk.insert(pk.end(), bo, bo + C);
        CK(cudaMemcpy(c->d_wf32, pk.data(), pk.size() * 4, cudaMemcpyHostToDevice));
        const float* d = c->d_wf32 + S * N + N;
        c->wf.W1 = d; d += B * N * N;
        c->wf.b1 = d; d += B * N;
        c->wf.W2 = d; d += B * N * N;
        c->wf.b2 = d; d += B * N;
        c->wf.Wo = d; d += N * C;
        c->wf.bo = d;
        c->wf.N = int(N); c->wf.B = int(B); c->wf.C = int(C);
    }
    // bf16 tensor-core operands: K-major ([out][in]) bf16, biases fp32, fp32 layer 0 (FFMA kernels)
    // plus layer 0 as a split-bf16 operand: W0 = W0h + W0m + W0l exactly (three bf16 pieces of the
    // 24-bit significand) and x = xh + xl exactly (x is 16-bit fixed point), so with
    // A0 = [xh | xl | xh | xl | xh | xl] and B0 = [W0h | W0h | W0m | W0m | W0l | W0l] (K = 42 of 48)
    // every product is exact and only the fp32 accumulation rounds (R22). B0 is rows
    // [2BN + Cp, 2BN + Cp + N) of the same [rows][N] tensor; only its first 48 columns are read.
    {
        const size_t nb16 = 2 * B * N * N + Cp * N + N * N;
        const size_t nf32 = S * N + N + 2 * B * N + Cp;
        if (first) {
            CK(cudaMalloc(&c->d_wbf, nb16 * 2 + nf32 * 4));
            c->device_bytes += nb16 * 2 + nf32 * 4;
        }
        std::vector<uint16_t> h16(nb16, 0);
        std::vector<float> h32;
        h32.reserve(nf32);
        for (size_t b = 0; b < B; ++b)
            for (size_t o = 0; o < N; ++o)
                for (size_t i = 0; i < N; ++i) {
                    h16[b * N * N + o * N + i] = f32_to_bf16_rne(W1[b * N * N + i * N + o]);
                    h16[(B + b) * N * N + o * N + i] = f32_to_bf16_rne(W2[b * N * N + i * N + o]);
                }
        for (size_t o = 0; o < C; ++o)
            for (size_t i = 0; i < N; ++i) h16[2 * B * N * N + o * N + i] = f32_to_bf16_rne(Wo[i * C + o]);
        {
            uint16_t* b0s = h16.data() + 2 * B * N * N + Cp * N;
            for (size_t o = 0; o < N; ++o)
                for (size_t f = 0; f < S; ++f) {
                    float rest = c->wblob[f * N + o];
                    for (size_t part = 0; part < 3; ++part) {
                        const uint16_t h = f32_to_bf16_rne(rest);
                        const uint32_t hb = uint32_t(h) << 16;
                        float hf;
                        std::memcpy(&hf, &hb, 4);
                        rest -= hf;                                   // exact (Sterbenz-style residual)
                        b0s[o * N + (2 * part) * S + f] = h;         // paired with xh
                        b0s[o * N + (2 * part + 1) * S + f] = h;     // paired with xl
                    }
                }
        }
        h32.insert(h32.end(), c->wblob.begin(), c->wblob.begin() + S * N + N);
        h32.insert(h32.end(), b1.begin(), b1.end());
        h32.insert(h32.end(), b2.begin(), b2.end());
        for (size_t o = 0; o < Cp; ++o) h32.push_back(o < C ? bo[o] : -3.0e38f);
        uint16_t* d16 = static_cast<uint16_t*>(c->d_wbf);
        float* d32 = reinterpret_cast<float*>(d16 + nb16);
        c->h_bias.assign(h32.begin() + S * N, h32.end());
        CK(cudaMemcpy(d16, h16.data(), nb16 * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d32, h32.data(), nf32 * 4, cudaMemcpyHostToDevice));
        c->wb.W1t = d16;
        c->wb.W2t = d16 + B * N * N;
        c->wb.Wot = d16 + 2 * B * N * N;
        c->wb.W0 = d32;
        c->wb.b0 = d32 + S * N;
        c->wb.b1 = d32 + S * N + N;
        c->wb.b2 = d32 + S * N + N + B * N;
        c->wb.bo = d32 + S * N + N + 2 * B * N;
        c->wb.N = int(N); c->wb.B = int(B); c->wb.C = int(C); c->wb.Cp = int(Cp);
    }
    if (c->cfg.mlp == TANG_MLP_FP8_TC || c->cfg.mlp == TANG_MLP_NVFP4_TC) {
        // e4m3 operands and folded power-of-two epilogue constants (R23); the NVFP4
        // chain (R24) shares the per-tensor scales, constants and layer-0 operand
        if (c->act_exp.size() != 2 * B + 1) return TANG_EMODEL;
        const size_t nq = (2 * B * N + Cp) * N, n0 = N * 64, nv = N + 2 * B * N + Cp;
        if (!c->d_wf8) {
            CK(cudaMalloc(&c->d_wf8, nq + n0 * 2 + nv * 4));
            c->device_bytes += nq + n0 * 2 + nv * 4;
        }
        std::vector<uint8_t> hq(nq, 0);
        std::vector<uint16_t> h0(n0, 0);
        std::vector<float> hv;
        hv.reserve(nv);
        auto amax = [](const float* w, size_t cnt) {
            double m = 0;
            for (size_t j = 0; j < cnt; ++j) m = std::max(m, double(std::fabs(w[j])));
            return m;
        };
        const float* W0 = c->wblob.data();
        const float* b0 = W0 + S * N;
        auto sc = [&](int k) { return std::ldexp(1.0, c->act_exp[k]); };
        WeightsF8& w = c->w8;
        w.N = int(N); w.B = int(B); w.C = int(C); w.Cp = int(Cp);
        w.inv_sh0 = float(1.0 / sc(0));
        for (size_t o = 0; o < N; ++o) hv.push_back(float(double(b0[o]) / sc(0)));
        std::vector<float> c2v, c2m;            // b2 / (s_u s_w2) (fp8), b2 / s_h' (nvfp4)
        float r2[kMaxBlocksF8] = {};             // s_h / s_h' (nvfp4 skip)
        double s_in = sc(0);
        for (size_t b = 0; b < B; ++b) {
            const float* W1 = b0 + N + b * (2 * N * N + 2 * N);
            const float* b1 = W1 + N * N;
            const float* W2 = b1 + N;
            const float* b2 = W2 + N * N;
            const double sw1 = std::ldexp(1.0, pow2_exp(amax(W1, N * N)));
            const double sw2 = std::ldexp(1.0, pow2_exp(amax(W2, N * N)));
            const double su = sc(1 + 2 * b), sout = sc(2 + 2 * b);
            for (size_t o = 0; o < N; ++o)
                for (size_t i = 0; i < N; ++i) {
                    hq[(b * N + o) * N + i] = to_e4m3_code(double(W1[i * N + o]) / sw1);
                    hq[((B + b) * N + o) * N + i] = to_e4m3_code(double(W2[i * N + o]) / sw2);
                }
            for (size_t o = 0; o < N; ++o) hv.push_back(float(double(b1[o]) / su));
            for (size_t o = 0; o < N; ++o) c2v.push_back(float(double(b2[o]) / (su * sw2)));
            for (size_t o = 0; o < N; ++o) c2m.push_back(float(double(b2[o]) / sout));
            r2[b] = float(s_in / sout);
            w.m1[b] = float(s_in * sw1 / su);
            w.k2[b] = float(s_in / (su * sw2));
            w.m2[b] = float(su * sw2 / sout);
            s_in = sout;
        }
        hv.insert(hv.end(), c2v.begin(), c2v.end());
        {
            const float* Wo = c->wblob.data() + S * N + N + B * (2 * N * N + 2 * N);
            const float* bo = Wo + N * C;
            const double swo = std::ldexp(1.0, pow2_exp(amax(Wo, N * C)));
            for (size_t o = 0; o < C; ++o)
                for (size_t i = 0; i < N; ++i) hq[(2 * B * N + o) * N + i] = to_e4m3_code(double(Wo[i * C + o]) / swo);
            w.mo = float(s_in * swo);
            for (size_t o = 0; o < Cp; ++o) hv.push_back(o < C ? bo[o] : -3.0e38f);
        }
        // layer-0 split operand (R22), [N][64] bf16
        auto split3 = [](float v, uint16_t* out) {
            for (int part = 0; part < 3; ++part) {
                out[part] = f32_to_bf16_rne(v);
                const uint32_t hb = uint32_t(out[part]) << 16;
                float hf;
                std::memcpy(&hf, &hb, 4);
                v -= hf;
            }
        };
        for (size_t o = 0; o < N; ++o)
            for (size_t f = 0; f < S; ++f) {
                uint16_t pc[3];
                split3(W0[f * N + o], pc);
                for (size_t part = 0; part < 3; ++part) {
                    h0[o * 64 + (2 * part) * S + f] = pc[part];
                    h0[o * 64 + (2 * part + 1) * S + f] = pc[part];
                }
            }
        uint8_t* d8 = static_cast<uint8_t*>(c->d_wf8);
        uint16_t* d0 = reinterpret_cast<uint16_t*>(d8 + nq);
        float* dv = reinterpret_cast<float*>(d0 + n0);
        CK(cudaMemcpy(d8, hq.data(), nq, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d0, h0.data(), n0 * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dv, hv.data(), nv * 4, cudaMemcpyHostToDevice));
        w.Wq = d8;
        w.B0 = d0;
        w.b0s = dv;
        w.b1s = dv + N;
        w.c2 = dv + N + B * N;
        w.bo = dv + N + 2 * B * N;
        if (c->f8) f8_plan_set_scales(c->f8, w);
        if (c->cfg.mlp == TANG_MLP_NVFP4_TC) {
            // NVFP4 operands (R24): e2m1 codes [2BN + Cp][N / 2] (value 2i in the low nibble of byte i)
            // and per pass (W1(b): slot b, W2(b): B + b, Wo pass q: 2B + q) 8 scale blocks of 512 B,
            // block 2j + h = K step j (inputs 64j..64j+63) x rows 128h..128h+127 of the pass, byte
            // (row % 32) * 16 + (row % 128 / 32) * 4 + (16-input block within the step)
            const size_t rows = 2 * B * N + Cp, nsf = (2 * B + 2) * 4096;
            if (!c->d_wf4) {
                CK(cudaMalloc(&c->d_wf4, rows * (N / 2) + nsf + nv * 4));
                c->device_bytes += rows * (N / 2) + nsf + nv * 4;
            }
            std::vector<uint8_t> h4(rows * (N / 2), 0), hsf(nsf, 0);
            // W [in = N][out] with per-tensor scale s: output o becomes packed row `row`, its pass
            // row (row - row0) the scale-block row
            auto put = [&](const float* W, size_t out_dim, double s, size_t row0, size_t slot0) {
                for (size_t o = 0; o < out_dim; ++o) {
                    const size_t row = row0 + o, q = o / 256, pr = o % 256;
                    for (size_t kb = 0; kb < N / 16; ++kb) {
                        double m = 0;
                        for (size_t i = 16 * kb; i < 16 * kb + 16; ++i)
                            m = std::max(m, std::fabs(double(W[i * out_dim + o]) / s));
                        const uint8_t sc = to_e4m3_code(m / 6.0);
                        const double sv = e4m3_value(sc);
                        hsf[(slot0 + q) * 4096 + (2 * (kb / 4) + pr / 128) * 512 + (pr % 32) * 16 + (pr % 128 / 32) * 4 +
                            kb % 4] = sc;
                        for (size_t i = 16 * kb; i < 16 * kb + 16; ++i) {
                            const uint8_t code = sv > 0 ? to_e2m1_code(double(W[i * out_dim + o]) / s / sv) : 0;
                            h4[row * (N / 2) + i / 2] |= uint8_t(code << (4 * (i & 1)));
                        }
                    }
                }
            };
            for (size_t b = 0; b < B; ++b) {
                const float* W1 = b0 + N + b * (2 * N * N + 2 * N);
                const float* W2 = W1 + N * N + N;
                put(W1, N, std::ldexp(1.0, pow2_exp(amax(W1, N * N))), b * N, b);
                put(W2, N, std::ldexp(1.0, pow2_exp(amax(W2, N * N))), (B + b) * N, B + b);
            }
            {
                const float* Wo = c->wblob.data() + S * N + N + B * (2 * N * N + 2 * N);
                put(Wo, C, std::ldexp(1.0, pow2_exp(amax(Wo, N * C))), 2 * B * N, 2 * B);
            }
            uint8_t* d4 = static_cast<uint8_t*>(c->d_wf4);
            CK(cudaMemcpy(d4, h4.data(), h4.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(d4 + h4.size(), hsf.data(), nsf, cudaMemcpyHostToDevice));
            // epilogue constants: fp8's with b2 / (s_u s_w2) replaced by b2 / s_h' (R24 GEMM2 form)
            std::vector<float> cv(hv.begin(), hv.begin() + N + B * N);
            cv.insert(cv.end(), c2m.begin(), c2m.end());
            cv.insert(cv.end(), hv.begin() + N + 2 * B * N, hv.end());
            float* dcv = reinterpret_cast<float*>(d4 + h4.size() + nsf);
            CK(cudaMemcpy(dcv, cv.data(), nv * 4, cudaMemcpyHostToDevice));
            c->w4.s = w;
            c->w4.Wq = d4;
            c->w4.SF = d4 + h4.size();
            c->w4.consts = dcv;
            for (size_t b = 0; b < B; ++b) c->w4.r2[b] = r2[b];
            if (c->f4) f4_plan_set_scales(c->f4, c->w4);
        }
    }
    return TANG_OK;
}

int upload(tang_ctx* c) {
    CK(cudaSetDevice(c->device));
    for (uint32_t r = 0; r < kNumRegions; ++r) {
        c->tab_bytes[r] = c->region_bytes(r);
        CK(cudaMalloc(&c->d_tab[r], c->tab_bytes[r]));
        CK(cudaMemcpy(c->d_tab[r], c->region_host(r), c->tab_bytes[r], cudaMemcpyHostToDevice));
        c->device_bytes += c->tab_bytes[r];
    }
    CK(cudaMalloc(&c->d_rejected, sizeof(uint32_t)));
    CK(cudaMemset(c->d_rejected, 0, sizeof(uint32_t)));
    int e = upload_weights(c);
    if (e) return e;
    // streams + scratch
    const uint32_t ns = c->cfg.streams;
    c->streams.resize(ns);
    for (auto& s : c->streams) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const size_t mb = c->cfg.max_batch;
    for (uint32_t q = 0; q <= ns; ++q) {
        Scratch sc;
        void* m;
        // deferred long-bucket entries: up to one per (packet, probed tuple); tang_classify_with_pred
        // may probe up to TANG_MAX_TOPK tuples whatever cfg.topk is
        const size_t k = TANG_MAX_TOPK;
        const size_t bytes = mb * 8 + mb * 16 * k + mb * 4 * TANG_MAX_TOPK + mb * 4 + mb * 8 + 64;
        CK(cudaMalloc(&m, bytes));
        c->scratch_mem.push_back(m);
        c->device_bytes += bytes;
        uint8_t* p = static_cast<uint8_t*>(m);
        sc.best_key = reinterpret_cast<unsigned long long*>(p); p += mb * 8;
        sc.long_ent = reinterpret_cast<uint4*>(p); p += mb * 16 * k;
        sc.pred = reinterpret_cast<uint32_t*>(p); p += mb * 4 * TANG_MAX_TOPK;
        sc.miss_idx = reinterpret_cast<uint32_t*>(p); p += mb * 4;
        sc.miss_bound = reinterpret_cast<uint32_t*>(p); p += mb * 8;
        sc.miss_count = reinterpret_cast<uint32_t*>(p);
        sc.long_count = sc.miss_count + 1;
        c->scratch.push_back(sc);
    }
    return TANG_OK;
}

void prof_begin(tang_ctx* c, const char* name, cudaStream_t s, cudaEvent_t* a) {
    if (!c->prof) return;
    *a = c->ev();
    cudaEventRecord(*a, s);
    (void)name;
}
void prof_end(tang_ctx* c, const char* name, cudaStream_t s, cudaEvent_t a) {
    if (!c->prof) return;
    cudaEvent_t b = c->ev();
    cudaEventRecord(b, s);
    c->prof_pending.push_back({name, a, b});
}

// one chunk (<= max_batch packets) of the hot path on stream s with scratch sc
int run_chunk(tang_ctx* c, const void* d_hdr, size_t n, uint32_t* d_rule_id, uint32_t* d_pred_out,
              float* d_logits, uint8_t* d_fell, const uint32_t* d_pred_in, uint32_t kin, bool use_pred,
              const Scratch& sc, cudaStream_t s) {
    const uint32_t k = use_pred ? kin : c->cfg.topk;
    const uint32_t* pred = d_pred_in;
    cudaEvent_t a = nullptr;
    if (!use_pred) {
        uint32_t* out = d_pred_out ? d_pred_out : sc.pred;
        prof_begin(c, "mlp", s, &a);
        if (c->cfg.mlp == TANG_MLP_FP32_FFMA) {
            launch_mlp_ffma(c->wf, d_hdr, n, k, out, d_logits, s);
        } else if (c->f8) {
            int e = launch_mlp_f8(c->f8, d_hdr, n, k, out, d_logits, s);
            if (e) return e;
        } else if (c->f4) {
            int e = launch_mlp_f4(c->f4, d_hdr, n, k, out, d_logits, s);
            if (e) return e;
        } else {
            int e = c->tc2 ? launch_mlp_tc2(c->tc2, d_hdr, n, k, out, d_logits, s)
                           : launch_mlp_tc(c->tc, d_hdr, n, k, out, d_logits, s);
            if (e) return e;
        }
        prof_end(c, "mlp", s, a);
        pred = out;
    }
    const Tables t = c->tables();
    prof_begin(c, "probe", s, &a);
    launch_probe(t, d_hdr, n, pred, k, c->cfg.mode, d_rule_id, d_fell, sc, s);
    prof_end(c, "probe", s, a);
    prof_begin(c, "fallback", s, &a);
    launch_fallback(t, d_hdr, n, d_rule_id, d_fell, sc, s);
    prof_end(c, "fallback", s, a);
    CK(cudaGetLastError());
    return TANG_OK;
}

int run_async(tang_ctx* c, const tang_header* d_hdr, size_t n, uint32_t* d_rule_id, uint32_t* d_pred,
              float* d_logits, uint8_t* d_fell, const uint32_t* d_pred_in, uint32_t kin, bool use_pred,
              cudaStream_t s, const Scratch& sc) {
    if (c->host_only) return TANG_ENODEV;
    if (n == 0) return TANG_OK;
    if (!d_hdr || !d_rule_id) return TANG_EINVAL;
    if ((reinterpret_cast<uintptr_t>(d_hdr) & 15u) != 0) return TANG_EINVAL;   // 16-B vector loads
    const size_t mb = c->cfg.max_batch;
    const uint32_t k = use_pred ? kin : c->cfg.topk;
    for (size_t o = 0; o < n; o += mb) {
        const size_t m = std::min(mb, n - o);
        int e = run_chunk(c, d_hdr + o, m, d_rule_id + o, d_pred ? d_pred + o * k : nullptr,
                          d_logits ? d_logits + o * c->C : nullptr, d_fell ? d_fell + o : nullptr,
                          use_pred ? d_pred_in + o * kin : nullptr, kin, use_pred, sc, s);
        if (e) return e;
    }
    return TANG_OK;
}

}  // namespace

// =========================================================================================
// C ABI
// =========================================================================================
extern "C" {

const char* tang_strerror(int code) {
    switch (code) {
        case TANG_OK: return "ok";
        case TANG_EINVAL: return "invalid argument";
        case TANG_EMODEL: return "invalid model blob";
        case TANG_ENOTUPLE: return "no candidate tuple for rule (rebuild required)";
        case TANG_ENOENT: return "unknown rule id";
        case TANG_ENOMEM: return "out of memory or table capacity";
        case TANG_ECUDA: return "CUDA error";
        case TANG_ENODEV: return "no CUDA device for this ctx";
        case TANG_ESTATE: return "operation not allowed in this ctx state";
        default: return "unknown error";
    }
}

int tang_build(const tang_rule* rules, size_t n_rules, const void* model_blob, size_t blob_len,
               const tang_config* cfg, tang_ctx** out) {
    if (!out || (n_rules && !rules)) return TANG_EINVAL;
    *out = nullptr;
    tang_ctx* c = new (std::nothrow) tang_ctx();
    if (!c) return TANG_ENOMEM;
    if (cfg) c->cfg = *cfg;
    else c->cfg.device = 0;
    if (c->cfg.topk == 0) c->cfg.topk = 1;
    if (c->cfg.max_batch == 0) c->cfg.max_batch = 1u << 20;
    if (c->cfg.batch == 0) c->cfg.batch = 1u << 18;
    if (c->cfg.streams == 0) c->cfg.streams = 4;
    if (c->cfg.ring_slots == 0) c->cfg.ring_slots = 2 * c->cfg.streams;
    if (c->cfg.rule_capacity == 0) c->cfg.rule_capacity = uint32_t(n_rules / 4 + 4096);
    if (c->cfg.topk > TANG_MAX_TOPK || c->cfg.mode > 1 || c->cfg.mlp > 3 || c->cfg.mlp_kernel > 6 ||
        c->cfg.batch > c->cfg.max_batch ||
        c->cfg.streams > 32) {
        delete c;
        return TANG_EINVAL;
    }
    int e = parse_blob(c, model_blob, blob_len);
    if (!e && c->cfg.topk > c->C) e = TANG_EINVAL;
    if (!e) e = build_tables(c, rules, n_rules);
    if (e) { delete c; return e; }
    c->host_only = c->cfg.device < 0;
    if (!c->host_only) {
        c->device = c->cfg.device;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || c->device >= ndev) { tang_destroy(c); return TANG_ENODEV; }
        e = upload(c);
        if (!e && c->cfg.mlp == TANG_MLP_BF16_TC) {
            if (c->cfg.mlp_kernel == TANG_KERNEL_PAIR || c->cfg.mlp_kernel == TANG_KERNEL_TS)
                e = TANG_EINVAL;                                               // variants removed (slower)
            else if (c->cfg.mlp_kernel == TANG_KERNEL_DUAL || (c->cfg.mlp_kernel == TANG_KERNEL_AUTO && c->N <= 256)) {
                c->tc2 = tc2_plan_create(c->wb, c->device, &e);
                // AUTO: a model whose two A tiles + biases leave no room for 2 weight stages runs the
                // one-tile kernel instead
                if (!c->tc2 && e == TANG_EMODEL && c->cfg.mlp_kernel == TANG_KERNEL_AUTO)
                    c->tc = tc_plan_create(c->wb, nullptr, c->device, 0, 2, &e);
            } else
                // AUTO = the fastest measured variant: 2SM (M = 256 cta_group::2 pairs) for N > 256 (r02f:
                // 1322 vs 1160 TFLOP/s single at N = 512), SINGLE for N <= 256 (r02_n256_ab: 646 vs 523)
                c->tc = tc_plan_create(c->wb, nullptr, c->device,
                                       c->cfg.mlp_kernel == TANG_KERNEL_2SM ||
                                           (c->cfg.mlp_kernel == TANG_KERNEL_AUTO && c->N > 256),
                                       c->cfg.mlp_kernel == TANG_KERNEL_WIDE ? 4 : 2, &e);
        }
        if (!e && c->cfg.mlp == TANG_MLP_FP8_TC) {
            if (c->act_exp.empty() || c->N % 128 || c->B > uint32_t(kMaxBlocksF8) || c->Cp > 512) e = TANG_EMODEL;
            else c->f8 = f8_plan_create(c->w8, c->device, c->cfg.mlp_kernel != TANG_KERNEL_SINGLE, &e);
        }
        if (!e && c->cfg.mlp == TANG_MLP_NVFP4_TC) {
            if (c->act_exp.empty() || c->N != 256 || c->B > uint32_t(kMaxBlocksF8) || c->Cp > 320) e = TANG_EMODEL;
            else c->f4 = f4_plan_create(c->w4, c->device, &e);
        }
        if (e) { tang_destroy(c); return e; }
    }
    *out = c;
    return TANG_OK;
}

void tang_destroy(tang_ctx* c) {
    if (!c) return;
    if (!c->host_only && c->device >= 0) {
        cudaSetDevice(c->device);
        for (auto& s : c->streams) cudaStreamSynchronize(s);
        cudaDeviceSynchronize();
        if (c->tc) tc_plan_destroy(c->tc);
        if (c->tc2) tc2_plan_destroy(c->tc2);
        if (c->f8) f8_plan_destroy(c->f8);
        if (c->d_wf8) cudaFree(c->d_wf8);
        if (c->f4) f4_plan_destroy(c->f4);
        if (c->d_wf4) cudaFree(c->d_wf4);
        for (auto p : c->d_tab) if (p) cudaFree(p);
        if (c->d_rejected) cudaFree(c->d_rejected);
        if (c->d_wf32) cudaFree(c->d_wf32);
        if (c->d_wbf) cudaFree(c->d_wbf);
        for (auto p : c->scratch_mem) cudaFree(p);
        if (c->d_delta) cudaFree(c->d_delta);
        if (c->h_delta_pinned) cudaFreeHost(c->h_delta_pinned);
        for (auto p : c->ring_hdr) cudaFreeHost(p);
        for (auto p : c->ring_out) cudaFreeHost(p);
        for (auto e : c->ring_done) cudaEventDestroy(e);
        for (auto p : c->dev_hdr) cudaFree(p);
        for (auto p : c->dev_out) cudaFree(p);
        for (auto& ev : c->lat_ev) for (auto e : ev) cudaEventDestroy(e);
        for (auto& pe : c->prof_pending) { cudaEventDestroy(pe.a); cudaEventDestroy(pe.b); }
        for (auto e : c->ev_pool) cudaEventDestroy(e);
        for (auto& s : c->streams) cudaStreamDestroy(s);
    }
    delete c;
}

int tang_stats(tang_ctx* c, tang_stats_t* o) {
    if (!c || !o) return TANG_EINVAL;
    std::memset(o, 0, sizeof(*o));
    o->tuples = c->C;
    o->rules = uint32_t(c->where.size());
    o->mismatch_count = c->mismatch;
    o->epoch = c->meta.epoch;
    o->device_bytes = c->device_bytes;
    for (uint32_t r = 0; r < kNumRegions; ++r) o->table_bytes += c->region_bytes(r);
    o->slots = uint32_t(c->slots.size());
    o->keys = c->keys;
    o->S = c->S; o->N = c->N; o->B = c->B; o->C = c->C;
    o->checksum = mirror_checksum(c);
    o->live_keys = c->live_keys;
    o->delta_rejected = c->host_rejected;
    if (!c->host_only && c->d_rejected) {
        uint32_t dr = 0;
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpy(&dr, c->d_rejected, sizeof(dr), cudaMemcpyDeviceToHost));
        o->delta_rejected += dr;
    }
    return TANG_OK;
}

int tang_classify_async(tang_ctx* c, const tang_header* d_hdr, size_t n, uint32_t* d_rule_id, void* stream) {
    if (!c) return TANG_EINVAL;
    if (c->host_only) return TANG_ENODEV;
    return run_async(c, d_hdr, n, d_rule_id, nullptr, nullptr, nullptr, nullptr, 0, false,
                     static_cast<cudaStream_t>(stream), c->scratch.back());
}

int tang_classify_ex(tang_ctx* c, const tang_header* d_hdr, size_t n, uint32_t* d_rule_id, uint32_t* d_pred,
                     float* d_logits, uint8_t* d_fell, void* stream) {
    if (!c) return TANG_EINVAL;
    if (c->host_only) return TANG_ENODEV;
    return run_async(c, d_hdr, n, d_rule_id, d_pred, d_logits, d_fell, nullptr, 0, false,
                     static_cast<cudaStream_t>(stream), c->scratch.back());
}

int tang_classify_with_pred(tang_ctx* c, const tang_header* d_hdr, size_t n, const uint32_t* d_pred, uint32_t k,
                            uint32_t* d_rule_id, uint8_t* d_fell, void* stream) {
    if (!c) return TANG_EINVAL;
    if (c->host_only) return TANG_ENODEV;
    if (k > TANG_MAX_TOPK || (k && !d_pred && n)) return TANG_EINVAL;
    return run_async(c, d_hdr, n, d_rule_id, nullptr, nullptr, d_fell, d_pred, k, true,
                     static_cast<cudaStream_t>(stream), c->scratch.back());
}

int tang_encode_async(tang_ctx* c, const tang_header* d_hdr, size_t n, float* d_feat, void* stream) {
    if (!c) return TANG_EINVAL;
    if (c->host_only) return TANG_ENODEV;
    if (n == 0) return TANG_OK;
    if (!d_hdr || !d_feat || (reinterpret_cast<uintptr_t>(d_hdr) & 15u) || (reinterpret_cast<uintptr_t>(d_feat) & 15u))
        return TANG_EINVAL;
    cudaEvent_t a = nullptr;
    prof_begin(c, "encode", static_cast<cudaStream_t>(stream), &a);
    launch_encode(d_hdr, n, d_feat, static_cast<cudaStream_t>(stream));
    prof_end(c, "encode", static_cast<cudaStream_t>(stream), a);
    CK(cudaGetLastError());
    return TANG_OK;
}

// Streaming classify over pinned host rings: chunk q uses ring slot q % R and
// stream q % S; H2D(q+1), kernels(q) and D2H(q-1) overlap across streams.
int tang_classify(tang_ctx* c, const tang_header* hdr, size_t n, uint32_t* rule_id) {
    if (!c) return TANG_EINVAL;
    if (c->host_only) return TANG_ENODEV;
    if (n == 0) return TANG_OK;
    if (!hdr || !rule_id) return TANG_EINVAL;
    CK(cudaSetDevice(c->device));
    const size_t bs = c->cfg.batch;
    const uint32_t S = c->cfg.streams, R = c->cfg.ring_slots;
    if (c->dev_hdr.empty()) {
        for (uint32_t s = 0; s < S; ++s) {
            void* p;
            CK(cudaMalloc(&p, bs * sizeof(tang_header)));
            c->dev_hdr.push_back(p);
            uint32_t* q;
            CK(cudaMalloc(&q, bs * 4));
            c->dev_out.push_back(q);
            c->device_bytes += bs * 20;
        }
    }
    cudaPointerAttributes ai{}, ao{};
    const bool pin_in = cudaPointerGetAttributes(&ai, hdr) == cudaSuccess && ai.type == cudaMemoryTypeHost;
    const bool pin_out = cudaPointerGetAttributes(&ao, rule_id) == cudaSuccess && ao.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if ((!pin_in || !pin_out) && c->ring_hdr.empty()) {
        for (uint32_t r = 0; r < R; ++r) {
            uint8_t* h;
            uint32_t* o;
            CK(cudaHostAlloc(reinterpret_cast<void**>(&h), bs * sizeof(tang_header), cudaHostAllocDefault));
            CK(cudaHostAlloc(reinterpret_cast<void**>(&o), bs * 4, cudaHostAllocDefault));
            c->ring_hdr.push_back(h);
            c->ring_out.push_back(o);
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->ring_done.push_back(e);
        }
    }
    // slot sizes ramp up bs/8, bs/4, bs/2, bs, bs, ...: the first H2D (not overlapped with any
    // compute) is short, later launches are full-size (a persistent grid pays fill/drain per launch)
    std::vector<std::pair<size_t, size_t>> chunk;        // (offset, packets)
    const size_t ramp_div = 8;                            // measured best of 1/4/8/16 (profiles/r01_ab_ring_ramp.txt)
    for (size_t o = 0, sz = std::min(bs, std::max<size_t>(bs / ramp_div, 8192)); o < n;) {
        const size_t m = std::min(sz, n - o);
        chunk.push_back({o, m});
        o += m;
        sz = std::min(bs, 2 * sz);
    }
    const size_t nchunks = chunk.size();
    while (c->lat_ev.size() < nchunks) {
        std::array<cudaEvent_t, 4> ev;
        for (auto& e : ev) CK(cudaEventCreate(&e));
        c->lat_ev.push_back(ev);
    }
    std::vector<long long> slot_chunk(R, -1);
    auto drain = [&](uint32_t r) -> int {
        if (slot_chunk[r] < 0) return TANG_OK;
        CK(cudaEventSynchronize(c->ring_done[r]));
        const size_t o = chunk[size_t(slot_chunk[r])].first, m = chunk[size_t(slot_chunk[r])].second;
        if (!pin_out) std::memcpy(rule_id + o, c->ring_out[r], m * 4);
        slot_chunk[r] = -1;
        return TANG_OK;
    };
    for (size_t q = 0; q < nchunks; ++q) {
        const size_t o = chunk[q].first, m = chunk[q].second;
        const uint32_t s = uint32_t(q % S);
        cudaStream_t st = c->streams[s];
        const void* src = hdr + o;
        uint32_t* dst = rule_id + o;
        if (!pin_in || !pin_out) {
            const uint32_t r = uint32_t(q % R);
            int e = drain(r);
            if (e) return e;
            if (!pin_in) { std::memcpy(c->ring_hdr[r], hdr + o, m * sizeof(tang_header)); src = c->ring_hdr[r]; }
            if (!pin_out) dst = c->ring_out[r];
            slot_chunk[r] = (long long)q;
        }
        CK(cudaEventRecord(c->lat_ev[q][0], st));
        CK(cudaMemcpyAsync(c->dev_hdr[s], src, m * sizeof(tang_header), cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(c->lat_ev[q][1], st));
        int e = run_async(c, static_cast<const tang_header*>(c->dev_hdr[s]), m, c->dev_out[s], nullptr, nullptr,
                          nullptr, nullptr, 0, false, st, c->scratch[s]);
        if (e) return e;
        CK(cudaEventRecord(c->lat_ev[q][2], st));
        CK(cudaMemcpyAsync(dst, c->dev_out[s], m * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(c->lat_ev[q][3], st));
        if (!pin_in || !pin_out) CK(cudaEventRecord(c->ring_done[q % R], st));
    }
    if (!pin_in || !pin_out)
        for (uint32_t r = 0; r < R; ++r) { int e = drain(r); if (e) return e; }
    for (auto& s : c->streams) CK(cudaStreamSynchronize(s));
    c->last_lat.resize(nchunks);
    c->last_timeline.resize(nchunks * 4);
    for (size_t q = 0; q < nchunks; ++q) {
        cudaEventElapsedTime(&c->last_lat[q], c->lat_ev[q][0], c->lat_ev[q][3]);
        for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&c->last_timeline[q * 4 + k], c->lat_ev[0][0], c->lat_ev[q][k]);
    }
    return TANG_OK;
}

int tang_timeline_read(tang_ctx* c, float* t, int cap) {
    if (!c) return TANG_EINVAL;
    const int n = int(c->last_timeline.size() / 4);
    for (int i = 0; i < 4 * n && i < 4 * cap; ++i) t[i] = c->last_timeline[i];
    return n;
}

int tang_debug_activations(tang_ctx* c, const tang_header* d_hdr, size_t n, void* d_act, uint32_t* d_pred,
                           float* d_logits, void* stream) {
    if (!c) return TANG_EINVAL;
    if (c->host_only) return TANG_ENODEV;
    if (!c->tc && !c->tc2 && !c->f8 && !c->f4) return TANG_ESTATE;
    if (n == 0) return TANG_OK;
    if (!d_hdr || !d_act || !d_pred || (reinterpret_cast<uintptr_t>(d_hdr) & 15u) || (reinterpret_cast<uintptr_t>(d_act) & 15u))
        return TANG_EINVAL;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    int e = c->f8   ? launch_mlp_f8(c->f8, d_hdr, n, c->cfg.topk, d_pred, d_logits, st, static_cast<uint8_t*>(d_act))
            : c->f4 ? launch_mlp_f4(c->f4, d_hdr, n, c->cfg.topk, d_pred, d_logits, st, static_cast<uint8_t*>(d_act))
            : c->tc2 ? launch_mlp_tc2(c->tc2, d_hdr, n, c->cfg.topk, d_pred, d_logits, st, static_cast<uint16_t*>(d_act))
                    : launch_mlp_tc(c->tc, d_hdr, n, c->cfg.topk, d_pred, d_logits, st, static_cast<uint16_t*>(d_act));
    if (e) return e;
    CK(cudaGetLastError());
    return TANG_OK;
}

// profiling hook (not in tang.h's stable surface): phase timestamps of block 0 of the single-CTA
// chain, d_trace[4 tiles][2B+1 layers][16] (bf16 kernel; 8 for the fp8 kernels) int64 clock64 values
extern "C" int tang_debug_trace(tang_ctx* c, const tang_header* d_hdr, size_t n, uint32_t* d_pred, long long* d_trace,
                                void* stream) {
    if (!c || (!c->tc && !c->f8 && !c->f4)) return TANG_ESTATE;
    if (c->f4)
        return launch_mlp_f4(c->f4, d_hdr, n, c->cfg.topk, d_pred, nullptr, static_cast<cudaStream_t>(stream), nullptr,
                             d_trace);
    if (c->f8)
        return launch_mlp_f8(c->f8, d_hdr, n, c->cfg.topk, d_pred, nullptr, static_cast<cudaStream_t>(stream), nullptr,
                             d_trace);
    return launch_mlp_tc(c->tc, d_hdr, n, c->cfg.topk, d_pred, nullptr, static_cast<cudaStream_t>(stream), nullptr,
                         d_trace);
}

// Deferred update: swap in new weights for the same tuple set at a batch boundary.
int tang_reload_model(tang_ctx* c, const void* blob, size_t len) {
    if (!c) return TANG_EINVAL;
    tang_ctx tmp;
    int e = parse_blob(&tmp, blob, len);
    if (e) return e;
    if (tmp.N != c->N || tmp.B != c->B || tmp.C != c->C || tmp.sigs != c->sigs) return TANG_EMODEL;
    if ((c->cfg.mlp == TANG_MLP_FP8_TC || c->cfg.mlp == TANG_MLP_NVFP4_TC) && tmp.act_exp.empty()) return TANG_EMODEL;
    c->wblob.swap(tmp.wblob);
    c->act_exp.swap(tmp.act_exp);
    if (c->host_only) return TANG_OK;
    CK(cudaSetDevice(c->device));
    for (auto& st : c->streams) CK(cudaStreamSynchronize(st));
    CK(cudaDeviceSynchronize());                       // no batch in flight sees a mix of weights
    e = upload_weights(c);
    if (e) return e;
    CK(cudaDeviceSynchronize());
    return TANG_OK;
}

int tang_latency_read(tang_ctx* c, float* ms, int cap) {
    if (!c) return TANG_EINVAL;
    const int n = int(c->last_lat.size());
    for (int i = 0; i < n && i < cap; ++i) ms[i] = c->last_lat[i];
    return n;
}

// ---- updates --------------------------------------------------------------------------
int tang_update_plan(tang_ctx* c, const tang_update_op* ops, size_t n, int32_t* status, const void** delta,
                     size_t* len) {
    if (!c || (n && !ops)) return TANG_EINVAL;
    if (c->follower) return TANG_ESTATE;
    bool dirty = false;
    int first_err = TANG_OK;
    for (size_t i = 0; i < n; ++i) {
        int32_t st = 0;
        int e;
        if (ops[i].kind == TANG_OP_INSERT) e = plan_insert(c, ops[i].rule, &st, true, &dirty);
        else if (ops[i].kind == TANG_OP_DELETE) e = plan_delete(c, ops[i].id, &dirty);
        else e = TANG_EINVAL;
        if (status) status[i] = e ? e : st;
        if (e && !first_err) first_err = e;
    }
    if (dirty) rebuild_order(c);
    c->meta.epoch++;
    touch(c, kRegMeta, 0, sizeof(MetaDev));
    emit_delta(c);
    if (delta) *delta = c->delta.data();
    if (len) *len = c->delta.size() * sizeof(DeltaWord);
    return status ? TANG_OK : first_err;   // without a status array the first failure is reported
}

int tang_apply_delta_host(tang_ctx* c, const void* delta, size_t len) {
    if (!c || (len && !delta) || len % sizeof(DeltaWord)) return TANG_EINVAL;
    const DeltaWord* d = static_cast<const DeltaWord*>(delta);
    const size_t nw = len / sizeof(DeltaWord);
    if (nw == 0) return TANG_OK;
    if (d[0].region != kDeltaHeader || d[0].word != layout_hash(c) || size_t(d[0].value) + 1 != nw) {
        c->host_rejected += uint32_t(nw);
        return TANG_EINVAL;
    }
    for (size_t i = 1; i < nw; ++i)                 // validate everything before writing anything
        if (d[i].region >= kNumRegions || size_t(d[i].word) * 4 >= c->region_bytes(d[i].region)) {
            c->host_rejected += uint32_t(nw);
            return TANG_EINVAL;
        }
    for (size_t i = 1; i < nw; ++i) static_cast<uint32_t*>(c->region_host(d[i].region))[d[i].word] = d[i].value;
    c->follower = true;   // planner indexes are now stale on this ctx
    return TANG_OK;
}

static void region_words(const tang_ctx* c, uint32_t* w) {
    for (uint32_t r = 0; r < kNumRegions; ++r) w[r] = uint32_t(c->tab_bytes[r] / 4);
}

int tang_apply_delta_async(tang_ctx* c, const void* d_delta, size_t len, void* stream) {
    if (!c || (len && !d_delta) || len % sizeof(DeltaWord)) return TANG_EINVAL;
    if (c->host_only) return TANG_ENODEV;
    CK(cudaSetDevice(c->device));
    uint32_t rw[kNumRegions];
    region_words(c, rw);
    launch_apply_delta(static_cast<const DeltaWord*>(d_delta), len / sizeof(DeltaWord), c->d_tab, rw, layout_hash(c),
                       c->d_rejected, static_cast<cudaStream_t>(stream));
    CK(cudaGetLastError());
    return TANG_OK;
}

int tang_update(tang_ctx* c, const tang_update_op* ops, size_t n, int32_t* status, void* stream) {
    if (!c) return TANG_EINVAL;
    const void* delta;
    size_t len;
    if (n && !ops) return TANG_EINVAL;
    if (c->follower) return TANG_ESTATE;
    const int plan_err = tang_update_plan(c, ops, n, status, &delta, &len);   // only per-op failures now
    if (c->host_only) return plan_err;
    CK(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // order after everything queued on the ctx's own streams
    for (auto& s : c->streams) {
        cudaEvent_t ev = c->ev();
        CK(cudaEventRecord(ev, s));
        CK(cudaStreamWaitEvent(st, ev, 0));
        c->ev_pool.push_back(ev);
    }
    const size_t nw = len / sizeof(DeltaWord);
    if (nw > c->d_delta_cap) {
        if (c->d_delta) cudaFree(c->d_delta);
        if (c->h_delta_pinned) cudaFreeHost(c->h_delta_pinned);
        c->d_delta_cap = nw * 2;
        CK(cudaMalloc(&c->d_delta, c->d_delta_cap * sizeof(DeltaWord)));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_delta_pinned), c->d_delta_cap * sizeof(DeltaWord),
                         cudaHostAllocDefault));
    }
    std::memcpy(c->h_delta_pinned, delta, len);
    CK(cudaMemcpyAsync(c->d_delta, c->h_delta_pinned, len, cudaMemcpyHostToDevice, st));
    uint32_t rw[kNumRegions];
    region_words(c, rw);
    launch_apply_delta(c->d_delta, nw, c->d_tab, rw, layout_hash(c), c->d_rejected, st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return plan_err;                       // the ops that succeeded are applied either way
}

int tang_device_checksum(tang_ctx* c, uint64_t* out) {
    if (!c || !out) return TANG_EINVAL;
    if (c->host_only) return TANG_ENODEV;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    uint64_t h = 1469598103934665603ull;
    for (uint32_t r = 0; r < kNumRegions; ++r) {
        std::vector<uint8_t> buf(c->tab_bytes[r]);
        CK(cudaMemcpy(buf.data(), c->d_tab[r], buf.size(), cudaMemcpyDeviceToHost));
        h = fnv1a(h, buf.data(), buf.size());
    }
    *out = h;
    return TANG_OK;
}

int tang_table_digest_async(tang_ctx* c, uint64_t* d_digest, void* stream) {
    if (!c || !d_digest) return TANG_EINVAL;
    if (c->host_only) return TANG_ENODEV;
    CK(cudaSetDevice(c->device));
    uint32_t rw[kNumRegions];
    region_words(c, rw);
    launch_table_digest(c->d_tab, rw, reinterpret_cast<unsigned long long*>(d_digest), static_cast<cudaStream_t>(stream));
    CK(cudaGetLastError());
    return TANG_OK;
}

int tang_mirror_digest(tang_ctx* c, uint64_t* out) {
    if (!c || !out) return TANG_EINVAL;
    uint64_t h = 0;
    for (uint32_t r = 0; r < kNumRegions; ++r) {
        const uint32_t* p = static_cast<const uint32_t*>(c->region_host(r));
        const size_t nw = c->region_bytes(r) / 4;
        for (size_t w = 0; w < nw; ++w) h += digest_word(r, uint32_t(w), p[w]);
    }
    *out = h;
    return TANG_OK;
}

int tang_debug_candidates(tang_ctx* c, uint32_t sip, uint32_t dip, uint32_t* words, uint32_t cap) {
    if (!c) return TANG_EINVAL;
    const uint32_t W = c->meta.cand_words;
    const uint32_t* rs = c->cand.data() + size_t(sip >> 16) * W;
    const uint32_t* rd = c->cand.data() + (size_t(65536) + (dip >> 16)) * W;
    for (uint32_t q = 0; q < W && q < cap && words; ++q) words[q] = rs[q] & rd[q];
    return int(W);
}

int tang_rule_tuple(tang_ctx* c, uint32_t id, uint32_t* tuple) {
    if (!c || !tuple) return TANG_EINVAL;
    auto it = c->where.find(id);
    if (it == c->where.end()) return TANG_ENOENT;
    *tuple = c->slots[it->second.slot].tup_cnt & kTupleMask;
    return TANG_OK;
}

int tang_profile_enable(tang_ctx* c, int on) {
    if (!c) return TANG_EINVAL;
    c->prof = on != 0;
    c->prof_acc.clear();
    for (auto& pe : c->prof_pending) { c->ev_pool.push_back(pe.a); c->ev_pool.push_back(pe.b); }
    c->prof_pending.clear();
    return TANG_OK;
}

// accumulated kernel time (ms) and launch count per kernel name since enable
int tang_profile_read(tang_ctx* c, const char** names, float* ms, uint64_t* counts, int cap) {
    if (!c) return TANG_EINVAL;
    for (auto& pe : c->prof_pending) {
        cudaEventSynchronize(pe.b);
        float t = 0.f;
        cudaEventElapsedTime(&t, pe.a, pe.b);
        auto& acc = c->prof_acc[pe.name];
        acc.first += t;
        acc.second += 1;
        c->ev_pool.push_back(pe.a);
        c->ev_pool.push_back(pe.b);
    }
    c->prof_pending.clear();
    int i = 0;
    static std::vector<std::string> keep;   // stable storage for returned names
    keep.clear();
    for (auto& kv : c->prof_acc) keep.push_back(kv.first);
    for (auto& kv : c->prof_acc) {
        if (i < cap) {
            if (names) names[i] = keep[size_t(i)].c_str();
            if (ms) ms[i] = float(kv.second.first);
            if (counts) counts[i] = kv.second.second;
        }
        ++i;
    }
    return i;
}

}  // extern "C"
