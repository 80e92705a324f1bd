/*
 * tang.h -- C ABI of libtang, the B200 (sm_100a) hot path of TaNG
 * ("Modeling Packet Classification with TSS-assisted Neural Networks on GPUs",
 * arXiv 2601.03187; PAPER.md is cited as P:<line> with its section).
 *
 * What the library computes:
 *   for each packet header P, stage 1 predicts the tuple(s) to search with a residual
 *   MLP over the 7 16-bit header segments (§6.2, Eq. 1-2, argmax P:383);
 *   stage 2 truncates P to each predicted tuple's prefix-length signature, looks the
 *   truncated key up in that tuple's hash table and compares the bucket's rules one by
 *   one (§5.1.1); if the predicted tuple(s) hold no match, post-verification
 *   searches the remaining tuples for the highest-priority match.  The result
 *   is the id of the matched rule, or TANG_NO_MATCH.
 *
 * Conventions for every entry point:
 *   - return 0 (TANG_OK) or a negative TANG_E* code; tang_strerror() names it.
 *   - "host" pointers are ordinary (pageable or pinned) CPU memory; "device" pointers
 *     are CUDA global memory on the ctx's device; `stream` is a cudaStream_t passed
 *     as void* (0 = the legacy default stream).
 *   - the caller owns every array it passes; the library copies rules and weights at
 *     build time and never retains caller pointers after a call returns (async calls:
 *     until the work queued on `stream` completes).
 *   - a tang_ctx is bound to one device and is not re-entrant: one host thread at a
 *     time per ctx.  Multi-GPU = one ctx per rank.
 *   - there is NO CPU classification path: a ctx built with device = -1 ("host-only",
 *     used to plan and replicate rule updates) returns TANG_ENODEV from every
 *     classify entry point.
 */
#ifndef TANG_H
#define TANG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque classifier context (tang_build / tang_destroy). */
struct tang_ctx;

#define TANG_OK          0
#define TANG_EINVAL     -1  /* bad argument: length, lo > hi, duplicate id, k out of range */
#define TANG_EMODEL     -2  /* model blob magic/version/dimensions invalid, S != 7        */
#define TANG_ENOTUPLE   -3  /* insert with no candidate tuple (needs a rebuild)     */
#define TANG_ENOENT     -4  /* delete of an unknown rule id                                */
#define TANG_ENOMEM     -5  /* host/device allocation failed or table capacity exhausted  */
#define TANG_ECUDA      -6  /* a CUDA runtime call failed                                  */
#define TANG_ENODEV     -7  /* classify on a host-only ctx, or no CUDA device              */
#define TANG_ESTATE     -8  /* operation not allowed in this ctx state (follower planning) */

#define TANG_NO_MATCH 0xFFFFFFFFu
#define TANG_BLOB_MAGIC 0x474E4154u   /* "TANG" little-endian */
#define TANG_BLOB_VERSION 1u
#define TANG_BLOB_F8_MAGIC 0x53413846u   /* "F8AS": optional fp8 activation-scale trailer */
#define TANG_MAX_TOPK 4

/* Packet header (§2.1; 5-tuple of P:389).  16 bytes, host byte order values. */
typedef struct tang_header {
    uint32_t sip, dip;      /* source / destination IPv4 address                        */
    uint16_t sp, dp;        /* source / destination port                                */
    uint8_t  proto;         /* IP protocol                                              */
    uint8_t  pad[3];        /* ignored                                                  */
} tang_header;

/* Rule (§2.1; Table 1).  32 bytes.
 * Smaller priority value = higher precedence; ties -> smaller id.
 * Prefix host bits are ignored (canonicalised at build).  Ranges inclusive, lo <= hi.
 * Protocol matches when (proto_of_packet & proto_mask) == (proto & proto_mask). */
typedef struct tang_rule {
    uint32_t id, priority;
    uint32_t sip, dip;
    uint16_t sp_lo, sp_hi, dp_lo, dp_hi;
    uint8_t  sip_len, dip_len;      /* prefix lengths 0..32                                */
    uint8_t  proto, proto_mask;
    uint32_t action;
} tang_rule;

/* Build-time configuration.  Zero fields take the defaults in brackets. */
typedef struct tang_config {
    int32_t  device;        /* CUDA device ordinal; -1 = host-only ctx (no classify)     */
    uint32_t mlp;           /* TANG_MLP_BF16_TC (default), TANG_MLP_FP32_FFMA, TANG_MLP_FP8_TC or
                               TANG_MLP_NVFP4_TC                                             */
    uint32_t topk;          /* tuples probed per packet, 1..TANG_MAX_TOPK [1 = paper]     */
    uint32_t mode;          /* TANG_MODE_PAPER [default] or TANG_MODE_STRICT              */
    uint32_t max_batch;     /* max packets per internal launch chunk [1<<20]             */
    uint32_t batch;         /* packets per ring slot of tang_classify() [1<<18]; the first
                               slots of a call ramp up from batch/8 (min 8192) by doubling  */
    uint32_t streams;       /* CUDA streams of tang_classify() [4, as P:453]             */
    uint32_t ring_slots;    /* pinned host ring slots of tang_classify() [2*streams]     */
    uint32_t rule_capacity; /* rule records reserved for inserts beyond the build [n/4+4096] */
    uint32_t mlp_kernel;    /* MLP kernel: TANG_KERNEL_AUTO [0], _SINGLE, _2SM, _WIDE, _DUAL (bf16);
                               AUTO or SINGLE (fp8: SINGLE = the single-tile kernel also for N <= 256) */
    uint32_t reserved[6];
} tang_config;

#define TANG_KERNEL_AUTO   0u   /* the fastest measured variant (2SM for N > 256, else DUAL)      */
#define TANG_KERNEL_SINGLE 1u   /* one CTA per 128-packet tile, full-N accumulator in TMEM; CTAs
                                   run in pairs (2-CTA clusters) sharing the weight stream by TMA
                                   multicast                                                      */
#define TANG_KERNEL_PAIR   2u   /* removed in round 2 (column-split pairs measured slower than 2SM):
                                   tang_build returns TANG_EINVAL                                 */
#define TANG_KERNEL_2SM    3u   /* 2-CTA cluster, M = 256 tcgen05 cta_group::2 MMAs, B split      */
#define TANG_KERNEL_WIDE   4u   /* SINGLE with 16 epilogue warps (4 per TMEM lane quadrant)       */
#define TANG_KERNEL_TS     5u   /* removed in round 2 (GEMM1 / output A operands in TMEM measured
                                   slower than 2SM, profiles/r02_ab_bf16_ts_kernel.txt):
                                   tang_build returns TANG_EINVAL                                 */
#define TANG_KERNEL_DUAL   6u   /* N <= 256: two 128-packet tiles in flight per CTA (one slot's
                                   epilogue overlaps the other's MMAs); AUTO for N <= 256         */

#define TANG_MLP_BF16_TC   0u   /* tcgen05/TMEM bf16 chain, fp32 accumulate (layer 0 fp32) */
#define TANG_MLP_FP32_FFMA 1u   /* fp32 CUDA-core reference chain (the "1e-5 path")          */
#define TANG_MLP_FP8_TC    2u   /* tcgen05 kind::f8f6f4 e4m3 chain (R23):
                                   needs the blob's fp8 trailer and N % 128 == 0, B <= 32         */
#define TANG_MLP_NVFP4_TC  3u   /* tcgen05 kind::mxf4nvf4 NVFP4 chain (R24, f2's NVFP4 stage):
                                   e2m1 codes with e4m3 scales per 16 inputs; needs the fp8 trailer
                                   (the same activation scales), N == 256, C <= 320, B <= 32
                                   (TMEM holds the accumulator and the scale vectors), else
                                   TANG_EMODEL                                                  */
#define TANG_MODE_PAPER    0u   /* scenario 1 left uncorrected, as the paper         */
#define TANG_MODE_STRICT   1u   /* also search tuples that could beat the in-tuple match     */

/* Immediate update (§5.2.1).  40 bytes. */
typedef struct tang_update_op {
    uint8_t   kind;         /* TANG_OP_INSERT or TANG_OP_DELETE                          */
    uint8_t   pad[3];
    uint32_t  id;           /* DELETE: rule id to remove                                  */
    tang_rule rule;         /* INSERT: the new rule (its id must be unused)               */
} tang_update_op;
#define TANG_OP_INSERT 1u
#define TANG_OP_DELETE 2u

typedef struct tang_stats_t {
    uint32_t tuples;         /* C, fixed by the model blob                                */
    uint32_t rules;          /* live rules                                                */
    uint32_t mismatch_count; /* rules placed in a non-exact tuple since build     */
    uint32_t epoch;          /* table epoch, +1 per applied update batch                  */
    uint64_t device_bytes;   /* device memory owned by the ctx                            */
    uint64_t table_bytes;    /* bytes of tuple + slot + rule tables (the L2 working set)  */
    uint32_t slots, keys;    /* hash slots, occupied keys                                 */
    uint32_t S, N, B, C;     /* model dimensions                                          */
    uint64_t checksum;       /* FNV-1a over the host mirror of all device tables          */
    uint32_t live_keys;      /* keys whose bucket holds >= 1 rule (keys - tombstones)      */
    uint32_t delta_rejected; /* delta words the device refused (layout mismatch / out of   *
                              * range, tang_apply_delta_async); reading it synchronises    */
} tang_stats_t;

/* ---------------------------------------------------------------------------------------
 * Build: tuples from the blob, rules placed, tables uploaded, weights converted.
 *   rules[n_rules] (host) -- each placed in its exact-signature tuple, else by restricted
 *       insertion; a rule with no candidate tuple fails the build (TANG_ENOTUPLE).
 *   model_blob (host), blob_len bytes -- little-endian:
 *       u32 magic, version, S, N, B, C;  C x {u8 lsip, u8 ldip} padded to 4 bytes;
 *       f32 W0[S][N], b0[N]; B x { W1[N][N], b1[N], W2[N][N], b2[N] }; Wo[N][C], bo[C]
 *       (weights [in][out], "x.w" of Eq. 1).  Class j of the model = tuple j = signature j.
 *       Optional trailer (required by TANG_MLP_FP8_TC / _NVFP4_TC): u32 TANG_BLOB_F8_MAGIC, u32 2B+1,
 *       i32 e[2B+1] -- the static activation scales 2^e of h0, u_1, h_1, ..., u_B, h_B
 *       (calibration, R23); weight scales are derived at build (per tensor, 2^e).
 *       S must be 7; N a multiple of 64 in [64, 512]; 1 <= C <= 1089 (<= 512 for the
 *       tcgen05 path).
 *   cfg (host, nullable = defaults); *out receives the ctx.
 * -------------------------------------------------------------------------------------*/
int  tang_build(const tang_rule* rules, size_t n_rules, const void* model_blob, size_t blob_len,
                const tang_config* cfg, struct tang_ctx** out);
void tang_destroy(struct tang_ctx* ctx);
const char* tang_strerror(int code);
int  tang_stats(struct tang_ctx* ctx, tang_stats_t* out);

/* ---------------------------------------------------------------------------------------
 * Classify (a1-a9).  rule_id[i] answers hdr[i]; TANG_NO_MATCH when no rule matches.
 * -------------------------------------------------------------------------------------*/
/* Host buffers; blocking.  Streams the batch through the ctx's pinned host rings:
 * H2D of slot r+1, kernels of slot r and D2H of slot r-1 overlap across cfg.streams
 * (the CPU-GPU streaming framework of P:300-306, with the search on the GPU). */
int tang_classify(struct tang_ctx* ctx, const tang_header* hdr, size_t n, uint32_t* rule_id);

/* Device buffers; queued on `stream`, returns without waiting. */
int tang_classify_async(struct tang_ctx* ctx, const tang_header* d_hdr, size_t n,
                        uint32_t* d_rule_id, void* stream);

/* Device buffers with diagnostics, each nullable:
 *   d_pred[n*topk] u32 predicted tuples (descending logit), d_logits[n*C] f32,
 *   d_fellback[n] u8 = 1 when post-verification searched other tuples. */
int tang_classify_ex(struct tang_ctx* ctx, const tang_header* d_hdr, size_t n, uint32_t* d_rule_id,
                     uint32_t* d_pred, float* d_logits, uint8_t* d_fellback, void* stream);

/* Stage 2 only, with externally supplied predictions d_pred[n*k] (device), 0 <= k <= 4.
 * k = 0 searches every tuple, i.e. returns the brute-force highest-priority rule. */
int tang_classify_with_pred(struct tang_ctx* ctx, const tang_header* d_hdr, size_t n,
                            const uint32_t* d_pred, uint32_t k, uint32_t* d_rule_id,
                            uint8_t* d_fellback, void* stream);

/* Step a2 alone: d_feat[n*7] f32 = [SIP_hi, SIP_lo, DIP_hi, DIP_lo, SP, DP, PRO]/65536.
 * (The production path fuses this into the MLP prologue.) */
int tang_encode_async(struct tang_ctx* ctx, const tang_header* d_hdr, size_t n, float* d_feat,
                      void* stream);

/* ---------------------------------------------------------------------------------------
 * Immediate updates (a10).  Updates are ordered after all work previously
 * queued on the ctx's streams and on `stream`; a batch sees table epoch e or e+1, never a mix.
 *   ops[n] (host); status[n] (host, nullable): tuple index for an insert / 0 for a delete,
 *   or a negative TANG_E* per op (failed ops change nothing).  With status != NULL the call
 *   returns TANG_OK and per-op failures are in status; with status == NULL it returns the
 *   first failing op's code (the ops that succeeded are still applied).
 *   Storage: records of relocated or emptied buckets are reused, a key whose bucket empties
 *   becomes a tombstone that a later insert on its probe path reuses, and the slot table is
 *   rehashed from the live keys (or the record pool repacked) when it would otherwise run out,
 *   so sustained insert/delete churn stays within the build's capacity.
 * -------------------------------------------------------------------------------------*/
int tang_update(struct tang_ctx* ctx, const tang_update_op* ops, size_t n, int32_t* status,
                void* stream);

/* Plan only: apply ops to the ctx's host mirror and expose the resulting table delta
 * (*delta, *len; library-owned, valid until the next call on ctx).  Used by the update
 * leader (rank 0), which broadcasts the delta (NCCL over NVLink) to every rank.  Return value
 * and status as tang_update; the delta is produced (and must be applied) either way.
 * The delta starts with a header word carrying a hash of the table layout (region sizes),
 * so it only applies to a ctx built with the same rules, blob and tang_config.rule_capacity. */
int tang_update_plan(struct tang_ctx* ctx, const tang_update_op* ops, size_t n, int32_t* status,
                     const void** delta, size_t* len);

/* Apply a delta produced by tang_update_plan on any ctx built from the same rules, blob and
 * rule_capacity: d_delta (device, len bytes) on `stream`.  Bumps the epoch.  The kernel checks
 * the header's layout hash and every word's region bounds; a mismatching delta writes nothing
 * and out-of-range words are dropped, both counted in tang_stats().delta_rejected. */
int tang_apply_delta_async(struct tang_ctx* ctx, const void* d_delta, size_t len, void* stream);

/* Apply a delta to the host mirror only (followers keep their mirror in step; marks the
 * ctx a follower: tang_update_plan then returns TANG_ESTATE).  TANG_EINVAL (nothing applied)
 * if the layout hash or any word is out of range. */
int tang_apply_delta_host(struct tang_ctx* ctx, const void* delta, size_t len);

/* Deferred update (§5.2.2): replace the model weights after an incremental fine-tune.
 * The blob must keep S, N, B, C and the C tuple signatures (the tuple set is fixed under
 * immediate updates; a changed tuple set is a full rebuild = tang_build).  Blocking:
 * synchronises the ctx, so every batch sees either the old or the new weights.
 * Errors: TANG_EMODEL (dimensions or signatures differ, bad blob). */
int tang_reload_model(struct tang_ctx* ctx, const void* model_blob, size_t blob_len);

/* FNV-1a over the DEVICE copy of the tables (copied back; synchronises the ctx). */
int tang_device_checksum(struct tang_ctx* ctx, uint64_t* out);

/* 64-bit order-independent digest of the DEVICE tables (sum over every 32-bit word of
 * splitmix64(region << 61 | word << 32 | value)), written to *d_digest (device, 8 bytes) on
 * `stream` without synchronising: after each update window, ranks all-gather these 8 bytes to
 * confirm every replica applied the same delta.  TANG_ENODEV host-only. */
int tang_table_digest_async(struct tang_ctx* ctx, uint64_t* d_digest, void* stream);

/* The same digest over the host mirror (leader / followers that keep mirrors). */
int tang_mirror_digest(struct tang_ctx* ctx, uint64_t* out);

/* Test hook: the candidate-tuple mask the post-verification search uses for a packet with these
 * addresses (words[q] bit b = tuple 32q + b may hold a match; a superset of the tuples that hold
 * the packet's key), from the host mirror.  Returns the word count W (fills min(W, cap) words). */
int tang_debug_candidates(struct tang_ctx* ctx, uint32_t sip, uint32_t dip, uint32_t* words, uint32_t cap);

/* Tuple (model class) hosting rule `id`, from the host mirror; TANG_ENOENT if absent. */
int tang_rule_tuple(struct tang_ctx* ctx, uint32_t id, uint32_t* tuple);

/* Per-kernel device time, for the roofline report: while enabled, every kernel the ctx
 * launches is bracketed by CUDA events on its launch stream.  tang_profile_read
 * synchronises, then returns the number of kernel names and fills up to `cap` entries
 * of names (static strings), ms (accumulated milliseconds) and counts (launches) since
 * the last tang_profile_enable.  Every argument array is nullable. */
int tang_profile_enable(struct tang_ctx* ctx, int on);
int tang_profile_read(struct tang_ctx* ctx, const char** names, float* ms, uint64_t* counts, int cap);

/* Test hook of the tcgen05 chains (bf16, fp8 or nvfp4 ctx, else TANG_ESTATE): runs stage 1 alone
 * on n <= max_batch packets and dumps every GEMM input activation, d_act[(2B+1)][n][...]
 * (h0, u_1, h_1, ..., u_B, h_B) as bf16 bits (bf16 ctx, N x 2 B) or e4m3 codes (fp8 ctx, N x 1 B,
 * unscaled) or NVFP4 (nvfp4 ctx, 144 B per row: 128 bytes of e2m1 codes, value 2i in the low
 * nibble of byte i, then the 16 ue4m3 block scales), plus d_pred[n*topk] and d_logits[n*C]
 * (nullable).
 * Lets tests check each layer against the exact result of its own inputs. */
int tang_debug_activations(struct tang_ctx* ctx, const tang_header* d_hdr, size_t n, void* d_act,
                           uint32_t* d_pred, float* d_logits, void* stream);

/* Per-chunk latency (H2D start -> D2H end, ms) of the last tang_classify call; returns the
 * chunk count and fills up to `cap` values. */
int tang_latency_read(struct tang_ctx* ctx, float* ms, int cap);

/* Streaming timeline of the last tang_classify call (Fig. 6: H2D of batch q+1,
 * kernels of q and D2H of q-1 overlap): t[4*q + k] = ms from chunk 0's H2D start to event k of
 * chunk q, k = 0 H2D start, 1 H2D end (kernels start), 2 kernels end (D2H start), 3 D2H end.
 * Returns the chunk count and fills up to `cap` chunks. */
int tang_timeline_read(struct tang_ctx* ctx, float* t, int cap);

#ifdef __cplusplus
}
#endif
#endif /* TANG_H */
