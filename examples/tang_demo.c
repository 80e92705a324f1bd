/* Plain-C use of the libtang ABI (include/tang.h), no Python involved.
 *
 * Builds the 8-rule classifier of the paper's Table 1 (two 3-bit fields X, Y,
 * embedded here as the top 3 bits of SIP and DIP), packs a model blob by hand (the layout
 * documented at tang_build), and
 *   host  (default, no GPU needed): builds a host-only ctx, reads its stats, plans an update
 *         (insert + delete) and checks that classification is refused with TANG_ENODEV;
 *   gpu   (argv[1] == "gpu"): builds on device 0 in strict mode (TANG_MODE_STRICT: the result is
 *         the highest-priority matching rule whatever the model predicts) and classifies all 64
 *         points of the X x Y universe through tang_classify, comparing every answer with a
 *         brute-force scan written here.
 * Exit status 0 on success.
 * Build: gcc -O2 -I include examples/tang_demo.c -L paper_2601_03187_b200 -ltang \
 *            -Wl,-rpath,$PWD/paper_2601_03187_b200 -o tang_demo */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tang.h"

static const struct { const char* name; uint32_t prio; const char *x, *y; } kTable1[8] = {
    {"R1", 1, "000", "011"}, {"R2", 2, "000", "101"}, {"R3", 3, "00*", "11*"}, {"R4", 4, "110", "***"},
    {"R5", 5, "111", "***"}, {"R6", 6, "***", "011"}, {"R7", 7, "***", "010"}, {"R8", 8, "0**", "0**"}};

/* "01*" -> value << 29 and the prefix length (the number of non-'*' bits) */
static void bits3(const char* pat, uint32_t* value, uint8_t* len) {
    uint32_t v = 0;
    uint8_t l = 0;
    for (int b = 0; b < 3; ++b) {
        v = (v << 1) | (pat[b] == '1');
        if (pat[b] != '*') ++l;
    }
    *value = v << 29;
    *len = l;
}

static int matches(const tang_rule* r, const tang_header* h) {
    const uint32_t ms = r->sip_len ? 0xFFFFFFFFu << (32 - r->sip_len) : 0u;
    const uint32_t md = r->dip_len ? 0xFFFFFFFFu << (32 - r->dip_len) : 0u;
    return ((h->sip ^ r->sip) & ms) == 0 && ((h->dip ^ r->dip) & md) == 0 && h->sp >= r->sp_lo &&
           h->sp <= r->sp_hi && h->dp >= r->dp_lo && h->dp <= r->dp_hi &&
           ((h->proto ^ r->proto) & r->proto_mask) == 0;
}

/* highest-priority (smallest priority, then smallest id) matching rule, TANG_NO_MATCH if none */
static uint32_t brute_force(const tang_rule* rules, int n, const tang_header* h) {
    int best = -1;
    for (int i = 0; i < n; ++i)
        if (matches(&rules[i], h) &&
            (best < 0 || rules[i].priority < rules[best].priority ||
             (rules[i].priority == rules[best].priority && rules[i].id < rules[best].id)))
            best = i;
    return best < 0 ? TANG_NO_MATCH : rules[best].id;
}

/* model blob: magic, version, S, N, B, C; C signatures; W0, b0; B x {W1, b1, W2, b2}; Wo, bo */
static uint8_t* pack_blob(const uint8_t (*sig)[2], uint32_t C, uint32_t N, uint32_t B, size_t* len) {
    const uint32_t S = 7;
    const size_t nf = (size_t)S * N + N + (size_t)B * (2 * (size_t)N * N + 2 * N) + (size_t)N * C + C;
    const size_t sig_bytes = (2 * C + 3) & ~(size_t)3;
    *len = 24 + sig_bytes + 4 * nf;
    uint8_t* blob = calloc(1, *len);
    const uint32_t head[6] = {TANG_BLOB_MAGIC, TANG_BLOB_VERSION, S, N, B, C};
    memcpy(blob, head, sizeof head);
    for (uint32_t j = 0; j < C; ++j) { blob[24 + 2 * j] = sig[j][0]; blob[24 + 2 * j + 1] = sig[j][1]; }
    float* w = (float*)(blob + 24 + sig_bytes);
    uint32_t state = 12345u;                       /* small deterministic pseudo-random weights */
    for (size_t i = 0; i < nf; ++i) {
        state = state * 1664525u + 1013904223u;
        w[i] = ((float)(state >> 8) / 16777216.0f - 0.5f) * 0.25f;
    }
    return blob;
}

static int check(int e, const char* what) {
    if (e != TANG_OK) fprintf(stderr, "%s: %s (%d)\n", what, tang_strerror(e), e);
    return e;
}

int main(int argc, char** argv) {
    const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
    tang_rule rules[8];
    memset(rules, 0, sizeof rules);
    for (int i = 0; i < 8; ++i) {
        rules[i].id = (uint32_t)(i + 1);
        rules[i].priority = kTable1[i].prio;
        bits3(kTable1[i].x, &rules[i].sip, &rules[i].sip_len);
        bits3(kTable1[i].y, &rules[i].dip, &rules[i].dip_len);
        rules[i].sp_hi = 0xFFFF;
        rules[i].dp_hi = 0xFFFF;
        rules[i].action = (uint32_t)i;
    }
    /* model classes = tuple signatures (lsip, ldip) in first-occurrence order (R10) */
    uint8_t sig[8][2];
    uint32_t C = 0;
    for (int i = 0; i < 8; ++i) {
        uint32_t j = 0;
        while (j < C && !(sig[j][0] == rules[i].sip_len && sig[j][1] == rules[i].dip_len)) ++j;
        if (j == C) { sig[C][0] = rules[i].sip_len; sig[C][1] = rules[i].dip_len; ++C; }
    }
    size_t blob_len = 0;
    uint8_t* blob = pack_blob((const uint8_t(*)[2])sig, C, 64, 1, &blob_len);

    tang_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.device = gpu ? 0 : -1;
    cfg.mode = TANG_MODE_STRICT;
    struct tang_ctx* ctx = NULL;
    if (check(tang_build(rules, 8, blob, blob_len, &cfg, &ctx), "tang_build")) return 1;
    tang_stats_t st;
    if (check(tang_stats(ctx, &st), "tang_stats")) return 1;
    printf("built: %u rules in %u tuples (model S=%u N=%u B=%u C=%u)\n", st.rules, st.tuples, st.S, st.N, st.B,
           st.C);
    if (st.rules != 8 || st.tuples != C) return 1;

    tang_header pts[64];
    memset(pts, 0, sizeof pts);
    for (uint32_t x = 0; x < 8; ++x)
        for (uint32_t y = 0; y < 8; ++y) { pts[8 * x + y].sip = x << 29; pts[8 * x + y].dip = y << 29; }
    uint32_t got[64];
    int bad = 0;
    if (!gpu) {
        /* host-only ctx: updates are planned on the host mirror, classification is refused */
        tang_update_op ops[2];
        memset(ops, 0, sizeof ops);
        ops[0].kind = TANG_OP_DELETE;
        ops[0].id = 8;
        ops[1].kind = TANG_OP_INSERT;
        ops[1].rule = rules[7];
        ops[1].rule.id = 100;
        ops[1].rule.priority = 9;
        int32_t status[2];
        if (check(tang_update(ctx, ops, 2, status, NULL), "tang_update")) return 1;
        if (check(tang_stats(ctx, &st), "tang_stats")) return 1;
        printf("after update: %u rules, epoch %u, status %d %d\n", st.rules, st.epoch, status[0], status[1]);
        if (st.rules != 8 || status[0] < 0 || status[1] < 0) return 1;
        const int e = tang_classify(ctx, pts, 64, got);
        printf("classify on a host-only ctx: %s\n", tang_strerror(e));
        bad = e != TANG_ENODEV;
    } else {
        if (check(tang_classify(ctx, pts, 64, got), "tang_classify")) return 1;
        for (int i = 0; i < 64; ++i) bad += got[i] != brute_force(rules, 8, &pts[i]);
        printf("classified the 64 points of Table 1's universe: %d mismatches against the brute-force scan\n", bad);
    }
    tang_destroy(ctx);
    free(blob);
    return bad ? 1 : 0;
}
