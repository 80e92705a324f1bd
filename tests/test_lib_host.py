"""CPU-side tests of libtang: symbol exports, blob validation, host-only ctx table builder and
update planner (placement against the paper's worked examples), delta replication."""
import ctypes
import os
import re

import numpy as np
import pytest

import tang_inputs as ti
from oracle import tss as otss
from paper_2601_03187_b200 import tang as T, train as TR

C = ctypes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _host_ctx(rules, sigs=None, w=None, **kw):
    sigs = sigs if sigs is not None else TR.tuple_signatures(rules)
    w = w or ti.random_weights(7, 64, 1, len(sigs), seed=0)
    return T.Ctx(rules, T.pack_blob(sigs, w), device=-1, **kw)


def test_every_declared_symbol_is_exported():
    decl = set(re.findall(r"\b(tang_[a-z_]+)\s*\(", open(os.path.join(ROOT, "include", "tang.h")).read()))
    lib = ctypes.CDLL(T.LIB_PATH)
    missing = [d for d in decl if not hasattr(lib, d)]
    assert not missing, missing
    assert set(T.EXPORTED) <= decl


def test_struct_sizes_match_header():
    assert T.HEADER_DTYPE.itemsize == 16 and T.RULE_DTYPE.itemsize == 32 and T.OP_DTYPE.itemsize == 40
    assert ctypes.sizeof(T.tang_config) == 64
    assert (ti.HEADER_DTYPE == T.HEADER_DTYPE) and (ti.RULE_DTYPE == T.RULE_DTYPE)


def test_table1_placement_matches_paper(table1):
    R = ti.table1_rules()
    ctx = _host_ctx(R)
    st = ctx.stats()
    assert st["tuples"] == 5 and st["rules"] == 8 and st["mismatch_count"] == 0
    names = [t[0] for t in table1["tuples"]]
    for j, (_, _, _, members) in enumerate(table1["tuples"]):
        for m in members:
            assert ctx.rule_tuple(int(m[1:])) == j, (m, names[j])
    # R9 -> T1, R10 -> T3 (restricted: mismatch +1)
    r9 = ti.make_rules([dict(id=9, priority=9, sip=0, sip_len=3, dip=0b100 << 29, dip_len=3)])
    r10 = ti.make_rules([dict(id=10, priority=10, sip=0b100 << 29, sip_len=3, dip=0, dip_len=1)])
    st9 = ctx.update(T.make_ops(r9))
    st10 = ctx.update(T.make_ops(r10))
    assert st9.tolist() == [0] and st10.tolist() == [2]
    assert ctx.stats()["mismatch_count"] == 1
    # delete R3: T2 becomes empty, tuple count fixed
    assert ctx.update(T.make_ops(deletes=[3])).tolist() == [0]
    assert ctx.stats()["tuples"] == 5
    with pytest.raises(T.TangError):
        ctx.rule_tuple(3)


def test_no_cpu_classify_path():
    ctx = _host_ctx(ti.table1_rules())
    with pytest.raises(T.TangError) as e:
        ctx.classify(ti.table1_universe())
    assert e.value.code == T.TANG_ENODEV


def test_build_errors():
    R = ti.table1_rules()
    sigs = TR.tuple_signatures(R)
    w = ti.random_weights(7, 64, 1, len(sigs), seed=0)
    blob = T.pack_blob(sigs, w)
    cfg = T.tang_config()
    cfg.device = -1
    for bad in (blob[:-4], b"XXXX" + blob[4:]):
        with pytest.raises(T.TangError) as e:
            T.tang_build(R, bad, cfg)
        assert e.value.code == T.TANG_EMODEL
    dup = R.copy()
    dup["id"][1] = dup["id"][0]
    with pytest.raises(T.TangError) as e:
        T.tang_build(dup, blob, cfg)
    assert e.value.code == T.TANG_EINVAL
    bad = R.copy()
    bad["sp_lo"][0], bad["sp_hi"][0] = 10, 5
    with pytest.raises(T.TangError):
        T.tang_build(bad, blob, cfg)
    # a rule whose lengths admit no tuple: (0, 0) with only (3,3)-style tuples
    only = [(3, 3)]
    w1 = ti.random_weights(7, 64, 1, 1, seed=0)
    with pytest.raises(T.TangError) as e:
        T.tang_build(ti.make_rules([dict(sip_len=0, dip_len=0)]), T.pack_blob(only, w1), cfg)
    assert e.value.code == T.TANG_ENOTUPLE


def test_update_errors_per_op():
    ctx = _host_ctx(ti.table1_rules())
    bad = ti.make_rules([dict(id=1, priority=1, sip=0, sip_len=3, dip=0, dip_len=3)])   # duplicate id 1
    st = ctx.update(T.make_ops(bad, deletes=[77]))
    assert st.tolist() == [T.TANG_ENOENT, T.TANG_EINVAL]


def test_planner_placement_equals_restricted_rule_on_generated_sets():
    """Every inserted rule lands in a tuple with l^T <= l^R of maximal sum, first index
     -- checked against the signatures directly."""
    R = ti.classbench_ruleset("acl", 3000, 21)
    sigs = TR.tuple_signatures(R[:1500])
    ctx = _host_ctx(R[:1500], sigs)
    st = ctx.update(T.make_ops(R[1500:]))
    for r, j in zip(R[1500:], st):
        ls, ld = int(r["sip_len"]), int(r["dip_len"])
        cands = [(a + b, -q) for q, (a, b) in enumerate(sigs) if a <= ls and b <= ld]
        if (ls, ld) in sigs:
            assert j == sigs.index((ls, ld))
        elif not cands:
            assert j == T.TANG_ENOTUPLE
        else:
            assert j == -max(cands)[1]


def test_delta_replicates_to_followers():
    """Leader plans, followers apply the delta to their mirrors: checksums agree."""
    R = ti.classbench_ruleset("fw", 2000, 3)
    sigs = TR.tuple_signatures(R)
    w = ti.random_weights(7, 64, 1, len(sigs), seed=0)
    blob = T.pack_blob(sigs, w)
    lead = T.Ctx(R, blob, device=-1)
    fol = T.Ctx(R, blob, device=-1)
    assert lead.stats()["checksum"] == fol.stats()["checksum"]
    rng = np.random.default_rng(0)
    new = ti.classbench_ruleset("fw", 300, 4)
    new["id"] += 10000
    for step in range(5):
        dels = rng.choice(R["id"][step * 100:(step + 1) * 100], 40, replace=False)
        st, delta = lead.update_plan(T.make_ops(new[step * 60:(step + 1) * 60], deletes=dels))
        assert (st[:40] == 0).all()
        fol.apply_delta_host(delta)
        assert lead.stats()["checksum"] == fol.stats()["checksum"]
    with pytest.raises(T.TangError) as e:
        fol.update_plan(T.make_ops(deletes=[1]))
    assert e.value.code == T.TANG_ESTATE


def test_fp8_blob_trailer_validation():
    """The optional fp8 activation-scale trailer (include/tang.h, R23)."""
    R = ti.table1_rules()
    sigs = TR.tuple_signatures(R)
    w = ti.random_weights(7, 128, 2, len(sigs), seed=0)
    cfg = T.tang_config()
    cfg.device = -1
    cfg.mlp = T.TANG_MLP_FP8_TC
    w["act_exp"] = [0, -1, 1, 2, -3]
    good = T.pack_blob(sigs, w)
    T.tang_destroy(T.tang_build(R, good, cfg))                  # parses (host-only: no upload)
    base = T.pack_blob(sigs, {k: v for k, v in w.items() if k != "act_exp"})
    assert len(good) == len(base) + 8 + 4 * 5
    bad_magic = base + np.array([0x12345678, 5], "<u4").tobytes() + good[-20:]
    bad_count = base + np.array([T.TANG_BLOB_F8_MAGIC, 3], "<u4").tobytes() + good[-20:]
    bad_exp = base + np.array([T.TANG_BLOB_F8_MAGIC, 5], "<u4").tobytes() + np.array([0, 0, 500, 0, 0], "<i4").tobytes()
    for bad in (bad_magic, bad_count, bad_exp, good[:-4], good + b"\0\0\0\0"):
        with pytest.raises(T.TangError) as e:
            T.tang_build(R, bad, cfg)
        assert e.value.code == T.TANG_EMODEL
    with pytest.raises(ValueError):
        T.pack_blob(sigs, dict(w, act_exp=[0, 0]))


def test_fp8_calibration_scale_is_minimal_power_of_two():
    import torch
    from paper_2601_03187_b200 import train as TR
    R = ti.classbench_ruleset("acl", 500, 3)
    sigs = TR.tuple_signatures(R)
    w = ti.random_weights(7, 64, 2, len(sigs), seed=1)
    H = ti.uniform_trace(R, 4096, 2)
    X = TR.features_torch(torch.from_numpy(H.view(np.uint8).copy()))
    ex = TR.calibrate_fp8(w, X)
    assert len(ex) == 5
    # recompute the maxima in float64 and check 448 * 2^(e-1) < max <= 448 * 2^e
    x = X.double().numpy()
    h = np.maximum(x @ np.asarray(w["W0"], np.float64) + w["b0"], 0)
    maxima = [h.max()]
    for i in range(2):
        u = np.maximum(h @ np.asarray(w["W1"][i], np.float64) + w["b1"][i], 0)
        h = np.maximum(u @ np.asarray(w["W2"][i], np.float64) + w["b2"][i] + h, 0)
        maxima += [u.max(), h.max()]
    for m, e in zip(maxima, ex):
        assert 448.0 * 2.0 ** (e - 1) < m * (1 + 1e-5) and m <= 448.0 * 2.0 ** e * (1 + 1e-5)


def _churn_windows(R, windows, size, seed):
    """Windows of `size` deletes of live rules + `size` inserts of new FW-shaped rules with random
    priorities (2,000 deleted + 2,000 inserted per window)."""
    extra = ti.classbench_ruleset("fw", windows * size, seed)
    extra["id"] += 1 << 24
    extra["priority"] = np.random.default_rng(seed).integers(0, R.size, extra.size)
    rng = np.random.default_rng(seed + 1)
    live = list(R["id"])
    for w in range(windows):
        pick = set(rng.choice(len(live), size, replace=False).tolist())
        dels = [live[i] for i in sorted(pick)]
        live = [x for i, x in enumerate(live) if i not in pick]
        ins = extra[w * size:(w + 1) * size]
        live += list(ins["id"])
        yield dels, ins


def test_long_churn_reuses_storage_and_matches_oracle_placement():
    """60 windows of +-400 rules on a 12k-rule set with the build's default headroom: every op
    succeeds (records of relocated / emptied buckets and tombstoned keys are reused, the slot table
    rehashes), a follower replaying the deltas stays byte-identical, and every live rule sits in
    the tuple the oracle's replay of the same sequence puts it in (O4/O5)."""
    R = ti.classbench_ruleset("acl", 12000, 31)
    sigs = otss.signatures_first_occurrence(R)
    blob = T.pack_blob(sigs, ti.random_weights(7, 64, 1, len(sigs), seed=0))
    lead, fol = T.Ctx(R, blob, device=-1), T.Ctx(R, blob, device=-1)
    tss = otss.Tss(sigs, R)
    for dels, ins in _churn_windows(R, 60, 400, 41):
        st, delta = lead.update_plan(T.make_ops(ins, deletes=dels))
        assert (st[:len(dels)] == 0).all()
        ok = st[len(dels):] >= 0
        assert (st[len(dels):][~ok] == T.TANG_ENOTUPLE).all()     # no ENOMEM, only tuple-less rules
        for d in dels:
            assert tss.delete(int(d))
        for r, good in zip(ins, ok):
            if good:
                tss.insert(r)
        fol.apply_delta_host(delta)
    s = lead.stats()
    assert s["rules"] == len(tss.where) and s["checksum"] == fol.stats()["checksum"]
    assert s["live_keys"] == sum(1 for v in tss.buckets.values() if v)
    for rid, key in list(tss.where.items())[::50]:
        assert lead.rule_tuple(rid) == key[0]


def test_delta_layout_hash_rejects_a_foreign_table_shape():
    """A delta only applies to tables of the leader's layout (same rules, blob, rule_capacity)."""
    R = ti.classbench_ruleset("acl", 2000, 5)
    sigs = otss.signatures_first_occurrence(R)
    blob = T.pack_blob(sigs, ti.random_weights(7, 64, 1, len(sigs), seed=0))
    lead = T.Ctx(R, blob, device=-1)
    other = T.Ctx(R, blob, device=-1, rule_capacity=12345)
    _, delta = lead.update_plan(T.make_ops(deletes=[int(R["id"][0])]))
    before = other.stats()["checksum"]
    with pytest.raises(T.TangError) as e:
        other.apply_delta_host(delta)
    assert e.value.code == T.TANG_EINVAL
    assert other.stats()["checksum"] == before and other.stats()["delta_rejected"] > 0


def test_update_without_status_reports_the_first_failure():
    """tang_update_plan with status == NULL returns the first failing op's code; the delta of the
    ops that succeeded is still produced."""
    R = ti.table1_rules()
    ctx = _host_ctx(R)
    ops = T.make_ops(deletes=[1, 77, 2])
    d, n = C.c_void_p(), C.c_size_t()
    rc = T._lib.tang_update_plan(ctx.h, ops.ctypes.data, ops.size, None, C.byref(d), C.byref(n))
    assert rc == T.TANG_ENOENT and n.value > 0
    assert ctx.stats()["rules"] == R.size - 2


@pytest.mark.parametrize("fam,seed", [("acl", 71), ("fw", 72), ("ipc", 73)])
def test_candidate_tuples_cover_every_matching_tuple_under_churn(fam, seed):
    """The post-verification search probes only the candidate tuples of a packet (kRegCand); they
    must include every tuple where the packet's truncated key has rules (a match lives in
    that bucket), at build and after insert/delete windows (deletes may leave extra candidates)."""
    R = ti.classbench_ruleset(fam, 3000, seed)
    sigs = otss.signatures_first_occurrence(R)
    ctx = T.Ctx(R, T.pack_blob(sigs, ti.random_weights(7, 64, 1, len(sigs), seed=0)), device=-1)
    tss = otss.Tss(sigs, R)

    def check(H):
        n_cand = []
        for h in H:
            cand = ctx.candidates(h["sip"], h["dip"])
            need = {j for j in range(len(sigs)) if tss.buckets.get(tss.key_of(j, int(h["sip"]), int(h["dip"])))}
            assert need <= cand, f"tuples {need - cand} hold the packet's key but are not candidates"
            n_cand.append(len(cand))
        return float(np.mean(n_cand))
    mean0 = check(np.concatenate([ti.uniform_trace(R, 400, seed), ti.random_headers(100, seed + 1)]))
    assert mean0 < len(sigs) / 2                                   # the filter actually filters
    for dels, ins in _churn_windows(R, 3, 300, seed + 5):
        st = ctx.update(T.make_ops(ins, deletes=dels))
        for d in dels:
            tss.delete(int(d))
        for r, s_ in zip(ins, st[len(dels):]):
            if s_ >= 0:
                tss.insert(r)
        check(np.concatenate([ti.uniform_trace(ins, 200, seed + 9), ti.uniform_trace(R, 200, seed + 10)]))
