"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(bf16 tcgen05 chain, 1M-packet launches, top-1, paper mode): sampled outputs against the
oracle one by one, and properties checked on every packet.

  configs[3]  512k-rule ACL/FW/IPC         -> test_512k_sampled_parity
  configs[2]  100k ACL uniform vs Zipf     -> test_100k_zipf_sampled_parity
  configs[4]  1M rules + insert/delete     -> test_1m_rules_update_windows
"""
import numpy as np
import pytest

import tang_inputs as ti
from oracle import pipeline as opipe, rules as orules, tss as otss
from tests._helpers import NM, headers_dev, model, require_cuda, u32_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    require_cuda()
    from paper_2601_03187_b200 import tang
    return tang


def _every_packet_properties(R, H, rid):
    """rule_id is NO_MATCH or the id of a rule that matches the packet (all packets)."""
    byid = np.argsort(R["id"])
    ids = R["id"][byid]
    m = rid != NM
    pos = np.searchsorted(ids, rid[m])
    assert (ids[pos] == rid[m]).all(), "rule id not in the ruleset"
    r = R[byid[pos]]
    h = H[m]
    mask = lambda l: np.where(l == 0, 0, (0xFFFFFFFF << (32 - l.astype(np.int64))) & 0xFFFFFFFF)
    ok = ((h["sip"].astype(np.int64) ^ r["sip"]) & mask(r["sip_len"]) == 0) & \
         ((h["dip"].astype(np.int64) ^ r["dip"]) & mask(r["dip_len"]) == 0) & \
         (h["sp"] >= r["sp_lo"]) & (h["sp"] <= r["sp_hi"]) & (h["dp"] >= r["dp_lo"]) & (h["dp"] <= r["dp_hi"]) & \
         ((h["proto"] & r["proto_mask"]) == (r["proto"] & r["proto_mask"]))
    assert ok.all(), f"{(~ok).sum()} packets got a rule that does not match them"


def _run(T, ctx, H):
    torch = require_cuda()
    n = H.size
    d = headers_dev(H)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    pred = torch.empty(n, dtype=torch.int32, device="cuda")
    fell = torch.zeros(n, dtype=torch.uint8, device="cuda")
    ctx.classify_ex(d, out, pred, None, fell)
    torch.cuda.synchronize()
    return u32_host(out), u32_host(pred), fell.cpu().numpy().astype(bool)


@pytest.mark.parametrize("fam,N,B", [(f, 512, 6) for f in ti.FAMILIES] + [("acl", 256, 2)])
def test_512k_sampled_parity(T, fam, N, B):
    """N = 512, B = 6: the paper-size 2SM kernel; N = 256, B = 2: the reduced model's dual-tile kernel."""
    R = ti.classbench_ruleset(fam, 524288, {"acl": 142, "fw": 152, "ipc": 162}[fam])
    H = ti.uniform_trace(R, 3_000_000, 5)
    sigs, w, blob = model(R, N, B, 3)
    ctx = T.Ctx(R, blob, mlp="bf16", max_batch=1 << 20)
    rid, pred, fell = _run(T, ctx, H)
    _every_packet_properties(R, H, rid)
    assert (rid != NM).all()                   # the trace only draws points inside rules
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(H.size, 1500, replace=False))
    tss = otss.Tss(sigs, R)
    want, wfell, _ = opipe.classify_with_pred(tss, H[idx], pred[idx, None], "paper")
    assert int((rid[idx] != want).sum()) == 0
    assert np.array_equal(fell[idx], wfell)
    truth = orules.brute_force(R, H[idx[:300]])
    host = np.array([tss.tuple_of(int(t)) for t in truth])
    G = wfell[:300] | (host == pred[idx[:300]])
    assert int((rid[idx[:300]][G] != truth[G]).sum()) == 0


def test_100k_zipf_sampled_parity(T):
    R = ti.classbench_ruleset("acl", 100000, 141)
    for H in (ti.uniform_trace(R, 2_000_000, 1), ti.zipf_trace(R, 2_000_000, 2)):
        sigs, w, blob = model(R, 256, 2, 4)
        ctx = T.Ctx(R, blob, mlp="bf16")
        rid, pred, fell = _run(T, ctx, H)
        _every_packet_properties(R, H, rid)
        idx = np.random.default_rng(1).choice(H.size, 2000, replace=False)
        tss = otss.Tss(sigs, R)
        want, _, _ = opipe.classify_with_pred(tss, H[idx], pred[idx, None], "paper")
        assert int((rid[idx] != want).sum()) == 0


def test_1m_rules_update_windows(T):
    """configs[4]: 1M-rule ACL, windows of 2,000 deletes + 2,000 inserts applied
    in place; after each window strict mode equals brute force on sampled packets and the
    device tables equal the host mirror."""
    torch = require_cuda()
    R = ti.classbench_ruleset("acl", 1 << 20, 143)
    extra = ti.classbench_ruleset("fw", 8000, 153)
    extra["id"] += 1 << 21
    extra["priority"] = np.random.default_rng(5).integers(0, 1 << 20, extra.size)
    sigs, w, blob = model(R, 256, 2, 6)
    ctx = T.Ctx(R, blob, mlp="bf16", mode="strict")
    live = np.ones(R.size, bool)
    cur_extra = []
    rng = np.random.default_rng(7)
    for win in range(3):
        dels = rng.choice(np.nonzero(live)[0], 2000, replace=False)
        live[dels] = False
        ins = extra[win * 2000:(win + 1) * 2000]
        st = ctx.update(T.make_ops(ins, deletes=R["id"][dels]))
        assert (st[:2000] == 0).all()
        cur_extra.append(ins[st[2000:] >= 0])
        assert ctx.device_checksum() == ctx.stats()["checksum"]
        cur = np.concatenate([R[live]] + cur_extra)
        H = np.concatenate([ti.uniform_trace(cur, 400, win), ti.uniform_trace(ins, 100, win + 10)])
        rid, _, _ = _run(T, ctx, H)
        assert np.array_equal(rid, orules.brute_force(cur, H))
    assert ctx.stats()["epoch"] == 3


def test_256k_long_churn_50_windows(T):
    """P:520-528 churn at scale: 50 windows of 2,000 deletes + 2,000 inserts on a 256k-rule ACL set,
    applied in place through the device deltas.  No op may fail for lack of storage (records and
    tombstoned slots are reused); at the end the device tables equal the host mirror, strict mode
    equals brute force, and paper mode equals the oracle replaying the same sequence (stage 2 on
    the GPU's predictions)."""
    torch = require_cuda()
    R = ti.classbench_ruleset("acl", 1 << 18, 144)
    windows, size = 50, 2000
    extra = ti.classbench_ruleset("fw", windows * size, 154)
    extra["id"] += 1 << 22
    extra["priority"] = np.random.default_rng(6).integers(0, R.size, extra.size)
    sigs, w, blob = model(R, 128, 2, 6)
    strict = T.Ctx(R, blob, mlp="bf16", mode="strict")
    paper = T.Ctx(R, blob, mlp="bf16", mode="paper")
    tss = otss.Tss(sigs, R)
    rng = np.random.default_rng(8)
    live = {int(i): r for i, r in zip(R["id"], R)}
    failed = 0
    for win in range(windows):
        ids = np.fromiter(live.keys(), dtype=np.int64)
        dels = rng.choice(ids, size, replace=False)
        ins = extra[win * size:(win + 1) * size]
        ops = T.make_ops(ins, deletes=dels)
        st = strict.update(ops)
        assert np.array_equal(paper.update(ops), st)
        assert (st[:size] == 0).all()
        assert (st[size:] >= 0).sum() + (st[size:] == T.TANG_ENOTUPLE).sum() == size   # no ENOMEM
        failed += int((st[size:] < 0).sum())
        for d in dels:
            tss.delete(int(d))
            del live[int(d)]
        for r, s in zip(ins, st[size:]):
            if s >= 0:
                tss.insert(r)
                live[int(r["id"])] = r
    for ctx in (strict, paper):
        assert ctx.device_checksum() == ctx.stats()["checksum"]
        assert ctx.stats()["delta_rejected"] == 0 and ctx.stats()["epoch"] == windows
    cur = np.array(list(live.values()), dtype=R.dtype)
    H = np.concatenate([ti.uniform_trace(cur, 1500, 21), ti.uniform_trace(extra[-size:], 500, 22)])
    rid_s, _, _ = _run(T, strict, H)
    assert np.array_equal(rid_s, orules.brute_force(cur, H))
    rid_p, pred_p, fell_p = _run(T, paper, H)
    want, wfell, _ = opipe.classify_with_pred(tss, H, pred_p[:, None], "paper")
    assert np.array_equal(rid_p, want) and np.array_equal(fell_p, wfell)
    print(f"churn: {windows} windows, {failed} inserts without a candidate tuple, "
          f"live keys {strict.stats()['live_keys']} / keys {strict.stats()['keys']}")


def test_512k_headline_trained_model_logits_and_rule_ids(T):
    """The bench's headline configuration: 512k-rule ACL, the committed trained paper-size model
    (models/acl-512k_paper.npz: N=512, B=6, C=300), bf16 chain in bench.py's launch configuration
    (AUTO kernel, 4M-packet launches).  P2: logits element-wise against the oracle's bf16 mode
    (R5) within R6's gate, and the error against the fp32 oracle reported beside it (north_star's
    1e-2); P3: every argmax flip is a near-tie; P4: rule ids equal the oracle's stage 2 on the
    GPU's predictions on >= 100k packets; P5 on a brute-force sample."""
    torch = require_cuda()
    from oracle import mlp as omlp
    from tests._helpers import order_spread
    path = ti.model_path("acl-512k", "paper")
    assert __import__("os").path.exists(path), "committed model missing: run scripts/train_model.py"
    R = ti.classbench_ruleset("acl", 524288, 142)
    sigs, w, meta = ti.load_model(path)
    assert sigs == otss.signatures_first_occurrence(R) and len(sigs) == 300
    blob = T.pack_blob(sigs, w)
    ctx = T.Ctx(R, blob, mlp="bf16", max_batch=1 << 22)
    H = ti.uniform_trace(R, 1 << 22, 1000 + 142 * 10)                 # bench.py's rank-0 trace seed
    rid, pred, fell = _run(T, ctx, H)
    _every_packet_properties(R, H, rid)
    # P2 on 4096 packets (logits are a debug output: a separate call on the same ctx)
    nl = 4096
    out, pl = torch.empty(nl, dtype=torch.int32, device="cuda"), torch.empty(nl, dtype=torch.int32, device="cuda")
    logits = torch.empty(nl * len(sigs), dtype=torch.float32, device="cuda")
    ctx.classify_ex(headers_dev(H[:nl]), out, pl, logits)
    torch.cuda.synchronize()
    L = logits.cpu().numpy().reshape(nl, -1).astype(np.float64)
    x = omlp.features(H[:nl])
    ref = omlp.forward(w, x, "bf16")
    ref32 = omlp.forward(w, x, "fp32")
    err, err32 = float(np.abs(L - ref).max()), float(np.abs(L - ref32).max())
    tol = max(1e-2, 4 * order_spread(w, x))
    print(f"headline logits: max|dlogit| vs bf16 oracle {err:.3e} (gate {tol:.3e}), vs fp32 oracle {err32:.3e}, "
          f"max|logit| {np.abs(ref).max():.1f}; north_star 1e-2 vs fp32 {'holds' if err32 <= 1e-2 else 'does not hold'}")
    assert err <= tol
    # north_star's 1e-2 holds for the bulk of the logits (the maximum is made by bf16 re-rounding
    # flips that propagate through the 13 layers, R6): report the fraction, gate the median
    dl = np.abs(L - ref)
    print(f"headline logits: {np.mean(dl <= 1e-2):.4f} within 1e-2 of the bf16 oracle, median {np.median(dl):.2e}; "
          f"{np.mean(np.abs(L - ref32) <= 1e-2):.4f} within 1e-2 of the fp32 oracle")
    assert np.median(dl) <= 1e-2 and np.mean(dl <= 1e-2) >= 0.95   # measured: 2.7e-5, 0.9878
    assert np.array_equal(u32_host(pl), pred[:nl])                    # same predictions as the full run
    srt = np.sort(ref, axis=1)
    flips = pred[:nl] != omlp.argmax(ref)
    assert np.all((srt[:, -1] - srt[:, -2])[flips] <= 2 * err + 1e-12)
    # P4 on 131072 packets
    n4 = 1 << 17
    tss = otss.Tss(sigs, R)
    want, wfell, _ = opipe.classify_with_pred(tss, H[:n4], pred[:n4, None], "paper")
    assert int((rid[:n4] != want).sum()) == 0 and np.array_equal(fell[:n4], wfell)
    # P5 on 512 packets against the brute force
    truth = orules.brute_force(R, H[:512])
    host = np.array([tss.tuple_of(int(t)) for t in truth])
    G = wfell[:512] | (host == pred[:512])
    assert int((rid[:512][G] != truth[G]).sum()) == 0
    print(f"headline: fallback rate {fell.mean():.4f}, model accuracy on the P5 sample {np.mean(host == pred[:512]):.4f}")
