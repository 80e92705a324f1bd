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


@pytest.mark.parametrize("fam", ti.FAMILIES)
def test_512k_sampled_parity(T, fam):
    R = ti.classbench_ruleset(fam, 524288, {"acl": 142, "fw": 152, "ipc": 162}[fam])
    H = ti.uniform_trace(R, 3_000_000, 5)
    sigs, w, blob = model(R, 512, 6, 3)
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
