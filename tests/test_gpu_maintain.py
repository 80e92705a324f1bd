"""Deferred update on the GPU (§7.3 dynamic scenario): immediate updates drift the
tuple boundaries, an incremental fine-tune on GPU-labelled fresh traffic is hot-swapped with
tang_reload_model, model accuracy recovers, and stage 2 stays bit-exact with the oracle."""
import numpy as np
import pytest

import tang_inputs as ti
from oracle import pipeline as opipe, tss as otss
from tests._helpers import headers_dev, require_cuda, u32_host

pytestmark = pytest.mark.gpu


def test_incremental_update_recovers_accuracy():
    torch = require_cuda()
    from paper_2601_03187_b200 import maintain as M, tang as T, train as TR
    R = ti.classbench_ruleset("acl", 10000, 140)
    sigs = otss.signatures_first_occurrence(R)
    tr = torch.from_numpy(ti.uniform_trace(R, 1 << 19, 7).view(np.uint8).copy()).cuda()
    lab_ctx = T.Ctx(R, T.pack_blob(sigs, ti.random_weights(7, 64, 1, len(sigs), 0)), mlp="fp32")
    w, _ = TR.train(R, sigs, 256, 2, tr, TR.gpu_labels(lab_ctx, tr, R, sigs), seconds=12.0)
    ctx = T.Ctx(R, T.pack_blob(sigs, w), mlp="bf16")
    tss = otss.Tss(sigs, R)

    # churn: delete 30 % of the rules, insert as many drawn from another family (restricted inserts)
    rng = np.random.default_rng(3)
    dels = rng.choice(R["id"], 3000, replace=False)
    ins = ti.classbench_ruleset("ipc", 3000, 77)
    ins["id"] += 1 << 20
    ins["priority"] = rng.integers(0, R.size, ins.size)
    st = ctx.update(T.make_ops(ins, deletes=dels))
    for d in dels:
        tss.delete(int(d))
    live = {int(r["id"]): r for r in R if int(r["id"]) not in set(dels.tolist())}
    for r, s in zip(ins, st[3000:]):
        if s >= 0:
            tss.insert(r)
            live[int(r["id"])] = r
    cur = np.array(list(live.values()), dtype=ti.RULE_DTYPE)
    assert ctx.stats()["mismatch_count"] > 0

    fresh = torch.from_numpy(ti.uniform_trace(cur, 1 << 19, 9).view(np.uint8).copy()).cuda()
    n = fresh.numel() // 16

    def model_acc():
        lab = TR.gpu_labels(ctx, fresh, cur, sigs, placed=True)
        pred = torch.empty(n, dtype=torch.int32, device="cuda")
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        ctx.classify_ex(fresh, out, pred)
        torch.cuda.synchronize()
        m = lab >= 0
        return float((pred.long()[m] == lab[m]).float().mean()), pred, out

    before, _, _ = model_acc()
    eng = M.UpdateEngine(tau=0.05, theta=10 ** 9)
    assert eng.observe(100.0, 0, cur.size) == "none"
    assert eng.observe(80.0, ctx.stats()["mismatch_count"], cur.size) == "incremental"
    M.incremental_update(ctx, cur, sigs, w, fresh, seconds=12.0)
    after, pred, out = model_acc()
    assert after > before, (before, after)

    # stage 2 after the hot swap: bit-exact with the oracle replaying the same updates
    idx = np.random.default_rng(5).choice(n, 1500, replace=False)
    H = fresh.cpu().numpy().view(ti.HEADER_DTYPE)[idx]
    gp = u32_host(pred)[idx]
    want, _, _ = opipe.classify_with_pred(tss, H, gp[:, None], "paper")
    assert int((u32_host(out)[idx] != want).sum()) == 0


def test_reload_same_weights_is_identity():
    torch = require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset("fw", 2000, 5)
    sigs = otss.signatures_first_occurrence(R)
    blob = T.pack_blob(sigs, ti.random_weights(7, 128, 2, len(sigs), 4))
    ctx = T.Ctx(R, blob, mlp="bf16")
    H = headers_dev(ti.uniform_trace(R, 20000, 1))
    a = torch.empty(20000, dtype=torch.int32, device="cuda")
    b = torch.empty_like(a)
    ctx.classify_async(H, a)
    ctx.reload_model(blob)
    ctx.classify_async(H, b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
