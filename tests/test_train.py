"""Host-side pins of the plain trainer (setup, off the hot path): class order, labels, the
alpha x10 retrain round (§6.2) and the committed-model format."""
import numpy as np
import torch

import tang_inputs as ti
from oracle import rules as orules, tss as otss
from paper_2601_03187_b200 import train as TR


def test_tuple_signatures_equal_oracle_first_occurrence():
    """The class order the trainer writes into the blob is the oracle's O3."""
    for fam, n, seed in (("acl", 2000, 1), ("fw", 2000, 2), ("ipc", 2000, 3)):
        R = ti.classbench_ruleset(fam, n, seed)
        assert TR.tuple_signatures(R) == otss.signatures_first_occurrence(R)
    R = ti.table1_rules()
    assert TR.tuple_signatures(R) == otss.signatures_first_occurrence(R)


def test_torch_labels_equal_brute_force_winner_tuple():
    """the label is the tuple of the highest-priority matching rule (O2), -1 if none."""
    R = ti.classbench_ruleset("acl", 1000, 101)
    H = np.concatenate([ti.uniform_trace(R, 2000, 5), ti.random_headers(500, 6)])
    sigs = otss.signatures_first_occurrence(R)
    got = TR.torch_labels(R, sigs, torch.from_numpy(H.view(np.uint8).copy()), chunk=97).numpy()
    truth = orules.brute_force(R, H)
    idx = {s: j for j, s in enumerate(sigs)}
    by_id = {int(r["id"]): idx[(int(r["sip_len"]), int(r["dip_len"]))] for r in R}
    want = np.array([by_id[int(t)] if t != orules.NO_MATCH else -1 for t in truth])
    assert (want == -1).any() and (want >= 0).any()
    assert np.array_equal(got, want)


def test_alpha_times_ten_round_is_reachable():
    """when the accuracy stays below beta, alpha grows x10 and the model is retrained."""
    R = ti.classbench_ruleset("acl", 200, 7)
    H = ti.uniform_trace(R, 4096, 8)
    sigs = TR.tuple_signatures(R)
    d = torch.from_numpy(H.view(np.uint8).copy())
    lab = TR.torch_labels(R, sigs, d)
    msgs = []
    TR.train(R, sigs, 16, 1, d, lab, seconds=12.0, alpha=10, beta=2.0, batch=256, log=msgs.append)
    assert len(msgs) == 2 and "alpha=10 " in msgs[0] and "alpha=100 " in msgs[1]


def test_model_file_roundtrip(tmp_path):
    w = ti.random_weights(7, 64, 2, 9, seed=3)
    sigs = [(i, 32 - i) for i in range(9)]
    wb = TR.round_weights_bf16(w)
    ti.save_model(str(tmp_path / "m.npz"), sigs, wb, {"k": 1})
    s2, w2, meta = ti.load_model(str(tmp_path / "m.npz"))
    assert s2 == sigs and meta == {"k": 1}
    bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy()
    assert np.array_equal(w2["W0"], w["W0"]) and np.array_equal(w2["bo"], w["bo"])
    for i in range(2):
        assert np.array_equal(w2["W1"][i], bf(w["W1"][i])) and np.array_equal(w2["b2"][i], w["b2"][i])
    assert np.array_equal(w2["Wo"], bf(w["Wo"]))


def test_nvfp4_fake_quant_matches_the_oracle_grid():
    """The trainer's NVFP4 fake quantisation (QAT, R24) lands on the oracle's NVFP4 values
    (codes x block scales) except where a value sits exactly on an e2m1 rounding midpoint (the trainer
    rounds those down, the oracle to even); the power-of-two tensor scale is applied exactly."""
    from oracle import mlp as omlp
    rng = np.random.default_rng(3)
    v = rng.normal(0, 1, (64, 256)).astype(np.float32) * 5
    for e in (0, -3, 4):
        got = TR.nvfp4_fake(torch.from_numpy(v), e).numpy().astype(np.float64)
        ref = omlp.nvfp4_values(v.astype(np.float64) / 2.0 ** e) * 2.0 ** e
        assert np.mean(got == ref) > 0.999, (e, np.mean(got == ref))
    # a value on a midpoint: 0.75 x sf rounds down here, to even (1.0) in the oracle
    blk = np.zeros((1, 16), np.float32)
    blk[0, 0], blk[0, 1] = 6.0, 0.75                     # sf = 1
    assert TR.nvfp4_fake(torch.from_numpy(blk), 0).numpy()[0, 1] == 0.5
    assert omlp.nvfp4_values(blk.astype(np.float64))[0, 1] == 1.0


def test_qat_forward_runs_and_trains():
    """The quantisation-aware forward is differentiable (straight-through) and lowers the loss."""
    torch.manual_seed(0)
    m = TR.TangMLP(7, 32, 1, 5)
    x = torch.rand(512, 7)
    y = torch.randint(0, 5, (512,))
    ae = [0, 0, 0]
    opt = torch.optim.Adam(m.parameters(), lr=1e-2)
    first = None
    for _ in range(60):
        loss = torch.nn.functional.cross_entropy(m(x, ae), y)
        first = float(loss) if first is None else first
        opt.zero_grad()
        loss.backward()
        opt.step()
    assert float(loss) < first
