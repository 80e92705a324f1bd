"""Pins of the oracle's bf16 mode: WHERE the quantisation points sit (R5, reading 5 of
SURVEY.md §8(c); "precision quantization", Eq. 1).

R5: W1, W2, Wo rounded to bf16 (RNE) once; layer 0 fp32; h0, u and h rounded to fp32 (the
accumulator) and then to bf16 as GEMM inputs; bias, skip-add and ReLU applied in fp32 before the
rounding; the skip adds the *rounded* block input hq.

Three kinds of evidence, none of which re-calls the oracle's own rounding helper:
  1. an independent torch implementation whose only rounding primitive is torch's own
     `.to(torch.bfloat16)` / `.float()` casts, placed at R5's points -> element-wise equality;
  2. mutation check: each plausible slip (unrounded skip, rounding before the bias, unrounded u,
     unrounded weights, no final rounding, bf16 layer 0, skip from h0, missing ReLU after the
     add) implemented in the same torch reference moves the logits well beyond the tolerance of
     (1), so (1) would catch it;
  3. a hand-derived network (dyadic values, exact by hand) where only R5's skip rounding gives
     the printed logit.
"""
import numpy as np
import pytest
import torch

import tang_inputs as ti
from oracle import mlp

D = torch.float64


def _ref(w, x, *, skip_rounded=True, bias_before_round=True, round_u=True, round_w=True, round_final=True,
         bf16_layer0=False, skip_from_h0=False, relu_after_add=True):
    """bf16-emulated forward in torch; the defaults are R5.  Sums of bf16 products are formed in
    float64 and rounded once to fp32 (`.float()`), as the GPU's fp32 accumulator does up to order."""
    t = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float32))
    bf = lambda a: a.float().to(torch.bfloat16).to(D)              # fp32 -> bf16 (RNE) -> exact in f64
    f32 = lambda a: a.float().to(D)                               # round to fp32
    qw = (lambda a: bf(t(a))) if round_w else (lambda a: t(a).to(D))
    X = t(x).to(D)
    if bf16_layer0:
        h = torch.relu(f32(bf(X) @ bf(t(w["W0"]))) + t(w["b0"]).to(D))
    else:
        h = torch.relu(X @ t(w["W0"]).to(D) + t(w["b0"]).to(D))
    h0q = bf(f32(h))
    for i in range(int(w["B"])):
        hq = bf(f32(h))
        mm = f32(hq @ qw(w["W1"][i]))
        b1 = t(w["b1"][i]).to(D)
        u = torch.relu(f32(mm + b1)) if bias_before_round else torch.relu(bf(mm) + b1)
        uq = bf(f32(u)) if (round_u and bias_before_round) else (f32(u) if not round_u else u)
        skip = h0q if skip_from_h0 else (hq if skip_rounded else f32(h))
        z = f32(uq @ qw(w["W2"][i])) + t(w["b2"][i]).to(D) + skip
        h = torch.relu(z) if relu_after_add else z
    hq = bf(f32(h)) if round_final else f32(h)
    return (f32(hq @ qw(w["Wo"])) + t(w["bo"]).to(D)).numpy()


def _nets():
    for S, N, B, C, seed in ((7, 64, 2, 9, 5), (7, 128, 3, 33, 6), (7, 48, 1, 5, 7)):
        w = ti.random_weights(S, N, B, C, seed=seed, gain=1.0)
        x = mlp.features(np.concatenate([ti.random_headers(300, seed + 10),
                                         ti.uniform_trace(ti.classbench_ruleset("acl", 300, seed), 300, seed)]))
        yield w, x


@pytest.mark.parametrize("k", range(3))
def test_bf16_mode_equals_independent_torch_reference(k):
    w, x = list(_nets())[k]
    got = mlp.forward(w, x, "bf16")
    ref = _ref(w, x)
    d = np.abs(got - ref)
    # both sides form the same float64 sums of bf16 products; BLAS blocking may change the last
    # float64 bits, which can move an fp32 rounding (then at most one bf16 flip downstream)
    assert d.max() <= 1e-6 * max(1.0, float(np.abs(ref).max()))
    assert (got == ref).mean() >= 0.999


MUTANTS = {
    "unrounded skip": dict(skip_rounded=False),
    "rounding before the bias": dict(bias_before_round=False),
    "u not rounded": dict(round_u=False),
    "weights not rounded": dict(round_w=False),
    "no rounding before the output FC": dict(round_final=False),
    "layer 0 in bf16": dict(bf16_layer0=True),
    "skip from h0": dict(skip_from_h0=True),
    "no ReLU after the add": dict(relu_after_add=False),
}


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_each_plausible_slip_is_detected(name):
    """Every mutant of R5 lands far outside the equality test's tolerance on some pinned net."""
    worst = 0.0
    for w, x in _nets():
        ref = _ref(w, x)
        worst = max(worst, float(np.abs(_ref(w, x, **MUTANTS[name]) - ref).max()) /
                    max(1.0, float(np.abs(ref).max())))
    assert worst > 1e-3, f"mutant '{name}' is indistinguishable ({worst:.2e})"


def test_hand_network_skip_adds_the_rounded_block_input():
    """S = N = C = 1, B = 1, x = 1.  bf16 has 8 significant bits: on [1, 2) the grid step is 2^-7.
         h0 = ReLU(1*1 + 3*2^-9)           = 1 + 3*2^-9            (fp32, layer 0 is not rounded)
         hq = bf16(h0)                     = 1 + 2^-7              (3*2^-9 is nearer 4*2^-9 than 0)
         u  = ReLU(hq*0 + 0) = 0,  uq = 0
         h  = ReLU(uq*0 + (-2^-9) + hq)    = 1 + 3*2^-9
         logit = bf16(h)*1 + 0             = 1 + 2^-7 = 1.0078125
       With the unrounded skip h0 instead, h = 1 + 2^-8, a tie that rounds to even: logit 1.0;
       the fp32 network gives 1 + 2^-8 = 1.00390625."""
    f = lambda *v: np.array(v, np.float32).reshape(1, -1)
    w = dict(S=1, N=1, B=1, C=1, W0=f(1.0), b0=np.array([3 * 2.0 ** -9], np.float32),
             W1=[f(0.0)], b1=[np.zeros(1, np.float32)], W2=[f(0.0)], b2=[np.array([-2.0 ** -9], np.float32)],
             Wo=f(1.0), bo=np.zeros(1, np.float32))
    x = np.ones((1, 1), np.float32)
    assert mlp.forward(w, x, "bf16")[0, 0] == 1.0078125
    assert mlp.forward(w, x, "fp32")[0, 0] == 1.00390625
    assert _ref(w, x)[0, 0] == 1.0078125 and _ref(w, x, skip_rounded=False)[0, 0] == 1.0
