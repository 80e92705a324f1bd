"""Pins for the oracle's fp8 mode (§8(f) row f2; R23).  Each pin is fixed by the
number format or by hand arithmetic, not by re-running the oracle's own formulas:
  * the e4m3 value set decoded independently from its bit fields (exhaustive),
  * ties-to-even / saturation / subnormal cases worked by hand,
  * torch's float8_e4m3fn conversion as an independent implementation (in range),
  * the power-of-two scale is the minimal one (checked by its defining inequality),
  * a hand-computed 2-2-2 network through one residual block,
  * networks whose every intermediate is e4m3-representable reduce to the exact forward."""
import numpy as np
import pytest

from oracle import mlp as omlp


def e4m3_table():
    """All finite e4m3fn values from the bit layout s.eeee.mmm, bias 7 (e=15, m=7 is NaN)."""
    vals = []
    for code in range(256):
        s, e, m = code >> 7, (code >> 3) & 15, code & 7
        if e == 15 and m == 7:
            continue
        v = (m / 8.0) * 2.0 ** -6 if e == 0 else (1 + m / 8.0) * 2.0 ** (e - 7)
        vals.append(-v if s else v)
    return np.unique(np.array(vals))


def test_table_and_identity():
    t = e4m3_table()
    assert t.max() == 448.0 and t.min() == -448.0 and 2.0 ** -9 in t
    assert np.array_equal(omlp.to_e4m3(t), t)


def test_rounds_to_nearest_table_value_ties_to_even():
    t = e4m3_table()
    rng = np.random.default_rng(8)
    x = rng.uniform(-460, 460, 200000) * 10.0 ** rng.integers(-4, 1, 200000)
    q = omlp.to_e4m3(x)
    assert np.isin(q, t).all()
    # nearest: no table value strictly closer
    idx = np.clip(np.searchsorted(t, x), 1, t.size - 1)
    best = np.minimum(np.abs(t[idx] - x), np.abs(t[idx - 1] - x))
    inr = np.abs(x) <= 448
    assert np.all(np.abs(q - x)[inr] <= best[inr])
    # midpoints go to the even mantissa (hand-worked)
    assert omlp.to_e4m3(1.0625) == 1.0 and omlp.to_e4m3(1.1875) == 1.25
    assert omlp.to_e4m3(2.0 ** -10) == 0.0 and omlp.to_e4m3(3 * 2.0 ** -10) == 2.0 ** -8
    assert omlp.to_e4m3(-3.3) == -3.25
    # saturation (satfinite) and the top binade
    assert omlp.to_e4m3(464.0) == 448.0 and omlp.to_e4m3(1e30) == 448.0 and omlp.to_e4m3(-1e30) == -448.0
    assert omlp.to_e4m3(431.9) == 416.0 and omlp.to_e4m3(440.0) == 448.0


def test_matches_torch_float8_in_range():
    torch = pytest.importorskip("torch")
    if not hasattr(torch, "float8_e4m3fn"):
        pytest.skip("no float8 in this torch")
    rng = np.random.default_rng(9)
    x = (rng.standard_normal(100000) * 10.0 ** rng.integers(-3, 3, 100000)).astype(np.float32)
    x = x[np.abs(x) <= 448]
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).to(torch.float64).numpy()
    assert np.array_equal(omlp.to_e4m3(x.astype(np.float64)), ref)


def test_pow2_scale_is_minimal():
    rng = np.random.default_rng(10)
    a = np.concatenate([rng.uniform(0, 1, 5000) * 10.0 ** rng.integers(-30, 30, 5000),
                        [448.0, 449.0, 896.0, 224.0, 448.0 * 2.0 ** -20]])
    e = omlp.pow2_scale_exp(a)
    assert np.all(a <= 448.0 * np.ldexp(1.0, e))
    assert np.all(a > 448.0 * np.ldexp(1.0, e - 1))
    assert omlp.pow2_scale_exp(0.0) == 0


def _net(N, B, C):
    return {"S": 7, "N": N, "B": B, "C": C}


def test_hand_computed_block():
    """N = 2, B = 1, C = 2, worked by hand (values in the comments)."""
    w = _net(2, 1, 2)
    w["W0"] = np.zeros((7, 2)); w["b0"] = np.array([1.1, 0.3])          # h0 = [1.1, 0.3]
    w["W1"] = np.array([np.eye(2)]); w["b1"] = np.zeros((1, 2))
    w["W2"] = np.array([0.5 * np.eye(2)]); w["b2"] = np.zeros((1, 2))
    w["Wo"] = np.array([[1.0, -1.0], [2.0, 0.0]]); w["bo"] = np.array([0.1, 0.0])
    w["act_exp"] = [0, -1, 0]
    # hq = q(h0 / 1) = [1.125, 0.3125]; W1 = I: s_w1 = 2^-8 (1 <= 1.75), W1q = 256 I
    # u = hq -> q(u / 0.5) = [2.25, 0.625]
    # W2 = I/2: s_w2 = 2^-9, W2q = 256 I; uq.W2q * (0.5 * 2^-9) = [0.5625, 0.15625]; + hq = [1.6875, 0.46875]
    # q(1.6875) = 1.75 (13.5 eighths -> 14, ties to even); q(0.46875) = 0.46875
    # Wo: max 2 -> s_wo = 2^-7, Woq = [[128, -128], [256, 0]] (exact)
    # logits: [1.75 * 1 + 0.46875 * 2 + 0.1, 1.75 * -1] = [2.7875, -1.75]
    dump = []
    got = omlp.forward_fp8(w, np.zeros((1, 7), np.float32), dump)
    assert np.array_equal(dump[0][0], [1.125, 0.3125])
    assert np.array_equal(dump[1][0], [2.25, 0.625])
    assert np.array_equal(dump[2][0], [1.75, 0.46875])
    assert np.allclose(got[0], [2.7875, -1.75], rtol=0, atol=1e-15)


def test_representable_network_reduces_to_exact_forward():
    """If every weight and activation is already an e4m3 multiple of its scale, quantisation
    is the identity and fp8 mode must equal the exact (fp32-mode, float64) forward."""
    rng = np.random.default_rng(11)
    found = 0
    for trial in range(400):
        N, B, C = 4, 2, 3
        w = _net(N, B, C)
        w["W0"] = np.zeros((7, N)); w["b0"] = rng.integers(0, 4, N).astype(np.float64)
        w["W1"] = rng.integers(-1, 2, (B, N, N)).astype(np.float64); w["b1"] = rng.integers(-1, 2, (B, N)) * 1.0
        w["W2"] = rng.integers(-1, 2, (B, N, N)).astype(np.float64); w["b2"] = rng.integers(-1, 2, (B, N)) * 1.0
        w["Wo"] = rng.integers(-2, 3, (N, C)).astype(np.float64); w["bo"] = rng.standard_normal(C)
        x = np.zeros((1, 7), np.float32)
        ref = omlp.forward(w, x, "fp32")
        # scales: 2^0 everywhere; check representability of the exact intermediates
        h = omlp.relu(w["b0"])
        ok = np.array_equal(omlp.to_e4m3(h), h)
        for i in range(B):
            u = omlp.relu(h @ w["W1"][i] + w["b1"][i])
            h = omlp.relu(u @ w["W2"][i] + w["b2"][i] + h)
            ok &= np.array_equal(omlp.to_e4m3(u), u) and np.array_equal(omlp.to_e4m3(h), h)
        if not ok:
            continue
        w["act_exp"] = [0] * (2 * B + 1)
        assert np.array_equal(omlp.forward_fp8(w, x), ref), trial
        found += 1
    assert found >= 20


def test_per_tensor_weight_scale_keeps_small_columns():
    """Per-tensor scale (R23): a column 1000x smaller than the tensor max is still quantised
    with e4m3's full 3-bit mantissa (relative error <= 2^-4), since it stays a normal."""
    W = np.array([[400.0, 0.4003], [-300.0, -0.2999]])
    Wq, s = omlp.quantize_weight_e4m3(W)
    assert s == 1.0                                   # 400 <= 448
    rel = np.abs(Wq * s - W) / np.abs(W)
    assert rel.max() <= 2.0 ** -4
