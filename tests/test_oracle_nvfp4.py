"""Pins for the oracle's nvfp4 mode (§8(f) row f2, NVFP4 stage; R24).  Each pin is fixed
by the number format, by brute force over the 8-value e2m1 set, or by hand arithmetic -- not by
re-running the oracle's own formulas:
  * the e2m1 value set decoded from its bit fields (exhaustive), ties-to-even / saturation cases,
  * every code is the nearest e2m1 value of v / sf (brute force), the block scale is the e4m3
    value nearest max|v| / 6 (brute force over the e4m3 set), blocks are independent,
  * torch's float4_e2m1fn_x2 as an independent decoder of packed codes (when this torch has it),
  * a hand-computed 2-2-2 network through one residual block,
  * networks whose every intermediate is NVFP4-representable reduce to the exact forward."""
import numpy as np
import pytest

from oracle import mlp as omlp
from tests.test_oracle_fp8 import e4m3_table, _net


def e2m1_table():
    """All e2m1 values from the bit layout s.ee.m, bias 1 (e = 0: subnormal m * 0.5)."""
    vals = []
    for code in range(16):
        s, e, m = code >> 3, (code >> 1) & 3, code & 1
        v = m * 0.5 if e == 0 else (1 + m / 2.0) * 2.0 ** (e - 1)
        vals.append(-v if s else v)
    return np.unique(np.array(vals))


def test_e2m1_table_and_identity():
    t = e2m1_table()
    assert list(t[t >= 0]) == [0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0]
    assert np.array_equal(omlp.to_e2m1(t), t)


def test_e2m1_nearest_ties_to_even_saturating():
    t = e2m1_table()
    rng = np.random.default_rng(40)
    x = rng.uniform(-7, 7, 100000)
    q = omlp.to_e2m1(x)
    assert np.isin(q, t).all()
    d = np.abs(t[None, :] - x[:, None]).min(axis=1)
    inr = np.abs(x) <= 6
    assert np.all(np.abs(q - x)[inr] <= d[inr])
    # midpoints, by hand: the even neighbour has mantissa bit 0 (codes 0, 2, 4, 6 of each sign)
    mids = {0.25: 0.0, 0.75: 1.0, 1.25: 1.0, 1.75: 2.0, 2.5: 2.0, 3.5: 4.0, 5.0: 4.0}
    for m, want in mids.items():
        assert omlp.to_e2m1(m) == want and omlp.to_e2m1(-m) == -want
    assert omlp.to_e2m1(6.9) == 6.0 and omlp.to_e2m1(1e9) == 6.0 and omlp.to_e2m1(-1e9) == -6.0


def test_torch_float4_decodes_the_same_values():
    torch = pytest.importorskip("torch")
    if not hasattr(torch, "float4_e2m1fn_x2"):
        pytest.skip("no float4 in this torch")
    codes = torch.arange(256, dtype=torch.uint8).view(torch.float4_e2m1fn_x2)
    try:
        # torch has no direct float4 -> float cast on CPU in every version: decode via the
        # bit fields is the pin then (test above); here only when the cast exists
        f = codes.to(torch.float32)
    except (RuntimeError, TypeError, NotImplementedError):
        pytest.skip("float4_e2m1fn_x2 has no float conversion in this torch")
    t = e2m1_table()
    assert np.isin(f.numpy().ravel(), t).all()


def test_block_scale_and_codes_by_brute_force():
    t4, t8 = e2m1_table(), e4m3_table()
    rng = np.random.default_rng(41)
    v = rng.standard_normal((300, 48)) * 10.0 ** rng.integers(-3, 3, (300, 1))
    v[5, :16] = 0.0                                    # an all-zero block
    v[6, 16:32] = 1e-6                                 # a block whose max / 6 rounds to e4m3 zero
    codes, sf = omlp.quantize_nvfp4(v)
    assert sf.shape == (300, 3) and codes.shape == v.shape
    for r in range(v.shape[0]):
        for j in range(3):
            blk = v[r, 16 * j:16 * j + 16]
            target = np.abs(blk).max() / 6.0
            # nearest e4m3 value to max/6 (ties: the even code; none occur in random data)
            dist = np.abs(t8 - target)
            assert abs(sf[r, j] - target) == dist.min()
            if sf[r, j] == 0:
                assert np.all(codes[r, 16 * j:16 * j + 16] == 0)
                continue
            y = blk / sf[r, j]
            dd = np.abs(t4[None, :] - y[:, None]).min(axis=1)
            c = codes[r, 16 * j:16 * j + 16]
            inr = np.abs(y) <= 6
            assert np.all(np.abs(c - y)[inr] <= dd[inr])
            assert np.all(c[~inr] == np.sign(y[~inr]) * 6)
            if sf[r, j] >= 2.0 ** -6:                  # normal scale: the block max maps to +-6
                assert np.abs(c).max() == 6.0
    assert np.all(sf[5, 0] == 0) and np.all(codes[5, :16] == 0)
    assert sf[6, 1] == 0 and np.all(codes[6, 16:32] == 0)


def test_blocks_are_independent_and_tail_block():
    rng = np.random.default_rng(42)
    v = rng.uniform(0, 1, (4, 36))                    # blocks 0-15, 16-31 and a 4-wide tail
    c0, s0 = omlp.quantize_nvfp4(v)
    assert s0.shape == (4, 3)
    w = v.copy()
    w[:, 3] = 100.0                                   # an outlier in block 0 only
    c1, s1 = omlp.quantize_nvfp4(w)
    assert np.array_equal(s1[:, 1:], s0[:, 1:]) and np.array_equal(c1[:, 16:], c0[:, 16:])
    assert np.all(s1[:, 0] > s0[:, 0])
    # the tail block alone equals quantising those 4 values as their own row
    ct, st = omlp.quantize_nvfp4(v[:, 32:])
    assert np.array_equal(ct, c0[:, 32:]) and np.array_equal(st[:, 0], s0[:, 2])


def test_weight_blocks_run_along_the_input_dimension():
    """x.W reduces over W's first axis (`in`): one block per 16 inputs of each output column."""
    W = np.full((32, 2), 0.5)
    W[0, 0] = 3.0                                     # outlier in column 0, inputs 0-15
    Wv, s = omlp.quantize_weight_nvfp4(W)
    assert s == 2.0 ** -7                              # 3 <= 448 * 2^-7 = 3.5 < 448 * 2^-8 * 2
    # column 1 / column 0 inputs 16-31: max 0.5 / s = 64 -> sf = e4m3(64 / 6) = 11 -> 64/11 = 5.8 -> 6
    assert np.all(Wv[16:, 0] == 66.0) and np.all(Wv[:, 1] == 66.0)
    # column 0 inputs 0-15: max 384 -> sf = e4m3(64) = 64 -> 64 / 64 = 1 -> value 64; 384 / 64 = 6
    assert Wv[0, 0] == 384.0 and np.all(Wv[1:16, 0] == 64.0)


def test_hand_computed_block():
    """N = 2, B = 1, C = 2 (the fp8 test's network), worked by hand; K = 2 blocks."""
    w = _net(2, 1, 2)
    w["W0"] = np.zeros((7, 2)); w["b0"] = np.array([1.1, 0.3])
    w["W1"] = np.array([np.eye(2)]); w["b1"] = np.zeros((1, 2))
    w["W2"] = np.array([0.5 * np.eye(2)]); w["b2"] = np.zeros((1, 2))
    w["Wo"] = np.array([[1.0, -1.0], [2.0, 0.0]]); w["bo"] = np.array([0.1, 0.0])
    w["act_exp"] = [0, -1, 0]
    # h0 = [1.1, 0.3]: sf = e4m3(1.1/6 = 0.1833) = 12/64 = 0.1875; codes 5.87 -> 6, 1.6 -> 1.5
    # W1 = I: s = 2^-8, W/s = 256 I: sf = e4m3(42.67) = 44, code 5.82 -> 6: value 264 I
    # u = [1.125, 0.28125] * 264 * 2^-8 = [1.16015625, 0.2900390625]; / 2^-1 = [2.3203125, 0.580078125]
    #   sf = e4m3(0.38671875) = 0.375; codes 6.19 -> 6 (sat), 1.546875 -> 1.5
    # W2 = I/2: s = 2^-9, same values 264 I; uq.W2v * 2^-10 = [0.580078125, 0.14501953125]
    # h = that + [1.125, 0.28125] = [1.705078125, 0.42626953125]: sf = e4m3(0.28418) = 0.28125
    #   codes 6.0625 -> 6, 1.515625 -> 1.5: hq = [1.6875, 0.421875]
    # Wo: s = 2^-7, W/s = [[128, -128], [256, 0]]; column 0 block [128, 256]: sf 44, codes 3, 6
    #   -> [132, 264]; column 1 block [-128, 0]: sf = e4m3(21.33) = 22, code -5.82 -> -6 -> -132
    # logits = [1.6875 * 1.03125 + 0.421875 * 2.0625 + 0.1, -1.6875 * 1.03125]
    dump = []
    got = omlp.forward_nvfp4(w, np.zeros((1, 7), np.float32), dump)
    assert np.array_equal(dump[0][0][0], [6.0, 1.5]) and dump[0][1][0, 0] == 0.1875
    assert np.array_equal(dump[1][0][0], [6.0, 1.5]) and dump[1][1][0, 0] == 0.375
    assert np.array_equal(dump[2][0][0], [6.0, 1.5]) and dump[2][1][0, 0] == 0.28125
    assert np.allclose(got[0], [2.7103515625, -1.740234375], rtol=0, atol=1e-15)
    assert np.array_equal(omlp.forward(w, np.zeros((1, 7), np.float32), "nvfp4"), got)


def test_representable_network_reduces_to_exact_forward():
    """If every weight and activation block is already NVFP4-representable (quantisation is the
    identity), nvfp4 mode must equal the exact (fp32-mode, float64) forward."""
    rng = np.random.default_rng(43)
    found = 0
    rep = lambda a: np.array_equal(omlp.nvfp4_values(a), a)
    for trial in range(600):
        N, B, C = 4, 2, 3
        w = _net(N, B, C)
        # values 0 / 6 (and -6 in Wo): a weight column's block max 6 = 384 * 2^-6 gets sf = 64 and
        # code 6 exactly; sums of 6 * 6 stay on grids like {36, 72, 108} whose block scales
        # (6, 12, 18) are e4m3 values -- the filter below keeps only fully representable trials
        w["W0"] = np.zeros((7, N)); w["b0"] = rng.choice([0.0, 6.0], N)
        w["W1"] = rng.choice([0.0, 6.0], (B, N, N), p=[0.7, 0.3])
        w["W2"] = rng.choice([0.0, 6.0], (B, N, N), p=[0.7, 0.3])
        w["Wo"] = rng.choice([-6.0, 0.0, 6.0], (N, C))
        w["b1"] = np.zeros((B, N)); w["b2"] = np.zeros((B, N))
        w["bo"] = rng.standard_normal(C)
        ok = all(rep((Wt / omlp.quantize_weight_nvfp4(Wt)[1]).T) for Wt in
                 [*w["W1"], *w["W2"], w["Wo"]])
        x = np.zeros((1, 7), np.float32)
        h = omlp.relu(w["b0"])[None, :]
        ok &= rep(h)
        for i in range(B):
            u = omlp.relu(h @ w["W1"][i] + w["b1"][i])
            h = omlp.relu(u @ w["W2"][i] + w["b2"][i] + h)
            ok &= rep(u) and rep(h)
        if not ok:
            continue
        w["act_exp"] = [0] * (2 * B + 1)
        assert np.array_equal(omlp.forward_nvfp4(w, x), omlp.forward(w, x, "fp32")), trial
        found += 1
    assert found >= 10, found


def test_nvfp4_error_is_bounded_against_fp32():
    """Sanity of the composition: on a random network the nvfp4 logits stay near fp32's (e2m1
    keeps 1 mantissa bit: relative element error <= 1/3 at the block scale), and argmax mostly
    agrees -- a dropped scale or a transposed block axis gives garbage."""
    import tang_inputs as ti
    w = ti.random_weights(7, 64, 1, 8, seed=5)
    x = np.random.default_rng(44).uniform(0, 1, (400, 7)).astype(np.float32)
    ref = omlp.forward(w, x, "fp32")
    w["act_exp"] = [int(omlp.pow2_scale_exp(a)) for a in (4.0, 4.0, 4.0)]
    got = omlp.forward_nvfp4(w, x)
    rel = np.abs(got - ref).max() / np.abs(ref).max()
    assert rel < 0.35, rel
    assert (omlp.argmax(got) == omlp.argmax(ref)).mean() > 0.6
