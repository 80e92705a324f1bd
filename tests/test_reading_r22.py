"""R22: layer 0 on the tensor core is exact up to fp32 accumulation because
(i) every feature x = v / 65536 (v < 2^16) equals xh + xl with xh = bf16_rne(x), xl = bf16_rne(x - xh),
(ii) every finite fp32 w equals the sum of three successive RNE bf16 residual pieces.
Both are properties of the number formats, checked here exhaustively / on a fuzzed sample."""
import numpy as np

from oracle import mlp as omlp


def _bf16(a):
    return omlp.to_bf16(np.asarray(a, np.float32)).astype(np.float32)


def test_feature_two_piece_split_is_exact_for_every_16_bit_value():
    v = np.arange(1 << 16, dtype=np.float64)
    x = (v / 65536.0).astype(np.float32)
    assert np.array_equal(x.astype(np.float64), v / 65536.0)          # x itself is exact in fp32
    xh = _bf16(x)
    xl = _bf16(x - xh)
    assert np.array_equal(xh.astype(np.float64) + xl.astype(np.float64), x.astype(np.float64))


def test_weight_three_piece_split_is_exact():
    rng = np.random.default_rng(22)
    w = np.concatenate([
        rng.standard_normal(200000).astype(np.float32),
        (rng.uniform(-1, 1, 100000) * 10.0 ** rng.integers(-30, 30, 100000)).astype(np.float32),
        np.array([0.0, -0.0, 1.0, -1.0, 3.0e38, -3.0e38, 1.1754944e-38, 0.33333334], np.float32),
    ])
    rest = w.copy()
    total = np.zeros(w.size, np.float64)
    for _ in range(3):
        piece = _bf16(rest)
        total += piece.astype(np.float64)
        rest = (rest - piece).astype(np.float32)
    assert np.array_equal(total, w.astype(np.float64))
    assert not np.any(rest)


def test_two_piece_weight_split_is_not_exact():
    """Why W0 needs three pieces: two bf16 pieces keep only 16 of fp32's 24 significand bits."""
    w = np.float32(1.0 + 2.0 ** -9 + 2.0 ** -20)     # bits spread over the full 24-bit significand
    wh = _bf16(w)[()]
    wl = _bf16(w - wh)[()]
    assert float(wh) + float(wl) != float(w)
