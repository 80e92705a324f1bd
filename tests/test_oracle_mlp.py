"""Pins of the oracle's features and MLP (§6.2, Eq. 1-2)."""
import numpy as np
import pytest
import torch

import tang_inputs as ti
from oracle import mlp


def test_feature_example():
    """192.168.1.1 / 10.0.0.1 / 1234 / 80 / 6 -> [49320, 257, 2560, 1, 1234, 80, 6]."""
    h = ti.make_headers((192 << 24) | (168 << 16) | (1 << 8) | 1, (10 << 24) | 1, 1234, 80, 6)
    want = np.array([[49320, 257, 2560, 1, 1234, 80, 6]], dtype=np.float64) / 65536.0
    got = mlp.features(h)
    assert got.dtype == np.float32
    assert (got.astype(np.float64) == want).all()      # exact: 16-bit / 2^16 is exact in fp32
    assert (mlp.features(ti.make_headers(0, 0)) == 0).all()


def test_bf16_rounding_against_torch_and_hand_values():
    one = 1.0
    assert mlp.to_bf16(np.float32(one + 2 ** -8)) == one                 # tie -> even
    assert mlp.to_bf16(np.float32(one + 3 * 2 ** -8)) == one + 2 ** -6   # tie -> even (up)
    assert mlp.to_bf16(np.float32(one + 2 ** -8 + 2 ** -12)) == one + 2 ** -7
    x = np.random.default_rng(0).standard_normal(100000).astype(np.float32) * 10
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert (mlp.to_bf16(x) == ref).all()


def _hand_weights():
    # S=2, N=2, B=1, C=2 with asymmetric matrices so a transposed operand changes the result
    return dict(S=2, N=2, B=1, C=2,
                W0=np.array([[2.0, 0.0], [1.0, -1.0]], np.float32), b0=np.array([-0.25, 0.5], np.float32),
                W1=[np.array([[1.0, 2.0], [0.0, 1.0]], np.float32)], b1=[np.array([-1.0, 0.0], np.float32)],
                W2=[np.array([[0.5, 0.0], [1.0, -3.0]], np.float32)], b2=[np.array([0.5, 0.25], np.float32)],
                Wo=np.array([[1.0, -1.0], [2.0, 0.5]], np.float32), bo=np.array([0.0, 2.0], np.float32))


def test_hand_computed_network():
    """x = [0.5, 0.25]:
       h0 = ReLU([1.0+0.25-0.25, 0-0.25+0.5])            = [1.0, 0.25]
       u  = ReLU(h0.W1 + b1) = ReLU([1-1, 2+0.25+0])      = [0.0, 2.25]
       h  = ReLU(u.W2 + b2 + h0) = ReLU([2.25+0.5+1, -6.75+0.25+0.25]) = [3.75, 0]
       logits = h.Wo + bo = [3.75, -3.75+2]               = [3.75, -1.75]"""
    w = _hand_weights()
    x = np.array([[0.5, 0.25]], np.float32)
    assert np.array_equal(mlp.forward(w, x, "fp32"), [[3.75, -1.75]])
    # every intermediate is a bf16 value, so bf16 mode gives the same result exactly
    assert np.array_equal(mlp.forward(w, x, "bf16"), [[3.75, -1.75]])
    assert mlp.argmax(mlp.forward(w, x))[0] == 0


def test_zero_blocks_are_identity():
    """zero block weights and biases make each block the identity on h0 >= 0."""
    w = ti.random_weights(7, 32, 3, 5, seed=1)
    for i in range(3):
        w["W1"][i][:] = 0
        w["W2"][i][:] = 0
        w["b1"][i][:] = 0
        w["b2"][i][:] = 0
    x = mlp.features(ti.random_headers(50, 2))
    h0 = np.maximum(x.astype(np.float64) @ w["W0"] + w["b0"], 0)
    assert np.allclose(mlp.forward(w, x, "fp32"), h0 @ w["Wo"] + w["bo"], rtol=0, atol=1e-12)


def test_matches_torch_float64_module():
    """Library reference: the same network as torch.nn modules in float64."""
    S, N, B, C = 7, 48, 3, 11
    w = ti.random_weights(S, N, B, C, seed=3)

    def lin(W, b):
        m = torch.nn.Linear(W.shape[0], W.shape[1]).double()
        m.weight.data = torch.from_numpy(W.T.astype(np.float64)).clone()
        m.bias.data = torch.from_numpy(b.astype(np.float64)).clone()
        return m

    l0 = lin(w["W0"], w["b0"])
    blocks = [(lin(w["W1"][i], w["b1"][i]), lin(w["W2"][i], w["b2"][i])) for i in range(B)]
    lo = lin(w["Wo"], w["bo"])
    x = mlp.features(ti.random_headers(64, 4))
    with torch.no_grad():
        h = torch.relu(l0(torch.from_numpy(x).double()))
        for a, b in blocks:
            h = torch.relu(b(torch.relu(a(h))) + h)
        ref = lo(h).numpy()
    assert np.allclose(mlp.forward(w, x, "fp32"), ref, rtol=0, atol=1e-12)


def test_bf16_mode_close_to_fp32_and_quantises():
    w = ti.random_weights(7, 64, 2, 9, seed=5)
    x = mlp.features(ti.random_headers(200, 6))
    a = mlp.forward(w, x, "fp32")
    b = mlp.forward(w, x, "bf16")
    assert not np.array_equal(a, b)
    assert np.max(np.abs(a - b)) < 0.05 * max(1.0, np.max(np.abs(a)))


def test_argmax_and_topk():
    L = np.array([[0.1, 2.3, -1.0], [1.0, 1.0, 1.0], [0.0, 5.0, 5.0]])
    assert mlp.argmax(L).tolist() == [1, 0, 1]
    assert mlp.argmax(L + 7.5).tolist() == [1, 0, 1]              # shift invariance
    assert mlp.topk(L, 2).tolist() == [[1, 0], [0, 1], [1, 2]]
