"""Shared helpers of the GPU parity tests (test code; may use the oracle)."""
import numpy as np

import tang_inputs as ti
from oracle import tss as otss

NM = 0xFFFFFFFF


def require_cuda():
    import torch
    assert torch.cuda.is_available(), "gpu test selected but no CUDA device"
    return torch


def to_dev(arr):
    """NumPy structured / plain array -> torch CUDA byte-compatible tensor."""
    torch = require_cuda()
    a = np.ascontiguousarray(arr)
    t = torch.from_numpy(a.view(np.uint8).copy()).cuda()
    return t


def headers_dev(h):
    return to_dev(h)            # uint8 [n*16]


def u32_dev(n, fill=0):
    torch = require_cuda()
    return torch.full((n,), fill, dtype=torch.int32, device="cuda")


def u32_host(t):
    return t.cpu().numpy().view(np.uint32)


def oracle_tss(rules, sigs):
    return otss.Tss(sigs, rules)


def model(rules, N, B, seed, sigs=None, gain=1.0):
    from paper_2601_03187_b200 import tang as T
    sigs = sigs if sigs is not None else T.tuple_signatures(rules)
    w = ti.random_weights(7, N, B, len(sigs), seed=seed, gain=gain)
    return sigs, w, T.pack_blob(sigs, w)


def order_spread(w, x):
    """Max |logit| difference between the oracle's bf16-emulated forward (fp64 sums) and the
    same quantisation points evaluated with fp32 BLAS sums in every layer: how far two valid fp32
    summation orders already land apart for these weights (reading R6)."""
    from oracle import mlp as omlp
    ref = omlp.forward(w, x, "bf16")
    q = lambda a: omlp.to_bf16(np.asarray(a, np.float32))
    # layer 0 in fp32 too (R5: layer 0 is an fp32 layer; its rounding also decides bf16 flips of h0)
    h = np.maximum((x.astype(np.float32) @ w["W0"].astype(np.float32)).astype(np.float32)
                   + w["b0"].astype(np.float32), 0).astype(np.float32)
    for i in range(int(w["B"])):
        hq = q(h)
        u = np.maximum((hq @ q(w["W1"][i])).astype(np.float32) + w["b1"][i], 0)
        h = np.maximum((q(u) @ q(w["W2"][i])).astype(np.float32) + w["b2"][i] + hq, 0)
    alt = (q(h) @ q(w["Wo"])).astype(np.float32) + w["bo"]
    return float(np.abs(alt - ref).max())


def bf16_bits_to_f64(u16):
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def check_rounded_layer(g, pre, terms, relu=True, eta=2.0 ** -14):
    """g = GPU bf16 output, pre = exact pre-activation (fp64) from the GPU's own inputs,
    terms = sum of |addends|.  The GPU sums in fp32 (error <= eta * terms) and rounds to bf16
    (error <= half an ulp), so |g - act(pre)| <= half_ulp + eta * terms must hold everywhere.
    Returns (violations, fraction bit-equal to bf16(act(pre)))."""
    from oracle import mlp as omlp
    e = np.maximum(pre, 0) if relu else pre
    mag = np.maximum(np.abs(e), np.abs(g))
    half_ulp = np.where(mag > 0, 2.0 ** (np.floor(np.log2(np.maximum(mag, 1e-30))) - 8), 0.0)
    viol = np.abs(g - e) > half_ulp + eta * terms + 1e-30
    same = omlp.to_bf16(e.astype(np.float32)).astype(np.float64) == g
    return int(viol.sum()), float(same.mean())
