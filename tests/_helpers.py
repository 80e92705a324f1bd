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
    # class order from the oracle's O3 (tests/test_oracle_table1.py pins it; the trainer's
    # tuple_signatures is asserted equal in tests/test_lib_host.py)
    sigs = sigs if sigs is not None else otss.signatures_first_occurrence(rules)
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


def decode_e4m3(codes):
    """e4m3fn codes (uint8) -> float64 from the bit fields s.eeee.mmm, bias 7 (no NaN expected)."""
    c = np.asarray(codes, dtype=np.uint8).astype(np.int64)
    s, e, m = c >> 7, (c >> 3) & 15, c & 7
    v = np.where(e == 0, (m / 8.0) * 2.0 ** -6, (1 + m / 8.0) * np.ldexp(1.0, (e - 7).astype(np.int64)))
    return np.where(s == 1, -v, v)


def fp8_scales(w):
    return [float(np.ldexp(1.0, int(e))) for e in w["act_exp"]]


def order_spread_fp8(w, x):
    """R23 analogue of order_spread: the oracle's fp8 forward (exact sums) vs the same
    quantisation points with float32 sums in every layer, in two valid fp32 orders (matmul first,
    then bias and skip; and skip + bias first, matmul added last -- the association the dual-tile
    kernel uses); the larger spread."""
    from oracle import mlp as omlp
    ref = omlp.forward_fp8(w, x)
    sc = fp8_scales(w)
    f32 = lambda a: np.asarray(a, np.float32)
    spread = 0.0
    for skip_first in (False, True):
        h = np.maximum(f32(x) @ f32(w["W0"]) + f32(w["b0"]), 0)
        hq, sh = omlp.to_e4m3(h / sc[0]), sc[0]
        for i in range(int(w["B"])):
            W1q, s1 = omlp.quantize_weight_e4m3(w["W1"][i])
            W2q, s2 = omlp.quantize_weight_e4m3(w["W2"][i])
            su, so = sc[1 + 2 * i], sc[2 + 2 * i]
            u = np.maximum((f32(hq) @ f32(W1q)) * np.float32(sh * s1) + f32(w["b1"][i]), 0)
            uq = omlp.to_e4m3(u / su)
            mm = (f32(uq) @ f32(W2q)) * np.float32(su * s2)
            if skip_first:
                h = np.maximum((f32(hq * sh) + f32(w["b2"][i])) + mm, 0)
            else:
                h = np.maximum(mm + f32(w["b2"][i]) + f32(hq * sh), 0)
            hq, sh = omlp.to_e4m3(h / so), so
        Woq, so_ = omlp.quantize_weight_e4m3(w["Wo"])
        alt = (f32(hq) @ f32(Woq)) * np.float32(sh * so_) + f32(w["bo"])
        spread = max(spread, float(np.abs(alt - ref).max()))
    return spread


def check_e4m3_layer(g, target, terms, eta=2.0 ** -14):
    """g = GPU e4m3 values (unscaled), target = exact ReLU(pre)/s_out from the GPU's own inputs,
    terms = sum of |addends| / s_out.  The GPU's fp32 sums are within eta * terms of target, so
    g must be the e4m3 rounding of some value in [target - eta*terms, target + eta*terms].
    Returns (violations, fraction equal to the exact rounding)."""
    from oracle import mlp as omlp
    exact = omlp.to_e4m3(np.maximum(target, 0))
    d = eta * terms + 1e-30
    lo = omlp.to_e4m3(np.maximum(target - d, 0))
    hi = omlp.to_e4m3(np.maximum(target + d, 0))
    ok = (g == exact) | ((g >= np.minimum(lo, hi)) & (g <= np.maximum(lo, hi)))
    return int((~ok).sum()), float((g == exact).mean())
