"""O6-O8: features, the residual MLP and argmax/top-k (test infrastructure only).

P:389 (§6.2): a 5-tuple header is split into 7 16-bit segments -- high and low
halves of SIP, of DIP, then SP, DP, PRO -- each converted to a 32-bit float.
Normalisation by 2^16 is SPEC.md:99's reading (SURVEY.md §8(c) reading 4); it is
exact in fp32.
P:371 (§6.1) + Eq. (1)-(2): an input FC S->N with ReLU, B residual
blocks B(x) = A(A(x.w1 + b1).w2 + b2 + x) with A = ReLU (the balanced reading of
the garbled Eq. 1, SURVEY.md §8(c) reading 1), and an output FC N->C; the
predicted tuple is argmax of the outputs, ties to the lowest index
(reading 6).  Weights are [in][out] ("x.w", reading 3).

Four precisions (fp8 and nvfp4 are §8(f) row f2):
  fp32 mode -- the weights as given (fp32 values), every product and sum in
               float64: the exact-arithmetic reference for the fp32 GPU path.
  bf16 mode -- the quantisation points of the bf16 GPU path (reading 5): W1, W2, Wo
               rounded to bf16 (round-to-nearest-even) once; layer 0 stays fp32;
               h0, u and h are rounded to fp32 (the accumulator) and then to bf16 as
               GEMM inputs; bias, skip-add and ReLU are applied before rounding.
               Products of bf16 values are exact in float64, so the only difference
               from the GPU is the fp32 summation order.
  fp8 mode  -- "precision quantization" read as TensorRT-style FP8 (R23):
               W1, W2, Wo quantised to e4m3 per tensor with a power-of-two scale
               s_w = 2^e, e the smallest integer with max |W| <= 448 * 2^e (e4m3's exponent
               range keeps entries down to 2^-14 of the maximum normal);
               activations h0, u_b, h_b quantised to e4m3 per layer with the static
               power-of-two scales 2^e_k carried by the model (calibration); layer 0 as in
               bf16 mode (fp32-accurate); bias, skip-add and ReLU in exact arithmetic on the
               dequantised values before each quantisation.
  nvfp4 mode -- f2's NVFP4 stage (R24): the fp8 mode with every e4m3 tensor
               replaced by NVFP4 blocks: along the reduction (K) dimension, each run of 16
               consecutive values v (already divided by the tensor's power-of-two scale) gets
               the block scale sf = e4m3(max|v| / 6) (an unsigned e4m3 value) and the codes
               e2m1(v / sf) (round to nearest even, saturating at 6; all zero when sf = 0); the
               value the tensor core multiplies is code * sf.  Weights keep the fp8 mode's
               per-tensor 2^e (max |W| <= 448 * 2^e); activations use the same calibrated 2^e_k
               as fp8 mode, so every block scale is <= 448 / 6 and inside e4m3's range.
"""
from __future__ import annotations

import numpy as np


def features(headers: np.ndarray) -> np.ndarray:
    """O6: [SIP_hi, SIP_lo, DIP_hi, DIP_lo, SP, DP, PRO] / 65536 as float32."""
    sip = headers["sip"].astype(np.uint64)
    dip = headers["dip"].astype(np.uint64)
    seg = np.stack([sip >> np.uint64(16), sip & np.uint64(0xFFFF),
                    dip >> np.uint64(16), dip & np.uint64(0xFFFF),
                    headers["sp"].astype(np.uint64), headers["dp"].astype(np.uint64),
                    headers["proto"].astype(np.uint64)], axis=1)
    return (seg.astype(np.float64) / 65536.0).astype(np.float32)


def to_bf16(x) -> np.ndarray:
    """Round float32 values to bfloat16 (round-to-nearest-even), returned as float32."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32).reshape(f.shape)


E4M3_MAX = 448.0


def to_e4m3(x) -> np.ndarray:
    """Round to the nearest FP8 E4M3 (OCP 'fn' variant: bias 7, no infinities, max 448,
    subnormals m * 2^-9) with ties to even, saturating to +-448; returned as float64."""
    v = np.asarray(x, dtype=np.float64)
    a = np.abs(v)
    _, ex = np.frexp(a)                                   # a = m * 2^ex, m in [0.5, 1)
    e = np.maximum(ex - 1, -6)                            # binade exponent (subnormals share -6)
    spacing = np.ldexp(1.0, (e - 3).astype(np.int64))     # 3 mantissa bits
    q = np.rint(a / spacing) * spacing                    # a / spacing is exact; rint = ties to even
    q = np.minimum(q, E4M3_MAX)
    return np.copysign(q, v)


def pow2_scale_exp(amax) -> np.ndarray:
    """Smallest integer e with amax <= 448 * 2^e (exact comparisons; amax <= 0 -> 0)."""
    a = np.asarray(amax, dtype=np.float64)
    _, ex = np.frexp(np.where(a > 0, a, 1.0))
    e = ex.astype(np.int64) - 9
    for _ in range(3):                                    # frexp puts e within one step
        e = np.where(a > np.ldexp(E4M3_MAX, e), e + 1, e)
        e = np.where((a > 0) & (a <= np.ldexp(E4M3_MAX, e - 1)), e - 1, e)
    return np.where(a > 0, e, 0)


def quantize_weight_e4m3(W):
    """Per-tensor e4m3 quantisation of W [in][out]: (Wq, s) with W ~ Wq * s, s a power of two."""
    W = np.asarray(W, dtype=np.float64)
    s = float(np.ldexp(1.0, int(pow2_scale_exp(np.abs(W).max()))))
    return to_e4m3(W / s), s


E2M1_MAX = 6.0


def to_e2m1(x) -> np.ndarray:
    """Round to the nearest FP4 E2M1 value (s.ee.m, bias 1: 0, 0.5, 1, 1.5, 2, 3, 4, 6) with
    ties to even, saturating to +-6 (cvt .satfinite); returned as float64."""
    v = np.asarray(x, dtype=np.float64)
    a = np.abs(v)
    _, ex = np.frexp(a)                                   # a = m * 2^ex, m in [0.5, 1)
    e = np.maximum(ex - 1, 0)                             # binade exponent (subnormals share 0)
    spacing = np.ldexp(1.0, (e - 1).astype(np.int64))     # 1 mantissa bit
    q = np.rint(a / spacing) * spacing                    # a / spacing is exact; rint = ties to even
    q = np.minimum(q, E2M1_MAX)
    return np.copysign(q, v)


NVFP4_BLOCK = 16


def quantize_nvfp4(v):
    """NVFP4 block quantisation of v [..., K] along the last axis (R24): blocks of 16 (the last
    one shorter when K % 16 != 0), sf = e4m3(max|v| / 6) per block, codes = e2m1(v / sf) (0 if
    sf = 0).  Returns (codes, sf): codes [..., K], sf [..., ceil(K / 16)], both float64; the
    quantised tensor is codes * sf repeated over each block."""
    v = np.asarray(v, dtype=np.float64)
    K = v.shape[-1]
    nb = (K + NVFP4_BLOCK - 1) // NVFP4_BLOCK
    codes = np.zeros_like(v)
    sf = np.zeros(v.shape[:-1] + (nb,))
    for j in range(nb):
        blk = v[..., j * NVFP4_BLOCK:(j + 1) * NVFP4_BLOCK]
        s = to_e4m3(np.abs(blk).max(axis=-1) / 6.0)
        sf[..., j] = s
        safe = np.where(s > 0, s, 1.0)[..., None]
        codes[..., j * NVFP4_BLOCK:(j + 1) * NVFP4_BLOCK] = np.where(s[..., None] > 0, to_e2m1(blk / safe), 0.0)
    return codes, sf


def nvfp4_values(v):
    """code * sf of quantize_nvfp4(v): the values the tensor core multiplies."""
    codes, sf = quantize_nvfp4(v)
    return codes * np.repeat(sf, NVFP4_BLOCK, axis=-1)[..., :codes.shape[-1]]


def quantize_weight_nvfp4(W):
    """W [in][out] -> (Wv, s): s = 2^e per tensor as in fp8 mode (max |W| <= 448 * 2^e), Wv the
    NVFP4 values of W / s with blocks of 16 along `in` (the K dimension of x.W), so W ~ Wv * s."""
    W = np.asarray(W, dtype=np.float64)
    s = float(np.ldexp(1.0, int(pow2_scale_exp(np.abs(W).max()))))
    return nvfp4_values((W / s).T).T, s


def relu(z):
    """Eq. (2): A(z) = max(0, z)."""
    return np.maximum(z, 0.0)


def forward(weights: dict, x: np.ndarray, mode: str = "fp32") -> np.ndarray:
    """O7: logits [n, C] (float64) of the residual MLP for features x [n, S]."""
    if mode == "fp8":
        return forward_fp8(weights, x)
    if mode == "nvfp4":
        return forward_nvfp4(weights, x)
    if mode not in ("fp32", "bf16"):
        raise ValueError(mode)
    f64 = lambda a: np.asarray(a, dtype=np.float64)
    q = (lambda a: f64(to_bf16(np.asarray(a, dtype=np.float32)))) if mode == "bf16" else f64
    acc = (lambda a: f64(np.asarray(a, dtype=np.float32))) if mode == "bf16" else (lambda a: a)

    # input FC + ReLU (fp32 in both modes: layer 0 is never quantised, reading 5)
    h = relu(f64(x) @ f64(weights["W0"]) + f64(weights["b0"]))
    for i in range(int(weights["B"])):
        hq = q(acc(h))                                          # GEMM input
        u = relu(acc(hq @ q(weights["W1"][i])) + f64(weights["b1"][i]))
        uq = q(acc(u))
        # B(x) = A(A(x.w1 + b1).w2 + b2 + x)   (Eq. 1); the skip x is the block input
        h = relu(acc(uq @ q(weights["W2"][i])) + f64(weights["b2"][i]) + hq)
    hq = q(acc(h))
    return acc(hq @ q(weights["Wo"])) + f64(weights["bo"])


def forward_fp8(weights: dict, x: np.ndarray, dump: list | None = None) -> np.ndarray:
    """O7, fp8 mode (R23): logits [n, C] in float64.  weights["act_exp"] = [e_h0, e_u0, e_h0',
    e_u1, e_h1', ...] (2B + 1 power-of-two activation-scale exponents, layer order).  Every
    product of e4m3 values and every scaling by a power of two is exact in float64.  If `dump`
    is a list, the quantised activations (e4m3 values, unscaled) are appended in layer order."""
    f64 = lambda a: np.asarray(a, dtype=np.float64)
    ex = [int(e) for e in weights["act_exp"]]
    B = int(weights["B"])
    if len(ex) != 2 * B + 1:
        raise ValueError("act_exp needs 2B+1 exponents")
    sc = [float(np.ldexp(1.0, e)) for e in ex]
    h = relu(f64(x) @ f64(weights["W0"]) + f64(weights["b0"]))          # layer 0: exact (R22)
    hq, sh = to_e4m3(h / sc[0]), sc[0]
    if dump is not None:
        dump.append(hq)
    for i in range(B):
        W1q, s1 = quantize_weight_e4m3(weights["W1"][i])
        W2q, s2 = quantize_weight_e4m3(weights["W2"][i])
        su, sh2 = sc[1 + 2 * i], sc[2 + 2 * i]
        u = relu((hq @ W1q) * (sh * s1) + f64(weights["b1"][i]))
        uq = to_e4m3(u / su)
        # B(x) = A(A(x.w1 + b1).w2 + b2 + x)   (Eq. 1); the skip is the dequantised block input
        h = relu((uq @ W2q) * (su * s2) + f64(weights["b2"][i]) + hq * sh)
        hq, sh = to_e4m3(h / sh2), sh2
        if dump is not None:
            dump += [uq, hq]
    Woq, so = quantize_weight_e4m3(weights["Wo"])
    return (hq @ Woq) * (sh * so) + f64(weights["bo"])


def forward_nvfp4(weights: dict, x: np.ndarray, dump: list | None = None) -> np.ndarray:
    """O7, nvfp4 mode (R24): forward_fp8 with quantize_nvfp4 in place of every e4m3 rounding
    (weights per quantize_weight_nvfp4, activation blocks along the feature axis, which is the
    next GEMM's K).  Products of NVFP4 values are exact in float64.  If `dump` is a list, each
    quantised activation is appended in layer order as (codes, sf)."""
    f64 = lambda a: np.asarray(a, dtype=np.float64)
    ex = [int(e) for e in weights["act_exp"]]
    B = int(weights["B"])
    if len(ex) != 2 * B + 1:
        raise ValueError("act_exp needs 2B+1 exponents")
    sc = [float(np.ldexp(1.0, e)) for e in ex]

    def q(v):
        codes, sf = quantize_nvfp4(v)
        if dump is not None:
            dump.append((codes, sf))
        return codes * np.repeat(sf, NVFP4_BLOCK, axis=-1)[..., :codes.shape[-1]]

    h = relu(f64(x) @ f64(weights["W0"]) + f64(weights["b0"]))          # layer 0: exact (R22)
    hq, sh = q(h / sc[0]), sc[0]
    for i in range(B):
        W1v, s1 = quantize_weight_nvfp4(weights["W1"][i])
        W2v, s2 = quantize_weight_nvfp4(weights["W2"][i])
        su, sh2 = sc[1 + 2 * i], sc[2 + 2 * i]
        u = relu((hq @ W1v) * (sh * s1) + f64(weights["b1"][i]))
        uq = q(u / su)
        # B(x) = A(A(x.w1 + b1).w2 + b2 + x)   (Eq. 1); the skip is the dequantised block input
        h = relu((uq @ W2v) * (su * s2) + f64(weights["b2"][i]) + hq * sh)
        hq, sh = q(h / sh2), sh2
    Wov, so = quantize_weight_nvfp4(weights["Wo"])
    return (hq @ Wov) * (sh * so) + f64(weights["bo"])


def argmax(logits: np.ndarray) -> np.ndarray:
    """O8: predicted tuple index, ties to the lowest index (reading 6)."""
    return np.argmax(logits, axis=1).astype(np.uint32)


def topk(logits: np.ndarray, k: int) -> np.ndarray:
    """O8: the k largest logits' indices, descending, ties to the lower index."""
    n, C = logits.shape
    idx = np.arange(C)
    out = np.empty((n, k), dtype=np.uint32)
    for i in range(n):
        order = sorted(range(C), key=lambda c: (-logits[i, c], idx[c]))
        out[i] = order[:k]
    return out
