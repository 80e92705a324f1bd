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

Two precisions:
  fp32 mode -- the weights as given (fp32 values), every product and sum in
               float64: the exact-arithmetic reference for the fp32 GPU path.
  bf16 mode -- the quantisation points of the bf16 GPU path (reading 5): W1, W2, Wo
               rounded to bf16 (round-to-nearest-even) once; layer 0 stays fp32;
               h0, u and h are rounded to fp32 (the accumulator) and then to bf16 as
               GEMM inputs; bias, skip-add and ReLU are applied before rounding.
               Products of bf16 values are exact in float64, so the only difference
               from the GPU is the fp32 summation order.
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


def relu(z):
    """Eq. (2): A(z) = max(0, z)."""
    return np.maximum(z, 0.0)


def forward(weights: dict, x: np.ndarray, mode: str = "fp32") -> np.ndarray:
    """O7: logits [n, C] (float64) of the residual MLP for features x [n, S]."""
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
