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
