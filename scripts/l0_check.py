#!/usr/bin/env python
"""Layer-0 accuracy of the tensor-core MLP: h0 dumped by tang_debug_activations vs the exact
h0 (fp64 x.W0 + b0, ReLU, RNE to bf16). Reports mismatch counts and the relative error of the
kernel's pre-activation implied by each mismatch (diagnostic for reading R22)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti
from oracle import mlp as omlp
from paper_2601_03187_b200 import tang as T, train as TR
from tests._helpers import bf16_bits_to_f64, headers_dev, model, u32_dev

for fam, nr, rs, N, B in (("acl", 3000, 1, 128, 1), ("acl", 3000, 1, 512, 2)):
    R = ti.classbench_ruleset(fam, nr, rs)
    H = ti.uniform_trace(R, 1500, 3)
    sigs, w, blob = model(R, N, B, 3)
    n = H.size
    for kern in ("single", "ffma"):
        ctx = T.Ctx(R, blob, mlp="bf16" if kern != "ffma" else "fp32", kernel="single")
        if kern == "ffma":
            continue
        act = torch.zeros((2 * B + 1) * n * N, dtype=torch.int16, device="cuda")
        T.tang_debug_activations(ctx.h, headers_dev(H), n, act, u32_dev(n))
        torch.cuda.synchronize()
        A = bf16_bits_to_f64(act.cpu().numpy().view(np.uint16)).reshape(2 * B + 1, n, N)
        x = omlp.features(H).astype(np.float64)
        pre = x @ w["W0"].astype(np.float64) + w["b0"]
        ex = omlp.to_bf16(np.maximum(pre, 0).astype(np.float32)).astype(np.float64)
        f32 = np.zeros_like(pre, dtype=np.float32) + w["b0"].astype(np.float32)
        for s in range(7):   # sequential fp32 FMA order of the FFMA kernel
            f32 = (x[:, s:s + 1].astype(np.float32) * w["W0"][s].astype(np.float32) + f32).astype(np.float32)
        ex32 = omlp.to_bf16(np.maximum(f32, 0)).astype(np.float64)
        mm = A[0] != ex
        print(f"{fam} N={N}: tc mismatches {int(mm.sum())} / {mm.size}; fp32-seq mismatches {int((ex32 != ex).sum())}")
        if mm.any():
            terms = np.abs(x) @ np.abs(w["W0"]) + np.abs(w["b0"])
            # the kernel's value lies past the rounding boundary: |pre - boundary| <= error
            mid = (A[0] + ex) / 2
            rel = np.abs(pre - mid)[mm] / terms[mm]
            print("   implied |err|/sum|terms| max %.3g  (2^%.1f)" % (rel.max(), np.log2(rel.max())))
