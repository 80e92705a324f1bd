#!/usr/bin/env python
"""Micro-benchmark of the MLP kernel alone (random paper-size weights, no training): the fast
iteration loop for kernel work and the ncu target.  Prints ms per 1M-packet launch and TFLOP/s."""
import argparse, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti
from paper_2601_03187_b200 import tang as T, train as TR

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=512)
ap.add_argument("--B", type=int, default=6)
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--kernel", default="auto")
ap.add_argument("--mlp", default="bf16", choices=["bf16", "fp8", "nvfp4"])
a = ap.parse_args()
R = ti.classbench_ruleset("acl", 100000, 141)
sigs = TR.tuple_signatures(R)
w = ti.random_weights(7, a.N, a.B, len(sigs), 3)
H = ti.uniform_trace(R, a.n, 1)
if a.mlp in ("fp8", "nvfp4"):
    from paper_2601_03187_b200 import train as TR
    w["act_exp"] = TR.calibrate_fp8(w, TR.features_torch(torch.from_numpy(H[:65536].view(np.uint8).copy()).cuda()))
ctx = T.Ctx(R, T.pack_blob(sigs, w), mlp=a.mlp, kernel=a.kernel)
d = torch.from_numpy(H.view(np.uint8).copy()).cuda()
out = torch.empty(a.n, dtype=torch.int32, device="cuda")
for _ in range(2):
    ctx.classify_async(d, out)
torch.cuda.synchronize()
ctx.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    ctx.classify_async(d, out)
e1.record(); e1.synchronize()
p = ctx.profile_read()
ms, cnt = p["mlp"]
flops = 2 * (7 * a.N + 2 * a.B * a.N * a.N + a.N * len(sigs)) * a.n * a.iters
print(f"{a.mlp} {a.kernel} mlp {a.n * a.iters / (ms / 1e3) / 1e6:.1f} Mpps-mlp-only; "
      f"{a.mlp} {a.kernel} N={a.N} B={a.B} C={len(sigs)}: total {e0.elapsed_time(e1)/a.iters:.3f} ms/step, "
      f"mlp {ms/cnt:.3f} ms/launch, {flops/(ms/1e3)/1e12:.1f} TFLOP/s, {a.n*a.iters/(e0.elapsed_time(e1)/1e3)/1e6:.1f} Mpps")
