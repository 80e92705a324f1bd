#!/usr/bin/env python
"""Micro-benchmark of stage 2 alone (probe + fallback) at the bench's scale: ACL 512k rules,
perfect predictions (the tuple of the brute-force winner, GPU k = 0 search), 4M packets per
launch.  Also a miss-heavy variant (predictions shifted by one tuple) for the fallback kernel.
Prints ms per launch of each stage and packets/s."""
import argparse, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti
from paper_2601_03187_b200 import tang as T, train as TR

ap = argparse.ArgumentParser()
ap.add_argument("--rules", type=int, default=1 << 19)
ap.add_argument("--fam", default="acl")
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--seed", type=int, default=142)          # bench.py's acl-512k ruleset seed
ap.add_argument("--noise", type=float, default=0.02)      # fraction of predictions replaced at random
a = ap.parse_args()
R = ti.classbench_ruleset(a.fam, a.rules, a.seed)
sigs = TR.tuple_signatures(R)
ctx = T.Ctx(R, T.pack_blob(sigs, ti.random_weights(7, 64, 1, len(sigs), 0)), mlp="fp32", max_batch=a.n)
H = ti.uniform_trace(R, a.n, 1000 + a.seed * 10)
d = torch.from_numpy(H.view(np.uint8).copy()).cuda()
lab = TR.gpu_labels(ctx, d, R, sigs).int()
out = torch.empty(a.n, dtype=torch.int32, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
noisy = lab.clamp(min=0).clone()
flip = torch.rand(a.n, device="cuda", generator=g) < a.noise
noisy[flip] = torch.randint(0, len(sigs), (int(flip.sum()),), device="cuda", generator=g, dtype=torch.int32)
for name, pred in (("perfect", lab.clamp(min=0)), (f"noisy{a.noise}", noisy),
                   ("shifted", (lab.clamp(min=0) + 1) % len(sigs))):
    for _ in range(2):
        ctx.classify_with_pred(d, pred, 1, out)
    torch.cuda.synchronize()
    ctx.profile(True)
    ctx.profile_read()
    for _ in range(a.iters):
        ctx.classify_with_pred(d, pred, 1, out)
    torch.cuda.synchronize()
    p = ctx.profile_read()
    ms = {k: v[0] / max(1, v[1]) for k, v in p.items()}
    tot = sum(ms.values())
    print(f"{name}: " + ", ".join(f"{k} {v:.3f} ms" for k, v in ms.items()) + f" -> {a.n / (tot / 1e3) / 1e9:.2f} Gpps (stage 2)")
    ctx.profile(False)
