#!/usr/bin/env python
"""Small invocations of every libtang kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): bf16 chain (single + 2SM with the forwarder warp), fp8 single- and dual-tile, NVFP4, fp32 path, probe /
long-bucket / fallback search, encode, and an in-place update (apply_delta), on tiny batches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti  # noqa: E402
from paper_2601_03187_b200 import tang as T, train as TR  # noqa: E402

R = ti.classbench_ruleset("acl", 2000, 101)
sigs = TR.tuple_signatures(R)
H = np.concatenate([ti.uniform_trace(R, 600, 1), ti.random_headers(40, 2)])
d = torch.from_numpy(H.view(np.uint8).copy()).cuda()
n = H.size
for N, B, mlp, kernel in ((256, 1, "bf16", "single"), (256, 1, "bf16", "2sm"), (512, 1, "bf16", "2sm"),
                          (256, 1, "fp8", "auto"), (512, 1, "fp8", "auto"), (256, 2, "nvfp4", "auto"),
                          (64, 1, "fp32", "auto")):
    w = ti.random_weights(7, N, B, len(sigs), seed=3)
    if mlp in ("fp8", "nvfp4"):
        w["act_exp"] = TR.calibrate_fp8(w, TR.features_torch(d))
    for mode in ("paper", "strict"):
        ctx = T.Ctx(R, T.pack_blob(sigs, w), mlp=mlp, kernel=kernel, mode=mode, topk=2 if mode == "strict" else 1)
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        pred = torch.empty(n * ctx.topk, dtype=torch.int32, device="cuda")
        lg = torch.empty(n * len(sigs), dtype=torch.float32, device="cuda")
        fell = torch.zeros(n, dtype=torch.uint8, device="cuda")
        ctx.classify_ex(d, out, pred, lg, fell)
        ctx.classify_async(d, out)
        ctx.classify_with_pred(d, None, 0, out)
        feat = torch.empty(n * 7, dtype=torch.float32, device="cuda")
        ctx.encode(d, feat)
        if mlp == "bf16" and kernel == "2sm" and mode == "paper":
            new = ti.classbench_ruleset("fw", 50, 9)
            new["id"] += 100000
            ctx.update(T.make_ops(new, deletes=R["id"][:50]))
            ctx.classify_async(d, out)
            h_out = np.empty(n, np.uint32)
            T.tang_classify(ctx.h, H, h_out)                 # streamed host path
        torch.cuda.synchronize()
        print(f"{mlp} {kernel} N={N} {mode}: ok", flush=True)
        ctx.close()
print("SANITIZE_DRIVER_DONE")
