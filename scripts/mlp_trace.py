#!/usr/bin/env python
"""Phase timeline of the single-CTA MLP kernel (block 0, first tiles) from clock64 stamps."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti
from paper_2601_03187_b200 import tang as T
N, B = int(os.environ.get('TRACE_N', 512)), int(os.environ.get('TRACE_B', 6))
R = ti.classbench_ruleset("acl", 100000, 141)
sigs = T.tuple_signatures(R)
kern = sys.argv[1] if len(sys.argv) > 1 else "single"
n = 1 << 20
H = ti.uniform_trace(R, n, 1)
w = ti.random_weights(7, N, B, len(sigs), 3)
if kern == "fp8":
    from paper_2601_03187_b200 import train as TR
    w["act_exp"] = TR.calibrate_fp8(w, TR.features_torch(torch.from_numpy(H[:65536].view(np.uint8).copy()).cuda()))
ctx = T.Ctx(R, T.pack_blob(sigs, w), mlp="fp8" if kern == "fp8" else "bf16",
            kernel="auto" if kern == "fp8" else kern)
d = torch.from_numpy(H.view(np.uint8).copy()).cuda()
pred = torch.empty(n, dtype=torch.int32, device="cuda")
L = 2 * B + 1
tr = torch.zeros(4 * L * 8, dtype=torch.int64, device="cuda")
f = T._lib.tang_debug_trace
f.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
for _ in range(3):
    assert f(ctx.h, d.data_ptr(), n, pred.data_ptr(), tr.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(4, L, 8)
for k in range(4):
    print(f"layer0 (tile {k}): start {t[k, 0, 5] - t[k, 0, 0]} duration {t[k, 0, 6] - t[k, 0, 5]}")
# block 0's first 4 tiles (0, grid, 2 grid, 3 grid)
base = t[0, 0, 0]
print("tile layer | mma_start mma_issued(+) wait_full | epi_start(+) epi_end(+) | gap act->mma")
for ti_ in range(4):
    for g in range(L):
        a = t[ti_, g]
        prev_end = t[ti_, g - 1, 4] if g > 0 else (t[ti_ - 1, L - 1, 4] if ti_ > 0 else a[0])
        print(f"{ti_} {g:2d} | {a[0]-base:8d} {a[1]-a[0]:6d} {a[2]:6d} | {a[3]-a[0]:6d} {a[4]-a[3]:6d} | {a[0]-prev_end:6d}")
