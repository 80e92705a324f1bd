#!/usr/bin/env python
"""Phase timeline of the NVFP4 MLP kernel (block 0, its first 4 tiles) from clock64 stamps
(kernels_mlp_f4.cu, p.trace): per (tile, layer l; l = 0 is layer 0, l = g + 1 GEMM g) 8 stamps:
  0 issuer saw act_ready (layer start)   1 issuer committed acc_full (all copies + MMAs issued)
  2 / 5 epilogue thread 0 / 511 woke on acc_full      4 / 7 thread 0 / 511 arrived act_ready
Printed relative to the layer start (slot 0)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti
from paper_2601_03187_b200 import tang as T, train as TR
B = int(os.environ.get('TRACE_B', 2))
R = ti.classbench_ruleset("acl", 100000, 141)
sigs = TR.tuple_signatures(R)
n = 1 << 20
H = ti.uniform_trace(R, n, 1)
w = ti.random_weights(7, 256, B, len(sigs), 3)
d = torch.from_numpy(H.view(np.uint8).copy()).cuda()
w["act_exp"] = TR.calibrate_fp8(w, TR.features_torch(d[:65536 * 16]))
ctx = T.Ctx(R, T.pack_blob(sigs, w), mlp="nvfp4")
pred = torch.empty(n, dtype=torch.int32, device="cuda")
L = 2 * B + 1
tr = torch.zeros(4 * (L + 1) * 8, dtype=torch.int64, device="cuda")
f = T._lib.tang_debug_trace
f.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
for _ in range(3):
    assert f(ctx.h, d.data_ptr(), n, pred.data_ptr(), tr.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(4, L + 1, 8)
print(f"nvfp4 N=256 B={B}: cycles relative to the layer start (issuer saw act_ready)")
print("tile l | period | iss_done | e0 wake  e0 mid  e0 done | e511 wake e511 mid e511 done   (mid: output layer argmax done)")
for k in range(4):
    for l in range(L + 1):
        a = t[k, l]
        nxt = t[k, l + 1, 0] if l < L else (t[k + 1, 0, 0] if k + 1 < 4 else 0)
        rel = lambda j: int(a[j] - a[0]) if a[j] else -1
        print(f"{k} {l:2d} | {int(nxt - a[0]) if nxt else -1:6d} | {rel(1):7d} | {rel(2):7d} {rel(3):7d} {rel(4):7d} | "
              f"{rel(5):7d} {rel(6):7d} {rel(7):7d}")
