#!/usr/bin/env python
"""Phase timeline of the fp8 dual-tile MLP kernel (mlp_f8x2_kernel, N <= 256): block 0, first two
tile pairs, from clock64 stamps: per job and slot the MMA issue window (after act_ready) and the
epilogue window (acc_full observed -> job done)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti
from paper_2601_03187_b200 import tang as T, train as TR
from paper_2601_03187_b200 import train as TR
N, B = int(os.environ.get('TRACE_N', 256)), int(os.environ.get('TRACE_B', 2))
R = ti.classbench_ruleset("acl", 100000, 141)
sigs = TR.tuple_signatures(R)
n = 1 << 20
H = ti.uniform_trace(R, n, 1)
w = ti.random_weights(7, N, B, len(sigs), 3)
w["act_exp"] = TR.calibrate_fp8(w, TR.features_torch(torch.from_numpy(H[:65536].view(np.uint8).copy()).cuda()))
ctx = T.Ctx(R, T.pack_blob(sigs, w), mlp="fp8")
d = torch.from_numpy(H.view(np.uint8).copy()).cuda()
pred = torch.empty(n, dtype=torch.int32, device="cuda")
Cp = (len(sigs) + 15) // 16 * 16
J = 1 + 2 * B + (Cp + N - 1) // N
tr = torch.zeros(4 * (2 * B + 1) * 8, dtype=torch.int64, device="cuda")
f = T._lib.tang_debug_trace
f.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
for _ in range(3):
    assert f(ctx.h, d.data_ptr(), n, pred.data_ptr(), tr.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
t = tr.cpu().numpy()[:2 * J * 2 * 4].reshape(2, J, 2, 4)
base = t[0, 0, 0, 0]
print(f"N={N} B={B} C={len(sigs)} J={J}: cycles relative to pair 0 job 0 MMA issue")
print("pair job slot | mma_issue  (+issue) | epi_start  epi_len | mma->epi  epi_end->next_mma")
for k in range(2):
    for j in range(J):
        for sl in range(2):
            a = t[k, j, sl]
            nxt = t[k, j + 1, sl, 0] if j + 1 < J else (t[k + 1, 0, sl, 0] if k + 1 < 2 else 0)
            print(f"{k} {j:2d} {sl} | {a[0]-base:9d} {a[1]-a[0]:6d} | {a[2]-base:9d} {a[3]-a[2]:6d} | "
                  f"{a[2]-a[1]:7d} {nxt - a[3] if nxt else 0:7d}")
print(f"pair 0 -> pair 1 (slot 0 job 0 MMA): {t[1, 0, 0, 0] - t[0, 0, 0, 0]} cycles")
