#!/usr/bin/env python
"""Phase timeline of the 2-CTA pair MLP kernel (cluster 0, first tile, both CTAs)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti
from paper_2601_03187_b200 import tang as T, train as TR
N, B = 512, 6
R = ti.classbench_ruleset("acl", 100000, 141)
sigs = TR.tuple_signatures(R)
ctx = T.Ctx(R, T.pack_blob(sigs, ti.random_weights(7, N, B, len(sigs), 3)), mlp="bf16", kernel="pair")
n = 1 << 20
H = ti.uniform_trace(R, n, 1)
d = torch.from_numpy(H.view(np.uint8).copy()).cuda()
pred = torch.empty(n, dtype=torch.int32, device="cuda")
L = 2 * B + 1
tr = torch.zeros(2 * 4 * L * 8, dtype=torch.int64, device="cuda")
f = T._lib.tang_debug_trace
f.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
for _ in range(3):
    assert f(ctx.h, d.data_ptr(), n, pred.data_ptr(), tr.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(2, 4, L, 8)
base = t[0, 0, 0, 0]
print("cta layer | mma_begin gate(+) mma_end(+) w_own w_peer w_full | epi_start(rel mma_begin) epi_len")
for x in range(2):
    for g in range(L):
        a = t[x, 0, g]
        print(f"{x} {g:2d} | {a[0]-base:8d} {a[1]-a[0]:6d} {a[2]-a[0]:6d} {a[3]:6d} {a[4]:6d} {a[5]:6d} | {a[6]-a[0]:6d} {a[7]-a[6]:6d}")
