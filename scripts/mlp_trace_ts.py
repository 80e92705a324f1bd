#!/usr/bin/env python
"""Phase timeline of the TS bf16 MLP kernel (kernels_mlp_ts.cu; block 0, its first 4 tiles) from clock64
stamps.  Per GEMM record: 0 issuer start, 1 issuer end (last MMA issued), 2/3 GEMM2 fold waits done,
4 cycles waiting on weight stages, 5 cycles waiting on the epilogue, 8+j T sub-pass j start; epilogue
unit ends 16+u (thread 0) / 32+u (thread 128), thread 0 woke for unit u at 48+u.  Cycles relative to
the record's issuer start."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti
from paper_2601_03187_b200 import tang as T, train as TR
N, B = 512, int(os.environ.get('TRACE_B', 6))
R = ti.classbench_ruleset("acl", 100000, 141)
sigs = TR.tuple_signatures(R)
n = 1 << 20
H = ti.uniform_trace(R, n, 1)
w = ti.random_weights(7, N, B, len(sigs), 3)
ctx = T.Ctx(R, T.pack_blob(sigs, w), mlp="bf16", kernel=sys.argv[1] if len(sys.argv) > 1 else "ts")
d = torch.from_numpy(H.view(np.uint8).copy()).cuda()
pred = torch.empty(n, dtype=torch.int32, device="cuda")
L = 2 * B + 2
S = 192
f = T._lib.tang_debug_trace
f.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
for _ in range(3):
    tr = torch.zeros(4 * L * S, dtype=torch.int64, device="cuda")
    assert f(ctx.h, d.data_ptr(), n, pred.data_ptr(), tr.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(4, L, S)
names = ["L0"] + [f"{'G1' if g % 2 else 'G2'}_{(g - 1) // 2}" for g in range(1, L - 1)] + ["OUT"]
for k in range(4):
    print(f"tile {k}")
    for g in range(L):
        a = t[k, g]
        nxt = t[k, g + 1, 0] if g + 1 < L else (t[k + 1, 0, 0] if k + 1 < 4 else 0)
        rel = lambda x: (x - a[0]) if x else None
        units0 = [rel(x) for x in a[16:24] if x]
        units1 = [rel(x) for x in a[32:40] if x]
        wakes = [rel(x) for x in a[48:56] if x]
        sp = [rel(x) for x in a[8:12] if x]
        print(f"  {names[g]:6s} period {nxt - a[0] if nxt else -1:6d} issue_end {rel(a[1])} wait_w {a[4]} wait_epi {a[5]}"
              f" folds {[rel(a[2]), rel(a[3])] if g % 2 == 0 and 0 < g < L - 1 else ''} subpass {sp}")
        print(f"         epi0 wake {wakes} end {units0}")
        print(f"         epi1 end {units1}")
print("\nweight stages 4-7 of each GEMM (tile 1): producer acquired the empty slot and issued the TMA /"
      " issuer saw it full (relative to the record start)")
for g in range(L):
    a = t[1, g]
    acq = [int(a[40 + i] - a[0]) if a[40 + i] else None for i in range(4)]
    ful = [int(a[24 + i] - a[0]) if a[24 + i] else None for i in range(4)]
    print(f"  {names[g]:6s} acquire {acq} full {ful}")

print("\nper-warp end of epilogue units 0-3 (tile 1), in ns (%globaltimer) relative to block 0 warp 0: block 0 warps 0-7 | block 1 warps 0-7")
for g in range(L):
    a = t[1, g]
    for u in range(4):
        v = a[64 + 16 * u: 64 + 16 * u + 16]
        ref = v[0]
        if not ref or not v.any():
            continue
        print(f"  {names[g]:6s} unit {u}: " + " ".join(f"{int(x - ref):6d}" for x in v[:8]) + " | " +
              " ".join(f"{int(x - ref):6d}" for x in v[8:]))

print("\nper-warp WAKE for epilogue units 0-3 (tile 1), ns relative to block 0 warp 0's wake: block 0 | block 1")
for g in range(L):
    a = t[1, g]
    for u in range(4):
        v = a[128 + 16 * u: 128 + 16 * u + 16]
        ref = v[0]
        if not ref or not v.any():
            continue
        print(f"  {names[g]:6s} unit {u}: " + " ".join(f"{int(x - ref):6d}" for x in v[:8]) + " | " +
              " ".join(f"{int(x - ref):6d}" for x in v[8:]))
