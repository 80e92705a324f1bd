#!/usr/bin/env python
"""Phase timeline of the bf16 MLP kernel (block 0, its first 4 tiles) from clock64 stamps.

Per (tile, layer) the kernel writes 16 stamps (kernels_mlp_tc.cu, kTraceSlots):
  0 issuer got half_ready (layer start)   1 issuer issued the last MMA   2 issuer cycles waiting on weights
  3 issuer got act_ready (whole A tile)
  4..7 epilogue thread 0 (column group 0): woke on acc_half/acc_full, a_lo_free, arrive half_ready, arrive act_ready
  8..11 the same for thread 128 (column group 1)
  12, 13 (layer 0 record only): tile start, layer-0 epilogue end (thread 0)
  14, 15 epilogue threads 0 / 128 woke on acc_full (split layers)
  16+i / 24+i producer of block 0 / block 1 issued the TMA of stage i (= q*KC + kc < 8) of the layer;
  48+i / 56+i they acquired the empty slot; 32+i the issuer (block 0) saw stage i full
Printed relative to the layer's start (slot 0)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tang_inputs as ti
from paper_2601_03187_b200 import tang as T, train as TR
N, B = int(os.environ.get('TRACE_N', 512)), int(os.environ.get('TRACE_B', 6))
R = ti.classbench_ruleset("acl", 100000, 141)
sigs = TR.tuple_signatures(R)
kern = sys.argv[1] if len(sys.argv) > 1 else "single"
n = 1 << 20
H = ti.uniform_trace(R, n, 1)
w = ti.random_weights(7, N, B, len(sigs), 3)
ctx = T.Ctx(R, T.pack_blob(sigs, w), mlp="bf16", kernel=kern)
d = torch.from_numpy(H.view(np.uint8).copy()).cuda()
pred = torch.empty(n, dtype=torch.int32, device="cuda")
L = 2 * B + 1
S = 64
tr = torch.zeros(4 * L * S, dtype=torch.int64, device="cuda")
f = T._lib.tang_debug_trace
f.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
for _ in range(3):
    assert f(ctx.h, d.data_ptr(), n, pred.data_ptr(), tr.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(4, L, S)
print(f"bf16 {kern} N={N} B={B}: per layer, cycles relative to the issuer's layer start")
print("tile g | period | iss_end wfull act_rdy | e0:wake lofree half act | e1:wake lofree half act")
rel = lambda a, k: (a[k] - a[0]) if a[k] else -1
for k in range(4):
    for g in range(L):
        a = t[k, g]
        nxt = t[k, g + 1, 0] if g + 1 < L else (t[k + 1, 0, 0] if k + 1 < 4 else 0)
        per = nxt - a[0] if nxt else -1
        print(f"{k} {g:2d} | {per:6d} | {rel(a,1):6d} {a[2]:5d} {rel(a,3):6d} | "
              f"{rel(a,4):6d} {rel(a,5):6d} {rel(a,6):6d} {rel(a,7):6d} | {rel(a,8):6d} {rel(a,9):6d} {rel(a,10):6d} {rel(a,11):6d}")
    print(f"  layer-0 epilogue: tile start {t[k,0,12]-t[k,0,0]:+d}, end {t[k,0,13]-t[k,0,0]:+d}")

print("\nper stage (tile 1, layers 2-3), relative to layer start: empty acquired / TMA issued by blocks 0 and 1,"
      " full seen by the issuer")
for g in (2, 3):
    a = t[1, g]
    print(f"layer {g}: e0 acc_half {a[4]-a[0]}, acc_full {a[14]-a[0]}, lofree {a[5]-a[0]}")
    for i in range(8):
        print(f"  stage {i}: b0 acq {a[48+i]-a[0]:7d} issue {a[16+i]-a[0]:7d} | b1 acq {a[56+i]-a[0]:7d} "
              f"issue {a[24+i]-a[0]:7d} | full {a[32+i]-a[0]:7d}  lat(b0) {a[32+i]-a[16+i]:6d}")
