#!/usr/bin/env python
"""Pinned host<->device copy bandwidth on this box (the e2e leg's PCIe ceiling): 64 MiB H2D and
16 MiB D2H (one 4M-packet step of headers / rule ids), alone and concurrently, CUDA events."""
import torch
h = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
ho = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
do = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / n
t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
t_d2h = timed(lambda: ho.copy_(do, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
t_both = timed(both)
print(f"H2D 64 MiB: {t_h2d:.3f} ms = {64 * 1.048576 / t_h2d:.1f} GB/s; D2H 16 MiB: {t_d2h:.3f} ms = "
      f"{16 * 1.048576 / t_d2h:.1f} GB/s; both concurrently: {t_both:.3f} ms")
