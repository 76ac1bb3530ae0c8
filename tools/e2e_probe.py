"""e2e path study: H2D + apply + D2H, plain vs slab-pipelined (apply_host)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_13131_b200 import MatrixFreeTangent
from paper_1904_13131_b200.workloads import make_workload
wl = make_workload(2, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
xh = torch.empty(wl.x.size, dtype=torch.float64, pin_memory=True); xh.copy_(torch.from_numpy(wl.x)); yh = torch.empty(wl.x.size, dtype=torch.float64, pin_memory=True)
xd = xh.cuda(); yd = torch.empty_like(xd)
def plain():
    xd.copy_(xh, non_blocking=True); op.apply_into(xd, yd); yh.copy_(yd, non_blocking=True)
def piped(ch):
    return lambda: op.apply_host(xh, yh, chunks=ch)
def t(f, reps=20):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); w1 = time.perf_counter()
    return e0.elapsed_time(e1) / reps * 1e3, (w1 - w0) / reps * 1e6
print("plain   dev %.1f us  wall %.1f us" % t(plain))
for ch in (1, 2, 4, 8, 16, 32):
    print(f"piped{ch}  dev %.1f us  wall %.1f us" % t(piped(ch)))
# launch-only cost of apply_host (no sync): how long does the host take to enqueue?
print("h2d only dev %.1f us wall %.1f" % t(lambda: xd.copy_(xh, non_blocking=True)))
print("d2h only dev %.1f us wall %.1f" % t(lambda: yh.copy_(yd, non_blocking=True)))
xh2 = torch.empty(xh.numel(), dtype=torch.float64, pin_memory=True); xh2.copy_(xh)
print("h2d fresh-pinned dev %.1f us" % t(lambda: xd.copy_(xh2, non_blocking=True))[0])
import numpy as np
print("apply only dev %.1f us" % t(lambda: op.apply_into(xd, yd))[0])
