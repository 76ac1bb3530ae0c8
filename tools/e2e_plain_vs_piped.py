"""Steady-state e2e step times on this host: plain (one H2D, the apply, one D2H on
one stream) against the slab pipeline (hf_tangent_apply_host), 40 synchronised
steps each, alternated twice.  python tools/e2e_plain_vs_piped.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

wl = make_workload(2, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
xh = torch.from_numpy(wl.x.copy()).pin_memory()
yh = torch.empty_like(xh).pin_memory()
xd = torch.empty(xh.shape, dtype=torch.float64, device="cuda")
yd = torch.empty_like(xd)


def plain():
    xd.copy_(xh, non_blocking=True)
    op.apply_into(xd, yd)
    yh.copy_(yd, non_blocking=True)
    torch.cuda.current_stream().synchronize()


def piped():
    op.apply(xh, out=yh)


def steps(f, k=40):
    for _ in range(3):
        f()
    t = []
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) * 1e3)
    return t


for rep in range(2):
    for name, f in (("plain", plain), ("piped", piped)):
        t = steps(f)
        print(f"{name} rep{rep}: median {np.median(t):.0f} us, min {np.min(t):.0f}, max {np.max(t):.0f}; "
              + " ".join(f"{v:.0f}" for v in t[:12]))
print(op.host_info())
