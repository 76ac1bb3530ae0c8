"""e2e step time through MatrixFreeTangent.apply(x_host, out=y_host) for pinned
buffers obtained different ways (torch pin_memory() copy vs torch.empty(pin_memory=True)
vs cudaHostAlloc via hf_host_register of numpy memory)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_13131_b200 import MatrixFreeTangent  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

wl = make_workload(2, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
n = wl.fine.n_dofs


def steps(xh, yh, k=20):
    for _ in range(3):
        op.apply(xh, out=yh)
    ts = []
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply(xh, out=yh)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return f"median {ts[len(ts) // 2]:.1f} us min {ts[0]:.1f} max {ts[-1]:.1f}"


ms, h2d, d2h = bench._e2e(op.apply_into, wl.x, 10, 5, public_apply=op.apply)
print(f"bench._e2e: {ms * 1e3:.1f} us per step")
a = torch.from_numpy(wl.x.copy()).pin_memory()
b = torch.empty_like(a).pin_memory()
print("from_numpy().pin_memory():", steps(a, b))
c = torch.empty(n, dtype=torch.float64, pin_memory=True)
c.copy_(torch.from_numpy(wl.x))
d = torch.empty(n, dtype=torch.float64, pin_memory=True)
print("torch.empty(pin_memory=True):", steps(c, d))
print("from_numpy().pin_memory() again:", steps(a, b))
for ch in (2, 4, 8):
    print(op.host_info())
    def f(ch=ch):
        op.apply_host(c, d, chunks=ch)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"apply_host chunks={ch}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
