"""Individual e2e step times (host-to-host apply through the public API) to see
their distribution on this host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

wl = make_workload(2, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
xh = torch.from_numpy(wl.x.copy()).pin_memory()
yh = torch.empty_like(xh).pin_memory()
for _ in range(5):
    op.apply(xh, out=yh)
print(op.host_info())
ev, wall = [], []
for _ in range(30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    op.apply(xh, out=yh)
    e1.record()
    torch.cuda.synchronize()
    wall.append((time.perf_counter() - t0) * 1e6)
    ev.append(e0.elapsed_time(e1) * 1e3)
print("event us:", " ".join(f"{v:.0f}" for v in ev))
print("wall  us:", " ".join(f"{v:.0f}" for v in wall))
print(f"median event {np.median(ev):.0f} us, min {min(ev):.0f}")
