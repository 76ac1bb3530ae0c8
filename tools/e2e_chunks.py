"""Host-to-host apply (hf_tangent_apply_host) step time vs the number of slabs
the pipeline cuts the cells into: python tools/e2e_chunks.py [chunks ...]"""
import json
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
ref = op.apply(torch.from_numpy(wl.x).cuda()).cpu()
out = {}
for chunks in [int(c) for c in sys.argv[1:]] or [2, 4, 6, 8, 12, 16]:
    yh = torch.empty_like(xh).pin_memory()  # a fresh buffer pair: its own calibration
    for _ in range(5):
        op.apply_host(xh, yh, chunks=chunks)
    t = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply_host(xh, yh, chunks=chunks)
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) * 1e3)
    assert torch.equal(yh, ref) or float((yh - ref).norm() / ref.norm()) < 1e-14
    out[chunks] = {"median_us": float(np.median(t)), "min_us": float(np.min(t)), "info": op.host_info()}
print(json.dumps(out))
