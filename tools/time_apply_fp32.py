"""Back-to-back apply time of the fp64 and the fp32-storage tangent (the
fp32 multigrid-level form) on one config: python tools/time_apply_fp32.py [cfg=4] [strategy=tensor4]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = sys.argv[2] if len(sys.argv) > 2 else "tensor4"
wl = make_workload(cfg, seed=0, with_x=False)
p = wl.fine
u = torch.zeros(p.n_dofs, dtype=torch.float64, device="cuda")
x = torch.randn(p.n_dofs, dtype=torch.float64, device="cuda")
out = {"cfg": cfg, "strategy": s}
for storage in ("fp64", "fp32"):
    op = MatrixFreeTangent(p, u, s, storage=storage)
    xx = x if storage == "fp64" else x.float()
    yy = torch.empty_like(xx)
    for _ in range(5):
        op.apply_into(xx, yy)
    reps = 30
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        op.apply_into(xx, yy)
    e1.record()
    torch.cuda.synchronize()
    out[storage + "_us"] = e0.elapsed_time(e1) / reps * 1e3
    out[storage + "_storage_MB"] = op.storage_bytes() / 1e6
    del op
print(json.dumps(out))
