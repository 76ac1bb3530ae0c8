"""Profiling driver: tangent applies of one config for ncu.
    python tools/prof_apply.py [strategy] [cfg] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

s = sys.argv[1] if len(sys.argv) > 1 else "tensor4"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
wl = make_workload(cfg, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, s)
x = torch.from_numpy(wl.x).cuda()
y = torch.empty_like(x)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(reps):
    flush.zero_()
    op.apply_into(x, y)
d = op.diagonal()
torch.cuda.synchronize()
print("ok", s, cfg, float(y.norm()), float(d.norm()))
