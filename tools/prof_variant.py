"""Run a few applies of one variant (the ncu target): python tools/prof_variant.py strategy cfg [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1904_13131_b200 import MatrixFreeTangent
from paper_1904_13131_b200.workloads import make_workload

s, cfg = sys.argv[1], int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
wl = make_workload(cfg, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, s)
x = torch.from_numpy(wl.x).cuda()
y = torch.empty_like(x)
for _ in range(n):
    op.apply_into(x, y)
torch.cuda.synchronize()
print("done", s, cfg, float(y.norm()))
