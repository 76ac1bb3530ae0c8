"""Apply on a small level (latency study): python tools/prof_small.py [m=4] [strategy] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_13131_b200 import MatrixFreeTangent
from paper_1904_13131_b200.workloads import make_workload, AMP_SOLVE
m = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = sys.argv[2] if len(sys.argv) > 2 else "tensor4"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
wl = make_workload(4, seed=0, m=m, amp=AMP_SOLVE)
op = MatrixFreeTangent(wl.fine, wl.ubar, s)
x = torch.from_numpy(wl.x).cuda(); y = torch.empty_like(x)
for _ in range(reps):
    op.apply_into(x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    op.apply_into(x, y)
e1.record(); torch.cuda.synchronize()
print("ok", m, s, e0.elapsed_time(e1) / reps * 1e3, "us/apply", float(y.norm()))
