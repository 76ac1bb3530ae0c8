"""Time MatrixFreeTangent.apply_into (L2 flushed) for one config/strategy: python tools/time_apply.py [strategy] [cfg]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_13131_b200 import MatrixFreeTangent
from paper_1904_13131_b200.workloads import make_workload
s = sys.argv[1] if len(sys.argv) > 1 else "tensor4"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = make_workload(cfg, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, s)
x = torch.from_numpy(wl.x).cuda(); y = torch.empty_like(x)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
ts = []
for k in range(25):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); op.apply_into(x, y); e1.record(); torch.cuda.synchronize()
    if k >= 5: ts.append(e0.elapsed_time(e1) * 1000)
ts.sort()
# back-to-back (no flush; the cache stream exceeds L2 at configs 2-5): resolution / reps
reps = 40
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    op.apply_into(x, y)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"strategy": s, "cfg": cfg, "env": {k: v for k, v in os.environ.items() if k.startswith("HF_")},
                  "median_us": ts[len(ts) // 2], "min_us": ts[0], "b2b_us": e0.elapsed_time(e1) / reps * 1e3,
                  "ynorm": float(y.norm())}))
