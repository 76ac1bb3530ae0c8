"""Time the cell kernel (fill + apply PDL pair) of every caching variant at
configs 2 and 3 three ways: back to back, after a 256 MiB L2 flush by WRITES
(the dirty lines are written back during the timed apply), and after a CLEAN
flush (write + read of the buffer before the timed region, so the timed apply
starts with L2 holding clean foreign lines).

    python tools/time_variants.py [cfg ...] [--strategies s1,s2] [--reps N]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1904_13131_b200 import MatrixFreeTangent
from paper_1904_13131_b200.workloads import algorithmic_bytes, make_workload

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfgs = [int(a) for a in args] or [2, 3]
strategies = ("tensor4", "tensor2", "scalar")
reps = 30
for a in sys.argv[1:]:
    if a.startswith("--strategies="):
        strategies = tuple(a.split("=", 1)[1].split(","))
    if a.startswith("--reps="):
        reps = int(a.split("=", 1)[1])
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
sink = torch.empty((), dtype=torch.float32, device="cuda")
hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "MEASURED_PEAKS.json")))["hbm_gbs"]


def timed(fn, pre, n):
    ts = []
    for _ in range(n):
        pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for cfg in cfgs:
    wl = make_workload(cfg, seed=0)
    p = wl.fine
    x = torch.from_numpy(wl.x).cuda()
    y = torch.empty_like(x)
    nqp = p.mesh.n_elements * p.n_qpoints_per_cell
    for s in strategies:
        op = MatrixFreeTangent(p, wl.ubar, s)
        for _ in range(5):
            op.apply_into(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            op.apply_into(x, y)
        e1.record()
        torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) / reps * 1e3
        wflush = timed(lambda: op.apply_into(x, y), lambda: flush.zero_(), reps)
        cflush = timed(lambda: op.apply_into(x, y), lambda: (flush.zero_(), torch.sum(flush, dim=0, out=sink)), reps)
        ab = algorithmic_bytes(s, 3, p.n_dofs, nqp)
        rec = {"cfg": cfg, "strategy": s, "b2b_us": round(b2b, 2), "write_flushed_us": round(wflush, 2),
               "clean_flushed_us": round(cflush, 2), "GDoF_s_b2b": round(p.n_dofs / b2b / 1e3, 2),
               "GDoF_s_clean": round(p.n_dofs / cflush / 1e3, 2), "frac_hbm_b2b": round(ab / b2b / 1e3 / hbm, 3),
               "frac_hbm_clean": round(ab / cflush / 1e3 / hbm, 3),
               "env": {k: v for k, v in os.environ.items() if k.startswith("HF_")}}
        print(json.dumps(rec), flush=True)
        del op
