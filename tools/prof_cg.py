"""Kernel-time breakdown of GMG-preconditioned CG iterations (torch.profiler / CUPTI).

    python tools/prof_cg.py [cfg=4] [iterations=5] [strategy=tensor4]

Builds the config's GMG hierarchy at the first Newton iterate of load step 1
(cfg 4) or at the synthetic SPD state (others), warms up, then profiles
``iterations`` CG iterations and prints per-kernel totals (JSON lines)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg, cg, compute_residual  # noqa: E402
from paper_1904_13131_b200.fespace import node_coordinates  # noqa: E402
from paper_1904_13131_b200.workloads import AMP_SOLVE, make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
its = int(sys.argv[2]) if len(sys.argv) > 2 else 5
strategy = sys.argv[3] if len(sys.argv) > 3 else "tensor4"
wl = make_workload(cfg, seed=0, levels=True, amp=AMP_SOLVE, with_x=(cfg != 4))
probs = wl.problems
fine = probs[-1]
if cfg == 4:
    X = node_coordinates(fine.mesh, fine.dofmap)
    u = torch.zeros(fine.n_dofs, dtype=torch.float64, device="cuda")
    u.view(-1, 3)[:, 2] += (-0.05 / 5) * torch.from_numpy(X[:, 2] / X[:, 2].max()).cuda()
    b = -compute_residual(fine, u)
    keep = True
else:
    u = torch.from_numpy(wl.ubar).cuda()
    b = MatrixFreeTangent(fine, u, "tensor4").apply(torch.from_numpy(wl.x).cuda())
    b[fine.mask_dev] = 0.0
    keep = False
op = MatrixFreeTangent(fine, u, strategy)
gmg = build_gmg(probs, u, strategy, seed=0, keep_constrained=keep, coarse_precision=os.environ.get("HF_COARSE_PRECISION", "fp64"))
cg(op, b, rel_tol=0.0, preconditioner=gmg, max_iterations=2)  # warm-up + graph capture
torch.cuda.synchronize()
t0 = time.perf_counter()
_, rep = cg(op, b, rel_tol=0.0, preconditioner=gmg, max_iterations=its)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    cg(op, b, rel_tol=0.0, preconditioner=gmg, max_iterations=its)
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    name = e.name[:90]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += e.device_time
tot = sum(v[1] for v in agg.values())
print(json.dumps({"cfg": cfg, "strategy": strategy, "levels": [p.mesh.cells[0] for p in probs], "iterations": its,
                  "wall_ms_per_iteration": wall / its * 1e3, "kernel_ms_per_iteration": tot / its / 1e3}))
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(json.dumps({"kernel": n, "count_per_it": c / its, "ms_per_it": t / its / 1e3, "share": t / tot}))
# per-level apply latency (warm, not L2-flushed: what the V-cycle sees)
for lv in gmg.levels:
    n = lv.problem.n_dofs
    xx = torch.randn(n, dtype=torch.float64, device="cuda")
    yy = torch.empty_like(xx)
    for _ in range(5):
        lv.op.apply_into(xx, yy)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        lv.op.apply_into(xx, yy)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"level_cells": lv.problem.mesh.cells[0], "n_dofs": n, "apply_us": e0.elapsed_time(e1) / 50 * 1e3}))
