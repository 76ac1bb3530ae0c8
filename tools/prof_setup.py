"""Newton-iteration setup breakdown at config 4 (64^3 Q2, levels 4..64):
per level the tangent build, the diagonal and the Lanczos range estimate(s),
then build_gmg as a whole.  python tools/prof_setup.py [cfg=4]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg, restrict_solution  # noqa: E402
from paper_1904_13131_b200.fespace import node_coordinates  # noqa: E402
from paper_1904_13131_b200.multigrid import estimate_eigenvalue_range  # noqa: E402
from paper_1904_13131_b200.workloads import AMP_SOLVE, make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = make_workload(cfg, seed=0, levels=True, amp=AMP_SOLVE, with_x=False)
probs = wl.problems
fine = probs[-1]
X = node_coordinates(fine.mesh, fine.dofmap)
u = torch.zeros(fine.n_dofs, dtype=torch.float64, device="cuda")
u.view(-1, fine.dim)[:, -1] += (-0.05 / 5) * torch.from_numpy(X[:, -1] / X[:, -1].max()).cuda()


def timed(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


build_gmg(probs, u, "tensor4", seed=0, keep_constrained=True)  # warm-up (allocator, module init)
us = restrict_solution(probs, u, keep_constrained=True)
for lvl, (p, ul) in enumerate(zip(probs, us)):
    op, t_build = timed(lambda: MatrixFreeTangent(p, ul, "tensor4"))
    d, t_diag = timed(lambda: op.diagonal())
    mask = p.constraints.mask
    _, t_l30 = timed(lambda: estimate_eigenvalue_range(op, d, seed=0, constrained=mask))
    rec = {"level": lvl, "cells": p.mesh.cells[0], "n_dofs": p.n_dofs, "build_ms": t_build, "diag_ms": t_diag,
           "lanczos30_ms": t_l30}
    if lvl == 0:
        _, t_l120 = timed(lambda: estimate_eigenvalue_range(op, d, seed=0, iterations=min(p.n_dofs, 120),
                                                            constrained=mask))
        rec["lanczos120_ms"] = t_l120
    print(json.dumps(rec), flush=True)
_, t_r = timed(lambda: restrict_solution(probs, u, keep_constrained=True))
_, t_g = timed(lambda: build_gmg(probs, u, "tensor4", seed=0, keep_constrained=True))
print(json.dumps({"restrict_solution_ms": t_r, "build_gmg_ms": t_g}))

if os.environ.get("PROF_LANCZOS"):
    from torch.profiler import ProfilerActivity, profile

    p, ul = probs[-1], us[-1]
    op = MatrixFreeTangent(p, ul, "tensor4")
    d = op.diagonal()
    estimate_eigenvalue_range(op, d, seed=0, constrained=p.constraints.mask)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        estimate_eigenvalue_range(op, d, seed=0, constrained=p.constraints.mask)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=12, max_name_column_width=60))
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=60))
