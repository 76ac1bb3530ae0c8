"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once on tiny problems.  python tools/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_13131_b200 import (AssembledTangent, MatrixFreeTangent, build_gmg, cg, compute_residual,  # noqa: E402
                                   energy)
from paper_1904_13131_b200.workloads import AMP_SOLVE, make_workload  # noqa: E402

for cfg, m in ((2, 4), (1, 4), (3, 2)):
    wl = make_workload(cfg, seed=0, m=m, amp=AMP_SOLVE, levels=(cfg != 3))
    p = wl.fine
    for s in ("scalar", "tensor2", "tensor4"):
        op = MatrixFreeTangent(p, wl.ubar, s)
        y = op.apply(wl.x)
        d = op.diagonal()
        y32 = MatrixFreeTangent(p, wl.ubar, s, storage="fp32").apply(wl.x)
    r = compute_residual(p, wl.ubar)
    e = energy(p, wl.ubar)
    if cfg != 3:
        AssembledTangent(p, wl.ubar).apply(wl.x)
        gmg = build_gmg(wl.problems, wl.ubar, "tensor4", seed=0)
        b = torch.from_numpy(y).cuda()
        b[p.mask_dev] = 0.0
        x, rep = cg(MatrixFreeTangent(p, wl.ubar, "tensor4"), b, rel_tol=1e-8, preconditioner=gmg)
        print("cfg", cfg, "cg iterations", rep.iterations)
    torch.cuda.synchronize()
print("sanitize case ok")
