cd $GRAFT_REPO_ROOT
timeout 1500 python - <<'PY' 2>&1 | grep -v Warn
import sys, json, time, gc
sys.argv=['bench.py']
import bench, torch
import numpy as np
from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg, build_transfers, cg, compute_residual
from paper_1904_13131_b200.fespace import node_coordinates
from paper_1904_13131_b200.workloads import make_workload
wl = make_workload(4, seed=0, levels=True, with_x=False)
probs = wl.problems; fine = probs[-1]
X = node_coordinates(fine.mesh, fine.dofmap)
transfers = build_transfers(probs)
def one(prec, disable_gc=False):
    u = torch.zeros(fine.n_dofs, dtype=torch.float64, device="cuda")
    u.view(-1, 3)[:, 2] += (-0.05 / 5) * torch.from_numpy(X[:, 2] / X[:, 2].max()).cuda()
    res = compute_residual(fine, u)
    torch.cuda.synchronize(); t0=time.perf_counter()
    op = MatrixFreeTangent(fine, u, "tensor4")
    gmg = build_gmg(probs, u, "tensor4", seed=0, transfers=transfers, keep_constrained=True, coarse_precision=prec)
    torch.cuda.synchronize(); t1=time.perf_counter()
    if disable_gc: gc.disable()
    du, rep = cg(op, -res, rel_tol=1e-6, preconditioner=gmg)
    torch.cuda.synchronize(); t2=time.perf_counter()
    # second solve with the same (already captured) preconditioner
    du, rep2 = cg(op, -res, rel_tol=1e-6, preconditioner=gmg)
    torch.cuda.synchronize(); t3=time.perf_counter()
    if disable_gc: gc.enable()
    print(prec, 'gc_off' if disable_gc else 'gc_on', 'setup %.1f ms  cg first %.2f ms/it  cg second %.2f ms/it  its %d'%((t1-t0)*1e3,(t2-t1)/rep.iterations*1e3,(t3-t2)/rep2.iterations*1e3,rep.iterations), flush=True)
    del op, gmg
for prec in ('fp64','fp32','fp32','fp64','fp32','fp32','fp32','fp64','fp32'):
    one(prec)
for prec in ('fp32','fp32','fp32','fp32'):
    one(prec, True)
PY
