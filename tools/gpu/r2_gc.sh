cd $GRAFT_REPO_ROOT
timeout 600 python - <<'PY' 2>&1 | grep -v Warn
import gc, weakref, numpy as np, torch
from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg, build_transfers, cg
from paper_1904_13131_b200.workloads import make_workload, AMP_SOLVE
gc.disable()
wl = make_workload(1, seed=0, levels=True, amp=AMP_SOLVE)
probs = wl.problems
u = torch.from_numpy(wl.ubar).cuda()
op = MatrixFreeTangent(probs[-1], u, "tensor4")
gmg = build_gmg(probs, u, "tensor4", seed=0)
b = op.apply(torch.from_numpy(wl.x).cuda()); b[probs[-1].mask_dev] = 0
cg(op, b, rel_tol=1e-8, preconditioner=gmg)
refs = {"op": weakref.ref(op), "gmg": weakref.ref(gmg), "level_op": weakref.ref(gmg.levels[-1].op), "level": weakref.ref(gmg.levels[-1])}
del op, gmg
print("alive after del (refcount only):", {k: r() is not None for k, r in refs.items()})
n = gc.collect()
print("gc.collect() found", n, "objects; alive:", {k: r() is not None for k, r in refs.items()})
PY
