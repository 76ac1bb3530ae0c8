import time, cProfile, pstats, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1904_13131_b200 import build_gmg, build_transfers
from paper_1904_13131_b200.fespace import node_coordinates
from paper_1904_13131_b200.workloads import make_workload
wl = make_workload(4, seed=0, levels=True, with_x=False)
probs = wl.problems; fine = probs[-1]
X = node_coordinates(fine.mesh, fine.dofmap)
tr = build_transfers(probs)
u = torch.zeros(fine.n_dofs, dtype=torch.float64, device="cuda")
u.view(-1, 3)[:, 2] += (-0.05 / 5) * torch.from_numpy(X[:, 2] / X[:, 2].max()).cuda()
for prec in ("fp64", "fp32", "fp64", "fp32"):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pr = cProfile.Profile(); pr.enable()
    g = build_gmg(probs, u, "tensor4", seed=0, transfers=tr, keep_constrained=True, coarse_precision=prec)
    torch.cuda.synchronize(); pr.disable()
    print(prec, "build_gmg %.1f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
    del g
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
