"""Kernel-time breakdown of build_gmg (the per-Newton-iteration setup) at config 4:
python tools/prof_gmg_build.py [strategy=tensor4].  Wall time against summed kernel time
shows how much of the setup the GPU idles behind the host."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1904_13131_b200 import build_gmg  # noqa: E402
from paper_1904_13131_b200.fespace import node_coordinates  # noqa: E402
from paper_1904_13131_b200.workloads import AMP_SOLVE, make_workload  # noqa: E402

strategy = sys.argv[1] if len(sys.argv) > 1 else "tensor4"
wl = make_workload(4, seed=0, levels=True, amp=AMP_SOLVE, with_x=False)
probs = wl.problems
fine = probs[-1]
X = node_coordinates(fine.mesh, fine.dofmap)
u = torch.zeros(fine.n_dofs, dtype=torch.float64, device="cuda")
u.view(-1, fine.dim)[:, -1] += (-0.05 / 5) * torch.from_numpy(X[:, -1] / X[:, -1].max()).cuda()
for _ in range(2):
    g = build_gmg(probs, u, strategy, seed=0, keep_constrained=True)
    del g
torch.cuda.synchronize()
walls = []
for _ in range(3):
    t0 = time.perf_counter()
    g = build_gmg(probs, u, strategy, seed=0, keep_constrained=True)
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
    del g
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g = build_gmg(probs, u, strategy, seed=0, keep_constrained=True)
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = tot.setdefault(e.name[:70], [0, 0.0])
        k[0] += 1
        k[1] += e.device_time / 1e3
ksum = sum(v[1] for v in tot.values())
print(json.dumps({"build_gmg_wall_ms": walls, "kernel_ms": ksum}))
for name, (n, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:16]:
    print(json.dumps({"kernel": name, "count": n, "ms": round(ms, 3)}))
