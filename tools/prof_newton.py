"""Per-iteration breakdown of the whole config-4 solve (newton_solve_prescribed):
setup (tangent + GMG build), CG, residual, and the caching allocator's cudaMalloc
count, so first-iteration overheads can be attributed.
python tools/prof_newton.py [cfg=4] [runs=1] [strategy=tensor4]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_13131_b200 import NewtonSettings, solver  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
strategy = sys.argv[3] if len(sys.argv) > 3 else "tensor4"
wl = make_workload(cfg, seed=0, levels=True, with_x=False)
log = []


def wrap(name, f):
    def g(*a, **k):
        torch.cuda.synchronize()
        m0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        m1 = torch.cuda.memory_stats().get("num_device_alloc", 0)
        log.append((name, time.perf_counter() - t0, m1 - m0))
        return r
    return g


solver._make_preconditioner = wrap("setup", solver._make_preconditioner)
solver.cg = wrap("cg", solver.cg)
solver.compute_residual = wrap("residual", solver.compute_residual)

for run in range(runs):
    log.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    marks = []

    def on_record(rec):
        torch.cuda.synchronize()
        marks.append(time.perf_counter())
        log.append(("--wall", marks[-1] - (marks[-2] if len(marks) > 1 else t0), 0))

    res = solver.newton_solve_prescribed(wl.problems, NewtonSettings(), -0.05, strategy=strategy, seed=0,
                                         on_record=on_record)
    torch.cuda.synchronize()
    print(f"{strategy} run {run}: total {time.perf_counter() - t0:.3f} s, {len(res.records)} Newton iterations")
    for name, dt, nalloc in log[:16]:
        print(f"  {name:9s} {dt * 1e3:8.1f} ms  cudaMallocs {nalloc}")

# build / destroy cost of one fine-level tangent and one GMG hierarchy
from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg  # noqa: E402

fine = wl.problems[-1]
u = res.u
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = MatrixFreeTangent(fine, u, strategy)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    del op
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    g = build_gmg(wl.problems, u, strategy, seed=0, keep_constrained=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    del g
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"fine tangent build {1e3 * (t1 - t0):.1f} ms destroy {1e3 * (t2 - t1):.1f} ms; "
          f"gmg build {1e3 * (t3 - t2):.1f} ms destroy {1e3 * (t4 - t3):.1f} ms")
