"""cProfile of the whole config-4 solve (host-side attribution of the wall time
outside setup/CG/residual).  python tools/prof_newton_cprof.py [runs=2]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_13131_b200 import NewtonSettings, solver  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = make_workload(4, seed=0, levels=True, with_x=False)
for run in range(runs):
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    solver.newton_solve_prescribed(wl.problems, NewtonSettings(), -0.05, seed=0)
    torch.cuda.synchronize()
    pr.disable()
    print(f"run {run}: {time.perf_counter() - t0:.3f} s")
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)
