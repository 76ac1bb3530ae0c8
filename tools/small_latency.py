"""Latency of small-level work inside a CUDA graph (what the V-cycle sees).

    python tools/small_latency.py [m ...]

For each m^3 Q2 level (config-4 recipe): the graph-replayed coarse solve
(99 applications + Chebyshev updates + norm checks), and a graph of 50 plain
applications (fill + cell kernel), each as us per application."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_13131_b200.multigrid import LevelOperator, _coarse_solve_into  # noqa: E402
from paper_1904_13131_b200.workloads import AMP_SOLVE, make_workload  # noqa: E402


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for m in [int(a) for a in sys.argv[1:]] or [4, 8, 16]:
    wl = make_workload(4, seed=0, m=m, amp=AMP_SOLVE)
    p = wl.fine
    lv = LevelOperator(p, torch.from_numpy(wl.ubar).cuda(), "tensor4", seed=0, level=0, is_coarsest=True)
    b = torch.from_numpy(wl.x).cuda()
    b[p.mask_dev] = 0.0
    x = torch.zeros_like(b)
    y = torch.empty_like(b)
    tc = graph_time(lambda: _coarse_solve_into(lv, b, x))

    def applies():
        for _ in range(50):
            lv.op.apply_into(b, y)

    ta = graph_time(applies)
    print(f"m={m} n_dofs={p.n_dofs} coarse_solve {tc:.1f} us ({tc / 99:.2f} us per application) "
          f"plain apply {ta / 50:.2f} us", flush=True)
