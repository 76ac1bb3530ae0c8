"""Time of one Chebyshev smoothing (2 steps x degree 4 = 8 applications and
updates, graph-replayed) on an m^3 Q2 level: python tools/smoother_time.py [m ...]
(HF_ALTERNATE=0 turns off the alternating sweep direction)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_13131_b200.multigrid import ChebyshevSettings, LevelOperator  # noqa: E402
from paper_1904_13131_b200.workloads import AMP_SOLVE, make_workload  # noqa: E402

for m in [int(a) for a in sys.argv[1:]] or [32, 64]:
    wl = make_workload(4, seed=0, m=m, amp=AMP_SOLVE)
    p = wl.fine
    lv = LevelOperator(p, torch.from_numpy(wl.ubar).cuda(), "tensor4", seed=0, level=1)
    b = torch.from_numpy(wl.x).cuda()
    b[p.mask_dev] = 0.0
    x = torch.zeros_like(b)

    def run():
        lv.smooth_into(b, x, 2, ChebyshevSettings(), x_zero=False)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"m={m} alternate={os.environ.get('HF_ALTERNATE', '1')} smoothing {e0.elapsed_time(e1) / 20 * 1e3:.1f} us "
          f"({e0.elapsed_time(e1) / 20 / 8 * 1e3:.1f} us per application + update)", flush=True)
