"""GPU timeline (CUPTI via torch.profiler) of one e2e step: plain copy/apply/copy
and the slab-pipelined apply_host, to see where the host->host step time goes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

wl = make_workload(2, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
xh = torch.empty(wl.x.size, dtype=torch.float64, pin_memory=True)
xh.copy_(torch.from_numpy(wl.x))
yh = torch.empty(wl.x.size, dtype=torch.float64, pin_memory=True)
xd = xh.cuda()
yd = torch.empty_like(xd)


def plain():
    xd.copy_(xh, non_blocking=True)
    op.apply_into(xd, yd)
    yh.copy_(yd, non_blocking=True)
    torch.cuda.synchronize()


variants = [("plain", plain)] + [(f"piped{c}", (lambda c=c: op.apply_host(xh, yh, chunks=c))) for c in
                                  (int(a) for a in (sys.argv[1:] or ["2", "4"]))]
for name, f in variants:
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            f()
        torch.cuda.synchronize()
    ev = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
    if not ev:
        continue
    # last step only: split at the largest gap-free group is fiddly; print all three steps
    t0 = ev[0].time_range.start
    print(f"== {name}")
    for e in ev:
        print(f"  {e.time_range.start - t0:8.1f} +{e.time_range.end - e.time_range.start:7.1f} us "
              f"stream {getattr(e, 'device_resource_id', '?')}  {e.name[:60]}")
