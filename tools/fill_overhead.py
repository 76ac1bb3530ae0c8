"""Back-to-back cost of the fill (y = mask ? x : 0, PDL primary) in the headline
step: apply_into (fill + cell kernel) vs apply_raw (cell kernel only) vs the fill alone."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent  # noqa: E402
from paper_1904_13131_b200 import device as dv  # noqa: E402
from paper_1904_13131_b200._lib import check, lib  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

wl = make_workload(2, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
x = torch.from_numpy(wl.x).cuda()
y = torch.empty_like(x)
mask = wl.fine.mask_ptr()


def t(f, reps=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print("fill + apply (PDL): %.1f us" % t(lambda: op.apply_into(x, y)))
print("apply only (raw):   %.1f us" % t(lambda: op.apply_raw(x, y)))
print("fill only:          %.1f us" % t(lambda: check(lib().hf_fill_masked(x.numel(), dv.ptr(y), dv.ptr(x), mask, 0.0,
                                                                         dv.stream()))))
