"""Host-side cost of one e2e step: wall time of MatrixFreeTangent.apply(x_host,
out=y_host) and of its pieces, against the GPU-side span of the graph."""
import ctypes as ct
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent  # noqa: E402
from paper_1904_13131_b200 import device as dv  # noqa: E402
from paper_1904_13131_b200._lib import check, lib  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

wl = make_workload(2, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
n = wl.fine.n_dofs
xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
xh.copy_(torch.from_numpy(wl.x))
yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
L = lib()


def wall(f, k=30):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e6


def raw():
    check(L.hf_tangent_apply_host(op._op, ct.c_void_p(xh.data_ptr()), ct.c_void_p(yh.data_ptr()), 4, dv.stream()))
    torch.cuda.current_stream().synchronize()


def raw_nosync():
    check(L.hf_tangent_apply_host(op._op, ct.c_void_p(xh.data_ptr()), ct.c_void_p(yh.data_ptr()), 4, dv.stream()))


print("public apply(x_host, out=y_host): %.1f us wall" % wall(lambda: op.apply(xh, out=yh)))
print("hf_tangent_apply_host + sync:     %.1f us wall" % wall(raw))
print("hf_tangent_apply_host, no sync:   %.1f us wall (queue-bound)" % wall(raw_nosync))
t0 = time.perf_counter()
for _ in range(100):
    xh.is_pinned()
print("is_pinned: %.1f us" % ((time.perf_counter() - t0) / 100 * 1e6))
print(op.host_info())
