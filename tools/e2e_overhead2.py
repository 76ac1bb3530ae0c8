"""Where the e2e step time goes beyond the C-level calibration: host wall time
of (a) the C call alone + stream sync, (b) MatrixFreeTangent.apply_host,
(c) MatrixFreeTangent.apply(x, out=y), (d) (c) bracketed by CUDA events as
bench.py times it.  python tools/e2e_overhead2.py"""
import ctypes as ct
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_13131_b200 import MatrixFreeTangent  # noqa: E402
from paper_1904_13131_b200 import device as dv  # noqa: E402
from paper_1904_13131_b200._lib import lib  # noqa: E402
from paper_1904_13131_b200.workloads import make_workload  # noqa: E402

wl = make_workload(2, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
xh = torch.from_numpy(wl.x.copy()).pin_memory()
yh = torch.empty_like(xh).pin_memory()
op.apply_host(xh, yh)
L = lib()
s = torch.cuda.current_stream()
sp = dv.stream()


def c_call():
    L.hf_tangent_apply_host(op._op, ct.c_void_p(xh.data_ptr()), ct.c_void_p(yh.data_ptr()), 4, sp)
    s.synchronize()


def host(fn, n=40, gap=0.0):
    t = []
    for _ in range(n):
        if gap:
            time.sleep(gap)
        t0 = time.perf_counter()
        fn()
        t.append((time.perf_counter() - t0) * 1e6)
    return round(float(np.median(t)), 1), round(float(np.min(t)), 1)


def evts(fn, n=40):
    t = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) * 1e3)
    return round(float(np.median(t)), 1), round(float(np.min(t)), 1)


out = {"info": op.host_info()}
out["c_call"] = host(c_call)
out["c_call_gap_1ms"] = host(c_call, gap=1e-3)
out["apply_host"] = host(lambda: op.apply_host(xh, yh))
out["apply_out"] = host(lambda: op.apply(xh, out=yh))
out["apply_out_events"] = evts(lambda: op.apply(xh, out=yh))
out["c_call_events"] = evts(c_call)
print(json.dumps(out))
