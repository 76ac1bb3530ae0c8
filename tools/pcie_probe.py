"""Host<->device bandwidth probe for the e2e path: one copy, K concurrent
copies on K streams, and a device kernel reading pinned host memory (UVA)."""
import torch
n = 823875
xh = torch.randn(n, dtype=torch.float64).pin_memory(); yh = torch.empty_like(xh).pin_memory()
xd = xh.cuda(); yd = xd.clone()
streams = [torch.cuda.Stream() for _ in range(8)]
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def split(dst, src, k):
    def f():
        cur = torch.cuda.current_stream()
        step = -(-n // k)
        for i in range(k):
            s = streams[i]; s.wait_stream(cur)
            with torch.cuda.stream(s):
                dst[i*step:(i+1)*step].copy_(src[i*step:(i+1)*step], non_blocking=True)
        for i in range(k): cur.wait_stream(streams[i])
    return f
for k in (1, 2, 4, 8):
    h = t(split(xd, xh, k)); d = t(split(yh, yd, k))
    print(f"k={k}: H2D {h*1e3:.1f} us ({n*8/h/1e6:.1f} GB/s)  D2H {d*1e3:.1f} us ({n*8/d/1e6:.1f} GB/s)")
# zero-copy kernel read: torch elementwise op on a host-mapped view is not allowed; use a raw pointer copy
import ctypes
from cuda.bindings import runtime as rt
err, dptr = rt.cudaHostGetDevicePointer(xh.data_ptr(), 0)
print("host device pointer", err)
