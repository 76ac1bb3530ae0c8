"""Device plumbing: torch fp64 CUDA tensors carry the vectors, libhf does the math."""

from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from ._lib import check, lib

F64 = torch.float64


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")


def stream() -> ct.c_void_p:
    """The current torch stream (also the capture stream inside torch.cuda.graph)."""
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def is_dev(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def as_dev(x, copy: bool = False) -> torch.Tensor:
    """numpy / torch -> contiguous fp64 CUDA tensor."""
    require_cuda()
    if isinstance(x, torch.Tensor):
        t = x.to(device="cuda", dtype=F64, non_blocking=x.is_pinned() if not x.is_cuda else False)
        t = t.contiguous()
        return t.clone() if (copy and t.data_ptr() == x.data_ptr()) else t
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to("cuda")


def like_input(y: torch.Tensor, x):
    """Return y in the flavour of the caller's input (numpy in -> numpy out)."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            return y
        out = torch.empty(y.shape, dtype=y.dtype, pin_memory=x.is_pinned())
        out.copy_(y, non_blocking=x.is_pinned())
        torch.cuda.current_stream().synchronize()
        return out
    return y.cpu().numpy()


def ptr(t) -> ct.c_void_p:
    return ct.c_void_p(0 if t is None else t.data_ptr())


class Workspace:
    """Reduction scratch + a small bank of device scalars (one per device)."""

    _inst: dict[int, "Workspace"] = {}

    def __init__(self):
        h = ct.c_void_p()
        check(lib().hf_ws_create(ct.byref(h)))
        self.handle = h

    @classmethod
    def get(cls) -> "Workspace":
        dev = torch.cuda.current_device()
        if dev not in cls._inst:
            cls._inst[dev] = Workspace()
        return cls._inst[dev]


def dot(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, skip=None) -> torch.Tensor:
    check(lib().hf_dot(Workspace.get().handle, a.numel(), ptr(a), ptr(b), ptr(out), ptr(skip), stream()))
    return out


def capture_graph(fn) -> torch.cuda.CUDAGraph:
    """Capture ``fn``'s launches into a CUDA graph on a side stream.

    ``torch.cuda.graph`` empties the caching allocator on entry; a Newton
    iteration captures a fresh V-cycle graph for every rebuilt hierarchy, and
    emptying the cache each time sent every later allocation back to
    cudaMalloc.  Capturing with ``capture_begin/capture_end`` directly keeps
    the cache."""
    import gc

    g = torch.cuda.CUDAGraph()
    cur = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(cur)
    # no cyclic GC while capturing: a collected libhf handle would free device
    # memory (a device synchronisation) in the middle of the capture
    was_enabled = gc.isenabled()
    gc.disable()
    try:
        with torch.cuda.stream(side):
            g.capture_begin()
            try:
                fn()
            finally:
                g.capture_end()
    finally:
        if was_enabled:
            gc.enable()
    cur.wait_stream(side)
    return g
