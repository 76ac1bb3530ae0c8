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


class LaunchGraph:
    """A launch sequence recorded through libhf (hf_graph_*) and replayed as one
    CUDA graph.  ``key`` names the shape of the sequence: when the graph is
    dropped its executable goes to an idle list under that key, and the next
    graph recorded under the same key updates it in place instead of
    instantiating a new one (a Newton iteration rebuilds the hierarchy with the
    same launch sequence and new pointers / coefficients: ~1 ms instead of
    3-9 ms, and none of the occasional 50-80 ms instantiations)."""

    _idle: dict = {}
    MAX_IDLE = 2

    def __init__(self, fn, key=None):
        import gc

        self.key = key
        self.updated = False
        idle = LaunchGraph._idle.get(key) if key is not None else None
        h = ct.c_void_p(idle.pop()) if idle else ct.c_void_p()
        reused = bool(h)
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        # no cyclic GC while recording: a collected libhf handle would free
        # device memory (a device synchronisation) in the middle of it
        was_enabled = gc.isenabled()
        gc.disable()
        upd = ct.c_int(0)
        try:
            with torch.cuda.stream(side):
                check(lib().hf_graph_begin(stream()))
                try:
                    fn()
                except BaseException:
                    dead = ct.c_void_p()
                    lib().hf_graph_end(stream(), ct.byref(dead), None)  # close the recording
                    if dead:
                        lib().hf_graph_destroy(dead)
                    raise
                check(lib().hf_graph_end(stream(), ct.byref(h), ct.byref(upd)))
        except BaseException:
            if reused and h:
                lib().hf_graph_destroy(h)
            raise
        finally:
            if was_enabled:
                gc.enable()
        cur.wait_stream(side)
        self._h = h
        self.updated = bool(upd.value)

    def replay(self) -> None:
        check(lib().hf_graph_launch(self._h, stream()))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if not h:
            return
        try:
            idle = LaunchGraph._idle.setdefault(self.key, []) if self.key is not None else None
            if idle is not None and len(idle) < self.MAX_IDLE:
                idle.append(h.value)  # later work queued on it has been launched; the executable stays valid
            else:
                lib().hf_graph_destroy(h)
        except Exception:  # interpreter teardown
            pass
