"""Multi-GPU slab decomposition of the matrix-free tangent, GMG and CG.

The reference is single-process; the paper partitioned cells
over MPI ranks.  Here one process drives one GPU:

* **Partition.**  Cells are cut into contiguous slabs along the last axis (z in
  3D, y in 2D), one slab per rank, nested across GMG levels (a rank's coarse
  slab is its fine slab halved).  With x fastest and the last axis slowest in
  the reference numbering (fespace.py:3-8), a slab's lattice nodes are a
  CONTIGUOUS range of global DoFs: the local vector of a rank is the slice
  ``global[offset : offset + n_local]``.  Neighbouring slabs share one node
  plane (the interface), which both ranks store.
* **Consistency.**  Every distributed vector keeps identical values in both
  copies of an interface plane.  Inputs of the operator are therefore
  complete; one exchange per application suffices: the reverse add of the
  partial sums on the interface plane (``SlabExchange.add``, NCCL send/recv,
  then ``hf_halo_add``).  Constrained rows hold the identity value on both
  ranks and are not added.
* **Dots.**  Summed over the OWNED DoFs (a rank does not own its lower
  interface plane), then all-reduced.
* **Coarse levels.**  Levels whose slabs would be thinner than ``min_cells``
  cells are replicated on every rank.  The restricted residual enters them
  through an all-reduce of the zero-padded partial sums; every rank runs the
  replicated V-cycle (the single-GPU ``GMGPreconditioner``, graph-captured) and
  prolongates from its own slice.

``Comm`` abstracts the transport: ``TorchComm`` over ``torch.distributed``
(NCCL on the GPU box; gloo stages through host memory, used to run several
ranks on one GPU in the tests), ``LocalComm`` for one rank.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import device as dv
from ._lib import check, lib
from .fespace import ConstraintSet
from .material import NonPositiveJacobian
from .mesh import Mesh, sub_box
from .multigrid import (ChebyshevSettings, GMGPreconditioner, TransferOperator, _cheb_coeffs, build_level_operators,
                        build_transfers)
from .operators import Material, MatrixFreeTangent, Problem, compute_residual


# ---------------------------------------------------------------------------
# transport
# ---------------------------------------------------------------------------


class LocalComm:
    """One rank: every collective is the identity."""

    rank, size = 0, 1

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        return t

    def exchange(self, sends: dict, recvs: dict) -> None:
        if sends or recvs:
            raise ValueError("a single rank has no neighbours")

    def exchange_start(self, sends: dict, recvs: dict):
        self.exchange(sends, recvs)
        return _Done()

    def barrier(self) -> None:
        pass


class _Done:
    def wait(self):
        pass


class _Works:
    def __init__(self, works):
        self.works = works

    def wait(self):
        for w in self.works:
            w.wait()


def _nccl_sms(exchange) -> int:
    """SMs left to a concurrent NCCL exchange kernel (HF_NCCL_SMS, default 4);
    0 for host-staged transports."""
    comm = getattr(exchange, "comm", None)
    if comm is None or getattr(comm, "staged", True):
        return 0
    return int(os.environ.get("HF_NCCL_SMS", "4"))


class TorchComm:
    """torch.distributed transport (nccl: device buffers; gloo: staged through host)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.staged = dist.get_backend(group) != "nccl"

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.staged and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)
        return t

    def exchange_start(self, sends: dict, recvs: dict):
        """Start the swap; returns a handle whose ``wait()`` orders the current
        stream after it (NCCL: asynchronous on the device; staged: completed here)."""
        if self.staged:
            self.exchange(sends, recvs)
            return _Done()
        dist = self.dist
        ops = [dist.P2POp(dist.isend, sends[p], p, self.group) for p in sorted(sends)]
        ops += [dist.P2POp(dist.irecv, recvs[p], p, self.group) for p in sorted(recvs)]
        return _Works(dist.batch_isend_irecv(ops) if ops else [])

    def exchange(self, sends: dict, recvs: dict) -> None:
        """Point-to-point swap: ``sends[peer]`` -> peer, ``recvs[peer]`` <- peer."""
        dist = self.dist
        if self.staged:
            s_h = {p: t.cpu() for p, t in sends.items()}
            r_h = {p: torch.empty(t.shape, dtype=t.dtype) for p, t in recvs.items()}
            ops = [dist.P2POp(dist.isend, s_h[p], p, self.group) for p in sorted(s_h)]
            ops += [dist.P2POp(dist.irecv, r_h[p], p, self.group) for p in sorted(r_h)]
            for w in dist.batch_isend_irecv(ops) if ops else []:
                w.wait()
            for p, t in recvs.items():
                t.copy_(r_h[p])
            return
        ops = [dist.P2POp(dist.isend, sends[p], p, self.group) for p in sorted(sends)]
        ops += [dist.P2POp(dist.irecv, recvs[p], p, self.group) for p in sorted(recvs)]
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()

    def barrier(self) -> None:
        self.dist.barrier(group=self.group)


class CommTimer:
    """Optional device-side timing of the collectives (config 5 reports the
    interface exchange and the dot-product all-reduce separately): CUDA event
    pairs on the current stream, summed when read."""

    def __init__(self):
        self.events = {"exchange": [], "allreduce": []}

    def span(self, kind: str):
        timer = self

        class _Span:
            def __enter__(self_):
                self_.e0 = torch.cuda.Event(enable_timing=True)
                self_.e1 = torch.cuda.Event(enable_timing=True)
                self_.e0.record()

            def __exit__(self_, *a):
                self_.e1.record()
                timer.events[kind].append((self_.e0, self_.e1))

        return _Span()

    def totals_ms(self) -> dict:
        torch.cuda.synchronize()
        return {k: float(sum(a.elapsed_time(b) for a, b in v)) for k, v in self.events.items()} | \
            {f"n_{k}": len(v) for k, v in self.events.items()}

    def reset(self):
        for v in self.events.values():
            v.clear()


class _NoTimer:
    def span(self, kind):
        return _NULL


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


_NULL = _Null()
NO_TIMER = _NoTimer()


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------


def slab_ranges(n_cells: int, size: int) -> list[tuple[int, int]]:
    """Balanced contiguous cell ranges along the slab axis, one per rank."""
    if size < 1 or n_cells < size:
        raise ValueError(f"cannot cut {n_cells} cell layers into {size} slabs")
    base, extra = divmod(n_cells, size)
    out, c = [], 0
    for r in range(size):
        n = base + (1 if r < extra else 0)
        out.append((c, c + n))
        c += n
    return out


@dataclass(frozen=True)
class Slab:
    """One rank's box of a level: cells [c0, c1) along the last axis."""

    dim: int
    degree: int
    cells: tuple  # global cells per axis
    c0: int
    c1: int

    @property
    def axis(self) -> int:
        return self.dim - 1

    @property
    def plane_nodes(self) -> int:
        return int(np.prod([c * self.degree + 1 for c in self.cells[:-1]]))

    @property
    def plane_dofs(self) -> int:
        return self.plane_nodes * self.dim

    @property
    def n_global_dofs(self) -> int:
        return self.plane_dofs * (self.cells[-1] * self.degree + 1)

    @property
    def dof_offset(self) -> int:
        """First global DoF of the slab (its lower node plane)."""
        return self.c0 * self.degree * self.plane_dofs

    @property
    def n_dofs(self) -> int:
        return ((self.c1 - self.c0) * self.degree + 1) * self.plane_dofs

    @property
    def has_lower(self) -> bool:
        return self.c0 > 0

    @property
    def has_upper(self) -> bool:
        return self.c1 < self.cells[-1]

    @property
    def owned(self) -> slice:
        """Local DoFs this rank owns (the lower interface plane belongs to the rank below)."""
        return slice(self.plane_dofs if self.has_lower else 0, self.n_dofs)

    def local(self, v_global):
        return v_global[self.dof_offset:self.dof_offset + self.n_dofs]

    def halved(self) -> "Slab":
        if self.c0 % 2 or self.c1 % 2 or any(c % 2 for c in self.cells):
            raise ValueError("slab does not coarsen 2:1")
        return Slab(self.dim, self.degree, tuple(c // 2 for c in self.cells), self.c0 // 2, self.c1 // 2)

    # --- the part interface shared with Box (DistProblem, DistGMG, DistHierarchy)
    @property
    def has_top(self) -> bool:
        return not self.has_upper

    def sub_mesh(self, global_mesh: Mesh) -> Mesh:
        return sub_box(global_mesh, self.axis, self.c0, self.c1)

    def put_local(self, full: torch.Tensor, part: torch.Tensor) -> None:
        full[self.dof_offset:self.dof_offset + self.n_dofs] = part

    def take_local(self, full: torch.Tensor) -> torch.Tensor:
        return full[self.dof_offset:self.dof_offset + self.n_dofs]

    def put_owned(self, full: torch.Tensor, part: torch.Tensor) -> None:
        o = self.owned
        full[self.dof_offset + o.start:self.dof_offset + o.stop] = part[o]

    def make_exchange(self, comm, mask_dev: torch.Tensor):
        return SlabExchange(self, comm, mask_dev)


def level_slabs(dim: int, degree: int, fine_cells: tuple, n_levels: int, rank: int, size: int,
                min_cells: int = 2) -> list:
    """Slabs of rank ``rank`` on every level, coarsest first.  A level is
    distributed while every rank's slab keeps >= ``min_cells`` cell layers and
    the slabs nest 2:1; the levels below, and always the coarsest, are
    replicated (None)."""
    ranges = slab_ranges(fine_cells[-1], size)
    if min(b - a for a, b in ranges) < min(min_cells, fine_cells[-1] // size):
        raise ValueError("the finest level is too thin to partition")
    cells = tuple(fine_cells)
    out = [Slab(dim, degree, cells, *ranges[rank])]
    for _ in range(n_levels - 2):
        ok = out[0] is not None and all(a % 2 == 0 and b % 2 == 0 for a, b in ranges) and \
            all(c % 2 == 0 for c in cells) and min(b - a for a, b in ranges) // 2 >= min_cells
        if ok:
            ranges = [(a // 2, b // 2) for a, b in ranges]
            cells = tuple(c // 2 for c in cells)
            out.insert(0, out[0].halved())
        else:
            out.insert(0, None)
    if n_levels > 1:
        out.insert(0, None)  # the coarsest level is always replicated
    return out


def morton_boxes(cells: tuple, size: int) -> list[tuple[tuple, tuple]]:
    """Cell boxes of a Morton (Z-order) partition into ``size`` = 2^k contiguous
    chunks of the space-filling curve (the paper's p4est
    partition).  On a box whose cell counts are divisible the
    chunks are boxes: the curve's first bisection halves the last axis, the
    next the one before it, and so on cyclically, so 2 ranks get z-halves, 4
    get (z, y) quarters and 8 get octants.  Returns [(lo, hi)] in rank (curve)
    order."""
    dim = len(cells)
    if size < 1 or size & (size - 1):
        raise ValueError(f"a Morton partition needs a power-of-two rank count, got {size}")
    boxes = [(tuple(0 for _ in cells), tuple(cells))]
    level = 0
    while len(boxes) < size:
        axis = dim - 1 - (level % dim)
        out = []
        for lo, hi in boxes:
            n = hi[axis] - lo[axis]
            if n < 2 or n % 2:
                raise ValueError(f"cannot bisect {n} cells along axis {axis}")
            mid = lo[axis] + n // 2
            out.append((lo, tuple(mid if a == axis else h for a, h in enumerate(hi))))
            out.append((tuple(mid if a == axis else l for a, l in enumerate(lo)), hi))
        boxes = out
        level += 1
    return boxes


@dataclass(frozen=True)
class Box:
    """One rank's box of a level in a general box partition: cells
    [lo_a, hi_a) on every axis.  ``boxes`` holds every rank's (lo, hi), so the
    owner and the neighbours of each interface node follow locally.  The rank's
    vector is its box's node lattice (interface nodes included), a gather of
    the global vector (``global_dofs``); a node is owned by the lowest rank
    whose closed box contains it."""

    dim: int
    degree: int
    cells: tuple   # global cells per axis
    rank: int
    boxes: tuple   # ((lo, hi), ...) of every rank

    @property
    def lo(self) -> tuple:
        return self.boxes[self.rank][0]

    @property
    def hi(self) -> tuple:
        return self.boxes[self.rank][1]

    @property
    def local_cells(self) -> tuple:
        return tuple(h - l for l, h in zip(self.lo, self.hi))

    @property
    def local_nodes(self) -> tuple:
        return tuple(c * self.degree + 1 for c in self.local_cells)

    @property
    def n_dofs(self) -> int:
        return int(np.prod(self.local_nodes)) * self.dim

    @property
    def n_global_dofs(self) -> int:
        return int(np.prod([c * self.degree + 1 for c in self.cells])) * self.dim

    @property
    def has_top(self) -> bool:
        """The box holds part of the domain's top face (the traction face)."""
        return self.hi[-1] == self.cells[-1]

    def _node_grid(self, lo_n, hi_n):
        """Global node ids of the node box [lo_n, hi_n] (inclusive), x fastest."""
        gn = [c * self.degree + 1 for c in self.cells]
        axes = [np.arange(l, h + 1) for l, h in zip(lo_n, hi_n)]
        strides = np.cumprod([1] + gn[:-1])
        idx = np.zeros((1,) * self.dim, dtype=np.int64)
        for a in range(self.dim):
            shape = [1] * self.dim
            shape[self.dim - 1 - a] = len(axes[a])
            idx = idx + (axes[a] * strides[a]).reshape(shape)
        return idx.reshape(-1)

    def _node_box(self, r: int):
        lo, hi = self.boxes[r]
        return tuple(l * self.degree for l in lo), tuple(h * self.degree for h in hi)

    @property
    def global_dofs(self) -> np.ndarray:
        """Global DoF of every local DoF (node-blocked, fespace.py:3-8)."""
        cache = self.__dict__.get("_gd")
        if cache is None:
            nodes = self._node_grid(*self._node_box(self.rank))
            cache = (nodes[:, None] * self.dim + np.arange(self.dim)[None, :]).reshape(-1)
            object.__setattr__(self, "_gd", cache)
        return cache

    @property
    def owned_mask(self) -> np.ndarray:
        """Local DoFs this rank owns: no lower rank's closed box contains the node."""
        cache = self.__dict__.get("_own")
        if cache is None:
            lo_n, hi_n = self._node_box(self.rank)
            coords = np.stack(np.meshgrid(*[np.arange(l, h + 1) for l, h in zip(lo_n, hi_n)], indexing="ij"), -1)
            coords = coords.transpose(tuple(reversed(range(self.dim))) + (self.dim,)).reshape(-1, self.dim)
            own = np.ones(len(coords), dtype=bool)
            for r in range(self.rank):
                rl, rh = self._node_box(r)
                own &= ~np.all((coords >= np.array(rl)) & (coords <= np.array(rh)), axis=1)
            cache = np.repeat(own, self.dim)
            object.__setattr__(self, "_own", cache)
        return cache

    def shared(self, peer: int):
        """Local DoF indices of the nodes shared with ``peer`` (ordered by global
        DoF, the same order on both ranks), or None."""
        a_lo, a_hi = self._node_box(self.rank)
        b_lo, b_hi = self._node_box(peer)
        lo = tuple(max(x, y) for x, y in zip(a_lo, b_lo))
        hi = tuple(min(x, y) for x, y in zip(a_hi, b_hi))
        if any(l > h for l, h in zip(lo, hi)):
            return None
        ln = self.local_nodes
        strides = np.cumprod([1] + list(ln[:-1]))
        axes = [np.arange(l - o, h - o + 1) for l, h, o in zip(lo, hi, a_lo)]
        idx = np.zeros((1,) * self.dim, dtype=np.int64)
        for a in range(self.dim):
            shape = [1] * self.dim
            shape[self.dim - 1 - a] = len(axes[a])
            idx = idx + (axes[a] * strides[a]).reshape(shape)
        nodes = idx.reshape(-1)
        return (nodes[:, None] * self.dim + np.arange(self.dim)[None, :]).reshape(-1)

    def peers(self) -> dict:
        out = {}
        for r in range(len(self.boxes)):
            if r != self.rank:
                s = self.shared(r)
                if s is not None:
                    out[r] = s
        return out

    def local(self, v_global):
        """This rank's part of a global vector (numpy or torch)."""
        idx = self.global_dofs
        if isinstance(v_global, torch.Tensor):
            return v_global[torch.from_numpy(idx).to(v_global.device)]
        return np.asarray(v_global)[idx]

    def sub_mesh(self, global_mesh: Mesh) -> Mesh:
        m = global_mesh
        for a in range(self.dim):  # each axis is cut once, in the global cell numbering
            m = sub_box(m, a, self.lo[a], self.hi[a])
        return m

    # --- device views for the coarse bridge (DistGMG) and owned dots
    def _dev(self, key, fn):
        d = self.__dict__.setdefault("_devcache", {})
        if key not in d:
            d[key] = fn()
        return d[key]

    def _gidx(self, device):
        return self._dev(("g", str(device)), lambda: torch.from_numpy(self.global_dofs).to(device))

    def put_local(self, full: torch.Tensor, part: torch.Tensor) -> None:
        """full[this part's DoFs] = part (zero-padded partial sums of a bridge)."""
        full[self._gidx(full.device)] = part

    def take_local(self, full: torch.Tensor) -> torch.Tensor:
        return full[self._gidx(full.device)]

    def put_owned(self, full: torch.Tensor, part: torch.Tensor) -> None:
        own = self._dev(("o", str(part.device)), lambda: torch.from_numpy(self.owned_mask).to(part.device))
        full[self._gidx(full.device)[own]] = part[own]

    def make_exchange(self, comm, mask_dev: torch.Tensor):
        return BoxExchange(self, comm, mask_dev)

    def halved(self) -> "Box":
        if any(c % 2 for c in self.cells) or any(v % 2 for lo, hi in self.boxes for v in lo + hi):
            raise ValueError("box partition does not coarsen 2:1")
        return Box(self.dim, self.degree, tuple(c // 2 for c in self.cells), self.rank,
                   tuple((tuple(v // 2 for v in lo), tuple(v // 2 for v in hi)) for lo, hi in self.boxes))

    def min_extent(self) -> int:
        return min(h - l for lo, hi in self.boxes for l, h in zip(lo, hi))


def partition_parts(dim: int, degree: int, cells: tuple, rank: int, size: int, partition: str = "slab"):
    """The finest level's part of ``rank``: a z-slab (``"slab"``) or a Morton box
    (``"morton"``, power-of-two rank counts; on 2 ranks it is the same z-half)."""
    if partition == "slab":
        return Slab(dim, degree, tuple(cells), *slab_ranges(cells[-1], size)[rank])
    if partition == "morton":
        return Box(dim, degree, tuple(cells), rank, tuple(morton_boxes(tuple(cells), size)))
    raise ValueError(f"unknown partition {partition!r}")


def level_parts(dim: int, degree: int, fine_cells: tuple, n_levels: int, rank: int, size: int,
                min_cells: int = 2, partition: str = "slab") -> list:
    """Parts of rank ``rank`` on every level, coarsest first (``level_slabs`` for
    either partition).  A level is distributed while every part keeps >=
    ``min_cells`` cells along every axis it is cut on and the parts nest 2:1;
    the levels below, and always the coarsest, are replicated (None)."""
    if partition == "slab":
        return level_slabs(dim, degree, fine_cells, n_levels, rank, size, min_cells)
    fine = partition_parts(dim, degree, fine_cells, rank, size, partition)
    if size > 1 and fine.min_extent() < min(min_cells, min(fine_cells)):
        raise ValueError("the finest level is too thin to partition")
    out = [fine]
    for _ in range(n_levels - 2):
        cur = out[0]
        try:
            nxt = cur.halved() if cur is not None else None
        except ValueError:
            nxt = None
        out.insert(0, nxt if (nxt is not None and nxt.min_extent() >= min_cells) else None)
    if n_levels > 1:
        out.insert(0, None)
    return out


# ---------------------------------------------------------------------------
# distributed level objects
# ---------------------------------------------------------------------------


def _halo_add_dev(y: torch.Tensor, recv: torch.Tensor, mask: torch.Tensor) -> None:
    check(lib().hf_halo_add(y.numel(), dv.ptr(y), dv.ptr(recv), dv.ptr(mask), dv.stream()))


class SlabExchange:
    """Reverse add of the interface-plane partial sums (the one exchange per apply).

    ``add_fn(y_plane, recv, mask_plane)`` performs y += recv on unconstrained
    entries; the product uses the libhf kernel (tests on CPU inject their own)."""

    def __init__(self, slab: Slab, comm, mask_dev: torch.Tensor, add_fn=_halo_add_dev):
        self.slab, self.comm, self.add_fn = slab, comm, add_fn
        self.timer = NO_TIMER
        pd = slab.plane_dofs
        self.pd = pd
        self.peers = {}
        if slab.has_lower:
            self.peers[comm.rank - 1] = slice(0, pd)
        if slab.has_upper:
            self.peers[comm.rank + 1] = slice(slab.n_dofs - pd, slab.n_dofs)
        self.recv = {p: torch.empty(pd, dtype=torch.float64, device=mask_dev.device) for p in self.peers}
        self.mask = {p: mask_dev[s] for p, s in self.peers.items()}

    def start(self, y: torch.Tensor):
        """Post the interface planes of y (their partial sums must be final);
        ``finish`` adds the neighbours' partials.  The interior cells may run in between."""
        sends = {p: y[s] for p, s in self.peers.items()}  # contiguous views: no copy
        return self.comm.exchange_start(sends, self.recv)

    def finish(self, handle, y: torch.Tensor) -> torch.Tensor:
        handle.wait()
        for p, s in self.peers.items():
            self.add_fn(y[s], self.recv[p], self.mask[p])
        return y

    def add(self, y: torch.Tensor) -> torch.Tensor:
        if not self.peers:
            return y
        with self.timer.span("exchange"):
            sends = {p: y[s].contiguous() for p, s in self.peers.items()}
            self.comm.exchange(sends, self.recv)
            for p, s in self.peers.items():
                self.add_fn(y[s], self.recv[p], self.mask[p])
        return y


def _pack_dev(y, idx, buf):
    check(lib().hf_halo_pack(idx.numel(), dv.ptr(idx), dv.ptr(y), dv.ptr(buf), dv.stream()))


def _unpack_add_dev(y, idx, buf, mask):
    check(lib().hf_halo_unpack_add(idx.numel(), dv.ptr(idx), dv.ptr(y), dv.ptr(buf), dv.ptr(mask), dv.stream()))


class BoxExchange:
    """Reverse add of the interface partial sums of a box partition: every
    node a rank shares with a neighbour (a face, an edge or a corner of its
    box) is packed, swapped over the transport (NCCL send/recv), and the
    neighbour's partials are added on the unconstrained DoFs.  A node shared
    by k ranks receives k - 1 partials, one per neighbour list.  ``pack_fn`` /
    ``unpack_fn`` are the libhf kernels; the CPU tests inject their own."""

    def __init__(self, box: "Box", comm, mask_dev: torch.Tensor, pack_fn=_pack_dev, unpack_fn=_unpack_add_dev):
        self.box, self.comm, self.mask = box, comm, mask_dev
        self.pack_fn, self.unpack_fn = pack_fn, unpack_fn
        self.timer = NO_TIMER
        dev = mask_dev.device
        self.idx = {p: torch.from_numpy(i.astype(np.int32)).to(dev) for p, i in box.peers().items()}
        self.send = {p: torch.empty(i.numel(), dtype=torch.float64, device=dev) for p, i in self.idx.items()}
        self.recv = {p: torch.empty(i.numel(), dtype=torch.float64, device=dev) for p, i in self.idx.items()}
        self.peers = self.idx

    def start(self, y: torch.Tensor):
        for p, i in self.idx.items():
            self.pack_fn(y, i, self.send[p])
        return self.comm.exchange_start(self.send, self.recv)

    def finish(self, handle, y: torch.Tensor) -> torch.Tensor:
        handle.wait()
        for p, i in self.idx.items():
            self.unpack_fn(y, i, self.recv[p], self.mask)
        return y

    def add(self, y: torch.Tensor) -> torch.Tensor:
        if not self.idx:
            return y
        with self.timer.span("exchange"):
            for p, i in self.idx.items():
                self.pack_fn(y, i, self.send[p])
            self.comm.exchange(self.send, self.recv)
            for p, i in self.idx.items():
                self.unpack_fn(y, i, self.recv[p], self.mask)
        return y


class DistProblem:
    """A rank's slab of one level: the local ``Problem`` plus its partition data."""

    def __init__(self, global_mesh: Mesh, degree: int, mat: Material, slab, comm, global_mask: np.ndarray,
                 basis_nodes: str = "equispaced"):
        """``slab``: this rank's part, a ``Slab`` or a ``Box`` (``self.part``)."""
        self.slab = self.part = slab
        self.comm = comm
        self.global_mesh = global_mesh
        self.local = Problem(slab.sub_mesh(global_mesh), degree, mat, basis_nodes=basis_nodes,
                             has_top_face=slab.has_top)
        mask = np.ascontiguousarray(slab.local(global_mask))
        self.local.constraints = ConstraintSet.from_dofs(self.local.n_dofs, np.flatnonzero(mask))
        self.mask_dev = torch.from_numpy(mask.astype(np.uint8)).cuda()
        self.exchange = slab.make_exchange(comm, self.mask_dev)
        self.own_dev = None
        if isinstance(slab, Box):
            self.own_dev = torch.from_numpy(slab.owned_mask.astype(np.uint8)).cuda()
            self._unowned = torch.from_numpy(~slab.owned_mask).cuda()
        self.timer = NO_TIMER

    def set_timer(self, timer) -> None:
        self.timer = timer
        self.exchange.timer = timer

    @property
    def n_dofs(self) -> int:
        return self.local.n_dofs

    @property
    def n_global_dofs(self) -> int:
        return self.slab.n_global_dofs

    def dot(self, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """Global dot product: owned DoFs on this rank, all-reduced (2 scalars max per call site)."""
        if self.own_dev is None:
            o = self.slab.owned
            dv.dot(a[o], b[o], out)
        else:
            check(lib().hf_dot_owned(dv.Workspace.get().handle, a.numel(), dv.ptr(a), dv.ptr(b), dv.ptr(self.own_dev),
                                     dv.ptr(out), dv.stream()))
        with self.timer.span("allreduce"):
            return self.comm.allreduce_(out)

    def zero_unowned_(self, r: torch.Tensor) -> torch.Tensor:
        """Zero the entries another rank owns (before a restriction, so every
        shared fine DoF enters the coarse interface sums once)."""
        if self.own_dev is None:
            if self.slab.has_lower:
                r[:self.slab.plane_dofs] = 0.0
        else:
            r.masked_fill_(self._unowned, 0.0)
        return r

    def residual(self, u: torch.Tensor, traction=None) -> torch.Tensor:
        """compute_residual (operators.py:205-224) on the slab + interface add."""
        return self.exchange.add(compute_residual(self.local, u, traction))


def _agree_jacobian(comm, exc: NonPositiveJacobian | None, level=None):
    """NonPositiveJacobian on any rank is raised on every rank."""
    flag = torch.tensor([1.0 if exc is not None else 0.0], dtype=torch.float64, device="cuda")
    comm.allreduce_(flag)
    if exc is not None:
        raise exc
    if flag.item() > 0:
        raise NonPositiveJacobian("det F <= 0 on another rank", element=-1, level=level)


class DistributedTangent:
    """MatrixFreeTangent on a slab: local cell kernel + reverse interface add."""

    def __init__(self, dp: DistProblem, u_local, strategy: str = "tensor4", level=None):
        self.dp = dp
        err = None
        try:
            self.local = MatrixFreeTangent(dp.local, u_local, strategy)
        except NonPositiveJacobian as e:
            err = e
        _agree_jacobian(dp.comm, err, level)
        self.strategy = strategy

        self._split = self._tile_split()

    def _tile_split(self):
        """(boundary tile ranges, interior tile range) of the slab: the boundary
        tiles hold every cell of the first / last cell layer that touches an
        interface plane, so the planes' partial sums are final after them."""
        sl = self.dp.slab
        if not isinstance(sl, Slab) or not (sl.has_lower or sl.has_upper):
            return None  # box partitions: apply, then exchange (no interior/boundary split)
        nt, cpt = self.local.tiles()
        cells = self.dp.local.mesh.cells
        layer = int(np.prod(cells[:-1]))
        n_el = self.dp.local.mesh.n_elements
        lo = -(-layer // cpt) if sl.has_lower else 0
        hi = (n_el - layer) // cpt if sl.has_upper else nt
        if lo >= hi:
            return None
        bounds = [(0, lo)] if lo > 0 else []
        if hi < nt:
            bounds.append((hi, nt))
        return bounds, (lo, hi)

    @property
    def n_dofs(self) -> int:
        return self.dp.n_dofs

    def apply_into(self, x: torch.Tensor, y: torch.Tensor, skip=None) -> torch.Tensor:
        """y = A x on the slab.  The interface exchange overlaps the interior cells:
        fill, boundary tiles, post the planes, interior tiles, add the partials."""
        if skip is not None or self._split is None:
            self.local.apply_into(x, y, skip)
            return self.dp.exchange.add(y)
        bounds, (i0, i1) = self._split
        check(lib().hf_fill_masked(x.numel(), dv.ptr(y), dv.ptr(x), dv.ptr(self.dp.mask_dev), 0.0, dv.stream()))
        for k, (t0, t1) in enumerate(bounds):
            self.local.apply_tiles(x, y, t0, t1, mode=1 if k == 0 else 0)
        ex = self.dp.exchange
        with ex.timer.span("exchange"):
            h = ex.start(y)
        # while NCCL's kernel holds a few SMs, launch the persistent interior
        # blocks on the others (a block queued behind it would finish late)
        self.local.apply_tiles(x, y, i0, i1, mode=0, reserve_sms=_nccl_sms(ex))
        with ex.timer.span("exchange"):
            ex.finish(h, y)
        return y

    def apply(self, x: torch.Tensor) -> torch.Tensor:
        y = torch.empty_like(x)
        return self.apply_into(x, y)

    __call__ = apply

    def diagonal_dev(self) -> torch.Tensor:
        return self.dp.exchange.add(self.local.diagonal_dev())

    diagonal = diagonal_dev


def dist_cg(dp: DistProblem, apply_fn, b: torch.Tensor, rel_tol: float = 1e-6, preconditioner=None,
            max_iterations: int | None = None):
    """PCG (solver.py:34-76) on slab vectors: local updates, all-reduced owned dots.
    Returns (x, iterations, relative residual, residual history)."""
    n = b.numel()
    if max_iterations is None:
        max_iterations = 10 * dp.n_global_dofs
    L = lib()
    s = torch.zeros(4, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    r = b.clone()
    ap = torch.empty_like(b)
    dp.dot(b, b, s[0:1])
    b_norm = float(np.sqrt(s[0].item()))
    history = [b_norm]
    if b_norm == 0.0:
        return x, 0, 0.0, history
    z = torch.empty_like(b)
    if preconditioner is not None:
        preconditioner.apply_into(r, z)
    else:
        z.copy_(r)
    p = z.clone()
    dp.dot(r, z, s[1:2])
    rz = s[1].item()
    from .solver import IndefiniteOperator

    for it in range(1, max_iterations + 1):
        apply_fn.apply_into(p, ap)
        dp.dot(p, ap, s[2:3])
        pap = s[2].item()
        if pap <= 0.0:
            raise IndefiniteOperator(f"p.Ap = {pap:.3e} <= 0 at iteration {it - 1}")
        alpha = rz / pap
        check(L.hf_axpby(n, alpha, dv.ptr(p), 1.0, dv.ptr(x), dv.stream()))
        check(L.hf_axpby(n, -alpha, dv.ptr(ap), 1.0, dv.ptr(r), dv.stream()))
        dp.dot(r, r, s[3:4])
        r_norm = float(np.sqrt(s[3].item()))
        history.append(r_norm)
        if r_norm <= rel_tol * b_norm:
            return x, it, r_norm / b_norm, history
        if preconditioner is not None:
            preconditioner.apply_into(r, z)
        else:
            z.copy_(r)
        dp.dot(r, z, s[1:2])
        rz_new = s[1].item()
        check(L.hf_axpby(n, 1.0, dv.ptr(z), rz_new / rz, dv.ptr(p), dv.stream()))
        rz = rz_new
    return x, max_iterations, history[-1] / b_norm, history


def dist_eigen_range(dp: DistProblem, op, diag: torch.Tensor, seed: int, iterations: int = 30):
    """estimate_eigenvalue_range (multigrid.py:112-166) with all-reduced dots;
    the Lanczos RHS is the rank's slice of the reference's global vector."""
    import scipy.linalg

    bg = np.random.default_rng(seed).standard_normal(dp.n_global_dofs)
    b = torch.from_numpy(np.ascontiguousarray(dp.slab.local(bg))).cuda()
    b[dp.mask_dev.bool()] = 0.0
    n = b.numel()
    L = lib()
    inv_d = torch.reciprocal(diag)
    s = torch.zeros(3, dtype=torch.float64, device="cuda")
    r = b.clone()
    z = inv_d * r
    p = z.clone()
    ap = torch.empty_like(r)
    dp.dot(r, z, s[0:1])
    rz = s[0].item()
    alphas, betas = [], []
    for _ in range(iterations):
        if rz <= 0.0 or not np.isfinite(rz):
            break
        op.apply_into(p, ap)
        dp.dot(p, ap, s[1:2])
        pap = s[1].item()
        if pap <= 0.0:
            break
        alpha = rz / pap
        check(L.hf_axpby(n, -alpha, dv.ptr(ap), 1.0, dv.ptr(r), dv.stream()))
        torch.mul(inv_d, r, out=z)
        dp.dot(r, z, s[2:3])
        rz_new = s[2].item()
        if rz_new <= 1e-28 * rz or not np.isfinite(rz_new):
            alphas.append(alpha)
            break
        beta = rz_new / rz
        alphas.append(alpha)
        betas.append(beta)
        check(L.hf_axpby(n, 1.0, dv.ptr(z), beta, dv.ptr(p), dv.stream()))
        rz = rz_new
    if not alphas:
        return 1.0, 1.0
    k = len(alphas)
    dt = np.empty(k)
    dt[0] = 1.0 / alphas[0]
    for i in range(1, k):
        dt[i] = 1.0 / alphas[i] + betas[i - 1] / alphas[i - 1]
    if k == 1:
        return float(dt[0]), float(dt[0])
    off = np.array([np.sqrt(betas[i]) / alphas[i] for i in range(k - 1)])
    ritz = scipy.linalg.eigvalsh_tridiagonal(dt, off)
    return float(ritz[0]), float(ritz[-1])


class DistLevel:
    """LevelOperator (multigrid.py:208-252) of a distributed level."""

    def __init__(self, dp: DistProblem, u_local, strategy: str, seed: int, level: int):
        self.dp, self.level = dp, level
        self.op = DistributedTangent(dp, u_local, strategy, level=level)
        self.diag = self.op.diagonal_dev()
        self.inv_diag = torch.reciprocal(self.diag)
        self.lam_min, self.lam_max = dist_eigen_range(dp, self.op, self.diag, seed)
        n = dp.n_dofs
        self.b = torch.zeros(n, dtype=torch.float64, device="cuda")
        self.x = torch.zeros_like(self.b)
        self.d = torch.zeros_like(self.b)
        self.ax = torch.zeros_like(self.b)
        self.r = torch.zeros_like(self.b)

    def smooth_into(self, b, x, steps: int, s: ChebyshevSettings, x_zero: bool):
        """Restarted Chebyshev smoothing in three-term form (multigrid._chebyshev_into):
        ``self.d`` is the second iterate buffer, every update writes x_{k+1} over
        x_{k-1}; elementwise, so both copies of an interface DoF stay identical."""
        theta, coefs = _cheb_coeffs(self.lam_max, s)
        n, L = x.numel(), lib()
        cur, oth = x, self.d
        prev_zero = False

        def update(first, th, cd, cz, zero):
            nonlocal cur, oth, prev_zero
            check(L.hf_cheb3_step(n, dv.ptr(cur), dv.ptr(oth), dv.ptr(b), None if zero else dv.ptr(self.ax),
                                  dv.ptr(self.inv_diag), first, th, cd, cz, int(zero), int(prev_zero), None, None, 64,
                                  0, dv.stream()))
            cur, oth = oth, cur
            prev_zero = zero

        for step in range(steps):
            zero = x_zero and step == 0
            if not zero:
                self.op.apply_into(cur, self.ax)
            update(1, theta, 0.0, 0.0, zero)
            for cd, cz in coefs:
                self.op.apply_into(cur, self.ax)
                update(0, 0.0, cd, cz, False)
        if cur is not x:
            x.copy_(cur)
        return x


class DistGMG:
    """V-cycle preconditioner (multigrid.py:309-351) over slab levels on top of
    replicated coarse levels."""

    def __init__(self, dist_levels: list, transfers: list, bridge: TransferOperator | None,
                 replicated: GMGPreconditioner | None, coarse_slab: Slab | None, comm,
                 smoothing_steps: int = 2, settings: ChebyshevSettings = ChebyshevSettings()):
        self.levels, self.transfers = dist_levels, transfers
        self.bridge, self.rep, self.cslab, self.comm = bridge, replicated, coarse_slab, comm
        self.steps, self.settings = smoothing_steps, settings
        self._graph = None  # None: not tried yet; False: eager
        self.graph_error = None
        if replicated is not None:
            n = coarse_slab.n_global_dofs
            self._cfull = torch.zeros(n, dtype=torch.float64, device="cuda")
            self._xfull = torch.zeros(n, dtype=torch.float64, device="cuda")
            self._cpart = torch.zeros(coarse_slab.n_dofs, dtype=torch.float64, device="cuda")

    def _vc(self, i: int, b: torch.Tensor, x: torch.Tensor):
        Lv = self.levels[i]
        Lv.smooth_into(b, x, self.steps, self.settings, x_zero=True)
        Lv.op.apply_into(x, Lv.ax)
        n = b.numel()
        check(lib().hf_resid_masked(n, dv.ptr(Lv.r), dv.ptr(b), dv.ptr(Lv.ax), dv.ptr(Lv.dp.mask_dev), dv.stream()))
        Lv.dp.zero_unowned_(Lv.r)  # a shared DoF enters the restriction once
        if i == 0:
            cs = self.cslab
            self.bridge.restrict_into(Lv.r, self._cpart, mode=1)
            self._cfull.zero_()
            cs.put_local(self._cfull, self._cpart)
            self.comm.allreduce_(self._cfull)
            self.rep.apply_into(self._cfull, self._xfull)
            self.bridge.prolong_into(cs.take_local(self._xfull).contiguous(), x, mode=2)
        else:
            C = self.levels[i - 1]
            self.transfers[i - 1].restrict_into(Lv.r, C.b, mode=1)
            C.dp.exchange.add(C.b)
            self._vc(i - 1, C.b, C.x)
            self.transfers[i - 1].prolong_into(C.x, x, mode=2)
        Lv.smooth_into(b, x, self.steps, self.settings, x_zero=False)
        return x

    def _eager(self, b: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        top = len(self.levels) - 1
        out.zero_()
        return self._vc(top, b, out)

    def _graph_wanted(self) -> bool:
        """Replay the V-cycle as one CUDA graph with the NCCL calls inside
        (NCCL supports stream capture; the host-staged gloo transport does not).
        Off while a CommTimer is attached (its events time each call eagerly)
        and with HF_DIST_GRAPH=0."""
        if os.environ.get("HF_DIST_GRAPH", "1") == "0" or getattr(self.comm, "staged", True):
            return False
        return all(lv.dp.timer is NO_TIMER for lv in self.levels)

    def apply_into(self, b: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        if self._graph is False or not self._graph_wanted():
            return self._eager(b, out)
        if self._graph is None:
            self._bs, self._xs = torch.empty_like(b), torch.empty_like(out)
            self._bs.copy_(b)
            self._eager(self._bs, self._xs)  # warm-up: communicators, the replicated levels' own graph
            graph, ok = None, 1.0
            rep_graph = self.rep.use_graph if self.rep is not None else None
            if self.rep is not None:
                self.rep.use_graph = False  # its launches go into this graph (a replay cannot be captured)
            try:
                graph = dv.capture_graph(lambda: self._eager(self._bs, self._xs))
            except Exception as e:  # the transport refused capture: every rank falls back together
                graph, ok = None, 0.0
                self.graph_error = f"{type(e).__name__}: {e}"
            finally:
                if self.rep is not None:
                    self.rep.use_graph = rep_graph
            flag = torch.tensor([ok], dtype=torch.float64, device=b.device)
            self.comm.allreduce_(flag)
            self._graph = graph if flag.item() == self.comm.size else False
            if self._graph is False:
                return self._eager(b, out)
        self._bs.copy_(b)
        self._graph.replay()
        out.copy_(self._xs)
        return out


class DistHierarchy:
    """The slab decomposition of a GMG hierarchy, built once and re-linearised
    every Newton iteration (the single-GPU path likewise keeps its Problems):
    distributed levels (DistProblem), their transfers, the replicated coarse
    Problems and the bridge between them."""

    def __init__(self, global_meshes: list, degree: int, mat: Material, global_masks: list, comm,
                 min_cells: int = 2, fine_dp: "DistProblem | None" = None, partition: str = "slab"):
        nlev = len(global_meshes)
        fine = global_meshes[-1]
        self.comm, self.degree, self.nlev = comm, degree, nlev
        self.partition = partition
        self.slabs = level_parts(fine.dim, degree, fine.cells, nlev, comm.rank, comm.size, min_cells, partition)
        first = next(i for i, s in enumerate(self.slabs) if s is not None)
        if first == 0:
            raise ValueError("the coarsest level must be replicated (min_cells too small for the hierarchy)")
        self.first = first
        self.dps = {i: (fine_dp if (i == nlev - 1 and fine_dp is not None) else
                        DistProblem(global_meshes[i], degree, mat, self.slabs[i], comm, global_masks[i]))
                    for i in range(first, nlev)}
        self.transfers = [TransferOperator(self.dps[i].local, self.dps[i + 1].local) for i in range(first, nlev - 1)]
        self.rep_probs = []
        for i in range(first):
            p = Problem(global_meshes[i], degree, mat)
            p.constraints = ConstraintSet.from_dofs(p.n_dofs, np.flatnonzero(global_masks[i]))
            self.rep_probs.append(p)
        self.rep_transfers = build_transfers(self.rep_probs)
        self.cslab = self.slabs[first].halved()
        cs = self.cslab
        self.coarse_local = Problem(cs.sub_mesh(global_meshes[first - 1]), degree, mat, has_top_face=cs.has_top)
        cmask = np.ascontiguousarray(cs.local(global_masks[first - 1]))
        self.coarse_local.constraints = ConstraintSet.from_dofs(self.coarse_local.n_dofs, np.flatnonzero(cmask))
        self.bridge = TransferOperator(self.coarse_local, self.dps[first].local)

    @property
    def fine(self) -> "DistProblem":
        return self.dps[self.nlev - 1]

    def build_gmg(self, u_fine_local, strategy: str = "tensor4", seed: int = 0, keep_constrained: bool = False):
        """Linearise every level at the injected fine state (multigrid.py:358-382).
        Returns (DistGMG, fine DistributedTangent)."""
        first, nlev, dps = self.first, self.nlev, self.dps
        u = {nlev - 1: dv.as_dev(u_fine_local)}
        for lvl in range(nlev - 1, first, -1):  # injection down the slabs (multigrid.py:76-92)
            uc = torch.empty(dps[lvl - 1].n_dofs, dtype=torch.float64, device="cuda")
            check(lib().hf_inject(dps[lvl - 1].local._space, dps[lvl].local._space, dv.ptr(u[lvl]), dv.ptr(uc),
                                  int(keep_constrained), dv.stream()))
            u[lvl - 1] = uc
        levels = [DistLevel(dps[i], u[i], strategy, seed + 7919 * i, i) for i in range(first, nlev)]
        # full state on the finest replicated level: owned slices, all-reduced
        cs = self.cslab
        uc_local = torch.empty(cs.n_dofs, dtype=torch.float64, device="cuda")
        check(lib().hf_inject(self.coarse_local._space, dps[first].local._space, dv.ptr(u[first]), dv.ptr(uc_local),
                              int(keep_constrained), dv.stream()))
        ufull = torch.zeros(cs.n_global_dofs, dtype=torch.float64, device="cuda")
        cs.put_owned(ufull, uc_local)
        self.comm.allreduce_(ufull)
        rep_levels = build_level_operators(self.rep_probs, ufull, strategy, seed, keep_constrained)
        replicated = GMGPreconditioner(rep_levels, self.rep_transfers)
        gmg = DistGMG(levels, self.transfers, self.bridge, replicated, cs, self.comm)
        return gmg, levels[-1].op


def build_dist_gmg(global_meshes: list, degree: int, mat: Material, global_masks: list, u_fine_local, comm,
                   strategy: str = "tensor4", seed: int = 0, min_cells: int = 2, keep_constrained: bool = False,
                   fine_dp: "DistProblem | None" = None, partition: str = "slab"):
    """Distributed analogue of build_gmg (multigrid.py:372-382).

    ``global_meshes``/``global_masks``: every level, coarsest first;
    ``partition``: "slab" (z-slabs) or "morton" (SFC boxes).  Returns
    (DistGMG, fine DistProblem, fine DistributedTangent)."""
    h = DistHierarchy(global_meshes, degree, mat, global_masks, comm, min_cells, fine_dp, partition)
    gmg, op = h.build_gmg(u_fine_local, strategy, seed, keep_constrained)
    gmg._hierarchy = h
    return gmg, h.fine, op


def newton_solve_prescribed_dist(h: DistHierarchy, settings, target: float, height_local: torch.Tensor,
                                 strategy: str = "tensor4", seed: int = 0, on_record=None):
    """Config-4 Newton (prescribed last-axis displacement) on the slab
    decomposition: the restatement of solver.py:143-201 that
    solver.newton_solve_prescribed runs on one GPU, with all-reduced norms.
    ``height_local``: X_last / max X_last on this rank's DoF slice (node-blocked)."""
    from .solver import MaxNewtonIterations, NewtonRecord

    dp = h.fine
    d = dp.local.dim
    u = torch.zeros(dp.n_dofs, dtype=torch.float64, device="cuda")
    s = torch.zeros(1, dtype=torch.float64, device="cuda")

    def norm(v):
        return float(np.sqrt(dp.dot(v, v, s).item()))

    records = []
    for step in range(1, settings.n_load_steps + 1):
        u.view(-1, d)[:, d - 1] += (target / settings.n_load_steps) * height_local
        residual = dp.residual(u)
        res0 = norm(residual)
        res_target = max(settings.residual_rel_tol * res0, settings.residual_abs_tol)
        for it in range(1, settings.max_newton_iterations + 1):
            gmg, op = h.build_gmg(u, strategy, seed, keep_constrained=True)
            t0 = time.perf_counter()
            du, its, _, _ = dist_cg(dp, op, -residual, rel_tol=settings.linear_rel_tol, preconditioner=gmg)
            t_cg = time.perf_counter() - t0
            u += du
            residual = dp.residual(u)
            res_norm, du_norm = norm(residual), norm(du)
            rec = NewtonRecord(step, step / settings.n_load_steps, it, res_norm, du_norm, its, t_cg)
            records.append(rec)
            if on_record:
                on_record(rec)
            if du_norm <= settings.update_tol and res_norm <= res_target:
                break
        else:
            raise MaxNewtonIterations("no convergence in the distributed prescribed-displacement Newton", records)
    return u, records
