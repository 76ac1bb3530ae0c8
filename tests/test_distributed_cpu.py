"""Multi-rank host logic of the slab decomposition (paper_1904_13131_b200.distributed),
run on CPU with the gloo backend at world size 2 and 3.

The per-rank cell kernel is stood in for by the CPU oracle on the rank's
sub-box (test infrastructure); everything else -- slab ranges, contiguous
local slices, the interface exchange over torch.distributed, owned dots, the
zero-padded coarse bridge -- is the product code.  The distributed results
must equal the oracle's global results.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hf_oracle as O
from paper_1904_13131_b200.distributed import LocalComm, Slab, SlabExchange, TorchComm, level_slabs, slab_ranges

MU = (1.0, 10.0)
LAM = (1.5, 15.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _global_case(dim, cells, degree, seed):
    rng = np.random.default_rng(seed)
    verts = O.uniform_vertices(cells)
    n_el = int(np.prod(cells))
    inc = rng.random(n_el) < 0.3
    mu = np.where(inc, MU[1], MU[0])
    lam = np.where(inc, LAM[1], LAM[0])
    n_nodes = int(np.prod([c * degree + 1 for c in cells]))
    mask = np.zeros(n_nodes * dim, dtype=bool)
    prob = O.OProblem(dim, degree, cells, verts, mu, lam, mask)
    mask = O.face_mask(prob, dim - 1, 0)  # clamp the bottom face
    mask |= rng.random(mask.size) < 0.02  # and a sprinkle of interior constraints
    prob = O.OProblem(dim, degree, cells, verts, mu, lam, mask)
    X = O.node_coordinates(prob)
    ubar = 0.01 * np.sin(3.0 * X[:, :1] + np.arange(dim)[None, :]).reshape(-1) * X[:, dim - 1].repeat(dim)
    x = rng.standard_normal(prob.n_dofs)
    return prob, ubar, x


def _sub_problem(prob, slab):
    """The oracle problem of one slab (cells of a z-slab are a contiguous cell range)."""
    d = prob.dim
    plane_cells = int(np.prod(prob.cells[:-1]))
    cells = tuple(prob.cells[:-1]) + (slab.c1 - slab.c0,)
    vplane = int(np.prod([c + 1 for c in prob.cells[:-1]]))
    verts = prob.vertices[slab.c0 * vplane:(slab.c1 + 1) * vplane]
    sl = slice(slab.c0 * plane_cells, slab.c1 * plane_cells)
    return O.OProblem(d, prob.degree, cells, verts, prob.mu_el[sl], prob.lam_el[sl], slab.local(prob.mask))


def _cpu_add(y, recv, mask):
    y += torch.where(mask.bool(), torch.zeros_like(recv), recv)


def _worker(rank, size, port, dim, cells, degree, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        comm = TorchComm()
        prob, ubar, x = _global_case(dim, cells, degree, seed=3)
        c0, c1 = slab_ranges(cells[-1], size)[rank]
        slab = Slab(dim, degree, tuple(cells), c0, c1)
        sub = _sub_problem(prob, slab)
        mask_t = torch.from_numpy(slab.local(prob.mask).astype(np.uint8))
        ex = SlabExchange(slab, comm, mask_t, add_fn=_cpu_add)
        res = {}
        for strategy in ("tensor4", "scalar"):
            y = torch.from_numpy(O.Tangent(sub, slab.local(ubar), strategy).apply(slab.local(x)))
            ex.add(y)
            yg = O.Tangent(prob, ubar, strategy).apply(x)
            res[f"apply_{strategy}"] = float(np.linalg.norm(y.numpy() - slab.local(yg)) / np.linalg.norm(yg))
        d = torch.from_numpy(O.Tangent(sub, slab.local(ubar), "tensor4").diagonal())
        ex.add(d)
        dg = O.Tangent(prob, ubar, "tensor4").diagonal()
        res["diagonal"] = float(np.abs(d.numpy() - slab.local(dg)).max() / np.abs(dg).max())
        r = torch.from_numpy(O.residual(sub, slab.local(ubar)))
        ex.add(r)
        rg = O.residual(prob, ubar)
        res["residual"] = float(np.linalg.norm(r.numpy() - slab.local(rg)) / np.linalg.norm(rg))
        # owned dot products, all-reduced
        a, b = slab.local(x), slab.local(np.cos(np.arange(prob.n_dofs)))
        o = slab.owned
        t = torch.tensor([float(a[o] @ b[o])], dtype=torch.float64)
        comm.allreduce_(t)
        full = float(x @ np.cos(np.arange(prob.n_dofs)))
        res["dot"] = abs(t.item() - full) / abs(full)
        # coarse bridge: partial restriction of the owned residual + all-reduce == global restriction
        coarse_cells = tuple(c // 2 for c in cells)
        cprob = O.OProblem(dim, degree, coarse_cells, O.uniform_vertices(coarse_cells), np.ones(int(np.prod(coarse_cells))),
                           np.ones(int(np.prod(coarse_cells))),
                           np.zeros(int(np.prod([c * degree + 1 for c in coarse_cells])) * dim, dtype=bool))
        cslab = slab.halved()
        csub = _sub_problem(cprob, cslab)
        rl = slab.local(x).copy()
        if slab.has_lower:
            rl[:slab.plane_dofs] = 0.0
        part = O.Transfer(csub, sub).restrict(rl)
        fullc = torch.zeros(cslab.n_global_dofs, dtype=torch.float64)
        fullc[cslab.dof_offset:cslab.dof_offset + cslab.n_dofs] = torch.from_numpy(part)
        comm.allreduce_(fullc)
        rcg = O.Transfer(cprob, prob).restrict(x)
        res["bridge_restrict"] = float(np.linalg.norm(fullc.numpy() - rcg) / np.linalg.norm(rcg))
        # prolongation from the replicated coarse vector is rank-local and consistent
        xc = np.sin(np.arange(cprob.n_dofs))
        pl = O.Transfer(csub, sub).prolong(cslab.local(xc))
        pg = O.Transfer(cprob, prob).prolong(xc)
        res["bridge_prolong"] = float(np.abs(pl - slab.local(pg)).max())
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _run(size, dim, cells, degree):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(size, port, dim, cells, degree, out), nprocs=size, join=True)
    return dict(out)


@pytest.mark.parametrize("size,dim,cells,degree", [(2, 3, (2, 2, 4), 2), (3, 3, (2, 2, 6), 2), (2, 2, (4, 4), 3)])
def test_slab_decomposition_matches_global_oracle(size, dim, cells, degree):
    out = _run(size, dim, cells, degree)
    assert sorted(out) == list(range(size))
    for rank, res in out.items():
        for k in ("apply_tensor4", "apply_scalar", "diagonal", "residual", "bridge_restrict"):
            assert res[k] < 1e-13, (rank, k, res[k])
        assert res["dot"] < 1e-13, (rank, res["dot"])
        assert res["bridge_prolong"] == 0.0


def test_slab_geometry_is_a_contiguous_dof_range():
    cells = (4, 3, 8)
    for size in (1, 2, 3, 4):
        ranges = slab_ranges(cells[-1], size)
        slabs = [Slab(3, 2, cells, a, b) for a, b in ranges]
        # owned ranges tile the global vector exactly once
        owned = np.zeros(slabs[0].n_global_dofs, dtype=int)
        for s in slabs:
            o = s.owned
            owned[s.dof_offset + o.start:s.dof_offset + o.stop] += 1
        assert (owned == 1).all()
        for s, t in zip(slabs, slabs[1:]):  # neighbours share exactly one node plane
            assert s.dof_offset + s.n_dofs - s.plane_dofs == t.dof_offset


def test_level_slabs_nest_and_replicate_the_coarsest():
    for size in (1, 2, 4, 8):
        sl = level_slabs(3, 2, (32, 32, 32), 4, size - 1, size)
        assert sl[0] is None
        for c, f in zip(sl, sl[1:]):
            if c is not None:
                assert (f.c0, f.c1) == (2 * c.c0, 2 * c.c1)
        assert sl[-1].c1 == 32
    with pytest.raises(ValueError):
        slab_ranges(3, 4)


def test_local_comm_has_no_neighbours():
    c = LocalComm()
    t = torch.ones(2, dtype=torch.float64)
    assert c.allreduce_(t) is t
    with pytest.raises(ValueError):
        c.exchange({1: t}, {})


# ---------------------------------------------------------------------------
# Box (Morton / space-filling-curve) partitions
# ---------------------------------------------------------------------------


def _box_problem(prob, box):
    """The oracle problem of one box of cells."""
    d = prob.dim
    vshape = tuple(c + 1 for c in reversed(prob.cells))
    vs = tuple(slice(box.lo[a], box.hi[a] + 1) for a in reversed(range(d)))
    cs = tuple(slice(box.lo[a], box.hi[a]) for a in reversed(range(d)))
    verts = prob.vertices.reshape(vshape + (d,))[vs].reshape(-1, d)
    mu = prob.mu_el.reshape(tuple(reversed(prob.cells)))[cs].reshape(-1)
    lam = prob.lam_el.reshape(tuple(reversed(prob.cells)))[cs].reshape(-1)
    return O.OProblem(d, prob.degree, box.local_cells, np.ascontiguousarray(verts), mu, lam, box.local(prob.mask))


def _cpu_pack(y, idx, buf):
    buf.copy_(y[idx.long()])


def _cpu_unpack(y, idx, buf, mask):
    i = idx.long()
    y.index_add_(0, i, torch.where(mask[i].bool(), torch.zeros_like(buf), buf))


def _box_worker(rank, size, port, dim, cells, degree, out):
    from paper_1904_13131_b200.distributed import Box, BoxExchange, morton_boxes

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        comm = TorchComm()
        prob, ubar, x = _global_case(dim, cells, degree, seed=4)
        box = Box(dim, degree, tuple(cells), rank, tuple(morton_boxes(tuple(cells), size)))
        sub = _box_problem(prob, box)
        mask_t = torch.from_numpy(box.local(prob.mask).astype(np.uint8))
        ex = BoxExchange(box, comm, mask_t, pack_fn=_cpu_pack, unpack_fn=_cpu_unpack)
        res = {"n_peers": len(ex.idx)}
        for strategy in ("tensor4", "tensor2"):
            y = torch.from_numpy(O.Tangent(sub, box.local(ubar), strategy).apply(box.local(x)))
            ex.add(y)
            yg = O.Tangent(prob, ubar, strategy).apply(x)
            res[f"apply_{strategy}"] = float(np.linalg.norm(y.numpy() - box.local(yg)) / np.linalg.norm(yg))
        d = torch.from_numpy(O.Tangent(sub, box.local(ubar), "tensor4").diagonal())
        ex.add(d)
        dg = O.Tangent(prob, ubar, "tensor4").diagonal()
        res["diagonal"] = float(np.abs(d.numpy() - box.local(dg)).max() / np.abs(dg).max())
        r = torch.from_numpy(O.residual(sub, box.local(ubar)))
        ex.add(r)
        rg = O.residual(prob, ubar)
        res["residual"] = float(np.linalg.norm(r.numpy() - box.local(rg)) / np.linalg.norm(rg))
        # owned dots: every global DoF is owned by exactly one rank
        a, b = box.local(x), box.local(np.cos(np.arange(prob.n_dofs)))
        o = box.owned_mask
        t = torch.tensor([float(a[o] @ b[o])], dtype=torch.float64)
        comm.allreduce_(t)
        full = float(x @ np.cos(np.arange(prob.n_dofs)))
        res["dot"] = abs(t.item() - full) / abs(full)
        # coarse bridge: restriction of the owned part + all-reduce == global restriction;
        # prolongation from the replicated coarse vector is box-local
        coarse_cells = tuple(c // 2 for c in cells)
        ones = np.ones(int(np.prod(coarse_cells)))
        cprob = O.OProblem(dim, degree, coarse_cells, O.uniform_vertices(coarse_cells), ones, ones,
                           np.zeros(int(np.prod([c * degree + 1 for c in coarse_cells])) * dim, dtype=bool))
        cbox = box.halved()
        csub = _box_problem(cprob, cbox)
        rl = box.local(x).copy()
        rl[~box.owned_mask] = 0.0
        part = O.Transfer(csub, sub).restrict(rl)
        fullc = torch.zeros(cbox.n_global_dofs, dtype=torch.float64)
        cbox.put_local(fullc, torch.from_numpy(part))
        comm.allreduce_(fullc)
        rcg = O.Transfer(cprob, prob).restrict(x)
        res["bridge_restrict"] = float(np.linalg.norm(fullc.numpy() - rcg) / np.linalg.norm(rcg))
        xc = np.sin(np.arange(cprob.n_dofs))
        pl = O.Transfer(csub, sub).prolong(cbox.take_local(torch.from_numpy(xc)).numpy())
        pg = O.Transfer(cprob, prob).prolong(xc)
        res["bridge_prolong"] = float(np.abs(pl - box.local(pg)).max())
        # the owned part of a replicated vector, all-reduced, rebuilds it
        uf = torch.zeros(box.n_global_dofs, dtype=torch.float64)
        box.put_owned(uf, torch.from_numpy(box.local(ubar)))
        comm.allreduce_(uf)
        res["put_owned"] = float(np.abs(uf.numpy() - ubar).max())
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("size,dim,cells,degree", [(2, 3, (4, 4, 4), 2), (4, 3, (4, 4, 4), 2), (8, 3, (4, 4, 4), 2),
                                                   (4, 2, (4, 4), 2), (8, 3, (4, 4, 8), 1)])
def test_morton_box_partition_matches_global_oracle(size, dim, cells, degree):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_box_worker, args=(size, port, dim, cells, degree, out), nprocs=size, join=True)
    out = dict(out)
    assert sorted(out) == list(range(size))
    for rank, res in out.items():
        for k in ("apply_tensor4", "apply_tensor2", "diagonal", "residual", "bridge_restrict", "dot"):
            assert res[k] < 1e-13, (rank, k, res[k])
        assert res["bridge_prolong"] == 0.0 and res["put_owned"] == 0.0
        assert res["n_peers"] == size - 1 or size > 8  # every octant touches every other one at 8 ranks


def test_morton_boxes_are_chunks_of_the_z_order_curve():
    from paper_1904_13131_b200.distributed import Box, level_parts, morton_boxes

    def key(c, bits):
        k = 0
        for b in range(bits):
            for a, v in enumerate(c):
                k |= ((v >> b) & 1) << (len(c) * b + a)
        return k

    for dim, m, bits in ((3, 8, 3), (2, 8, 3)):
        cells = [tuple(int(v) for v in c) for c in np.ndindex(*(m,) * dim)]
        cells = [tuple(reversed(c)) for c in cells]  # (x, y[, z])
        order = sorted(cells, key=lambda c: key(c, bits))
        for size in (1, 2, 4, 8):
            boxes = morton_boxes((m,) * dim, size)
            n = len(order) // size
            for r, (lo, hi) in enumerate(boxes):
                assert all(all(lo[a] <= c[a] < hi[a] for a in range(dim)) for c in order[r * n:(r + 1) * n])
    # owned DoFs tile the global vector exactly once; the levels nest 2:1
    for size in (2, 4, 8):
        parts = [Box(3, 2, (8, 8, 8), r, tuple(morton_boxes((8, 8, 8), size))) for r in range(size)]
        cnt = np.zeros(parts[0].n_global_dofs, dtype=int)
        for p in parts:
            np.add.at(cnt, p.global_dofs[p.owned_mask], 1)
        assert (cnt == 1).all()
        lv = level_parts(3, 2, (32, 32, 32), 4, size - 1, size, partition="morton")
        assert lv[0] is None
        for c, f in zip(lv, lv[1:]):
            if c is not None:
                assert tuple(2 * v for v in c.lo) == f.lo and tuple(2 * v for v in c.hi) == f.hi
    with pytest.raises(ValueError):
        morton_boxes((8, 8, 8), 3)
