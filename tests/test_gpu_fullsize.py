"""Parity at the BASELINE sizes: the CPU oracle is run where it
finishes in seconds (config 1 2D 32^2 Q2, 3D 16^3 Q2), and size-independent
properties are checked at configs 2 and 3 (823,875 DoFs): the three caching
strategies agree, the operator is symmetric and linear, and it is the identity
on the constrained subspace (operators.py:331-339)."""

import numpy as np
import pytest
import torch

from oracle import hf_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _oracle_of(p):
    inc = p.mesh.material_id == 1
    from paper_1904_13131_b200.workloads import MATERIAL

    mu = np.where(inc, MATERIAL.inclusion.mu, MATERIAL.matrix.mu)
    lam = np.where(inc, MATERIAL.inclusion.lam, MATERIAL.matrix.lam)
    return O.OProblem(p.dim, p.degree, p.mesh.cells, p.mesh.vertices, mu, lam, p.constraints.mask)


def _rel(a, b):
    return float(torch.linalg.norm(a - b) / torch.linalg.norm(b))


@pytest.mark.parametrize("cfg,m", [(1, None), (2, 16)])
def test_apply_diagonal_residual_vs_oracle_at_size(cfg, m):
    from paper_1904_13131_b200 import MatrixFreeTangent, compute_residual
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(cfg, seed=5, m=m)
    p = wl.fine
    op_ = _oracle_of(p)
    for s in ("scalar", "tensor2", "tensor4"):
        y = MatrixFreeTangent(p, wl.ubar, s).apply(wl.x)
        yo = O.Tangent(op_, wl.ubar, s).apply(wl.x)
        assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < TOL, s
    r = compute_residual(p, wl.ubar)
    ro = O.residual(op_, wl.ubar)
    assert np.linalg.norm(r - ro) / np.linalg.norm(ro) < TOL
    if cfg == 1:
        d = MatrixFreeTangent(p, wl.ubar, "tensor4").diagonal().cpu().numpy()
        do = O.Tangent(op_, wl.ubar, "tensor4").diagonal()
        assert np.linalg.norm(d - do) / np.linalg.norm(do) < TOL


@pytest.mark.parametrize("cfg", [2, 3])
def test_properties_at_full_size(cfg):
    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(cfg, seed=0)
    p = wl.fine
    x = torch.from_numpy(wl.x).cuda()
    z = torch.from_numpy(np.random.default_rng(9).standard_normal(p.n_dofs)).cuda()
    mask = p.mask_dev
    ys = {}
    for s in ("tensor4", "tensor2", "scalar"):
        op = MatrixFreeTangent(p, wl.ubar, s)
        ys[s] = op.apply(x)
        if s == "tensor4":
            az = op.apply(z)
            # symmetric: <Ax, z> = <x, Az>
            lhs, rhs = float(ys[s] @ z), float(x @ az)
            assert abs(lhs - rhs) <= 1e-12 * float(torch.linalg.norm(ys[s]) * torch.linalg.norm(z))
            # linear
            a, b = 0.7, -1.3
            assert _rel(op.apply(a * x + b * z), a * ys[s] + b * az) < TOL
            # identity on the constrained subspace, exactly; atomics reorder sums only
            assert torch.equal(ys[s][mask], x[mask])
            assert _rel(op.apply(x), ys[s]) < 1e-14
            assert op.storage_bytes() == 8 * p.mesh.n_elements * p.n_qpoints_per_cell * (6 + 21 + 9 + 1)
    assert _rel(ys["tensor2"], ys["tensor4"]) < TOL
    assert _rel(ys["scalar"], ys["tensor4"]) < TOL


def test_pinned_host_apply_pipeline_matches_device_apply():
    """MatrixFreeTangent.apply on pinned host tensors (slab-pipelined H2D /
    tile-range kernels / D2H) equals the device apply up to summation order."""
    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(2, seed=3)
    op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
    xh = torch.from_numpy(wl.x.copy()).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    yd = op.apply(xh.cuda())
    for _ in range(2):
        yh.zero_()
        op.apply(xh, out=yh)
        assert _rel(yh.cuda(), yd) < 1e-14
        assert torch.equal(yh[wl.fine.constraints.mask], xh[wl.fine.constraints.mask])
    # pageable host tensors (or one of them): the device-buffer path, same result
    xp, yp = xh.clone(), torch.empty_like(xh)
    assert not xp.is_pinned() and not yp.is_pinned()
    for x_, y_ in ((xp, yp), (xh, yp), (xp, yh)):
        y_.zero_()
        assert op.apply(x_, out=y_) is y_
        assert _rel(y_.cuda(), yd) < 1e-14


@pytest.mark.parametrize("cfg,m", [(1, None), (2, 6), (3, 3)])
def test_host_apply_graph_chunks_and_buffers(cfg, m):
    """hf_tangent_apply_host: every slab count (incl. more slabs than cell
    layers), new data through a cached graph, more buffer pairs than the graph
    cache holds, and numpy memory page-locked with hf_host_register."""
    import ctypes as ct

    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200._lib import HfError, check, lib
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(cfg, seed=5, m=m)
    op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
    n = op.n_dofs
    pairs = [(torch.empty(n, dtype=torch.float64).pin_memory(), torch.empty(n, dtype=torch.float64).pin_memory())
             for _ in range(6)]
    rng = np.random.default_rng(11)
    for rep in range(2):
        for k, (xh, yh) in enumerate(pairs):
            for chunks in (1, 3, 8, 1000):
                xh.copy_(torch.from_numpy(rng.standard_normal(n)))
                yh.fill_(np.nan)
                op.apply_host(xh, yh, chunks=chunks)
                yd = op.apply(xh.cuda())
                assert _rel(yh.cuda(), yd) < 1e-14, (rep, k, chunks)
    # pageable memory is refused, registered numpy memory accepted
    xa = rng.standard_normal(n)
    ya = np.zeros(n)
    with pytest.raises(HfError):
        check(lib().hf_tangent_apply_host(op._op, ct.c_void_p(xa.ctypes.data), ct.c_void_p(ya.ctypes.data), 4, None))
    check(lib().hf_host_register(ct.c_void_p(xa.ctypes.data), xa.nbytes))
    check(lib().hf_host_register(ct.c_void_p(ya.ctypes.data), ya.nbytes))
    try:
        check(lib().hf_tangent_apply_host(op._op, ct.c_void_p(xa.ctypes.data), ct.c_void_p(ya.ctypes.data), 4, None))
        torch.cuda.synchronize()
        yd = op.apply(torch.from_numpy(xa).cuda())
        assert _rel(torch.from_numpy(ya).cuda(), yd) < 1e-14
    finally:
        check(lib().hf_host_unregister(ct.c_void_p(xa.ctypes.data)))
        check(lib().hf_host_unregister(ct.c_void_p(ya.ctypes.data)))


def test_host_apply_recalibration():
    """hf_tangent_apply_host recalibrates each buffer pair's pipeline once
    after HostPipe::RECAL_AT (256) calls: results stay exact across it and the
    pipeline info reports a variant afterwards."""
    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(2, seed=3, m=4)
    op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
    n = op.n_dofs
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    yh = torch.empty(n, dtype=torch.float64).pin_memory()
    rng = np.random.default_rng(2)
    for call in range(300):
        if call % 50 == 0 or 254 <= call <= 258:
            xh.copy_(torch.from_numpy(rng.standard_normal(n)))
            yh.fill_(np.nan)
            op.apply(xh, out=yh)
            assert _rel(yh.cuda(), op.apply(xh.cuda())) < 1e-14, call
        else:
            op.apply(xh, out=yh)
    info = op.host_info()
    assert info["variant"] in ("graph+overlap", "graph+serial", "direct+overlap", "direct+serial")
    assert all(v > 0 for v in info["calibration_us"].values())


def test_tile_range_apply_with_reserved_sms():
    """hf_tangent_apply_tiles_ex: tile ranges launched on fewer SMs (room for a
    concurrent NCCL kernel) accumulate the same result as the full apply."""
    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200._lib import check, lib
    from paper_1904_13131_b200 import device as dv
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(2, seed=6, m=12)
    op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
    x = torch.from_numpy(wl.x).cuda()
    ref = op.apply(x)
    nt, _ = op.tiles()
    for reserve in (0, 4, 100):
        y = torch.empty_like(x)
        check(lib().hf_fill_masked(x.numel(), dv.ptr(y), dv.ptr(x), dv.ptr(wl.fine.mask_dev), 0.0, dv.stream()))
        cut = nt // 3
        op.apply_tiles(x, y, 0, cut, reserve_sms=reserve)
        op.apply_tiles(x, y, cut, nt, reserve_sms=reserve)
        assert _rel(y, ref) < 1e-14
