"""Parity at the BASELINE sizes.

* Configs 2 and 3 (823,875 DoFs): apply (all three caching strategies) and
  residual against the whole-problem CPU oracle, the diagonal against the
  oracle on sub-boxes, and apply / residual against the unmodified reference
  itself (oracle/_ref) -- all 1e-12 relative L2.
* Config 4's fine level (64^3, 6.44M DoFs): apply and residual vs the oracle.
* Config 5 (128^3, 50.9M DoFs): apply, diagonal and residual vs the oracle on
  sub-boxes of the full-size problem.
* Size-independent properties at configs 2 and 3: the strategies agree, the
  operator is symmetric and linear and the identity on the constrained
  subspace (operators.py:331-339)."""

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


def _subbox(p, ubar, x, lo, k):
    """The oracle problem of the k^dim cells starting at cell ``lo`` of the
    product problem ``p`` (same vertices, material, mask, u_bar and x), and
    the map from its DoFs to global DoFs with a flag for "complete" DoFs: nodes
    all of whose cells lie in the sub-box, where the sub-box apply / diagonal /
    residual must equal the global ones (every quantity is a sum over cells)."""
    from paper_1904_13131_b200.workloads import MATERIAL

    d, deg, m = p.dim, p.degree, p.mesh.cells
    nv = tuple(c + 1 for c in m)
    V = p.mesh.vertices.reshape(tuple(reversed(nv)) + (d,))
    vs = tuple(slice(lo[a], lo[a] + k + 1) for a in reversed(range(d)))
    cs = tuple(slice(lo[a], lo[a] + k) for a in reversed(range(d)))
    inc = (p.mesh.material_id == 1).reshape(tuple(reversed(m)))[cs].reshape(-1)
    mu = np.where(inc, MATERIAL.inclusion.mu, MATERIAL.matrix.mu)
    lam = np.where(inc, MATERIAL.inclusion.lam, MATERIAL.matrix.lam)
    n1 = tuple(c * deg + 1 for c in m)
    gid = np.arange(p.n_dofs).reshape(tuple(reversed(n1)) + (d,))
    ns = tuple(slice(lo[a] * deg, (lo[a] + k) * deg + 1) for a in reversed(range(d)))
    sub = gid[ns].reshape(-1)
    li = np.indices((k * deg + 1,) * d).reshape(d, -1)[::-1]  # li[a]: local lattice index along axis a
    full = np.ones(li.shape[1], dtype=bool)
    for a in range(d):
        full &= ((li[a] > 0) | (lo[a] == 0)) & ((li[a] < k * deg) | (lo[a] + k == m[a]))
    full = np.repeat(full, d)
    op_ = O.OProblem(d, deg, (k,) * d, np.ascontiguousarray(V[vs].reshape(-1, d)), mu, lam, p.constraints.mask[sub])
    return op_, sub, full, np.ascontiguousarray(ubar[sub]), np.ascontiguousarray(x[sub])


def _subboxes(m, k):
    """A corner box on the clamped face, one in the middle, one at the far corner."""
    return [(0, 0, 0), (m // 2 - k // 2,) * 3, (m - k,) * 3]


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_size_vs_oracle(cfg):
    """Configs 2 (32^3 Q2) and 3 (16^3 Q4) at their BASELINE size: apply for all
    three caching strategies and the residual (with and without traction)
    against the CPU oracle of the whole problem (operators.py:205-224,
    331-339), 1e-12; the diagonal (operators.py:395-410) of every strategy
    against the oracle on sub-boxes at the full-size geometry (complete DoFs)."""
    from paper_1904_13131_b200 import MatrixFreeTangent, compute_residual
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(cfg, seed=0)
    p = wl.fine
    op_ = _oracle_of(p)
    traction = np.array([0.01, -0.02, 0.03])
    for s in ("scalar", "tensor2", "tensor4"):
        op = MatrixFreeTangent(p, wl.ubar, s)
        y = op.apply(wl.x)
        yo = O.Tangent(op_, wl.ubar, s).apply(wl.x)
        assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < TOL, s
        d = op.diagonal(as_numpy=True)
        k = 4 if cfg == 2 else 2
        for lo in _subboxes(p.mesh.cells[0], k):
            sp, sub, full, ub, _ = _subbox(p, wl.ubar, wl.x, lo, k)
            do = O.Tangent(sp, ub, s).diagonal()
            assert np.linalg.norm(d[sub][full] - do[full]) / np.linalg.norm(do[full]) < TOL, (s, lo)
        del op
    for tr in (None, traction):
        r = compute_residual(p, wl.ubar, tr)
        ro = O.residual(op_, wl.ubar, tr)
        assert np.linalg.norm(r - ro) / np.linalg.norm(ro) < TOL


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_size_vs_reference_itself(cfg):
    """The same configs against the UNMODIFIED reference (oracle/_ref, run on
    this host): MatrixFreeTangent.apply (tensor4 and tensor2) and
    compute_residual with traction, 1e-12."""
    from oracle import ref
    from paper_1904_13131_b200 import MatrixFreeTangent, compute_residual
    from paper_1904_13131_b200.workloads import CONFIGS, make_workload

    if not ref.available():
        pytest.skip("oracle/_ref not installed")
    hf = ref.hyperfree()
    wl = make_workload(cfg, seed=0)
    p = wl.fine
    c = CONFIGS[cfg]
    rp = ref.problem(hf, 3, c["m"], c["degree"], wl.centres, c["radius"], p.constraints.mask)
    assert np.array_equal(rp.mu_el[:, 0], p.mu_el[:, 0])
    for s in ("tensor4", "tensor2"):
        y = MatrixFreeTangent(p, wl.ubar, s).apply(wl.x)
        yr = hf.operators.MatrixFreeTangent(rp, wl.ubar, s).apply(wl.x)
        assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < TOL, s
    traction = np.array([0.01, -0.02, 0.03])
    r = compute_residual(p, wl.ubar, traction)
    rr = hf.operators.compute_residual(rp, wl.ubar, traction)
    assert np.linalg.norm(r - rr) / np.linalg.norm(rr) < TOL


def test_config4_fine_level_64_vs_oracle():
    """vmult and residual parity up to 64^3 -- the config-4 fine
    level (6,440,067 DoFs), tensor4 and tensor2 apply and the residual at the
    first load increment, against the whole-problem CPU oracle (1e-12)."""
    from paper_1904_13131_b200 import MatrixFreeTangent, compute_residual
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(4, seed=0)
    p = wl.fine
    op_ = _oracle_of(p)
    for s in ("tensor4", "tensor2"):
        y = MatrixFreeTangent(p, wl.ubar, s).apply(wl.x)
        yo = O.Tangent(op_, wl.ubar, s).apply(wl.x)
        assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < TOL, s
        del yo
    r = compute_residual(p, wl.ubar)
    ro = O.residual(op_, wl.ubar)
    assert np.linalg.norm(r - ro) / np.linalg.norm(ro) < TOL


def test_config5_128_subboxes_vs_oracle():
    """Config 5 (128^3 Q2, 50.9M DoFs) is beyond a whole-problem CPU oracle
    (SURVEY H9), but every entry of y = A x, diag(A) and the residual is a sum
    over the cells around its node: on sub-boxes of the full-size problem the
    oracle gives the exact value at every DoF whose cells all lie in the box."""
    from paper_1904_13131_b200 import MatrixFreeTangent, compute_residual
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(5, seed=0)
    p = wl.fine
    op = MatrixFreeTangent(p, wl.ubar, "tensor4")
    y = op.apply(wl.x)
    d = op.diagonal(as_numpy=True)
    del op
    r = compute_residual(p, wl.ubar)
    k = 6
    for lo in _subboxes(p.mesh.cells[0], k):
        sp, sub, full, ub, xs = _subbox(p, wl.ubar, wl.x, lo, k)
        to = O.Tangent(sp, ub, "tensor4")
        yo = to.apply_unconstrained_input(np.where(sp.mask, 0.0, xs))
        yo[sp.mask] = xs[sp.mask]
        assert np.linalg.norm(y[sub][full] - yo[full]) / np.linalg.norm(yo[full]) < TOL, lo
        do = to.diagonal()
        assert np.linalg.norm(d[sub][full] - do[full]) / np.linalg.norm(do[full]) < TOL, lo
        ro = O.residual(sp, ub)
        assert np.linalg.norm(r[sub][full] - ro[full]) / np.linalg.norm(ro[full]) < TOL, lo


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


def test_numpy_apply_repeated_uses_staging():
    """apply(ndarray) -> fresh ndarray (operators.py:331-339): from the third
    call the tangent stages through page-locked buffers and the host pipeline;
    results equal the device apply, x is untouched, y is a fresh array."""
    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(2, seed=4, m=8)
    op = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4")
    rng = np.random.default_rng(3)
    outs = []
    for k in range(6):
        x = rng.standard_normal(op.n_dofs)
        x0 = x.copy()
        y = op.apply(x)
        assert isinstance(y, np.ndarray) and np.array_equal(x, x0)
        yd = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.linalg.norm(y - yd) / np.linalg.norm(yd) < 1e-14, k
        outs.append(y)
    assert all(a is not b and not np.shares_memory(a, b) for a, b in zip(outs, outs[1:]))


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


def test_host_apply_recalibration(monkeypatch):
    """With HF_E2E_RECAL=1, hf_tangent_apply_host recalibrates each buffer
    pair's pipeline once after HostPipe::RECAL_AT (256) calls: results stay
    exact across it and the pipeline info reports a variant afterwards."""
    monkeypatch.setenv("HF_E2E_RECAL", "1")
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


@pytest.mark.parametrize("dim,degree,m", [(2, 5, 6), (2, 6, 5), (2, 7, 5), (2, 8, 4), (3, 1, 7), (3, 3, 5)])
def test_every_instantiated_degree_vs_oracle_and_reference(dim, degree, m):
    """The degrees the golden files do not hold (2D Q5-Q8: warp tiles of 5, 4, 4
    and 3 cells; 3D Q1 and Q3 on a mesh whose cell count is not a multiple of the
    tile): apply of every caching variant, diagonal and residual against the
    oracle, and apply / residual against the unmodified reference itself."""
    from oracle import ref
    from paper_1904_13131_b200 import MatrixFreeTangent, Problem, build_benchmark_mesh, compute_residual
    from paper_1904_13131_b200.workloads import MATERIAL, clamp_weighted_sine, constrain

    rng = np.random.default_rng(degree * 10 + dim)
    centres = rng.random((3, dim))
    radius = 0.2
    p = Problem(build_benchmark_mesh(dim, m, [(c, radius) for c in centres], side=1.0), degree, MATERIAL)
    constrain(p, 0)
    ubar = clamp_weighted_sine(dim, m, degree, 2.0 * np.pi * rng.random((dim, dim)), 0.03, 0)
    x = rng.standard_normal(p.n_dofs)
    op_ = _oracle_of(p)
    for s in O.STRATEGIES:
        op = MatrixFreeTangent(p, ubar, s)
        y = op.apply(x)
        yo = O.Tangent(op_, ubar, s).apply(x)
        assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < TOL, s
        d = np.asarray(op.diagonal())
        do = O.Tangent(op_, ubar, s).diagonal()
        assert np.linalg.norm(d - do) / np.linalg.norm(do) < TOL, s
    traction = np.array([0.01, -0.02, 0.03])[:dim]
    r = compute_residual(p, ubar, traction)
    ro = O.residual(op_, ubar, traction)
    assert np.linalg.norm(r - ro) / np.linalg.norm(ro) < TOL
    if ref.available():
        hf = ref.hyperfree()
        rp = ref.problem(hf, dim, m, degree, centres, radius, p.constraints.mask)
        yr = hf.operators.MatrixFreeTangent(rp, ubar, "tensor4").apply(x)
        assert np.linalg.norm(MatrixFreeTangent(p, ubar, "tensor4").apply(x) - yr) / np.linalg.norm(yr) < TOL
        rr = hf.operators.compute_residual(rp, ubar, traction)
        assert np.linalg.norm(r - rr) / np.linalg.norm(rr) < TOL
