"""fp32 multigrid levels (BASELINE north_star: 1e-5 for
the optional fp32 levels): fp32-storage tangents against fp64, mixed-precision
transfers, and GMG-CG with every level below the finest in fp32."""

import numpy as np
import pytest
import torch

from _cases import golden, product_levels, product_problem, rel

pytestmark = pytest.mark.gpu
TOL32 = 1e-5


@pytest.mark.parametrize("name", ["ops_2d_q2.npz", "ops_3d_q2.npz", "ops_3d_q4.npz", "ops_2d_q4_gl.npz"])
@pytest.mark.parametrize("strategy", ["scalar", "tensor2", "tensor4"])
def test_fp32_storage_tangent(name, strategy):
    from paper_1904_13131_b200 import MatrixFreeTangent

    g = golden(name)
    p = product_problem(g)
    op32 = MatrixFreeTangent(p, g["ubar"], strategy, storage="fp32")
    assert op32.cache.payload_nbytes * 2 == MatrixFreeTangent(p, g["ubar"], strategy).cache.payload_nbytes
    y = op32.apply(g["x"])  # public apply: fp64 in, fp64 out
    assert rel(y, g[f"y_{strategy}"]) < TOL32
    x32 = torch.from_numpy(g["x"]).float().cuda()
    y32 = torch.empty_like(x32)
    op32.apply_into(x32, y32)
    assert y32.dtype == torch.float32
    assert rel(y32.double().cpu().numpy(), g[f"y_{strategy}"]) < TOL32
    with pytest.raises(Exception):
        op32.diagonal()


def test_fp32_at_config2_size():
    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(2, seed=0)
    y64 = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4").apply(wl.x)
    y32 = MatrixFreeTangent(wl.fine, wl.ubar, "tensor4", storage="fp32").apply(wl.x)
    assert rel(y32, y64) < TOL32


def test_mixed_precision_transfers():
    from paper_1904_13131_b200 import build_transfers

    g = golden("mg_3d_8.npz")
    probs = product_levels(g)
    t = build_transfers(probs)[-1]
    rf = torch.from_numpy(g["restrict_in_0"] if "restrict_in_0" in g else np.random.default_rng(1).standard_normal(
        probs[-1].n_dofs)).cuda()
    ref = t.restrict_into(rf, torch.empty(probs[-2].n_dofs, dtype=torch.float64, device="cuda"))
    r32 = t.restrict_into(rf, torch.empty(probs[-2].n_dofs, dtype=torch.float32, device="cuda"))
    assert rel(r32.double().cpu().numpy(), ref.cpu().numpy()) < 1e-7
    xc = torch.randn(probs[-2].n_dofs, dtype=torch.float64, device="cuda")
    pf = t.prolong_into(xc, torch.zeros(probs[-1].n_dofs, dtype=torch.float64, device="cuda"))
    p32 = t.prolong_into(xc.float(), torch.zeros(probs[-1].n_dofs, dtype=torch.float64, device="cuda"))
    assert rel(p32.cpu().numpy(), pf.cpu().numpy()) < 1e-7


@pytest.mark.parametrize("name", ["mg_2d_32_cfg1.npz", "mg_3d_8.npz", "mg_2d_16.npz"])
def test_gmg_cg_with_fp32_levels(name):
    from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg, cg

    g = golden(name)
    probs = product_levels(g)
    op = MatrixFreeTangent(probs[-1], g["ubar"], str(g["strategy"]))
    gmg = build_gmg(probs, g["ubar"], str(g["strategy"]), seed=0, coarse_precision="fp32")
    assert all(lv.x.dtype == torch.float32 for lv in gmg.levels[1:-1])
    assert gmg.levels[-1].x.dtype == torch.float64 and gmg.levels[0].x.dtype == torch.float64
    x, rep = cg(op, g["b"], rel_tol=1e-8, preconditioner=gmg)
    assert rep.converged
    assert rep.iterations <= int(g["cg_iterations"]) + 2
    # fp32 levels: BASELINE north_star's 1e-5 tolerance (the CG stops at
    # ||r|| <= 1e-8 ||b||; the iterate's distance from the fp64 run's is
    # cond(A) x that, ~1e-6 for these levels)
    assert rel(x, g["cg_solution"]) < 1e-5
