"""GPU parity of the multigrid/CG path against the reference golden runs:
transfers, injection, Lanczos range, Chebyshev, coarse solve, V-cycle, GMG-CG."""

import numpy as np
import pytest

from _cases import golden, product_levels, rel

pytestmark = pytest.mark.gpu
MG = ["mg_2d_16.npz", "mg_3d_8.npz", "mg_2d_32_cfg1.npz"]


@pytest.fixture(scope="module", params=MG)
def case(request):
    from paper_1904_13131_b200 import build_gmg, build_transfers

    g = golden(request.param)
    probs = product_levels(g)
    for i, p in enumerate(probs):
        assert np.array_equal(p.mu_el[:, 0], g[f"mu_{i}"]), "per-level centroid material differs"
    transfers = build_transfers(probs)
    gmg = build_gmg(probs, g["ubar"], str(g["strategy"]), seed=0, transfers=transfers)
    return g, probs, transfers, gmg


def test_transfers(case):
    g, probs, transfers, _ = case
    for i, t in enumerate(transfers):
        assert rel(t.prolong(g[f"prolong_in_{i}"]), g[f"prolong_out_{i}"]) < 1e-14
        assert rel(t.restrict(g[f"restrict_in_{i}"]), g[f"restrict_out_{i}"]) < 1e-14


def test_injection(case):
    from paper_1904_13131_b200 import restrict_solution

    g, probs, _, _ = case
    for i, v in enumerate(restrict_solution(probs, g["ubar"])):
        assert np.array_equal(v, g[f"inject_{i}"])


def test_level_setup(case):
    g, probs, _, gmg = case
    for i, lv in enumerate(gmg.levels):
        assert rel(lv.diag.cpu().numpy(), g[f"diag_{i}"]) < 1e-12
        assert abs(lv.lam_max - float(g[f"lam_max_{i}"])) <= 1e-9 * abs(float(g[f"lam_max_{i}"]))
        # lam_min of the coarsest level comes from 120 Lanczos steps without
        # re-orthogonalisation (multigrid.py:231-242): rounding-sensitive
        assert abs(lv.lam_min - float(g[f"lam_min_{i}"])) <= 1e-4 * abs(float(g[f"lam_min_{i}"]))


def test_chebyshev_and_coarse(case):
    from paper_1904_13131_b200 import ChebyshevSettings, chebyshev_apply, coarse_solve

    g, probs, _, gmg = case
    lv = gmg.levels[-1]
    out = chebyshev_apply(lv.op, lv.inv_diag, lv.lam_max, g["b"], g["cheb_x0"], ChebyshevSettings(), 2)
    assert rel(out, g["cheb_out"]) < 1e-10
    # the coarse Chebyshev polynomial depends on lam_min (see test_level_setup)
    assert rel(coarse_solve(gmg.levels[0], g["coarse_b"]), g["coarse_out"]) < 1e-4


def test_vcycle(case):
    g, probs, _, gmg = case
    z = gmg.apply(g["b"])
    assert rel(z, g["vcycle"]) < 1e-5
    z2 = gmg.apply(g["b"])  # graph replay: same result up to fp64 atomic ordering
    assert rel(z2, z) < 1e-11


def test_vcycle_vs_oracle_same_spectrum(case):
    """Oracle V-cycle with the GPU's eigenvalue estimates: isolates the V-cycle
    arithmetic from the Lanczos rounding sensitivity (tight tolerance)."""
    from oracle import hf_oracle as O

    g, probs, _, gmg = case
    if probs[-1].n_dofs > 20000:
        pytest.skip("oracle diagonal too slow for this size")
    oprobs = [O.OProblem(p.dim, 2, p.mesh.cells, p.mesh.vertices, p.mu_el, p.lam_el, p.constraints.mask)
              for p in probs]
    og = O.GMG(oprobs, g["ubar"], str(g["strategy"]), 0)
    for lo, lv in zip(og.levels, gmg.levels):
        lo.lam_min, lo.lam_max = lv.lam_min, lv.lam_max
    assert rel(gmg.apply(g["b"]), og.apply(g["b"])) < 1e-11


def test_gmg_cg(case):
    from paper_1904_13131_b200 import MatrixFreeTangent, cg

    g, probs, _, gmg = case
    op = MatrixFreeTangent(probs[-1], g["ubar"], str(g["strategy"]))
    x, rep = cg(op, g["b"], rel_tol=1e-8, preconditioner=gmg)
    assert abs(rep.iterations - int(g["cg_iterations"])) <= 1
    assert rel(x, g["cg_solution"]) < 1e-6
    h = np.array(rep.residual_history)
    k = min(len(h), len(g["cg_history"]))
    assert np.allclose(h[:k], g["cg_history"][:k], rtol=1e-5)


def test_chained_chebyshev_update_matches_plain_launch(case, monkeypatch):
    """On small levels the Chebyshev update is launched as the cell kernel's
    programmatic dependent (hf_cheb_step_after_apply); with the threshold at
    zero every update is a plain launch.  Same arithmetic: the smoothed
    iterates agree to the rounding of the scatter's atomic order."""
    from paper_1904_13131_b200 import ChebyshevSettings, chebyshev_apply, multigrid

    g, _, _, gmg = case
    lv = gmg.levels[-1]
    assert lv.problem.n_dofs <= multigrid._PDL_CHEB_MAX_DOFS
    chained = chebyshev_apply(lv.op, lv.inv_diag, lv.lam_max, g["b"], g["cheb_x0"], ChebyshevSettings(), 2)
    monkeypatch.setattr(multigrid, "_PDL_CHEB_MAX_DOFS", 0)
    plain = chebyshev_apply(lv.op, lv.inv_diag, lv.lam_max, g["b"], g["cheb_x0"], ChebyshevSettings(), 2)
    assert rel(chained, plain) < 1e-12
    assert rel(chained, g["cheb_out"]) < 1e-10


@pytest.mark.parametrize("degree,steps", [(3, 1), (4, 1), (5, 3), (2, 1), (1, 3)])
def test_three_term_chebyshev_matches_stored_direction(case, degree, steps, monkeypatch):
    """The product smoother keeps x_{k-1} instead of the direction
    (hf_cheb3_step, d = x_k - x_{k-1}); hf_cheb_step* store d as the reference
    does (multigrid.py:195-204).  Same iterates to rounding, for even and odd
    numbers of updates (an odd count ends in the second buffer and is copied)."""
    from paper_1904_13131_b200 import ChebyshevSettings, chebyshev_apply, multigrid

    g, _, _, gmg = case
    lv = gmg.levels[-1]
    s = ChebyshevSettings(degree=degree)
    three = chebyshev_apply(lv.op, lv.inv_diag, lv.lam_max, g["b"], g["cheb_x0"], s, steps)
    monkeypatch.setattr(multigrid, "_CHEB3", False)
    stored = chebyshev_apply(lv.op, lv.inv_diag, lv.lam_max, g["b"], g["cheb_x0"], s, steps)
    assert rel(three, stored) < 1e-12


def test_cg_fused_p_update_matches_plain_launches(case):
    """cg on the tangent itself fuses the p update with the next A p's
    initialisation and chains that apply as a programmatic dependent
    (hf_cg_update_p_fill); through a plain ``apply_into`` wrapper it launches
    the update, the fill and the apply separately.  Same iteration, so the
    residual histories agree to rounding (the scatter's atomic order)."""
    from paper_1904_13131_b200 import MatrixFreeTangent, cg

    g, probs, _, gmg = case
    op = MatrixFreeTangent(probs[-1], g["ubar"], str(g["strategy"]))

    class Plain:
        def apply_into(self, x, y):
            return op.apply_into(x, y)

    x1, r1 = cg(op, g["b"], rel_tol=1e-8, preconditioner=gmg)
    x2, r2 = cg(Plain(), g["b"], rel_tol=1e-8, preconditioner=gmg)
    assert r1.iterations == r2.iterations
    assert np.allclose(r1.residual_history, r2.residual_history, rtol=1e-6)
    assert rel(x1, x2) < 1e-8


def test_newton_traction_reference():
    """The reference's own newton_solve (traction) on a tiny 2D problem."""
    from paper_1904_13131_b200 import LoadSpec, NewtonSettings, newton_solve

    g = golden("newton_traction_2d.npz")
    g["dim"] = 2
    probs = product_levels(g)
    res = newton_solve(probs, NewtonSettings(n_load_steps=int(g["n_steps"])),
                       LoadSpec(float(g["magnitude"]), tuple(g["direction"])), "gmg", "tensor4", seed=0)
    recs = np.array([(r.load_step, r.fraction, r.iteration, r.residual_norm, r.update_norm, r.cg_iterations)
                     for r in res.records])
    ref = g["records"]
    assert recs.shape == ref.shape
    assert np.array_equal(recs[:, [0, 2]], ref[:, [0, 2]])
    assert np.all(np.abs(recs[:, 5] - ref[:, 5]) <= 1)
    big = ref[:, 3] > 1e-9
    assert np.allclose(recs[big, 3], ref[big, 3], rtol=1e-4)
    assert rel(res.u.cpu().numpy(), g["u"]) < 1e-8


def test_newton_load_bisection_reference():
    """One load step whose full increment inverts an element: newton_solve
    catches NonPositiveJacobian and bisects the step once (solver.py:196-199),
    keeping the failed attempt's records, as the reference run did."""
    from paper_1904_13131_b200 import LoadSpec, NewtonSettings, newton_solve

    g = golden("newton_bisect_2d.npz")
    g["dim"] = 2
    probs = product_levels(g)
    res = newton_solve(probs, NewtonSettings(n_load_steps=int(g["n_steps"])),
                       LoadSpec(float(g["magnitude"]), tuple(g["direction"])), "gmg", "tensor4", seed=0)
    recs = np.array([(r.load_step, r.fraction, r.iteration, r.residual_norm, r.update_norm, r.cg_iterations)
                     for r in res.records])
    ref = g["records"]
    assert 0.5 in ref[:, 1]
    assert recs.shape == ref.shape
    assert np.array_equal(recs[:, :3], ref[:, :3])  # step, fraction (bisected), iteration
    assert np.all(np.abs(recs[:, 5] - ref[:, 5]) <= 1)
    big = ref[:, 3] > 1e-9
    assert np.allclose(recs[big, 3], ref[big, 3], rtol=1e-4)
    assert rel(res.u.cpu().numpy(), g["u"]) < 1e-8


def test_newton_matrix_based_with_gmg():
    """strategy="matrix_based" with the GMG preconditioner: the fine operator
    is the assembled CSR, the GMG levels are tensor4 (solver.py:128-135)."""
    from paper_1904_13131_b200 import LoadSpec, NewtonSettings, newton_solve

    g = golden("newton_traction_2d.npz")
    g["dim"] = 2
    probs = product_levels(g)
    res = newton_solve(probs, NewtonSettings(n_load_steps=int(g["n_steps"])),
                       LoadSpec(float(g["magnitude"]), tuple(g["direction"])), "gmg", "matrix_based", seed=0)
    ref = g["records"]
    assert len(res.records) == len(ref)
    assert rel(res.u.cpu().numpy(), g["u"]) < 1e-8


def test_newton_prescribed_golden():
    """Config-4 restatement (prescribed top displacement) vs the
    golden run driven by reference primitives (tests/golden/make_golden.py)."""
    from paper_1904_13131_b200 import NewtonSettings, newton_solve_prescribed

    g = golden("newton_prescribed_3d.npz")
    g["dim"] = 3
    probs = product_levels(g)
    res = newton_solve_prescribed(probs, NewtonSettings(n_load_steps=int(g["n_steps"])), float(g["target"]))
    recs = np.array([(r.load_step, r.iteration, r.residual_norm, r.update_norm, r.cg_iterations) for r in res.records])
    ref = g["records"]
    assert recs.shape == ref.shape
    assert np.array_equal(recs[:, :2], ref[:, :2])
    assert np.all(np.abs(recs[:, 4] - ref[:, 4]) <= 1)
    assert np.allclose(recs[:, 2], ref[:, 2], rtol=1e-3, atol=1e-11)
    assert rel(res.u.cpu().numpy(), g["u"]) < 1e-8


def _coarse_reference(A, inv_d, b, lv, rel_target, max_applications=100):
    """coarse_solve (multigrid.py:255-306) in extended precision (np.longdouble)
    on the assembled level matrix: the yardstick for both fp64 paths."""
    from paper_1904_13131_b200.multigrid import ChebyshevSettings

    s = lv.coarse_settings(ChebyshevSettings())
    ld = np.longdouble
    theta = ld(0.5) * (ld(s.range_hi) + ld(s.range_lo)) * ld(lv.lam_max)
    delta = ld(0.5) * (ld(s.range_hi) - ld(s.range_lo)) * ld(lv.lam_max)
    sigma = theta / delta
    A, inv_d, b = A.astype(ld), inv_d.astype(ld), b.astype(ld)
    target = ld(rel_target) * np.sqrt(b @ b)
    d = inv_d * b / theta
    x = d.copy()
    rho_old = 1 / sigma
    for step in range(2, max_applications + 1):
        ax = A @ x
        if step % s.degree == 0 and np.sqrt((b - ax) @ (b - ax)) <= target:
            return x.astype(np.float64), True
        rho = 1 / (2 * sigma - rho_old)
        d = rho * rho_old * d + 2 * rho / delta * (inv_d * (b - ax))
        x = x + d
        rho_old = rho
    return x.astype(np.float64), False


@pytest.mark.parametrize("single", ["1", "0"])
def test_coarse_kernel_matches_launches(case, single, monkeypatch):
    """The one-kernel coarse solve (hf_coarse_cheb_solve on the assembled level
    matrix) against the per-application launches on the matrix-free operator
    and an extended-precision restatement of the same iteration.  The coarse
    levels of these cases are ill-conditioned: a 99-application Chebyshev
    iterate amplifies fp64 rounding (summation order of CSR vs matrix-free
    applies) to ~1e-6, so the check is that the kernel is as close to the
    extended-precision iterate as the launches are.  The stop/cap flag agrees,
    b = 0 returns x = 0, and GMG-CG takes the same number of iterations."""
    from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg, cg
    from paper_1904_13131_b200.multigrid import LevelOperator, coarse_solve, restrict_solution
    from paper_1904_13131_b200.operators import AssembledTangent

    g, probs, transfers, _ = case
    monkeypatch.setenv("HF_COARSE_SINGLE", single)  # single-CTA form where the level fits, or always multi-CTA
    u0 = restrict_solution(probs, g["ubar"])[0]
    lv = {}
    for mode in ("kernel", "launches"):
        monkeypatch.setenv("HF_COARSE", mode)
        lv[mode] = LevelOperator(probs[0], u0, str(g["strategy"]), seed=0, level=0, is_coarsest=True)
    assert lv["kernel"].coarse is not None and lv["launches"].coarse is None
    A = AssembledTangent(probs[0], u0).matrix.to_dense().cpu().numpy()
    inv_d = lv["kernel"].inv_diag.cpu().numpy()
    rng = np.random.default_rng(4)
    for rel_target in (1e-3, 1e-9):
        b = rng.standard_normal(probs[0].n_dofs)
        b[probs[0].constraints.mask] = 0.0
        xk = coarse_solve(lv["kernel"], b, rel_target=rel_target)
        xl = coarse_solve(lv["launches"], b, rel_target=rel_target)
        xr, converged = _coarse_reference(A, inv_d, b, lv["kernel"], rel_target)
        ek, el = rel(xk, xr), rel(xl, xr)
        assert ek < max(1e-11, 10 * el), (rel_target, ek, el)
        assert ek < 1e-4
        assert lv["kernel"].cap_reached() == lv["launches"].cap_reached() == (not converged)
    z = coarse_solve(lv["kernel"], np.zeros(probs[0].n_dofs))
    assert not np.any(z) and not lv["kernel"].cap_reached()
    its = {}
    for mode in ("kernel", "launches"):
        monkeypatch.setenv("HF_COARSE", mode)
        gmg = build_gmg(probs, g["ubar"], str(g["strategy"]), seed=0, transfers=transfers)
        assert (gmg.levels[0].coarse is not None) == (mode == "kernel")
        op = MatrixFreeTangent(probs[-1], g["ubar"], str(g["strategy"]))
        its[mode] = cg(op, g["b"], rel_tol=1e-8, preconditioner=gmg)
    assert abs(its["kernel"][1].iterations - its["launches"][1].iterations) <= 1
    assert rel(its["kernel"][0], its["launches"][0]) < 1e-6


def test_vcycle_graph_updated_in_place_for_a_rebuilt_hierarchy():
    """A second hierarchy of the same shape (another linearisation point: new
    caches, diagonals and Chebyshev coefficients) reuses the first one's
    executable graph through hf_graph_end's in-place update; its replayed
    V-cycle equals its own eager run, and the first hierarchy's result is not
    what it returns."""
    import gc

    from paper_1904_13131_b200 import build_gmg, build_transfers

    import ctypes as ct

    from paper_1904_13131_b200 import device as dv
    from paper_1904_13131_b200._lib import lib

    for handles in dv.LaunchGraph._idle.values():  # start without idle graphs from earlier tests
        for h in handles:
            lib().hf_graph_destroy(ct.c_void_p(h))
    dv.LaunchGraph._idle.clear()
    g = golden("mg_3d_8.npz")
    probs = product_levels(g)
    transfers = build_transfers(probs)
    b = g["b"]
    first = build_gmg(probs, g["ubar"], "tensor4", seed=0, transfers=transfers)
    z1 = first.apply(b)
    assert not first._graph.updated
    del first
    gc.collect()
    u2 = 0.5 * g["ubar"]
    second = build_gmg(probs, u2, "tensor4", seed=0, transfers=transfers)
    z2 = second.apply(b)
    assert second._graph.updated, "the idle executable graph of the same shape was not reused"
    # the same hierarchy run eagerly (two separately built hierarchies differ by ~1e-7: the coarsest
    # level's lam_min comes from 120 Lanczos steps without re-orthogonalisation, multigrid.py:231-242)
    import torch

    second._b.copy_(torch.from_numpy(b).cuda())
    second._run()
    ze = second._x.cpu().numpy()
    assert rel(z2, ze) < 1e-11
    assert rel(z2, z1) > 1e-6  # a different operator: the update carried the new pointers and coefficients
    assert rel(second.apply(b), ze) < 1e-11  # replay
