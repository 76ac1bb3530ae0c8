"""Generate golden input/output vectors by running the UNMODIFIED reference.

Run in the build container (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--newton]

It imports ``hyperfree`` read-only from ``/root/reference/pkg/src`` and writes
small ``.npz`` fixtures next to this file.  Inputs follow the synthetic recipe
of SURVEY.md §8(d) (seeded inclusion centres, clamp-weighted sine state,
N(0,1) vector) and are stored in the fixtures too, so tests never need to
re-derive them.  The constraint overrides of SURVEY H2/H5 are applied by
replacing ``Problem.constraints`` with ``ConstraintSet.from_dofs``.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from hyperfree import fespace, material, mesh as rmesh, multigrid, operators, solver  # noqa: E402
from hyperfree.flops import FLOPS, counting  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
MAT = operators.Material(
    matrix=material.NeoHookeanParams.from_shear_and_poisson(1.0, 0.3),
    inclusion=material.NeoHookeanParams.from_shear_and_poisson(10.0, 0.3),
)


def synth(dim, m, n_inc, radius, seed, amp, clamp_axis, degree=2, node_rule="equispaced", perturb=0.0):
    """SURVEY §8(d) recipe: one rng, draws in a fixed order."""
    rng = np.random.default_rng(seed)
    centres = rng.random((n_inc, dim))
    phases = 2.0 * np.pi * rng.random((dim, dim))
    msh = rmesh.build_benchmark_mesh(dim, m, [(c, radius) for c in centres], side=1.0)
    if perturb:
        # interior vertex jitter (general multilinear geometry path)
        v = msh.vertices.copy()
        inner = np.all((v > 1e-12) & (v < 1 - 1e-12), axis=1)
        v[inner] += perturb / m * (rng.random((inner.sum(), dim)) - 0.5)
        import dataclasses

        msh = dataclasses.replace(msh, vertices=v)
    prob = operators.Problem(msh, degree, MAT, basis_nodes=node_rule)
    X = fespace.node_coordinates(msh, prob.dofmap)
    u = np.empty((prob.dofmap.n_nodes, dim))
    for c in range(dim):
        u[:, c] = amp * X[:, clamp_axis] * np.prod(np.sin(np.pi * X + phases[c][None, :]), axis=1)
    x = rng.standard_normal(prob.n_dofs)
    return prob, msh, centres, phases, u.reshape(-1), x


def clamp(prob, axis, comps=None, extra=None):
    dm = prob.dofmap
    idx = rmesh.lex_grid_indices((dm.nodes_per_side,) * prob.dim)
    nodes = np.flatnonzero(idx[:, axis] == 0)
    comps = range(prob.dim) if comps is None else comps
    dofs = [nodes * prob.dim + c for c in comps]
    if extra is not None:
        dofs.append(extra)
    prob.constraints = fespace.ConstraintSet.from_dofs(prob.n_dofs, np.concatenate(dofs))
    return prob.constraints.mask


def top_z_dofs(prob):
    dm = prob.dofmap
    idx = rmesh.lex_grid_indices((dm.nodes_per_side,) * prob.dim)
    nodes = np.flatnonzero(idx[:, prob.dim - 1] == dm.nodes_per_side - 1)
    return nodes * prob.dim + (prob.dim - 1)


def op_case(name, dim, m, degree, n_inc, radius, seed, amp, clamp_axis, node_rule="equispaced", perturb=0.0):
    prob, msh, centres, phases, ubar, x = synth(dim, m, n_inc, radius, seed, amp, clamp_axis, degree, node_rule, perturb)
    mask = clamp(prob, clamp_axis)
    out = dict(dim=dim, m=m, degree=degree, seed=seed, amp=amp, clamp_axis=clamp_axis, node_rule=node_rule,
               vertices=msh.vertices, material_id=msh.material_id, mu_el=prob.mu_el[:, 0], lam_el=prob.lam_el[:, 0],
               mask=mask, centres=centres, phases=phases, ubar=ubar, x=x, radius=radius,
               jac_inv=prob.geometry.jac_inv, jxw=prob.geometry.jxw)
    for s in operators.STRATEGIES:
        op = operators.MatrixFreeTangent(prob, ubar, s)
        out[f"y_{s}"] = op.apply(x)
        FLOPS.reset()
        with counting():
            op.apply(x)
        out[f"flops_{s}"] = FLOPS.count
        out[f"storage_{s}"] = op.storage_bytes()
        out[f"diag_{s}"] = op.diagonal()
    traction = np.linspace(0.01, 0.03, dim)
    out["traction"] = traction
    out["residual"] = operators.compute_residual(prob, ubar, traction)
    out["residual_notraction"] = operators.compute_residual(prob, ubar)
    out["surface_weights"] = prob.surface_weights
    out["jrange"] = np.array(operators.jacobian_range(prob, ubar))
    out["energy"] = operators.energy(prob, ubar, traction)
    # an inverted state for the error path
    Xn = fespace.node_coordinates(msh, prob.dofmap)
    bad = ubar.copy()
    bad.reshape(-1, dim)[:, 0] -= 3.0 * Xn[:, 0] ** 2 * (1.0 + 0.5 * Xn[:, 1] + 0.25 * Xn[:, -1])
    try:
        operators.MatrixFreeTangent(prob, bad, "tensor4")
        out["bad_element"] = -1
    except material.NonPositiveJacobian as e:
        out["bad_element"] = e.element
    out["bad_state"] = bad
    np.savez_compressed(os.path.join(HERE, f"ops_{name}.npz"), **out)
    print("wrote", name, prob.n_dofs, flush=True)


def hierarchy_problems(dim, levels_m, degree, centres, radius):
    """One Problem per level with per-level centroid material."""
    meshes = [rmesh.build_benchmark_mesh(dim, mm, [(c, radius) for c in centres], side=1.0) for mm in levels_m]
    return [operators.Problem(mm, degree, MAT) for mm in meshes]


def mg_case(name, dim, levels_m, n_inc, radius, seed, amp, clamp_axis, strategy="tensor4", full_cg=True):
    rng = np.random.default_rng(seed)
    centres = rng.random((n_inc, dim))
    phases = 2.0 * np.pi * rng.random((dim, dim))
    problems = hierarchy_problems(dim, levels_m, 2, centres, radius)
    masks = [clamp(p, clamp_axis) for p in problems]
    fine = problems[-1]
    X = fespace.node_coordinates(fine.mesh, fine.dofmap)
    u = np.empty((fine.dofmap.n_nodes, dim))
    for c in range(dim):
        u[:, c] = amp * X[:, clamp_axis] * np.prod(np.sin(np.pi * X + phases[c][None, :]), axis=1)
    ubar = u.reshape(-1)
    x = rng.standard_normal(fine.n_dofs)
    out = dict(dim=dim, levels_m=np.array(levels_m), n_inc=n_inc, radius=radius, seed=seed, amp=amp,
               clamp_axis=clamp_axis, centres=centres, phases=phases, ubar=ubar, x=x, strategy=strategy)
    for i, mk in enumerate(masks):
        out[f"mask_{i}"] = mk
        out[f"mu_{i}"] = problems[i].mu_el[:, 0]
        out[f"lam_{i}"] = problems[i].lam_el[:, 0]
    transfers = multigrid.build_transfers(problems)
    # transfers on random vectors
    trng = np.random.default_rng(seed + 1)
    for i, t in enumerate(transfers):
        xc = trng.standard_normal(problems[i].n_dofs)
        xf = trng.standard_normal(problems[i + 1].n_dofs)
        out[f"prolong_in_{i}"], out[f"prolong_out_{i}"] = xc, t.prolong(xc)
        out[f"restrict_in_{i}"], out[f"restrict_out_{i}"] = xf, t.restrict(xf)
    ul = multigrid.restrict_solution(problems, ubar)
    for i, v in enumerate(ul):
        out[f"inject_{i}"] = v
    t0 = time.time()
    gmg = multigrid.build_gmg(problems, ubar, strategy, seed=0, transfers=transfers)
    out["setup_s"] = time.time() - t0
    for i, lv in enumerate(gmg.levels):
        out[f"lam_min_{i}"], out[f"lam_max_{i}"] = lv.lam_min, lv.lam_max
        out[f"diag_{i}"] = lv.diag
    op = operators.MatrixFreeTangent(fine, ubar, strategy)
    b = op.apply(x)
    b[fine.constraints.mask] = 0.0
    out["b"] = b
    out["vcycle"] = gmg.apply(b)
    # one smoother application on the finest level from a random start
    lv = gmg.levels[-1]
    x0 = trng.standard_normal(fine.n_dofs)
    out["cheb_x0"] = x0
    out["cheb_out"] = multigrid.chebyshev_apply(lv.op.apply, lv.inv_diag, lv.lam_max, b, x0, multigrid.ChebyshevSettings(), 2)
    out["coarse_b"] = trng.standard_normal(problems[0].n_dofs) * (~problems[0].constraints.mask)
    out["coarse_out"] = multigrid.coarse_solve(gmg.levels[0], out["coarse_b"])
    if full_cg:
        t0 = time.time()
        sol, rep = solver.cg(op.apply, b, rel_tol=1e-8, preconditioner=gmg.apply)
        out["cg_s"] = time.time() - t0
        out["cg_iterations"] = rep.iterations
        out["cg_history"] = np.array(rep.residual_history)
        out["cg_solution"] = sol
    np.savez_compressed(os.path.join(HERE, f"mg_{name}.npz"), **out)
    print("wrote", name, out.get("cg_iterations"), flush=True)


def newton_traction_case():
    """The reference's own newton_solve (traction load) on a tiny 2D problem."""
    rng = np.random.default_rng(11)
    centres = rng.random((3, 2))
    problems = hierarchy_problems(2, (2, 4), 2, centres, 0.2)
    load = solver.LoadSpec(magnitude=0.05, direction=(1.0, 0.0))
    res = solver.newton_solve(problems, solver.NewtonSettings(n_load_steps=2), load, "gmg", "tensor4", seed=0)
    recs = np.array([(r.load_step, r.fraction, r.iteration, r.residual_norm, r.update_norm, r.cg_iterations)
                     for r in res.records])
    out = dict(centres=centres, radius=0.2, levels_m=np.array((2, 4)), magnitude=0.05, direction=np.array((1.0, 0.0)),
               n_steps=2, records=recs, u=res.u)
    for i, p in enumerate(problems):
        out[f"mu_{i}"] = p.mu_el[:, 0]
        out[f"lam_{i}"] = p.lam_el[:, 0]
    np.savez_compressed(os.path.join(HERE, "newton_traction_2d.npz"), **out)
    print("wrote newton_traction", recs[:, 2].max(), len(recs), flush=True)


def newton_bisect_case():
    """The reference's newton_solve with one load step whose full increment
    inverts an element: the NonPositiveJacobian path bisects the step once
    (solver.py:196-199) and reaches the load through the midpoint."""
    rng = np.random.default_rng(11)
    centres = rng.random((3, 2))
    problems = hierarchy_problems(2, (2, 4), 2, centres, 0.2)
    load = solver.LoadSpec(magnitude=0.6, direction=(0.0, -1.0))
    res = solver.newton_solve(problems, solver.NewtonSettings(n_load_steps=1), load, "gmg", "tensor4", seed=0)
    recs = np.array([(r.load_step, r.fraction, r.iteration, r.residual_norm, r.update_norm, r.cg_iterations)
                     for r in res.records])
    assert 0.5 in recs[:, 1], "the load step was not bisected"
    out = dict(centres=centres, radius=0.2, levels_m=np.array((2, 4)), magnitude=0.6, direction=np.array((0.0, -1.0)),
               n_steps=1, records=recs, u=res.u)
    for i, p in enumerate(problems):
        out[f"mu_{i}"] = p.mu_el[:, 0]
        out[f"lam_{i}"] = p.lam_el[:, 0]
    np.savez_compressed(os.path.join(HERE, "newton_bisect_2d.npz"), **out)
    print("wrote newton_bisect", len(recs), flush=True)


def newton_prescribed_case(levels_m=(4, 8), n_inc=160, radius=0.04, seed=0, target=-0.05, n_steps=5):
    """Config-4 restatement driven by reference primitives:
    bottom clamp + prescribed top-z displacement, smooth lifting of each load
    increment, GMG levels injected WITH prescribed values kept."""
    rng = np.random.default_rng(seed)
    centres = rng.random((n_inc, 3))
    problems = hierarchy_problems(3, levels_m, 2, centres, radius)
    for p in problems:
        clamp(p, 2, extra=top_z_dofs(p))
    fine = problems[-1]
    X = fespace.node_coordinates(fine.mesh, fine.dofmap)
    height = X[:, 2] / X[:, 2].max()
    transfers = multigrid.build_transfers(problems)

    def inject_keep(u_f):
        levels = [u_f]
        for lvl in range(len(problems) - 1, 0, -1):
            mf = problems[lvl].dofmap.nodes_per_side
            g = levels[0].reshape((mf,) * 3 + (3,))
            levels.insert(0, g[::2, ::2, ::2].reshape(-1).copy())
        return levels

    u = np.zeros(fine.n_dofs)
    recs = []
    t0 = time.time()
    for step in range(1, n_steps + 1):
        u = u.copy()
        u.reshape(-1, 3)[:, 2] += (target / n_steps) * height
        R = operators.compute_residual(fine, u)
        rt = max(1e-8 * np.linalg.norm(R), 1e-8)
        for it in range(1, 31):
            op = operators.MatrixFreeTangent(fine, u, "tensor4")
            ul = inject_keep(u)
            levels = [multigrid.LevelOperator(p, v, "tensor4", seed=7919 * l, level=l, is_coarsest=(l == 0))
                      for l, (p, v) in enumerate(zip(problems, ul))]
            gmg = multigrid.GMGPreconditioner(levels, transfers)
            du, rep = solver.cg(op.apply, -R, rel_tol=1e-6, preconditioner=gmg.apply)
            u = u + du
            R = operators.compute_residual(fine, u)
            rn, dn = np.linalg.norm(R), np.linalg.norm(du)
            recs.append((step, it, rn, dn, rep.iterations))
            print("  newton", recs[-1], f"{time.time() - t0:.0f}s", flush=True)
            if dn <= 1e-5 and rn <= rt:
                break
    out = dict(levels_m=np.array(levels_m), n_inc=n_inc, radius=radius, seed=seed, target=target, n_steps=n_steps,
               centres=centres, records=np.array(recs), u=u)
    for i, p in enumerate(problems):
        out[f"mu_{i}"] = p.mu_el[:, 0]
        out[f"lam_{i}"] = p.lam_el[:, 0]
        out[f"mask_{i}"] = p.constraints.mask
    np.savez_compressed(os.path.join(HERE, "newton_prescribed_3d.npz"), **out)
    print("wrote newton_prescribed", len(recs), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--newton", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    if a.only in (None, "ops"):
        op_case("2d_q2", 2, 4, 2, 5, 0.1, 0, 0.05, 0)
        op_case("2d_q1", 2, 6, 1, 3, 0.15, 1, 0.05, 0)
        op_case("2d_q3", 2, 3, 3, 3, 0.2, 2, 0.05, 0)
        op_case("2d_q4_gl", 2, 2, 4, 2, 0.3, 3, 0.05, 0, node_rule="gauss_lobatto")
        op_case("2d_q2_perturbed", 2, 4, 2, 4, 0.15, 4, 0.03, 0, perturb=0.3)
        op_case("3d_q2", 3, 3, 2, 20, 0.08, 5, 0.05, 2)
        op_case("3d_q1", 3, 4, 1, 6, 0.2, 6, 0.05, 2)
        op_case("3d_q3", 3, 2, 3, 4, 0.25, 7, 0.05, 2)
        op_case("3d_q4", 3, 2, 4, 20, 0.08, 8, 0.05, 2)
        op_case("3d_q2_perturbed", 3, 3, 2, 5, 0.2, 9, 0.03, 2, perturb=0.3)
    if a.only in (None, "mg"):
        mg_case("2d_16", 2, (4, 8, 16), 5, 0.1, 0, 0.005, 0)
        mg_case("2d_32_cfg1", 2, (4, 8, 16, 32), 5, 0.1, 0, 0.005, 0)
        mg_case("3d_8", 3, (4, 8), 20, 0.08, 0, 0.005, 2)
    if a.only in (None, "newton_t"):
        newton_traction_case()
    if a.only in (None, "newton_b"):
        newton_bisect_case()
    if a.newton or a.only == "newton_p":
        newton_prescribed_case()


if __name__ == "__main__":
    main()
