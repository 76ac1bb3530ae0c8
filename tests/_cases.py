"""Shared helpers: load golden fixtures and turn them into oracle problems."""

import glob
import os

import numpy as np

from oracle import hf_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def op_case_names():
    return sorted(os.path.basename(f) for f in glob.glob(os.path.join(GOLDEN, "ops_*.npz")))


def oracle_problem(g):
    dim, m, p = int(g["dim"]), int(g["m"]), int(g["degree"])
    return O.OProblem(dim, p, (m,) * dim, g["vertices"], g["mu_el"], g["lam_el"], g["mask"],
                      node_rule=str(g["node_rule"]))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def product_problem(g, degree=None):
    """The B200 Problem for a golden op case (same mesh, material, constraints)."""
    from paper_1904_13131_b200.fespace import ConstraintSet
    from paper_1904_13131_b200.mesh import Mesh
    from paper_1904_13131_b200.operators import Problem
    from paper_1904_13131_b200.workloads import MATERIAL

    dim, m = int(g["dim"]), int(g["m"])
    mesh = Mesh(dim=dim, side=1.0, cells=(m,) * dim, vertices=g["vertices"], material_id=g["material_id"])
    p = Problem(mesh, int(g["degree"]) if degree is None else degree, MATERIAL, basis_nodes=str(g["node_rule"]))
    p.constraints = ConstraintSet.from_dofs(p.n_dofs, np.flatnonzero(g["mask"]))
    return p


def product_levels(g, key_mask="mask_"):
    """B200 problems of a golden multigrid case, one per level, golden masks applied."""
    from paper_1904_13131_b200.fespace import ConstraintSet
    from paper_1904_13131_b200.mesh import build_benchmark_mesh
    from paper_1904_13131_b200.operators import Problem
    from paper_1904_13131_b200.workloads import MATERIAL

    dim = int(g.get("dim", 3))
    spec = [(c, float(g["radius"])) for c in g["centres"]]
    probs = []
    for i, m in enumerate(g["levels_m"]):
        p = Problem(build_benchmark_mesh(dim, int(m), spec, side=1.0), 2, MATERIAL)
        if f"{key_mask}{i}" in g:
            p.constraints = ConstraintSet.from_dofs(p.n_dofs, np.flatnonzero(g[f"{key_mask}{i}"]))
        probs.append(p)
    return probs
