"""Golden outputs of the reference's matrix-based tangent (AssembledTangent,
operators.py:494-516) for the op cases that the GPU assembly supports.

Run in the build container (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_matrix.py

For every ``ops_<case>.npz`` it rebuilds the reference Problem from the stored
mesh, constraints and state, runs the unmodified ``AssembledTangent`` and
writes ``mb_<case>.npz``: y = A x, diag(A), storage_bytes and nnz.
"""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from hyperfree import fespace, material, mesh as rmesh, operators  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
MAT = operators.Material(
    matrix=material.NeoHookeanParams.from_shear_and_poisson(1.0, 0.3),
    inclusion=material.NeoHookeanParams.from_shear_and_poisson(10.0, 0.3),
)
CASES = ["2d_q1", "2d_q2", "2d_q2_perturbed", "2d_q3", "3d_q1", "3d_q2", "3d_q2_perturbed"]


def main():
    for name in CASES:
        g = dict(np.load(os.path.join(HERE, f"ops_{name}.npz")))
        dim, m, p = int(g["dim"]), int(g["m"]), int(g["degree"])
        msh = rmesh.build_benchmark_mesh(dim, m, [(c, float(g["radius"])) for c in g["centres"]], side=1.0)
        msh = dataclasses.replace(msh, vertices=g["vertices"], material_id=g["material_id"])
        prob = operators.Problem(msh, p, MAT, basis_nodes=str(g["node_rule"]))
        prob.constraints = fespace.ConstraintSet.from_dofs(prob.n_dofs, np.flatnonzero(g["mask"]))
        op = operators.AssembledTangent(prob, g["ubar"])
        out = dict(y=op.apply(g["x"]), diag=op.diagonal(), storage=op.storage_bytes(), nnz=op.matrix.nnz)
        np.savez_compressed(os.path.join(HERE, f"mb_{name}.npz"), **out)
        print("wrote", name, prob.n_dofs, op.matrix.nnz, flush=True)


if __name__ == "__main__":
    main()
