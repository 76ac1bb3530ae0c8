"""Host-side logic of the product (mesh, lattice numbering, constraints, 1D
tables, transfer matrices, workload recipe, FLOP/byte meters) against the
reference golden fixtures and the oracle.  CPU only."""

import numpy as np
import pytest

from _cases import golden, op_case_names, oracle_problem, rel
from oracle import hf_oracle as O
from paper_1904_13131_b200 import fespace, mesh, workloads


@pytest.mark.parametrize("name", op_case_names())
def test_material_and_lattice(name):
    g = golden(name)
    if "perturbed" in name:
        pytest.skip("vertices perturbed after meshing")
    d, m = int(g["dim"]), int(g["m"])
    msh = mesh.build_benchmark_mesh(d, m, [(c, float(g["radius"])) for c in g["centres"]], side=1.0)
    assert np.array_equal(msh.material_id, g["material_id"])
    assert np.allclose(msh.vertices, g["vertices"], rtol=0, atol=1e-15)
    dm = fespace.build_dof_map(msh, int(g["degree"]), d)
    assert np.array_equal(dm.cell_nodes, oracle_problem(g).cell_nodes())


@pytest.mark.parametrize("name", op_case_names())
def test_basis_tables(name):
    g = golden(name)
    op_ = oracle_problem(g)
    q = fespace.gauss_legendre(int(g["degree"]) + 1)
    b = fespace.lagrange_basis(int(g["degree"]), q, str(g["node_rule"]))
    assert np.allclose(b.values, op_.V, atol=1e-15) and np.allclose(b.derivatives, op_.D, atol=1e-13)


def test_constraints_faces():
    msh = mesh.build_benchmark_mesh(2, 4, [], side=1.0)
    dm = fespace.build_dof_map(msh, 2, 2)
    bottom = fespace.bottom_constraints(msh, dm)
    assert len(bottom.dofs) == 9 * 2
    X = fespace.node_coordinates(msh, dm)
    assert np.all(X[bottom.dofs // 2, 1] == 0.0)
    left = fespace.face_dofs(dm, 0, 0)
    assert np.all(X[left // 2, 0] == 0.0) and len(left) == 18
    top_y = fespace.face_dofs(dm, 1, 1, components=[1])
    assert np.all(X[top_y // 2, 1] == 1.0) and np.all(top_y % 2 == 1)


@pytest.mark.parametrize("p,m", [(1, 3), (2, 2), (2, 4), (4, 2)])
def test_interpolation_matrix(p, m):
    nodes = np.arange(p + 1) / p
    assert np.allclose(fespace.interpolation_matrix_1d(p, m, nodes), O.interpolation_1d(p, m, nodes), atol=1e-15)


@pytest.mark.parametrize("name", op_case_names())
def test_meter_flops_matches_reference_count(name):
    g = golden(name)
    d, p, m = int(g["dim"]), int(g["degree"]), int(g["m"])
    for s in ("scalar", "tensor2", "tensor4"):
        assert workloads.meter_flops(d, p, m**d, s) == int(g[f"flops_{s}"])


def test_algorithmic_bytes_survey_formula():
    # cfg2 tensor4 333.9 B/DoF, tensor2 170.6, scalar 118.5 (JxW stored)
    nd, nqp = 823875, 32**3 * 27
    for s, bpd in (("tensor4", 333.9), ("tensor2", 170.6), ("scalar", 118.5)):
        assert abs(workloads.algorithmic_bytes(s, 3, nd, nqp, reference_fields=True) / nd - bpd) < 0.05
    # this design folds JxW into the tensor4 / tensor2 fields: one double less per q-point
    for s in ("tensor4", "tensor2"):
        assert workloads.algorithmic_bytes(s, 3, nd, nqp, True) - workloads.algorithmic_bytes(s, 3, nd, nqp) == 8 * nqp
    assert workloads.algorithmic_bytes("scalar", 3, nd, nqp, True) == workloads.algorithmic_bytes("scalar", 3, nd, nqp)


def test_workload_recipe():
    """Clamp-weighted sine vanishes on the clamp and equals the
    direct formula at the lattice nodes."""
    ph = 2 * np.pi * np.random.default_rng(0).random((3, 3))
    u = workloads.clamp_weighted_sine(3, 4, 2, ph, 0.05, 2).reshape(-1, 3)
    msh = mesh.build_benchmark_mesh(3, 4, [], side=1.0)
    X = fespace.node_coordinates(msh, fespace.build_dof_map(msh, 2, 3))
    ref = np.stack([0.05 * X[:, 2] * np.prod(np.sin(np.pi * X + ph[c]), axis=1) for c in range(3)], axis=1)
    assert np.allclose(u, ref, atol=1e-15)
    assert np.all(u[X[:, 2] == 0.0] == 0.0)


def test_sub_box_partition_roundtrip():
    msh = mesh.build_benchmark_mesh(3, 8, [((0.3, 0.5, 0.5), 0.2)], side=1.0)
    parts = [mesh.sub_box(msh, 2, a, b) for a, b in ((0, 3), (3, 8))]
    assert sum(pp.n_elements for pp in parts) == msh.n_elements
    assert np.array_equal(np.concatenate([pp.material_id for pp in parts]), msh.material_id)
    assert parts[1].cell_offset == (0, 0, 3)
    assert np.allclose(parts[1].vertices[0], [0, 0, 3 / 8])


@pytest.mark.parametrize("dim,m,p", [(2, 5, 2), (3, 4, 2), (3, 3, 4), (2, 4, 3), (3, 2, 1)])
def test_node_coordinates_separable_matches_cell_map(dim, m, p):
    """node_coordinates refines the vertex lattice axis by axis; it equals the
    per-cell multilinear map (fespace.py:142-151) evaluated at every cell's
    local nodes, also on a perturbed mesh."""
    import dataclasses

    msh = mesh.build_benchmark_mesh(dim, m, [], side=1.0)
    rng = np.random.default_rng(3)
    msh = dataclasses.replace(msh, vertices=msh.vertices + 0.02 * rng.standard_normal(msh.vertices.shape))
    dm = fespace.build_dof_map(msh, p, dim)
    loc = fespace.lex_grid_points([np.arange(p + 1) / p] * dim)
    off = fespace.lex_grid_indices((2,) * dim)
    q1 = np.ones((2**dim, len(loc)))
    for k in range(dim):
        q1 *= np.where(off[:, k:k + 1] == 1, loc[None, :, k], 1.0 - loc[None, :, k])
    per_el = np.einsum("eci,cn->eni", msh.element_corners(), q1)
    ref = np.zeros((dm.n_nodes, dim))
    ref[dm.cell_nodes.reshape(-1)] = per_el.reshape(-1, dim)
    assert np.allclose(fespace.node_coordinates(msh, dm), ref, rtol=0, atol=1e-15)
