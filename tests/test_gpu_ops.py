"""GPU parity of the hot path (apply, cache build, diagonal, residual, geometry)
against the reference golden vectors and the CPU oracle.  Tolerances: 1e-12
relative L2 (BASELINE north_star) for vmult/residual; geometry 1e-13."""

import numpy as np
import pytest
import torch

from _cases import golden, op_case_names, oracle_problem, product_problem, rel
from oracle import hf_oracle as O

pytestmark = pytest.mark.gpu
CASES = op_case_names()
TOL = 1e-12


@pytest.fixture(scope="module")
def lib_loaded():
    from paper_1904_13131_b200 import _lib

    return _lib.lib()


@pytest.mark.parametrize("name", CASES)
def test_geometry(name, lib_loaded):
    g = golden(name)
    p = product_problem(g)
    geo = p.geometry
    assert rel(geo.jac_inv, g["jac_inv"]) < 1e-13
    assert rel(geo.jxw, g["jxw"]) < 1e-13


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("strategy", ["scalar", "tensor2", "tensor4"])
def test_apply_vs_reference(name, strategy, lib_loaded):
    from paper_1904_13131_b200 import MatrixFreeTangent

    g = golden(name)
    p = product_problem(g)
    op = MatrixFreeTangent(p, g["ubar"], strategy)
    y = op.apply(g["x"])
    assert isinstance(y, np.ndarray)
    assert rel(y, g[f"y_{strategy}"]) < TOL
    # identity on the constrained subspace, exactly
    assert np.array_equal(y[g["mask"]], g["x"][g["mask"]])
    assert op.storage_bytes() == int(g[f"storage_{strategy}"])
    # device in -> device out, x untouched
    xd = torch.from_numpy(g["x"]).cuda()
    x0 = xd.clone()
    yd = op.apply(xd)
    assert yd.is_cuda and torch.equal(xd, x0)
    assert rel(yd.cpu().numpy(), g[f"y_{strategy}"]) < TOL


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("strategy", ["scalar", "tensor2", "tensor4"])
def test_diagonal_vs_reference(name, strategy, lib_loaded):
    from paper_1904_13131_b200 import MatrixFreeTangent

    g = golden(name)
    p = product_problem(g)
    d = MatrixFreeTangent(p, g["ubar"], strategy).diagonal(as_numpy=True)
    assert rel(d, g[f"diag_{strategy}"]) < TOL
    assert np.all(d[g["mask"]] == 1.0)


@pytest.mark.parametrize("name", CASES)
def test_residual_vs_reference(name, lib_loaded):
    from paper_1904_13131_b200 import compute_residual, jacobian_range

    g = golden(name)
    p = product_problem(g)
    assert rel(p.surface_weights, g["surface_weights"]) < 1e-14
    assert rel(compute_residual(p, g["ubar"], g["traction"]), g["residual"]) < TOL
    assert rel(compute_residual(p, g["ubar"]), g["residual_notraction"]) < TOL
    lo, hi = jacobian_range(p, g["ubar"])
    assert np.allclose([lo, hi], g["jrange"], rtol=1e-13)


@pytest.mark.parametrize("name", CASES)
def test_inversion_raises_reference_exception(name, lib_loaded):
    from paper_1904_13131_b200 import MatrixFreeTangent, NonPositiveJacobian, compute_residual

    g = golden(name)
    p = product_problem(g)
    with pytest.raises(NonPositiveJacobian) as ei:
        MatrixFreeTangent(p, g["bad_state"], "tensor4")
    assert ei.value.element == int(g["bad_element"])
    with pytest.raises(NonPositiveJacobian):
        compute_residual(p, g["bad_state"])


@pytest.mark.parametrize("name", ["ops_3d_q2.npz", "ops_2d_q2.npz", "ops_3d_q4.npz"])
def test_apply_vs_oracle_random_states(name, lib_loaded):
    """Fresh seeded inputs (not in the golden file) against the CPU oracle."""
    from paper_1904_13131_b200 import MatrixFreeTangent

    g = golden(name)
    p = product_problem(g)
    op_ = oracle_problem(g)
    rng = np.random.default_rng(123)
    for _ in range(2):
        x = rng.standard_normal(p.n_dofs)
        u = g["ubar"] * (0.5 + rng.random())
        for s in O.STRATEGIES:
            y = MatrixFreeTangent(p, u, s).apply(x)
            yo = O.Tangent(op_, u, s).apply(x)
            assert rel(y, yo) < TOL


def test_unknown_strategy(lib_loaded):
    from paper_1904_13131_b200 import MatrixFreeTangent

    g = golden("ops_2d_q2.npz")
    p = product_problem(g)
    with pytest.raises(ValueError):
        MatrixFreeTangent(p, g["ubar"], "tensor3")


def test_constraints_override_changes_device_mask(lib_loaded):
    """Problem.constraints is mutable in the reference."""
    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200.fespace import ConstraintSet

    g = golden("ops_2d_q2.npz")
    p = product_problem(g)
    y1 = MatrixFreeTangent(p, g["ubar"], "tensor4").apply(g["x"])
    p.constraints = ConstraintSet.from_dofs(p.n_dofs, np.array([], dtype=np.int64))
    y2 = MatrixFreeTangent(p, g["ubar"], "tensor4").apply(g["x"])
    op_ = oracle_problem(g)
    op_.mask = np.zeros(p.n_dofs, dtype=bool)
    assert rel(y2, O.Tangent(op_, g["ubar"], "tensor4").apply(g["x"])) < TOL
    assert rel(y1, g["y_tensor4"]) < TOL


@pytest.mark.parametrize("name", CASES)
def test_energy_vs_reference(name, lib_loaded):
    """Total potential energy (operators.py:227-236) against the reference value."""
    from paper_1904_13131_b200 import NonPositiveJacobian, energy

    g = golden(name)
    p = product_problem(g)
    e = energy(p, g["ubar"], g["traction"])
    assert abs(e - float(g["energy"])) <= 1e-12 * abs(float(g["energy"]))
    with pytest.raises(NonPositiveJacobian):
        energy(p, g["bad_state"])


@pytest.mark.parametrize("name", ["ops_2d_q2.npz", "ops_3d_q2.npz"])
def test_residual_is_energy_gradient(name, lib_loaded):
    """verify.py:107-121: central differences of the energy along a direction
    that vanishes on the constraints reproduce residual . v."""
    from paper_1904_13131_b200 import compute_residual, energy

    g = golden(name)
    p = product_problem(g)
    v = np.random.default_rng(4).standard_normal(p.n_dofs)
    v[g["mask"]] = 0.0
    eps = 1e-6
    fd = (energy(p, g["ubar"] + eps * v, g["traction"]) - energy(p, g["ubar"] - eps * v, g["traction"])) / (2 * eps)
    r = compute_residual(p, g["ubar"], g["traction"])
    assert abs(fd - r @ v) <= 1e-6 * max(1.0, abs(r @ v))


def test_device_pool_reuses_freed_blocks(lib_loaded):
    """A rebuilt tangent takes its cache from the pool (hf_pool_*), and the
    reused (stale) block gives the same result as a fresh one (up to the
    order of the fp64 atomic adds, which varies from launch to launch)."""
    import ctypes as ct

    from paper_1904_13131_b200 import MatrixFreeTangent

    L = lib_loaded
    g = golden(CASES[0])
    p = product_problem(g)

    def info():
        pooled, live = ct.c_longlong(), ct.c_longlong()
        assert L.hf_pool_info(ct.byref(pooled), ct.byref(live)) == 0
        return pooled.value, live.value

    assert L.hf_pool_release() == 0
    y0 = MatrixFreeTangent(p, g["ubar"], "tensor4").apply(g["x"])  # built, applied, destroyed
    pooled, live = info()
    assert pooled > 0
    op = MatrixFreeTangent(p, g["ubar"], "tensor4")
    pooled2, live2 = info()
    assert pooled2 < pooled and live2 > live
    assert rel(op.apply(g["x"]), y0) < 1e-14
    del op
    assert L.hf_pool_release() == 0
    assert info()[0] == 0
