"""The drop-in boundary exercised from the reference side.

The ctypes stub of INTEGRATION.md (extracted verbatim from that file) is loaded
as ``hyperfree._b200`` inside the UNMODIFIED reference installed in
``oracle/_ref``; ``install()`` rebinds ``operators.MatrixFreeTangent`` and
``multigrid.MatrixFreeTangent`` (multigrid.py:22, 223; operators.py:519-522).
The reference's own ``build_gmg`` (multigrid.py:372-382) and ``cg``
(solver.py:34-76) then run config 1 on top of libhf.so, and the result is
checked against the golden reference run (mg_2d_32_cfg1.npz: 20 iterations).
"""

import os
import re
import sys
import types

import numpy as np
import pytest

from _cases import golden, rel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def stub_source() -> str:
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"```python\n(# hyperfree/_b200\.py.*?)```", text, re.S)
    assert m, "INTEGRATION.md has no hyperfree/_b200.py block"
    return m.group(1)


@pytest.fixture(scope="module")
def refside():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not installed (python oracle/build_ref.py)")
    from paper_1904_13131_b200 import _lib

    hf = ref.hyperfree()
    os.environ["HF_LIBRARY"] = _lib.LIB_PATH
    mod = types.ModuleType("hyperfree._b200")
    mod.__package__ = "hyperfree"
    mod.__file__ = os.path.join(ref.REF_DIR, "hyperfree", "_b200.py")
    sys.modules["hyperfree._b200"] = mod
    exec(compile(stub_source(), mod.__file__, "exec"), mod.__dict__)
    saved = (hf.operators.MatrixFreeTangent, hf.multigrid.MatrixFreeTangent)
    mod.reference_operator = saved[0]  # the reference's own class, for side-by-side checks
    mod.install()
    yield hf, mod
    hf.operators.MatrixFreeTangent, hf.multigrid.MatrixFreeTangent = saved


def cfg1_problems(hf, g):
    from oracle import ref

    return [ref.problem(hf, 2, int(m), 2, g["centres"], float(g["radius"]), g[f"mask_{i}"])
            for i, m in enumerate(g["levels_m"])]


def test_stub_apply_and_diagonal(refside):
    hf, mod = refside
    g = golden("mg_2d_32_cfg1.npz")
    probs = cfg1_problems(hf, g)
    op = hf.operators.make_tangent(probs[-1], g["ubar"], "tensor4")
    assert isinstance(op, mod.MatrixFreeTangent)
    x = g["x"].copy()
    y = op.apply(x)
    assert np.array_equal(x, g["x"]), "apply must leave x untouched"
    yb = y.copy()
    yb[probs[-1].constraints.mask] = 0.0
    assert rel(yb, g["b"]) < 1e-12
    d = op.diagonal()
    assert isinstance(d, np.ndarray)
    assert rel(d, g["diag_3"]) < 1e-12
    with pytest.raises(ValueError):
        mod.MatrixFreeTangent(probs[-1], g["ubar"], "tensor3")


def test_reference_gmg_cg_on_libhf(refside):
    hf, mod = refside
    g = golden("mg_2d_32_cfg1.npz")
    probs = cfg1_problems(hf, g)
    transfers = hf.multigrid.build_transfers(probs)
    gmg = hf.multigrid.build_gmg(probs, g["ubar"], "tensor4", seed=0, transfers=transfers)
    assert all(isinstance(lv.op, mod.MatrixFreeTangent) for lv in gmg.levels)
    for i, lv in enumerate(gmg.levels):
        assert lv.lam_max == pytest.approx(float(g[f"lam_max_{i}"]), rel=1e-9)
    op = hf.operators.make_tangent(probs[-1], g["ubar"], "tensor4")
    sol, rep = hf.solver.cg(op.apply, g["b"], rel_tol=1e-8, preconditioner=gmg.apply)
    assert abs(rep.iterations - int(g["cg_iterations"])) <= 1
    n = min(len(rep.residual_history), len(g["cg_history"]), 8)
    np.testing.assert_allclose(rep.residual_history[:n], g["cg_history"][:n], rtol=1e-6)
    assert rel(sol, g["cg_solution"]) < 1e-6


def test_reference_nonpositive_jacobian_through_stub(refside):
    hf, mod = refside
    g = golden("ops_2d_q2.npz")
    from oracle import ref

    prob = ref.problem(hf, 2, int(g["m"]), 2, g["centres"], float(g["radius"]), g["mask"])
    with pytest.raises(hf.material.NonPositiveJacobian) as ei:
        hf.operators.make_tangent(prob, g["bad_state"], "tensor4")
    assert ei.value.element == int(g["bad_element"])


# the reference's own self-checks (verify.py) that construct MatrixFreeTangent:
# strategies vs the reference's assembled matrix (verify.py:70-84), the tangent
# vs central differences of the reference's residual (87-104), the diagonal vs
# the assembled one (158-165), the cache payload counts (168-178)
VERIFY_CHECKS = ["check_strategy_equivalence", "check_tangent_fd", "check_diagonal", "check_payload_counts"]


@pytest.mark.parametrize("check", VERIFY_CHECKS)
def test_reference_verify_checks_on_libhf(refside, check, monkeypatch):
    """``hyperfree verify`` (verify.py:199-217) with the B200 operator bound:
    the reference's own thresholds, its own AssembledTangent / compute_residual
    on the CPU as the independent side."""
    hf, mod = refside
    import importlib

    verify = importlib.import_module("hyperfree.verify")
    built = []

    class Counting(mod.MatrixFreeTangent):
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            built.append(self.strategy)

    monkeypatch.setattr(verify, "MatrixFreeTangent", mod.reference_operator)
    want = getattr(verify, check)(0)  # the unmodified reference, on the CPU
    monkeypatch.setattr(verify, "MatrixFreeTangent", Counting)
    rec = getattr(verify, check)(0)
    assert built, "the check did not construct the B200 operator"
    # same verdict as the reference's own operator, and the same measured value
    # where the value is a convergence order (the reference's finite-difference
    # slope check fails its own 1.8 threshold at this seed: 1.69, SURVEY 8(c)
    # calls it fragile; the B200 operator must reproduce that number)
    assert bool(rec.passed) == bool(want.passed), (rec, want)
    if check == "check_tangent_fd":
        assert rec.value == pytest.approx(want.value, rel=1e-5), (rec, want)
    else:
        assert rec.passed, f"{rec.name}: {rec.value} against the reference's threshold {rec.threshold}"

