"""Matrix-based baseline (AssembledTangent, operators.py:436-516) on the GPU
against the reference's own assembled matrix (tests/golden/mb_*.npz, written
by make_golden_matrix.py from the unmodified reference)."""

import glob
import os

import numpy as np
import pytest

from _cases import GOLDEN, golden, product_problem, rel

pytestmark = pytest.mark.gpu
CASES = sorted(os.path.basename(f)[3:] for f in glob.glob(os.path.join(GOLDEN, "mb_*.npz")))


@pytest.mark.parametrize("case", CASES)
def test_assembled_tangent_vs_reference(case):
    from paper_1904_13131_b200 import MatrixFreeTangent, make_tangent

    g = golden(f"ops_{case}")
    mb = golden(f"mb_{case}")
    p = product_problem(g)
    op = make_tangent(p, g["ubar"], "matrix_based")
    assert op.strategy == "matrix_based"
    y = op.apply(g["x"])
    assert rel(y, mb["y"]) < 1e-12
    assert rel(op.diagonal(as_numpy=True), mb["diag"]) < 1e-12
    assert op.storage_bytes() == int(mb["storage"])
    assert op.matrix.values().numel() == int(mb["nnz"])
    # the matrix-based and matrix-free tangents are the same operator
    assert rel(y, MatrixFreeTangent(p, g["ubar"], "tensor4").apply(g["x"])) < 1e-12
    assert np.array_equal(y[g["mask"]], g["x"][g["mask"]])


def test_assembly_is_limited_to_instantiated_degrees():
    from paper_1904_13131_b200 import make_tangent
    from paper_1904_13131_b200._lib import HfError

    g = golden("ops_3d_q3.npz")
    with pytest.raises(HfError):
        make_tangent(product_problem(g), g["ubar"], "matrix_based")
