"""Benchmark records in the reference's formats (bench.py:87-141, 248-300)."""

import json

import pytest

from paper_1904_13131_b200 import harness as H


def _rec(**kw):
    base = dict(dim=3, degree=2, q=3, refinements=2, coarse_cells=4, strategy="tensor4", preconditioner="gmg",
                material="benchmark", load="benchmark", seed=0, n_dofs=823875, n_elements=32768)
    base.update(kw)
    return H.MetricsRecord(**base)


def test_columns_follow_the_reference_order():
    assert H.metrics_columns()[:10] == ("dim", "degree", "q", "refinements", "coarse_cells", "strategy",
                                        "preconditioner", "material", "load", "seed")
    assert H.metrics_columns()[10:] == ("n_dofs", "n_elements", "flops_per_apply", "flops_per_dof", "storage_bytes",
                                        "storage_bytes_per_dof", "mv_seconds", "mv_seconds_per_dof",
                                        "cg_iterations_mean", "newton_iterations_total", "solver_seconds",
                                        "solver_seconds_per_dof")
    assert "mv_seconds" not in H.metrics_columns(timings=False)
    assert H.newton_log_columns(True)[-1] == "cg_seconds"


def test_csv_and_json_rendering():
    r = _rec(mv_seconds=1.0 / 3.0, flops_per_apply=528216576)
    cols = H.metrics_columns()
    text = H.render_csv([r], cols)
    head, row = text.splitlines()
    assert head.split(",") == list(cols)
    vals = dict(zip(cols, row.split(",")))
    assert vals["mv_seconds"] == format(1.0 / 3.0, ".17g")
    assert vals["solver_seconds"] == ""  # None -> empty field
    assert vals["flops_per_apply"] == "528216576"
    js = json.loads(H.render_json([r], cols))
    assert js[0]["mv_seconds"] == 1.0 / 3.0 and js[0]["solver_seconds"] is None


@pytest.mark.gpu
def test_mv_record_on_gpu():
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(2, seed=0, m=8)
    for s in ("tensor4", "matrix_based"):
        rec = H.mv_record(wl.fine, wl.ubar, s, n_runs=3)
        assert rec.n_dofs == wl.fine.n_dofs and rec.mv_seconds > 0 and rec.storage_bytes > 0
        assert rec.flops_per_apply > 0
