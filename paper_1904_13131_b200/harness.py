"""Benchmark records in the reference's formats.

The reference's harness (bench.py:87-141, 187-300) reports one
``MetricsRecord`` per run with a stable column order (configuration fields
first, then metrics), floats at 17 significant digits, and a per-iteration
Newton log.  This module keeps those records, columns and renderers, and fills
them from the B200 operators:

* ``mv_record``: one tangent application timed as the reference times it
  (one warm-up, mean of ``n_runs``; bench.py:187-219), with device
  synchronisation around the timed loop.  The FLOP count is the reference
  meter's (``workloads.meter_flops``; flops.py).
* ``solver_record``: a full incremental Newton solve (bench.py:222-245).

Presets (paper-scale material, traction loads) are not part of the hot path
and are not restated; callers pass the problems and the load.
"""

from __future__ import annotations

import csv
import dataclasses
import io
import json
import time
from dataclasses import dataclass

import numpy as np
import torch

CONFIG_COLUMNS = ("dim", "degree", "q", "refinements", "coarse_cells", "strategy", "preconditioner", "material",
                  "load", "seed")
METRIC_COLUMNS = ("n_dofs", "n_elements", "flops_per_apply", "flops_per_dof", "storage_bytes",
                  "storage_bytes_per_dof", "mv_seconds", "mv_seconds_per_dof", "cg_iterations_mean",
                  "newton_iterations_total", "solver_seconds", "solver_seconds_per_dof")
TIMING_COLUMNS = ("mv_seconds", "mv_seconds_per_dof", "solver_seconds", "solver_seconds_per_dof")


@dataclass
class MetricsRecord:
    """One benchmark row (bench.py:118-141)."""

    dim: int
    degree: int
    q: int
    refinements: int
    coarse_cells: int
    strategy: str
    preconditioner: str
    material: str
    load: str
    seed: int
    n_dofs: int
    n_elements: int
    flops_per_apply: int | None = None
    flops_per_dof: float | None = None
    storage_bytes: int | None = None
    storage_bytes_per_dof: float | None = None
    mv_seconds: float | None = None
    mv_seconds_per_dof: float | None = None
    cg_iterations_mean: float | None = None
    newton_iterations_total: int | None = None
    solver_seconds: float | None = None
    solver_seconds_per_dof: float | None = None


def metrics_columns(timings: bool = True) -> tuple:
    cols = CONFIG_COLUMNS + METRIC_COLUMNS
    return cols if timings else tuple(c for c in cols if c not in TIMING_COLUMNS)


def newton_log_columns(timings: bool = False) -> tuple:
    cols = ("load_step", "fraction", "iteration", "residual_norm", "update_norm", "cg_iterations")
    return cols + ("cg_seconds",) if timings else cols


def _value(v) -> str:
    if v is None:
        return ""
    if isinstance(v, float):
        return format(v, ".17g")
    return str(v)


def _as_dict(rec) -> dict:
    return dataclasses.asdict(rec) if dataclasses.is_dataclass(rec) else dict(rec)


def records_to_rows(records, columns) -> list:
    return [[_value(_as_dict(r).get(c)) for c in columns] for r in records]


def render_csv(records, columns) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(columns)
    w.writerows(records_to_rows(records, columns))
    return buf.getvalue()


def render_json(records, columns) -> str:
    return json.dumps([{c: _as_dict(r).get(c) for c in columns} for r in records], indent=2) + "\n"


def emit_results(records, path: str, fmt: str = "csv", columns=None) -> None:
    columns = metrics_columns() if columns is None else columns
    with open(path, "w") as f:
        f.write(render_csv(records, columns) if fmt == "csv" else render_json(records, columns))


def _base(problem, strategy, preconditioner, refinements, coarse_cells, material, load, seed) -> MetricsRecord:
    return MetricsRecord(dim=problem.dim, degree=problem.degree, q=problem.quadrature.n_points,
                         refinements=refinements, coarse_cells=coarse_cells, strategy=strategy,
                         preconditioner=preconditioner, material=material, load=load, seed=seed,
                         n_dofs=problem.n_dofs, n_elements=problem.mesh.n_elements)


def mv_record(problem, u_bar, strategy: str = "tensor4", n_runs: int = 10, seed: int = 0, refinements: int = 0,
              coarse_cells: int = 0, material: str = "benchmark", load: str = "benchmark",
              preconditioner: str = "gmg") -> MetricsRecord:
    """One operator application at ``u_bar``, timed as bench.py:187-219."""
    from .operators import make_tangent
    from .workloads import meter_flops

    op = make_tangent(problem, u_bar, strategy)
    x = torch.from_numpy(np.random.default_rng(seed).standard_normal(problem.n_dofs)).cuda()
    y = torch.empty_like(x)
    op.apply_into(x, y)  # warm up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n_runs):
        op.apply_into(x, y)
    torch.cuda.synchronize()
    elapsed = (time.perf_counter() - t0) / n_runs
    rec = _base(problem, strategy, preconditioner, refinements, coarse_cells, material, load, seed)
    if strategy != "matrix_based":
        flops = meter_flops(problem.dim, problem.degree, problem.mesh.n_elements, strategy)
    else:
        flops = 2 * int(op.matrix.values().numel())  # AssembledTangent.apply (operators.py:507-509)
    rec.flops_per_apply = flops
    rec.flops_per_dof = flops / problem.n_dofs
    rec.storage_bytes = op.storage_bytes()
    rec.storage_bytes_per_dof = op.storage_bytes() / problem.n_dofs
    rec.mv_seconds = elapsed
    rec.mv_seconds_per_dof = elapsed / problem.n_dofs
    return rec


def solver_record(problems, settings, load_spec, strategy: str = "tensor4", preconditioner: str = "gmg",
                  seed: int = 0, refinements: int = 0, coarse_cells: int = 0, material: str = "benchmark",
                  load: str = "benchmark"):
    """Full incremental Newton solve (bench.py:222-245): (record, Newton log)."""
    from .solver import newton_solve

    fine = problems[-1]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    result = newton_solve(problems, settings, load_spec, preconditioner=preconditioner, strategy=strategy, seed=seed)
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    rec = _base(fine, strategy, preconditioner, refinements, coarse_cells, material, load, seed)
    its = [r.cg_iterations for r in result.records]
    rec.cg_iterations_mean = float(np.mean(its)) if its else 0.0
    rec.newton_iterations_total = len(result.records)
    rec.solver_seconds = elapsed
    rec.solver_seconds_per_dof = elapsed / fine.n_dofs
    return rec, result.records
