"""The UNMODIFIED reference (``hyperfree``, installed into ``oracle/_ref`` by
``oracle/build_ref.py``) set up on the BASELINE configs -- test infrastructure.

Used as the checker by the ``-m gpu`` parity tests and as the reference arm /
CPU baseline of ``bench.py``; never on the product path.  Everything here calls
the reference's own public API:

* ``build_benchmark_mesh(dim, m, spec, side=1.0)`` (mesh.py:170-204), one mesh
  per level with per-level centroid material;
* ``Problem(mesh, degree, MAT)`` (operators.py:83-105), its ``constraints``
  replaced by ``ConstraintSet.from_dofs`` (fespace.py:162-167);
* ``MatrixFreeTangent(problem, u_bar, strategy).apply / .diagonal``
  (operators.py:319-410), ``compute_residual`` (205-224), ``build_gmg``
  (multigrid.py:372-382), ``cg`` (solver.py:34-76).

The synthetic inputs are drawn exactly as ``paper_1904_13131_b200.workloads``
draws them (one ``default_rng(seed)``: inclusion centres, phases, then x), so
the reference and the GPU product see the same configuration.
"""

from __future__ import annotations

import importlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "hyperfree"))


def hyperfree():
    """Import the installed reference package (from oracle/_ref only)."""
    if not available():
        raise ImportError("oracle/_ref is not installed (python oracle/build_ref.py in the build container)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    mod = importlib.import_module("hyperfree")
    if not os.path.abspath(mod.__file__).startswith(REF_DIR):
        raise ImportError(f"hyperfree resolved to {mod.__file__}, not oracle/_ref")
    for sub in ("fespace", "material", "mesh", "multigrid", "operators", "solver"):
        importlib.import_module(f"hyperfree.{sub}")
    return mod


def material(hf):
    """BASELINE material: matrix mu 1, inclusion mu 10, nu 0.3."""
    P = hf.material.NeoHookeanParams
    return hf.operators.Material(matrix=P.from_shear_and_poisson(1.0, 0.3),
                                 inclusion=P.from_shear_and_poisson(10.0, 0.3))


def problem(hf, dim: int, m: int, degree: int, centres: np.ndarray, radius: float, mask: np.ndarray):
    """A reference Problem on the unit box with the given constraint mask."""
    msh = hf.mesh.build_benchmark_mesh(dim, m, [(c, radius) for c in centres], side=1.0)
    prob = hf.operators.Problem(msh, degree, material(hf))
    prob.constraints = hf.fespace.ConstraintSet.from_dofs(prob.n_dofs, np.flatnonzero(mask))
    return prob


def face_mask(dim: int, m: int, degree: int, clamp_axis: int, top_last: bool = False) -> np.ndarray:
    """All components on the face ``clamp_axis`` = 0, plus the last
    component on the top face (config 4, H5); lexicographic nodes, x fastest."""
    n1 = m * degree + 1
    idx = np.indices((n1,) * dim).reshape(dim, -1)[::-1]  # idx[a] = lattice index along axis a
    mask = np.zeros((n1**dim, dim), dtype=bool)
    mask[idx[clamp_axis] == 0, :] = True
    if top_last:
        mask[idx[dim - 1] == n1 - 1, dim - 1] = True
    return mask.reshape(-1)


# BASELINE.json configs (same table as paper_1904_13131_b200.workloads.CONFIGS)
CONFIGS = {
    1: dict(dim=2, m=32, degree=2, n_inc=5, radius=0.1, clamp_axis=0),
    2: dict(dim=3, m=32, degree=2, n_inc=20, radius=0.08, clamp_axis=2),
    3: dict(dim=3, m=16, degree=4, n_inc=20, radius=0.08, clamp_axis=2),
    4: dict(dim=3, m=64, degree=2, n_inc=160, radius=0.04, clamp_axis=2, top_last=True),
    5: dict(dim=3, m=128, degree=2, n_inc=1280, radius=0.02, clamp_axis=2),
}


def clamp_weighted_sine(hf, prob, phases: np.ndarray, amp: float, clamp_axis: int) -> np.ndarray:
    """u_c = amp X_clamp prod_a sin(pi X_a + phi[c, a]) at the reference's node
    coordinates (fespace.py:142-151)."""
    X = hf.fespace.node_coordinates(prob.mesh, prob.dofmap)
    d = prob.dim
    u = np.empty((X.shape[0], d))
    for c in range(d):
        u[:, c] = amp * X[:, clamp_axis] * np.prod(np.sin(np.pi * X + phases[c][None, :]), axis=1)
    return u.reshape(-1)


def config_problem(cfg_id: int, seed: int = 0, amp: float = 0.05, m: int | None = None):
    """(reference module, fine Problem, u_bar, x) of a BASELINE config, drawn as
    ``workloads.make_workload(cfg_id, seed, amp)`` draws it."""
    hf = hyperfree()
    c = dict(CONFIGS[cfg_id])
    if m is not None:
        c["m"] = m
    rng = np.random.default_rng(seed)
    centres = rng.random((c["n_inc"], c["dim"]))
    phases = 2.0 * np.pi * rng.random((c["dim"], c["dim"]))
    mask = face_mask(c["dim"], c["m"], c["degree"], c["clamp_axis"], c.get("top_last", False))
    prob = problem(hf, c["dim"], c["m"], c["degree"], centres, c["radius"], mask)
    ubar = clamp_weighted_sine(hf, prob, phases, amp, c["clamp_axis"])
    x = rng.standard_normal(prob.n_dofs)
    return hf, prob, ubar, x


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"
