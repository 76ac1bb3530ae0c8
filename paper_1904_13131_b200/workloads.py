"""Seeded synthetic inputs of the BASELINE configs.

One ``np.random.default_rng(seed)`` draws, in this order: inclusion centres
(n_inc, d), phases 2*pi*U(d, d), then x ~ N(0, 1)^N_dof.  The linearisation
point is u_c(X) = A * X_clamp * prod_a sin(pi X_a + phi[c, a]) (the
clamp-weighted sine of SURVEY H3); X_clamp = x (2D, left clamp) or z (3D,
bottom clamp).  Materials: matrix mu = 1, nu = 0.3; inclusion mu = 10,
nu = 0.3 (H7), unit square/cube, per-level centroid material (H6).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .fespace import ConstraintSet, face_dofs
from .material import NeoHookeanParams
from .mesh import build_benchmark_mesh
from .operators import Material, Problem

MATERIAL = Material(matrix=NeoHookeanParams.from_shear_and_poisson(1.0, 0.3),
                    inclusion=NeoHookeanParams.from_shear_and_poisson(10.0, 0.3))

# BASELINE.json configs[0..4]
CONFIGS = {
    1: dict(name="cfg1_2d_32_q2", dim=2, m=32, degree=2, n_inc=5, radius=0.1, clamp_axis=0, coarsest=4),
    2: dict(name="cfg2_3d_32_q2", dim=3, m=32, degree=2, n_inc=20, radius=0.08, clamp_axis=2, coarsest=4),
    3: dict(name="cfg3_3d_16_q4", dim=3, m=16, degree=4, n_inc=20, radius=0.08, clamp_axis=2, coarsest=4),
    4: dict(name="cfg4_3d_64_q2_newton", dim=3, m=64, degree=2, n_inc=160, radius=0.04, clamp_axis=2, coarsest=4,
            top_z=True),
    5: dict(name="cfg5_3d_128_q2", dim=3, m=128, degree=2, n_inc=1280, radius=0.02, clamp_axis=2, coarsest=4),
}
AMP_VMULT = 0.05  # BASELINE amplitude (vmult timing)
AMP_SOLVE = 0.005  # SPD at every level


def lattice_1d(m: int, degree: int) -> np.ndarray:
    """Node coordinates along one axis of the unit interval: cell map of the
    equispaced local nodes, (1 - l/p) x_e + (l/p) x_{e+1}."""
    xv = np.linspace(0.0, 1.0, m + 1)
    e = np.repeat(np.arange(m), degree)
    l = np.tile(np.arange(degree), m) / degree
    out = np.empty(m * degree + 1)
    out[:-1] = (1.0 - l) * xv[e] + l * xv[e + 1]
    out[-1] = 1.0
    return out


def clamp_weighted_sine(dim: int, m, degree: int, phases: np.ndarray, amp: float, clamp_axis: int) -> np.ndarray:
    """u_c = amp X_clamp prod_a sin(pi X_a + phi[c,a]) on the node lattice, node-blocked.

    ``m`` is the cells per axis (an int for the unit cube, or a per-axis tuple:
    each axis' lattice spans [0, 1])."""
    ms = (m,) * dim if np.isscalar(m) else tuple(m)
    x1 = [lattice_1d(mm, degree) for mm in ms]
    shape_all = tuple(len(x1[a]) for a in reversed(range(dim)))
    u = np.empty(shape_all + (dim,))  # array axes (z, y, x) / (y, x)
    for c in range(dim):
        f = np.ones(shape_all)
        for a in range(dim):
            shape = [1] * dim
            shape[dim - 1 - a] = len(x1[a])
            fac = np.sin(np.pi * x1[a] + phases[c, a])
            if a == clamp_axis:
                fac = fac * x1[a]
            f = f * fac.reshape(shape)
        u[..., c] = amp * f
    return u.reshape(-1)


def constrain(problem: Problem, clamp_axis: int, top_last_component: bool = False) -> ConstraintSet:
    """Clamp every component on the face ``clamp_axis`` = 0 (H2); optionally also
    the last component on the top face (config 4, H5)."""
    dm = problem.dofmap
    dofs = [face_dofs(dm, clamp_axis, 0)]
    if top_last_component:
        dofs.append(face_dofs(dm, dm.dim - 1, 1, components=[dm.dim - 1]))
    cs = ConstraintSet.from_dofs(dm.n_dofs, np.concatenate(dofs))
    problem.constraints = cs
    return cs


@dataclass
class Workload:
    cfg: dict
    centres: np.ndarray
    phases: np.ndarray
    problems: list = field(default_factory=list)
    ubar: np.ndarray | None = None
    x: np.ndarray | None = None

    @property
    def fine(self) -> Problem:
        return self.problems[-1]


def make_workload(cfg_id: int, seed: int = 0, amp: float = AMP_VMULT, levels: bool = False, m: int | None = None,
                  coarsest: int | None = None, with_x: bool = True) -> Workload:
    """Problems (one per GMG level when ``levels``), linearisation point and input vector."""
    cfg = dict(CONFIGS[cfg_id])
    if m is not None:
        cfg["m"] = m
    if coarsest is not None:
        cfg["coarsest"] = coarsest
    dim, p = cfg["dim"], cfg["degree"]
    rng = np.random.default_rng(seed)
    centres = rng.random((cfg["n_inc"], dim))
    phases = 2.0 * np.pi * rng.random((dim, dim))
    ms = [cfg["m"]]
    if levels:
        while ms[0] // 2 >= cfg["coarsest"] and ms[0] % 2 == 0:
            ms.insert(0, ms[0] // 2)
    wl = Workload(cfg, centres, phases)
    spec = [(c, cfg["radius"]) for c in centres]
    for mm in ms:
        prob = Problem(build_benchmark_mesh(dim, mm, spec, side=1.0), p, MATERIAL)
        constrain(prob, cfg["clamp_axis"], cfg.get("top_z", False))
        wl.problems.append(prob)
    wl.ubar = clamp_weighted_sine(dim, cfg["m"], p, phases, amp, cfg["clamp_axis"])
    if with_x:
        wl.x = rng.standard_normal(wl.fine.n_dofs)
    return wl


@dataclass
class HostWorkload:
    """Host-only description of a BASELINE config (for the multi-GPU path: every
    rank derives its slab from the same global meshes, masks and vectors)."""

    cfg: dict
    meshes: list        # global mesh per level, coarsest first
    masks: list         # global constraint mask per level
    ubar: np.ndarray    # global linearisation point (finest level)
    x: np.ndarray | None


def host_workload(cfg_id: int, seed: int = 0, amp: float = AMP_VMULT, levels: bool = False, m: int | None = None,
                  coarsest: int | None = None, with_x: bool = True, stack: int = 1) -> HostWorkload:
    """Same draws as ``make_workload``; ``stack`` > 1 stacks copies of the cell
    layers along the last axis (weak-scaling meshes of ``stack`` GPUs)."""
    from .fespace import build_dof_map

    cfg = dict(CONFIGS[cfg_id])
    if m is not None:
        cfg["m"] = m
    if coarsest is not None:
        cfg["coarsest"] = coarsest
    dim, p = cfg["dim"], cfg["degree"]
    rng = np.random.default_rng(seed)
    centres = rng.random((cfg["n_inc"], dim))
    phases = 2.0 * np.pi * rng.random((dim, dim))
    ms = [cfg["m"]]
    if levels:
        while ms[0] // 2 >= cfg["coarsest"] and ms[0] % 2 == 0:
            ms.insert(0, ms[0] // 2)
    spec = [(c, cfg["radius"]) for c in centres]
    meshes, masks = [], []
    for mm in ms:
        mesh = build_benchmark_mesh(dim, mm, spec, side=1.0)
        if stack > 1:
            mesh = stack_mesh(mesh, stack)
        dm = build_dof_map(mesh, p, dim)
        dofs = [face_dofs(dm, cfg["clamp_axis"], 0)]
        if cfg.get("top_z"):
            dofs.append(face_dofs(dm, dim - 1, 1, components=[dim - 1]))
        mask = np.zeros(dm.n_dofs, dtype=bool)
        mask[np.concatenate(dofs)] = True
        meshes.append(mesh)
        masks.append(mask)
    # stacked meshes: the same smooth field over the whole stack (its last axis mapped onto [0, 1])
    ubar = clamp_weighted_sine(dim, meshes[-1].cells, p, phases, amp, cfg["clamp_axis"])
    n_dofs = int(np.prod([c * p + 1 for c in meshes[-1].cells])) * dim
    x = rng.standard_normal(n_dofs) if with_x else None
    return HostWorkload(cfg, meshes, masks, ubar, x)


def stack_mesh(mesh, k: int):
    """``k`` copies of a box mesh stacked along the last axis (shifted by its side)."""
    from dataclasses import replace

    d = mesh.dim
    vg = mesh.vertices.reshape(tuple(c + 1 for c in reversed(mesh.cells)) + (d,))
    parts = []
    for i in range(k):
        v = vg[: -1 if i < k - 1 else None].copy()
        v[..., d - 1] += i * mesh.side
        parts.append(v)
    verts = np.concatenate(parts, axis=0).reshape(-1, d)
    mat = np.tile(mesh.material_id.reshape(mesh.cells[-1], -1), (k, 1)).reshape(-1)
    cells = tuple(mesh.cells[:-1]) + (mesh.cells[-1] * k,)
    return replace(mesh, cells=cells, vertices=np.ascontiguousarray(verts), material_id=mat)


def algorithmic_bytes(strategy: str, dim: int, n_dofs: int, n_qp: int, reference_fields: bool = False) -> int:
    """Bytes one apply must move: 8 (v N_dof + P N_qp).  The
    cache of this design folds JxW into the tensor4 / tensor2 fields (P = 36 /
    17 in 3D); ``reference_fields`` gives SURVEY's P = 37 / 18 (JxW stored)."""
    nv = dim * (dim + 1) // 2
    jxw = 1 if reference_fields else 0
    P = {"tensor4": nv + nv * (nv + 1) // 2 + dim * dim + jxw, "tensor2": 2 + nv + dim * dim + jxw,
         "scalar": 1 + dim * dim + 1}[strategy]
    v = 3 if strategy == "scalar" else 2
    return 8 * (v * n_dofs + P * n_qp)


def meter_flops(dim: int, degree: int, n_el: int, strategy: str) -> int:
    """The reference FLOPS meter of one MatrixFreeTangent.apply (flops.py:28-47
    as tallied by fespace.py / operators.py:341-393); pinned in tests against
    the reference's own count."""
    n = q = degree + 1
    C, nq, nv = dim, q**dim, dim * (dim + 1) // 2
    qp = n_el * nq
    ev = sum(2 * n_el * C * q ** (k + 1) * n ** (dim - k - 1) * n for _ in range(dim) for k in range(dim))
    f = ev
    if strategy == "scalar":
        f += ev + 2 * qp * dim**3 * 3 + 2 * qp * dim * dim
    f += 2 * qp * dim**3 + 2 * qp * dim * dim
    f += 2 * qp * nv * nv if strategy == "tensor4" else 4 * qp * dim * dim
    f += 2 * qp * dim**3 + 2 * qp * dim**3 + qp * dim * dim + qp * C * dim
    f += sum(2 * n_el * C * n ** (k + 1) * q ** (dim - k - 1) * q for _ in range(dim) for k in range(dim))
    f += n_el * n**dim * C
    return int(f)
