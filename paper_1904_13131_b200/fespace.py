"""Tensor-product Lagrange spaces, host side (reference fespace.py:1-175).

Only the small 1D tables, the closed-form DoF numbering and the constraint
sets live here; gather / sum-factorisation / scatter run on the device
(csrc/hf_cell.cuh).  Vector DoF = node * n_components + component, nodes on
the lexicographic (cells*p+1)^dim lattice (fespace.py:3-8, 125-139).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

from .mesh import Mesh, lex_grid_indices, lex_grid_points


@dataclass(frozen=True)
class Quadrature1D:
    points: np.ndarray
    weights: np.ndarray

    @property
    def n_points(self) -> int:
        return len(self.points)


def gauss_legendre(q: int) -> Quadrature1D:
    """Gauss-Legendre rule on [0, 1] (fespace.py:33-37)."""
    if not 1 <= q <= 16:
        raise ValueError(f"number of quadrature points must be in [1, 16], got {q}")
    t, w = np.polynomial.legendre.leggauss(q)
    return Quadrature1D(points=(t + 1.0) * 0.5, weights=w * 0.5)


def lagrange_values(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """(n_nodes, n_x) Lagrange basis values (fespace.py:40-47)."""
    x = np.asarray(x, dtype=float)
    n = len(nodes)
    out = np.ones((n, len(x)))
    for i in range(n):
        for j in range(n):
            if j != i:
                out[i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
    return out


def lagrange_derivatives(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """(n_nodes, n_x) first derivatives (fespace.py:50-62)."""
    x = np.asarray(x, dtype=float)
    n = len(nodes)
    out = np.zeros((n, len(x)))
    for i in range(n):
        for k in range(n):
            if k == i:
                continue
            term = np.full(len(x), 1.0 / (nodes[i] - nodes[k]))
            for j in range(n):
                if j != i and j != k:
                    term *= (x - nodes[j]) / (nodes[i] - nodes[j])
            out[i] += term
    return out


@dataclass(frozen=True)
class Basis1D:
    degree: int
    nodes: np.ndarray
    quadrature: Quadrature1D
    values: np.ndarray  # (p+1, q)
    derivatives: np.ndarray  # (p+1, q)

    @property
    def n_nodes_1d(self) -> int:
        return self.degree + 1


def lagrange_basis(degree: int, quadrature: Quadrature1D, nodes: str = "equispaced") -> Basis1D:
    """Equispaced (default) or Gauss-Lobatto Lagrange basis (fespace.py:85-102)."""
    if degree < 1:
        raise ValueError("degree must be at least 1")
    if nodes == "equispaced":
        pts = np.arange(degree + 1) / degree
    elif nodes == "gauss_lobatto":
        inner = np.polynomial.legendre.Legendre.basis(degree).deriv().roots()
        pts = np.concatenate(([0.0], 0.5 * (np.sort(inner) + 1.0), [1.0]))
    else:
        raise ValueError(f"unknown node rule {nodes!r}")
    return Basis1D(degree, pts, quadrature, lagrange_values(pts, quadrature.points),
                   lagrange_derivatives(pts, quadrature.points))


@dataclass(frozen=True)
class DoFMap:
    """Closed-form numbering of the scalar lattice nodes plus vector blocking."""

    dim: int
    degree: int
    components: int
    nodes_per_axis: tuple

    @property
    def nodes_per_side(self) -> int:
        return self.nodes_per_axis[0]

    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.nodes_per_axis))

    @property
    def n_dofs(self) -> int:
        return self.n_nodes * self.components

    @property
    def n_local_nodes(self) -> int:
        return (self.degree + 1) ** self.dim

    @cached_property
    def cell_nodes(self) -> np.ndarray:
        """(n_el, (p+1)^dim) global node ids; the device computes these on the fly."""
        cells = tuple((n - 1) // self.degree for n in self.nodes_per_axis)
        strides = np.cumprod((1,) + self.nodes_per_axis[:-1])
        e = lex_grid_indices(cells)
        loc = lex_grid_indices((self.degree + 1,) * self.dim)
        return (e[:, None, :] * self.degree + loc[None, :, :]) @ strides


def build_dof_map(mesh: Mesh, degree: int, components: int) -> DoFMap:
    return DoFMap(mesh.dim, degree, components, tuple(c * degree + 1 for c in mesh.cells))


def node_coordinates(mesh: Mesh, dofmap: DoFMap) -> np.ndarray:
    """Physical node coordinates via the multilinear cell map (fespace.py:142-151).

    The cell map is the tensor product of 1D linear interpolations between
    the cell corners, so the node lattice is the vertex lattice refined by
    p-1 interpolated points per cell, one axis after the other (no per-cell
    gather: 20 ms instead of 0.4 s at 64^3 Q2)."""
    d, p = mesh.dim, dofmap.degree
    V = np.asarray(mesh.vertices, dtype=np.float64).reshape(tuple(c + 1 for c in reversed(mesh.cells)) + (d,))
    t = np.arange(p) / p
    for A in range(d):  # array axis A (x is the last array axis: lexicographic, x fastest)
        m = V.shape[A] - 1
        out = np.empty(V.shape[:A] + (p * m + 1,) + V.shape[A + 1:])

        def ax(sl, A=A):
            return (slice(None),) * A + (sl,)

        lo, hi = V[ax(slice(0, m))], V[ax(slice(1, m + 1))]
        for j in range(p):
            out[ax(slice(j, p * m, p))] = lo * (1.0 - t[j]) + hi * t[j] if j else lo
        out[ax(slice(p * m, p * m + 1))] = V[ax(slice(m, m + 1))]
        V = out
    return V.reshape(-1, d)


@dataclass(frozen=True)
class ConstraintSet:
    """Homogeneous Dirichlet DoFs (fespace.py:154-167)."""

    n_dofs: int
    dofs: np.ndarray
    mask: np.ndarray

    @classmethod
    def from_dofs(cls, n_dofs: int, dofs) -> "ConstraintSet":
        dofs = np.unique(np.asarray(dofs, dtype=np.int64))
        mask = np.zeros(n_dofs, dtype=bool)
        mask[dofs] = True
        return cls(n_dofs=n_dofs, dofs=dofs, mask=mask)


def face_dofs(dofmap: DoFMap, axis: int, side: int, components=None) -> np.ndarray:
    """DoFs of every lattice node on the face ``axis`` = min (side 0) / max (side 1)."""
    npa = dofmap.nodes_per_axis
    idx = [np.arange(n) for n in npa]
    idx[axis] = np.array([0 if side == 0 else npa[axis] - 1])
    strides = np.cumprod((1,) + npa[:-1])
    grids = np.meshgrid(*idx, indexing="ij")
    nodes = np.sort(sum(g.reshape(-1) * s for g, s in zip(grids, strides)))
    comps = range(dofmap.components) if components is None else components
    return np.sort(np.concatenate([nodes * dofmap.components + c for c in comps]))


def bottom_constraints(mesh: Mesh, dofmap: DoFMap) -> ConstraintSet:
    """All components on the face of minimal last coordinate (fespace.py:170-175)."""
    return ConstraintSet.from_dofs(dofmap.n_dofs, face_dofs(dofmap, dofmap.dim - 1, 0))


def interpolation_matrix_1d(degree: int, n_coarse_cells: int, nodes: np.ndarray) -> np.ndarray:
    """Coarse -> 2:1 refined 1D nodal interpolation, (n_fine, n_coarse) (multigrid.py:58-73)."""
    p, m = degree, n_coarse_cells
    nf = 2 * m * p + 1
    mat = np.zeros((nf, m * p + 1))
    f = np.arange(nf)
    cell = np.minimum(f // (2 * p), m - 1)
    xi = (f - 2 * p * cell) / (2.0 * p)
    for c in range(m):
        sel = np.flatnonzero(cell == c)
        if len(sel):
            mat[sel[None, :], (c * p + np.arange(p + 1))[:, None]] = lagrange_values(nodes, xi[sel])
    return mat
