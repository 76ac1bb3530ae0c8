"""Structured quad/hex meshes (reference mesh.py), host side.

Conventions as in the reference (mesh.py:1-13): lexicographic numbering with x
fastest; corner c = c1 + 2 c2 + 4 c3; the face of minimal last coordinate is
"bottom", the opposite one "top".  Meshes here are boxes of ``cells[a]`` cells
per axis (cubes in the reference; boxes are the slabs of a multi-GPU
partition).  Connectivity is implicit in the lattice, so only vertices and
per-cell material are stored.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Sequence

import numpy as np

MATRIX = 0
INCLUSION = 1
BOTTOM, TOP, OTHER = "bottom", "top", "other"


def lex_grid_points(axes: Sequence[np.ndarray]) -> np.ndarray:
    """Tensor grid of 1D coordinate arrays, (prod(len), dim), x fastest (mesh.py:30-42)."""
    dim = len(axes)
    grids = np.meshgrid(*[np.asarray(a, dtype=float) for a in reversed(axes)], indexing="ij")
    return np.stack([grids[dim - 1 - k].reshape(-1) for k in range(dim)], axis=1)


def lex_grid_indices(counts: Sequence[int]) -> np.ndarray:
    """Integer multi-indices of a tensor grid, x fastest (mesh.py:45-54)."""
    return lex_grid_points([np.arange(c) for c in counts]).astype(np.int64)


@dataclass(frozen=True)
class Mesh:
    """One structured level: ``cells`` per axis, vertices (n_vertices, dim)."""

    dim: int
    side: float
    cells: tuple
    vertices: np.ndarray
    material_id: np.ndarray
    cell_offset: tuple = (0, 0, 0)  # position of this box inside a partitioned global mesh

    @property
    def n_cells_per_side(self) -> int:
        return self.cells[0]

    @property
    def n_elements(self) -> int:
        return int(np.prod(self.cells))

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    def element_corners(self) -> np.ndarray:
        """(n_el, 2^dim, dim) corner coordinates (mesh.py:84-86)."""
        vstr = np.cumprod((1,) + tuple(c + 1 for c in self.cells[:-1]))
        e = lex_grid_indices(self.cells)
        off = lex_grid_indices((2,) * self.dim)
        return self.vertices[(e[:, None, :] + off[None, :, :]) @ vstr]

    def centroids(self) -> np.ndarray:
        return self.element_corners().mean(axis=1)


@dataclass(frozen=True)
class MeshHierarchy:
    """Nested levels, coarsest first (mesh.py:96-114)."""

    levels: tuple
    parent_index: tuple = ()
    child_index: tuple = ()

    @classmethod
    def from_coarse(cls, mesh: Mesh) -> "MeshHierarchy":
        return cls(levels=(mesh,))

    @property
    def n_levels(self) -> int:
        return len(self.levels)

    @property
    def finest(self) -> Mesh:
        return self.levels[-1]


def _uniform_vertices(cells, side) -> np.ndarray:
    return lex_grid_points([np.linspace(0.0, side, c + 1) for c in cells])


def inclusion_material(dim: int, cells, side: float, inclusion_spec, cell_offset=(0, 0, 0), global_cells=None):
    """Centroid-in-sphere material of a uniform lattice (mesh.py:198-204).

    Only the cells inside each inclusion's bounding box are tested, so the cost
    is O(n_el + n_inclusions * cells_per_ball) instead of O(n_el * n_inclusions).
    """
    gcells = tuple(global_cells) if global_cells is not None else tuple(cells)
    h = np.array([side / g for g in gcells])
    mat = np.full(tuple(reversed(cells)), MATRIX, dtype=np.int64)  # (z, y, x) indexing
    for center, radius in inclusion_spec:
        c = np.asarray(center, dtype=float)
        lo = [max(int(np.floor((c[a] - radius) / h[a] - 0.5)) - cell_offset[a], 0) for a in range(dim)]
        hi = [min(int(np.ceil((c[a] + radius) / h[a] - 0.5)) + 1 - cell_offset[a], cells[a]) for a in range(dim)]
        if any(l >= u for l, u in zip(lo, hi)):
            continue
        axes = [((np.arange(lo[a], hi[a]) + cell_offset[a]) + 0.5) * h[a] - c[a] for a in range(dim)]
        d2 = np.zeros(tuple(hi[a] - lo[a] for a in reversed(range(dim))))
        for a in range(dim):
            shape = [1] * dim
            shape[dim - 1 - a] = -1
            d2 = d2 + axes[a].reshape(shape) ** 2
        inside = np.sqrt(d2) <= radius
        sl = tuple(slice(lo[a], hi[a]) for a in reversed(range(dim)))
        sub = mat[sl]
        sub[inside] = INCLUSION
    return mat.reshape(-1)


def build_benchmark_mesh(dim: int, n_cells_per_side: int, inclusion_spec, side: float = 1e-3) -> Mesh:
    """Structured grid on [0, side]^dim with centroid-test inclusions (mesh.py:170-204)."""
    if dim not in (2, 3):
        raise ValueError(f"dim must be 2 or 3, got {dim}")
    if n_cells_per_side < 2:
        raise ValueError("n_cells_per_side must be at least 2")
    spec = []
    for center, radius in inclusion_spec:
        c = np.asarray(center, dtype=float)
        if c.shape != (dim,):
            raise ValueError(f"inclusion center {center} does not have dim {dim}")
        if np.any(c < 0.0) or np.any(c > side):
            raise ValueError(f"inclusion center {center} lies outside the domain")
        if radius <= 0.0:
            raise ValueError("inclusion radius must be positive")
        spec.append((c, float(radius)))
    cells = (n_cells_per_side,) * dim
    mat = inclusion_material(dim, cells, side, spec)
    return Mesh(dim=dim, side=side, cells=cells, vertices=_uniform_vertices(cells, side), material_id=mat)


def refine_globally(hierarchy: MeshHierarchy, times: int) -> MeshHierarchy:
    """2:1 refinement with inherited material and midpoint vertices (mesh.py:225-264)."""
    if times < 0:
        raise ValueError("times must be non-negative")
    levels = list(hierarchy.levels)
    parents, children = list(hierarchy.parent_index), list(hierarchy.child_index)
    for _ in range(times):
        m = levels[-1]
        d = m.dim
        grid = m.vertices.reshape(tuple(c + 1 for c in reversed(m.cells)) + (d,))
        for ax in range(d):
            n = grid.shape[ax]
            shape = list(grid.shape)
            shape[ax] = 2 * n - 1
            out = np.empty(shape)
            sl = [slice(None)] * grid.ndim
            sl[ax] = slice(0, None, 2)
            out[tuple(sl)] = grid
            lo = [slice(None)] * grid.ndim
            lo[ax] = slice(0, n - 1)
            hi = [slice(None)] * grid.ndim
            hi[ax] = slice(1, n)
            sl[ax] = slice(1, None, 2)
            out[tuple(sl)] = 0.5 * (grid[tuple(lo)] + grid[tuple(hi)])
            grid = out
        cells2 = tuple(2 * c for c in m.cells)
        fe = lex_grid_indices(cells2)
        parent = (fe // 2) @ np.cumprod((1,) + m.cells[:-1])
        child = (fe % 2) @ (2 ** np.arange(d))
        levels.append(Mesh(d, m.side, cells2, grid.reshape(-1, d), m.material_id[parent]))
        parents.append(parent)
        children.append(child)
    return MeshHierarchy(tuple(levels), tuple(parents), tuple(children))


def sub_box(mesh: Mesh, axis: int, start: int, stop: int) -> Mesh:
    """Cells [start, stop) along ``axis`` as a stand-alone box mesh (a partition slab)."""
    d = mesh.dim
    cells = list(mesh.cells)
    cells[axis] = stop - start
    vgrid = mesh.vertices.reshape(tuple(c + 1 for c in reversed(mesh.cells)) + (d,))
    sl = [slice(None)] * d
    sl[d - 1 - axis] = slice(start, stop + 1)
    verts = vgrid[tuple(sl)].reshape(-1, d)
    mgrid = mesh.material_id.reshape(tuple(reversed(mesh.cells)))
    sl[d - 1 - axis] = slice(start, stop)
    mat = mgrid[tuple(sl)].reshape(-1)
    off = list(mesh.cell_offset)
    off[axis] += start
    return replace(mesh, cells=tuple(cells), vertices=np.ascontiguousarray(verts), material_id=mat,
                   cell_offset=tuple(off))
