"""Problem, matrix-free tangent and residual on the B200 (reference operators.py).

Host objects keep the reference API (operators.py:83-116, 205-224, 319-417,
519-522); every numeric step runs in libhf.so:

* ``Problem``         -> ``hf_space``   (1D tables, lattice, J^-1/JxW computed on device)
* ``MatrixFreeTangent``-> ``hf_tangent``(q-point caches built on device; apply/diagonal kernels)
* ``compute_residual``-> ``hf_residual``

Vectors may be numpy arrays (copied to/from the device around the call, the
reference's calling convention) or CUDA fp64 torch tensors (stay on device).
"""

from __future__ import annotations

import ctypes as ct
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import device as dv
from ._lib import HF_ERR_ARG, HF_ERR_JACOBIAN, STRATEGY_CODE, HfErrorInfo, check, lib
from .fespace import (ConstraintSet, bottom_constraints, build_dof_map, gauss_legendre, lagrange_basis)
from .material import NeoHookeanParams, NonPositiveJacobian, n_sym
from .mesh import INCLUSION, Mesh, MeshHierarchy, lex_grid_indices, lex_grid_points

STRATEGIES = ("scalar", "tensor2", "tensor4")


@dataclass(frozen=True)
class Material:
    """Two-phase material (operators.py:75-80)."""

    matrix: NeoHookeanParams
    inclusion: NeoHookeanParams


@dataclass(frozen=True)
class GeometryCache:
    """Host copy of the device geometry (mesh.py:117-130)."""

    jac_inv: np.ndarray  # (n_el, nq, dim, dim)
    jxw: np.ndarray  # (n_el, nq)

    @property
    def nbytes(self) -> int:
        return self.jac_inv.nbytes + self.jxw.nbytes


class Problem:
    """One discretisation level (operators.py:83-116), resident on the GPU."""

    def __init__(self, mesh: Mesh, degree: int, mat: Material, n_qpoints: int | None = None,
                 basis_nodes: str = "equispaced", has_top_face: bool = True):
        dv.require_cuda()
        self.mesh = mesh
        self.degree = degree
        self.quadrature = gauss_legendre(n_qpoints if n_qpoints is not None else degree + 1)
        self.basis = lagrange_basis(degree, self.quadrature, nodes=basis_nodes)
        self.dofmap = build_dof_map(mesh, degree, components=mesh.dim)
        self.material = mat
        inc = mesh.material_id == INCLUSION
        self.mu_el = np.where(inc, mat.inclusion.mu, mat.matrix.mu)[:, None]
        self.lam_el = np.where(inc, mat.inclusion.lam, mat.matrix.lam)[:, None]
        self.has_top_face = has_top_face
        self._constraints = bottom_constraints(mesh, self.dofmap)
        q = self.quadrature.n_points
        cells = (ct.c_int * 3)(*(list(mesh.cells) + [1] * (3 - mesh.dim)))
        h = ct.c_void_p()
        vals = np.ascontiguousarray(self.basis.values)
        ders = np.ascontiguousarray(self.basis.derivatives)
        verts = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        mu = np.ascontiguousarray(self.mu_el[:, 0])
        lam = np.ascontiguousarray(self.lam_el[:, 0])
        mask = np.ascontiguousarray(self._constraints.mask.astype(np.uint8))
        rc = lib().hf_space_create(mesh.dim, degree, q, cells, vals.ctypes.data, ders.ctypes.data,
                                   self.quadrature.points.ctypes.data, self.quadrature.weights.ctypes.data,
                                   verts.ctypes.data, mu.ctypes.data, lam.ctypes.data, mask.ctypes.data,
                                   dv.stream(), ct.byref(h))
        if rc == 5:
            raise ValueError(lib().hf_last_error().decode())
        check(rc)
        self._space = h
        self._geometry = None
        self._sw = None
        self._sw_dev = None
        self._mask_dev = None

    def __del__(self):
        try:
            if getattr(self, "_space", None):
                lib().hf_space_destroy(self._space)
                self._space = None
        except Exception:
            pass

    # --- reference attributes
    @property
    def dim(self) -> int:
        return self.mesh.dim

    @property
    def n_dofs(self) -> int:
        return self.dofmap.n_dofs

    @property
    def n_qpoints_per_cell(self) -> int:
        return self.quadrature.n_points ** self.dim

    def zero_vector(self) -> np.ndarray:
        return np.zeros(self.n_dofs)

    @property
    def constraints(self) -> ConstraintSet:
        return self._constraints

    @constraints.setter
    def constraints(self, cs: ConstraintSet) -> None:
        if cs.n_dofs != self.n_dofs:
            raise ValueError("constraint set does not match the DoF count")
        self._constraints = cs
        m = np.ascontiguousarray(cs.mask.astype(np.uint8))
        check(lib().hf_space_set_mask(self._space, m.ctypes.data, dv.stream()))
        self._mask_dev = None

    @property
    def mask_dev(self) -> torch.Tensor:
        """Device bool mask (torch) of the constrained DoFs."""
        if self._mask_dev is None:
            self._mask_dev = torch.from_numpy(self._constraints.mask.copy()).to("cuda")
        return self._mask_dev

    def mask_ptr(self) -> ct.c_void_p:
        m = ct.c_void_p()
        check(lib().hf_space_pointers(self._space, None, None, ct.byref(m)))
        return m

    @property
    def geometry(self) -> GeometryCache:
        """Download J^-1 and JxW (computed on the device) in the reference layout."""
        if self._geometry is None:
            d, nel, nq = self.dim, self.mesh.n_elements, self.n_qpoints_per_cell
            nqp = nel * nq
            a = torch.empty(d * d * nqp, dtype=torch.float64, device="cuda")
            b = torch.empty(nqp, dtype=torch.float64, device="cuda")
            check(lib().hf_space_geometry_copy(self._space, dv.ptr(a), dv.ptr(b), dv.stream()))
            jinv = a.cpu().numpy().reshape(d, d, nel, nq).transpose(2, 3, 0, 1).copy()
            self._geometry = GeometryCache(jinv, b.cpu().numpy().reshape(nel, nq))
        return self._geometry

    @property
    def surface_weights(self) -> np.ndarray:
        if self._sw is None:
            self._sw = top_surface_weights(self) if self.has_top_face else np.zeros(self.dofmap.n_nodes)
        return self._sw

    @property
    def surface_weights_dev(self) -> torch.Tensor:
        if self._sw_dev is None:
            self._sw_dev = dv.as_dev(self.surface_weights)
        return self._sw_dev


def build_problem_hierarchy(hierarchy: MeshHierarchy, degree: int, mat: Material, n_qpoints: int | None = None):
    """One Problem per mesh level, coarsest first (operators.py:119-126)."""
    return [Problem(m, degree, mat, n_qpoints=n_qpoints) for m in hierarchy.levels]


def top_surface_weights(problem: Problem) -> np.ndarray:
    """s_n = int_top N_n dS per lattice node (operators.py:129-167); host setup."""
    mesh, basis = problem.mesh, problem.basis
    d = mesh.dim
    fd = d - 1
    surf = np.zeros(problem.dofmap.n_nodes)
    e = lex_grid_indices(mesh.cells)
    top = np.flatnonzero(e[:, d - 1] == mesh.cells[d - 1] - 1)
    if len(top) == 0:
        return surf
    quad = basis.quadrature
    pts = lex_grid_points([quad.points] * fd)
    wts = lex_grid_points([quad.weights] * fd).prod(axis=1)
    off = lex_grid_indices((2,) * d)
    fc = np.flatnonzero(off[:, d - 1] == 1)
    corners = mesh.element_corners()[top][:, fc]
    foff = lex_grid_indices((2,) * fd)
    dn = np.ones((2**fd, len(pts), fd))
    for k in range(fd):
        fac = np.where(foff[:, k : k + 1] == 1, pts[None, :, k], 1.0 - pts[None, :, k])
        dfac = np.where(foff[:, k : k + 1] == 1, 1.0, -1.0)
        for a in range(fd):
            dn[:, :, a] *= dfac if a == k else fac
    tang = np.einsum("fci,cqk->fqik", corners, dn)
    if d == 2:
        ds = np.linalg.norm(tang[..., 0], axis=-1)
    else:
        ds = np.linalg.norm(np.cross(tang[..., 0], tang[..., 1]), axis=-1)
    n1 = basis.n_nodes_1d
    nm = lex_grid_indices((n1,) * fd)
    qm = lex_grid_indices((quad.n_points,) * fd)
    nface = np.ones((n1**fd, quad.n_points**fd))
    for k in range(fd):
        nface *= basis.values[nm[:, k][:, None], qm[:, k][None, :]]
    local = np.einsum("nq,fq->fn", nface, wts[None, :] * ds)
    # top-face lattice nodes of each top cell (local last index = p)
    npa = problem.dofmap.nodes_per_axis
    p = problem.degree
    strides = np.cumprod((1,) + npa[:-1])
    loc = lex_grid_indices((n1,) * fd)
    base = e[top] * p
    nodes = np.zeros((len(top), n1**fd), dtype=np.int64)
    for a in range(fd):
        nodes += (base[:, a][:, None] + loc[None, :, a]) * strides[a]
    nodes += (base[:, d - 1][:, None] + p) * strides[d - 1]
    np.add.at(surf, nodes, local)
    return surf


# ---------------------------------------------------------------------------


def _raise_jacobian(err: HfErrorInfo, level=None):
    raise NonPositiveJacobian(lib().hf_last_error().decode(), element=int(err.element), level=level)


def jacobian_range(problem: Problem, u) -> tuple[float, float]:
    """Min and max of det F over all quadrature points (operators.py:192-196)."""
    ud = dv.as_dev(u)
    lo, hi = ct.c_double(), ct.c_double()
    check(lib().hf_jacobian_range(problem._space, dv.ptr(ud), dv.stream(), ct.byref(lo), ct.byref(hi), None, None))
    return lo.value, hi.value


def compute_residual(problem: Problem, u, traction=None):
    """Internal Kirchhoff-stress force minus the top traction, constrained
    entries zeroed (operators.py:205-224)."""
    ud = dv.as_dev(u)
    out = torch.empty_like(ud)
    err = HfErrorInfo()
    if traction is not None:
        t = np.ascontiguousarray(np.asarray(traction, dtype=np.float64).reshape(-1))
        rc = lib().hf_residual(problem._space, dv.ptr(ud), t.ctypes.data, dv.ptr(problem.surface_weights_dev),
                               dv.ptr(out), dv.stream(), ct.byref(err))
    else:
        rc = lib().hf_residual(problem._space, dv.ptr(ud), None, None, dv.ptr(out), dv.stream(), ct.byref(err))
    if rc == HF_ERR_JACOBIAN:
        _raise_jacobian(err)
    check(rc)
    return dv.like_input(out, u)


def energy(problem: Problem, u, traction=None) -> float:
    """Total potential energy: strain energy minus the top traction work
    (operators.py:227-236); the finite-difference oracle of the residual."""
    ud = dv.as_dev(u)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    err = HfErrorInfo()
    rc = lib().hf_energy(problem._space, dv.ptr(ud), dv.ptr(out), dv.stream(), ct.byref(err))
    if rc == HF_ERR_JACOBIAN:
        _raise_jacobian(err)
    check(rc)
    total = float(out.item())
    if traction is not None:
        t = torch.as_tensor(np.asarray(traction, dtype=np.float64).reshape(-1), device="cuda")
        work = problem.surface_weights_dev @ ud.view(-1, problem.dim)  # (dim,)
        total -= float(t @ work)
    return total


@dataclass
class CacheInfo:
    """What the reference exposes of its quadrature caches (operators.py:244-289)."""

    strategy: str
    payload_scalars_per_qpoint: int
    payload_nbytes: int


class MatrixFreeTangent:
    """Apply-only tangent backed by one of the three q-point caches (operators.py:319-417)."""

    def __init__(self, problem: Problem, u_bar, strategy: str = "tensor4", storage: str = "fp64"):
        """``storage="fp32"`` keeps the q-point cache -- and the x / y vectors of
        ``apply_into`` -- in float (mixed-precision multigrid levels, SURVEY §8(f)
        row 1); all arithmetic stays fp64."""
        if strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {strategy!r}")
        if storage not in ("fp64", "fp32"):
            raise ValueError(f"unknown storage {storage!r}")
        self.problem = problem
        self.strategy = strategy
        self.storage = storage
        self.dtype = torch.float32 if storage == "fp32" else torch.float64
        # numpy u_bar -> numpy results from diagonal() (the reference's calling
        # convention, operators.py:395-410; multigrid.py:226-227 does 1.0 / diag)
        self._host_io = isinstance(u_bar, np.ndarray)
        ud = dv.as_dev(u_bar)
        h = ct.c_void_p()
        err = HfErrorInfo()
        rc = lib().hf_tangent_create_ex(problem._space, STRATEGY_CODE[strategy], 32 if storage == "fp32" else 64,
                                        dv.ptr(ud), dv.stream(), ct.byref(h), ct.byref(err))
        if rc == HF_ERR_JACOBIAN:
            _raise_jacobian(err)
        check(rc)
        self._op = h
        sb, ps, pb = ct.c_longlong(), ct.c_int(), ct.c_longlong()
        check(lib().hf_tangent_storage(h, ct.byref(sb), ct.byref(ps), ct.byref(pb)))
        self._storage = sb.value
        self.cache = CacheInfo(strategy, ps.value, pb.value)

    def __del__(self):
        try:
            if getattr(self, "_op", None):
                lib().hf_tangent_destroy(self._op)
                self._op = None
        except Exception:
            pass

    @property
    def n_dofs(self) -> int:
        return self.problem.n_dofs

    def apply_into(self, x: torch.Tensor, y: torch.Tensor, skip: torch.Tensor | None = None) -> torch.Tensor:
        """y = A x on device buffers (no allocation; graph-capturable)."""
        check(lib().hf_tangent_apply_flagged(self._op, dv.ptr(x), dv.ptr(y), dv.ptr(skip), dv.stream()))
        return y

    def apply_after_fill(self, x: torch.Tensor, y: torch.Tensor, skip: torch.Tensor | None = None) -> torch.Tensor:
        """Cell kernel of y = A x when the previous kernel on the stream already
        wrote x and y = mask ? x : 0 (hf_cheb_step_fill); programmatic dependent launch."""
        check(lib().hf_tangent_apply_after_fill(self._op, dv.ptr(x), dv.ptr(y), dv.ptr(skip), dv.stream()))
        return y

    def tiles(self) -> tuple[int, int]:
        """(number of tiles, cells per tile) of the cell kernel's work decomposition."""
        nt, cpt = ct.c_longlong(), ct.c_int()
        check(lib().hf_tangent_tiles(self._op, ct.byref(nt), ct.byref(cpt)))
        return nt.value, cpt.value

    def apply_tiles(self, x: torch.Tensor, y: torch.Tensor, tile0: int, tile1: int, mode: int = 0,
                    reserve_sms: int = 0) -> torch.Tensor:
        """y += A_loc x over the cells of tiles [tile0, tile1) (constrained rows dropped);
        mode 1/2: programmatic dependent of the fill / of an x-and-y producer;
        reserve_sms: launch on that many fewer SMs (a concurrent NCCL kernel)."""
        check(lib().hf_tangent_apply_tiles_ex(self._op, dv.ptr(x), dv.ptr(y), None, tile0, tile1, mode, reserve_sms,
                                              dv.stream()))
        return y

    def apply_raw(self, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        """y += sum over cells of A_loc x (constrained rows dropped), no init."""
        check(lib().hf_tangent_apply_raw(self._op, dv.ptr(x), dv.ptr(y), None, dv.stream()))
        return y

    def apply(self, x, out=None):
        """y = A x: zero-in / identity-out on the constrained subspace (operators.py:331-339).

        numpy in -> numpy out; CUDA tensor in -> CUDA tensor out; a pinned CPU
        tensor in with a pinned ``out`` runs the host-to-host pipeline
        (``apply_host``)."""
        if (out is not None and isinstance(x, torch.Tensor) and isinstance(out, torch.Tensor) and not x.is_cuda
                and not out.is_cuda and self.storage == "fp64"):
            # host tensors: the host pipeline when both are page-locked (libhf
            # checks that itself, so no torch is_pinned() queries on this path)
            if self._apply_host(x, out, 4, must=False):
                return out
        if isinstance(x, np.ndarray) and out is None and self.storage == "fp64" and x.size == self.n_dofs and \
                self._count_numpy_apply() > 2:
            # the reference's convention (numpy in, fresh numpy out), applied
            # repeatedly: x is copied into page-locked staging owned by the
            # tangent, the slab-pipelined host apply runs from there (calibrated
            # once per tangent), and y is copied out of it
            xs, ys = self._staging()
            np.copyto(xs.numpy(), x.reshape(-1), casting="same_kind")
            self._apply_host(xs, ys, 4, must=True)
            return ys.numpy().copy().reshape(x.shape)
        xd = dv.as_dev(x)
        if self.storage == "fp32":  # the public apply stays fp64 in, fp64 out
            y32 = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
            self.apply_into(xd.float(), y32)
            y = y32.double()
        else:
            y = torch.empty_like(xd)
            self.apply_into(xd, y)
        if out is not None:
            out.copy_(y, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return out
        return dv.like_input(y, x)

    def _count_numpy_apply(self) -> int:
        self._numpy_applies = getattr(self, "_numpy_applies", 0) + 1
        return self._numpy_applies

    def _staging(self):
        """Page-locked host x / y staging of the numpy apply (allocated once)."""
        st = getattr(self, "_host_staging", None)
        if st is None:
            st = self._host_staging = (torch.empty(self.n_dofs, dtype=torch.float64).pin_memory(),
                                       torch.empty(self.n_dofs, dtype=torch.float64).pin_memory())
        return st

    def apply_host(self, xh: torch.Tensor, yh: torch.Tensor, chunks: int = 4) -> torch.Tensor:
        """y = A x between page-locked host buffers (hf_tangent_apply_host): the
        H2D copy of each slab's node planes, the slab's cell kernel and the D2H
        copy of finished planes overlap on three streams; the pipeline is a
        CUDA graph captured on first use per buffer pair and replayed after."""
        self._apply_host(xh, yh, chunks, must=True)
        return yh

    def _apply_host(self, xh: torch.Tensor, yh: torch.Tensor, chunks: int, must: bool) -> bool:
        """hf_tangent_apply_host + stream synchronisation.  With ``must=False``
        returns False (nothing run) when the buffers are not page-locked."""
        if xh.dtype != torch.float64 or yh.dtype != torch.float64 or xh.numel() != self.n_dofs \
                or yh.numel() != self.n_dofs or not (xh.is_contiguous() and yh.is_contiguous()):
            if must:
                raise ValueError("apply_host needs contiguous float64 host vectors of n_dofs entries")
            return False
        s = torch.cuda.current_stream()
        rc = lib().hf_tangent_apply_host(self._op, xh.data_ptr(), yh.data_ptr(), chunks, s.cuda_stream)
        if rc == HF_ERR_ARG and not must:
            return False  # not page-locked: the caller copies through device buffers
        check(rc)
        s.synchronize()
        return True

    def host_info(self) -> dict:
        """How the host pipeline runs on this host (hf_tangent_host_info): the
        variant kept and the calibration step times (us) of all four."""
        v, us = ct.c_int(), (ct.c_float * 4)()
        check(lib().hf_tangent_host_info(self._op, ct.byref(v), us))
        names = ["graph+overlap", "graph+serial", "direct+overlap", "direct+serial"]
        return {"variant": names[v.value] if v.value >= 0 else None,
                "calibration_us": {names[i]: round(us[i], 1) for i in range(4)}}

    def __call__(self, x):
        return self.apply(x)

    def diagonal(self, as_numpy: bool | None = None):
        """diag(A), constrained entries 1 (operators.py:395-410); fp64 storage only.

        Returns an ndarray when the tangent was built from an ndarray ``u_bar``
        (the reference's convention) or ``as_numpy`` is set, else a CUDA tensor."""
        d = self.diagonal_dev()
        return d.cpu().numpy() if (self._host_io if as_numpy is None else as_numpy) else d

    def diagonal_dev(self) -> torch.Tensor:
        """diag(A) as a CUDA fp64 tensor (the form the device-side callers use)."""
        d = torch.empty(self.n_dofs, dtype=torch.float64, device="cuda")
        check(lib().hf_tangent_diagonal(self._op, dv.ptr(d), dv.stream()))
        return d

    def storage_bytes(self) -> int:
        """Strategy payload plus geometry (operators.py:412-417)."""
        return self._storage


class AssembledTangent:
    """Matrix-based tangent: CSR on the device, used as baseline and second
    oracle (operators.py:436-516).

    Element matrices come from libhf (``hf_tangent_assemble_local``, formed
    from the tensor4 q-point cache); duplicates are summed and the CSR built
    with torch's sort/coalesce; constrained rows and columns are cleared and
    replaced by a unit diagonal (operators.py:481-490); ``apply`` is a
    cuSPARSE SpMV.  Host-side plumbing only: a baseline, not the hot path."""

    strategy = "matrix_based"

    def __init__(self, problem: Problem, u_bar):
        self.problem = problem
        self._host_io = isinstance(u_bar, np.ndarray)
        op4 = MatrixFreeTangent(problem, u_bar, "tensor4")  # NonPositiveJacobian propagates
        nel, d = problem.mesh.n_elements, problem.dim
        nld = problem.n_qpoints_per_cell * d
        vals = torch.empty(nel * nld * nld, dtype=torch.float64, device="cuda")
        check(lib().hf_tangent_assemble_local(op4._op, dv.ptr(vals), dv.stream()))
        dofs = torch.empty(nel * nld, dtype=torch.int64, device="cuda")
        check(lib().hf_space_cell_dofs(problem._space, dv.ptr(dofs), dv.stream()))
        del op4
        dofs = dofs.view(nel, nld)
        rows = dofs[:, :, None].expand(nel, nld, nld).reshape(-1)
        cols = dofs[:, None, :].expand(nel, nld, nld).reshape(-1)
        mask = problem.mask_dev
        keep = ~(mask[rows] | mask[cols])
        fixed = torch.nonzero(mask).reshape(-1)
        rows = torch.cat([rows[keep], fixed])
        cols = torch.cat([cols[keep], fixed])
        vals = torch.cat([vals[keep], torch.ones(fixed.numel(), dtype=torch.float64, device="cuda")])
        n = problem.n_dofs
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)  # torch: sparse invariant checks off / CSR "beta"
            coo = torch.sparse_coo_tensor(torch.stack([rows, cols]), vals, (n, n), check_invariants=False).coalesce()
            del rows, cols, vals, keep
            self.matrix = coo.to_sparse_csr()
        self._diag = None

    @property
    def n_dofs(self) -> int:
        return self.problem.n_dofs

    def apply_into(self, x: torch.Tensor, y: torch.Tensor, skip=None) -> torch.Tensor:
        y.copy_(torch.mv(self.matrix, x))
        return y

    def apply(self, x):
        xd = dv.as_dev(x)
        return dv.like_input(torch.mv(self.matrix, xd), x)

    __call__ = apply

    def diagonal(self, as_numpy: bool | None = None):
        d = self.diagonal_dev()
        return d.cpu().numpy() if (self._host_io if as_numpy is None else as_numpy) else d

    def diagonal_dev(self) -> torch.Tensor:
        if self._diag is None:
            m = self.matrix
            crow, col, val = m.crow_indices(), m.col_indices(), m.values()
            row = torch.repeat_interleave(torch.arange(self.n_dofs, device="cuda"), crow[1:] - crow[:-1])
            d = torch.zeros(self.n_dofs, dtype=torch.float64, device="cuda")
            on = row == col
            d.index_add_(0, row[on], val[on])
            self._diag = d
        return self._diag

    def storage_bytes(self) -> int:
        """CSR bytes with 32-bit indices, as scipy stores the reference matrix (operators.py:514-516)."""
        nnz = self.matrix.values().numel()
        return 8 * nnz + 4 * nnz + 4 * (self.n_dofs + 1)


def make_tangent(problem: Problem, u_bar, strategy: str):
    """(operators.py:519-522)"""
    if strategy == "matrix_based":
        return AssembledTangent(problem, u_bar)
    return MatrixFreeTangent(problem, u_bar, strategy)
