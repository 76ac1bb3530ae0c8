"""Geometric multigrid on the B200 (reference multigrid.py:1-382).

Same algorithm and API as the reference: level tangents linearised at the
nodal injection of the fine state, Kronecker 1D transfers (restriction = the
transpose), CG/Lanczos eigenvalue range, restarted Chebyshev smoothing of
degree 4 on [0.6, 1.2] lambda_max, continuous Chebyshev coarse solve to 1e-3
with a 100-application cap, V-cycle with 2 pre/post steps.

Device design: every vector lives in a per-level preallocated buffer; each
step is one fused libhf kernel (apply, Chebyshev update, masked residual,
transfer passes).  The coarse solve's convergence test is evaluated on the
device (a flag that turns the remaining kernels into no-ops), so one whole
V-cycle is a fixed launch sequence that ``GMGPreconditioner`` captures once
into a CUDA graph and replays per application.

Deviation (documented in DESIGN.md): the first operator application of the
pre-smoother acts on the zero vector and is skipped (A 0 = 0 exactly).
"""

from __future__ import annotations

import ctypes as ct
import os
import logging
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import torch

from . import device as dv
from ._lib import HF_ERR_UNSUPPORTED, HfError, check, lib
from .fespace import interpolation_matrix_1d
from .material import NonPositiveJacobian
from .operators import AssembledTangent, MatrixFreeTangent, Problem

log = logging.getLogger(__name__)


def _bits(t: torch.Tensor) -> int:
    return 32 if t.dtype == torch.float32 else 64


def _apply_into(op, x, y, skip=None):
    if hasattr(op, "apply_into"):
        return op.apply_into(x, y, skip)
    y.copy_(op(x))
    return y


class TransferOperator:
    """Embedding of a coarse tensor-product space into the 2:1 refined one (multigrid.py:27-55)."""

    def __init__(self, coarse: Problem, fine: Problem):
        if any(f != 2 * c for f, c in zip(fine.mesh.cells, coarse.mesh.cells)):
            raise ValueError("transfer requires a 2:1 refined pair of levels")
        self.coarse, self.fine = coarse, fine
        self.dim = coarse.dim
        self.components = coarse.dofmap.components
        self.coarse_nodes_1d = coarse.dofmap.nodes_per_side
        self.fine_nodes_1d = fine.dofmap.nodes_per_side
        self.matrices_1d = [np.ascontiguousarray(interpolation_matrix_1d(coarse.degree, m, coarse.basis.nodes))
                            for m in coarse.mesh.cells]
        self.matrix_1d = self.matrices_1d[0]
        ptrs = (ct.c_void_p * 3)(*[m.ctypes.data for m in self.matrices_1d] + [None] * (3 - self.dim))
        h = ct.c_void_p()
        check(lib().hf_transfer_create(coarse._space, fine._space, ptrs, ct.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().hf_transfer_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def prolong_into(self, xc, xf, mode: int = 0):
        """fp64 or fp32 vectors on either side (mixed-precision levels)."""
        check(lib().hf_prolong_ex(self._h, dv.ptr(xc), _bits(xc), dv.ptr(xf), _bits(xf), mode, dv.stream()))
        return xf

    def restrict_into(self, rf, rc, mode: int = 0):
        check(lib().hf_restrict_ex(self._h, dv.ptr(rf), _bits(rf), dv.ptr(rc), _bits(rc), mode, dv.stream()))
        return rc

    def prolong(self, x_coarse):
        xc = dv.as_dev(x_coarse)
        out = torch.empty(self.fine.n_dofs, dtype=torch.float64, device="cuda")
        return dv.like_input(self.prolong_into(xc, out), x_coarse)

    def restrict(self, r_fine):
        rf = dv.as_dev(r_fine)
        out = torch.empty(self.coarse.n_dofs, dtype=torch.float64, device="cuda")
        return dv.like_input(self.restrict_into(rf, out), r_fine)


def restrict_solution(problems: list[Problem], u_fine, keep_constrained: bool = False):
    """Nodal injection of the finest displacement onto every level (multigrid.py:76-92).

    ``keep_constrained`` keeps prescribed Dirichlet values on the levels
    (needed for non-homogeneous constraints); the reference resets
    them to zero."""
    levels = [dv.as_dev(u_fine)]
    for lvl in range(len(problems) - 1, 0, -1):
        fp, cp = problems[lvl], problems[lvl - 1]
        uc = torch.empty(cp.n_dofs, dtype=torch.float64, device="cuda")
        check(lib().hf_inject(cp._space, fp._space, dv.ptr(levels[0]), dv.ptr(uc), int(keep_constrained),
                              dv.stream()))
        levels.insert(0, uc)
    if not isinstance(u_fine, torch.Tensor):
        return [v.cpu().numpy() for v in levels]
    return levels


_RHS_CACHE: dict = {}


def _lanczos_rhs(n: int, seed: int, mask) -> torch.Tensor:
    """b = default_rng(seed).standard_normal(n), constrained = 0 (multigrid.py:121-124).  The
    unmasked draw is cached on the device per (n, seed); the mask (numpy or device bool) is
    applied on the device."""
    key = (n, seed)
    if key not in _RHS_CACHE:
        _RHS_CACHE[key] = dv.as_dev(np.random.default_rng(seed).standard_normal(n))
    b = _RHS_CACHE[key]
    if mask is None:
        return b.clone()
    m = mask if isinstance(mask, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(mask, dtype=bool))
    return b.masked_fill(m.to(device=b.device, dtype=torch.bool), 0.0)


def _ritz_extremes(alphas, betas) -> tuple[float, float]:
    """Extreme eigenvalues of the Lanczos tridiagonal (multigrid.py:156-166)."""
    k = len(alphas)
    if k == 0:
        return 1.0, 1.0
    diag_t = np.empty(k)
    diag_t[0] = 1.0 / alphas[0]
    for i in range(1, k):
        diag_t[i] = 1.0 / alphas[i] + betas[i - 1] / alphas[i - 1]
    off_t = np.array([np.sqrt(betas[i]) / alphas[i] for i in range(k - 1)])
    if k == 1:
        return float(diag_t[0]), float(diag_t[0])
    ritz = scipy.linalg.eigvalsh_tridiagonal(diag_t, off_t)
    return float(ritz[0]), float(ritz[-1])


def lanczos_coefficients(apply_fn, diagonal, seed: int = 0, iterations: int = 30, constrained=None):
    """alpha_k, beta_k of the Jacobi-PCG run of estimate_eigenvalue_range
    (multigrid.py:112-155).  All iterations are enqueued without a host round
    trip: the scalars, the stopping tests and the recording live on the device
    (hf_lanczos_step); the application is skipped once the run has stopped.
    One synchronisation at the end reads the coefficients."""
    diag = dv.as_dev(diagonal)
    n = diag.numel()
    r = _lanczos_rhs(n, seed, constrained)
    inv_d = torch.reciprocal(diag)
    z = torch.empty_like(r)
    ap = torch.empty_like(r)
    scal = torch.zeros(4, dtype=torch.float64, device="cuda")
    st = torch.zeros(2, dtype=torch.int32, device="cuda")
    ab = torch.zeros(2 * max(iterations, 1), dtype=torch.float64, device="cuda")
    ws = dv.Workspace.get().handle
    L = lib()
    check(L.hf_jacobi_dot(ws, n, dv.ptr(z), dv.ptr(r), dv.ptr(inv_d), dv.ptr(scal[0:1]), dv.stream()))
    p = z.clone()
    check(L.hf_lanczos_init(dv.ptr(scal), dv.ptr(st), dv.stream()))
    # the tangent itself: the p update also writes the next application's
    # initialisation (ap = mask ? p : 0) and that application runs as its
    # programmatic dependent; r update, Jacobi scaling and r.z are one pass
    # (hf_lanczos_step_fill: 5 launches per iteration instead of 7)
    fused = _LANCZOS_FUSED and isinstance(apply_fn, MatrixFreeTangent) and apply_fn.storage == "fp64"
    mask_ptr = apply_fn.problem.mask_ptr() if fused else None
    for it in range(iterations):
        if fused and it > 0:
            apply_fn.apply_after_fill(p, ap, st)
        else:
            _apply_into(apply_fn, p, ap, st)
        if fused:
            check(L.hf_lanczos_step_fill(ws, n, dv.ptr(r), dv.ptr(z), dv.ptr(p), dv.ptr(ap), dv.ptr(inv_d),
                                         dv.ptr(scal), dv.ptr(ab), dv.ptr(st), mask_ptr, dv.ptr(ap), dv.stream()))
        else:
            check(L.hf_lanczos_step(ws, n, dv.ptr(r), dv.ptr(z), dv.ptr(p), dv.ptr(ap), dv.ptr(inv_d), dv.ptr(scal),
                                    dv.ptr(ab), dv.ptr(st), dv.stream()))
    k = int(st[1].item())
    abh = ab[: 2 * k].cpu().numpy()
    return abh[0::2].copy(), abh[1::2][: max(k - 1, 0)].copy()


def estimate_eigenvalue_range(apply_fn, diagonal, seed: int = 0, iterations: int = 30,
                              constrained=None) -> tuple[float, float]:
    """Smallest and largest Ritz values of D^-1 A from a Jacobi-PCG/Lanczos run
    (multigrid.py:112-166).  Vector work, dots and the stopping tests on the
    device; the k x k tridiagonal eigenproblem on the host with the reference's
    scipy call."""
    return _ritz_extremes(*lanczos_coefficients(apply_fn, diagonal, seed, iterations, constrained))


def estimate_lambda_max(apply_fn, diagonal, seed=0, iterations=30, constrained=None) -> float:
    return estimate_eigenvalue_range(apply_fn, diagonal, seed, iterations, constrained)[1]


@dataclass(frozen=True)
class ChebyshevSettings:
    degree: int = 4
    range_lo: float = 0.6
    range_hi: float = 1.2


def _cheb_coeffs(lam_max: float, s: ChebyshevSettings):
    theta = 0.5 * (s.range_hi + s.range_lo) * lam_max
    delta = 0.5 * (s.range_hi - s.range_lo) * lam_max
    sigma = theta / delta
    coefs = []
    rho_old = 1.0 / sigma
    for _ in range(s.degree - 1):
        rho = 1.0 / (2.0 * sigma - rho_old)
        coefs.append((rho * rho_old, 2.0 * rho / delta))
        rho_old = rho
    return theta, coefs


_PDL_CHEB_MAX_DOFS = int(os.environ.get("HF_PDL_CHEB_MAX_DOFS", 1 << 18))
_LANCZOS_FUSED = os.environ.get("HF_LANCZOS_FUSED", "1") != "0"  # A/B switch of hf_lanczos_step_fill
_CHEB3 = os.environ.get("HF_CHEB3", "1") != "0"  # three-term Chebyshev updates (hf_cheb3_step)


def _apply_maybe_filled(apply_fn, x, ax, prefilled: bool, skip=None):
    if prefilled:
        return apply_fn.apply_after_fill(x, ax, skip)
    return _apply_into(apply_fn, x, ax, skip)


def _chebyshev_into(apply_fn, inv_d, lam_max, b, x, d, ax, s: ChebyshevSettings, steps: int, x_zero: bool,
                    mask=None, fill_last: bool = False):
    """In-place restarted Chebyshev on device buffers (multigrid.py:176-205).

    With ``mask`` (and an operator that has ``apply_after_fill``), every
    Chebyshev update also writes ax = mask ? x : 0 for the next operator
    application, which then runs as its programmatic dependent launch;
    ``fill_last`` does so after the final update too (the V-cycle's residual
    apply follows the pre-smoother).

    The updates run in three-term form (hf_cheb3_step): ``d`` is not the stored
    direction but the second iterate buffer; each update reads x_k and x_{k-1}
    and writes x_{k+1} over x_{k-1}, one vector write less than the
    stored-direction form.  The result ends in ``x`` (copied there after an odd
    number of updates).  ``HF_CHEB3=0`` keeps the stored direction
    (hf_cheb_step*)."""
    theta, coefs = _cheb_coeffs(lam_max, s)
    n = x.numel()
    L = lib()
    fuse = mask is not None and hasattr(apply_fn, "apply_after_fill")
    # The launch before an update is libhf's cell kernel: on small levels the
    # update runs as its programmatic dependent (hf_cheb_step_after_apply),
    # which hides its launch latency: a smoothing at 8^3 49.4 -> 47.3 us, at
    # 16^3 86.2 -> 84.2 us, the config-1 solve 12.5 -> 11.9 ms.  On large levels
    # the early-resident update blocks slow the cell kernel (64^3: +3 %), so
    # those keep the plain launch (profiles/r02/experiments/ab_pdl_cheb.txt).
    chained = isinstance(apply_fn, MatrixFreeTangent) and n <= _PDL_CHEB_MAX_DOFS
    filled = False
    n_upd = steps * (1 + len(coefs))
    k = 0
    cur, oth = x, d          # three-term form: x_k and the buffer x_{k+1} goes to
    prev_zero = False        # x_{k-1} = 0 (the update after one from x = 0)

    def update(first, th, cd, cz, zero):
        nonlocal filled, k, cur, oth, prev_zero
        k += 1
        fill = fuse and (k < n_upd or fill_last)
        if _CHEB3:
            check(L.hf_cheb3_step(n, dv.ptr(cur), dv.ptr(oth), dv.ptr(b), None if zero else dv.ptr(ax), dv.ptr(inv_d),
                                  first, th, cd, cz, int(zero), int(prev_zero), mask if fill else None,
                                  dv.ptr(ax) if fill else None, _bits(x), int(chained and not zero), dv.stream()))
            cur, oth = oth, cur
            prev_zero = zero
            filled = fill
            return
        if chained and not zero:
            check(L.hf_cheb_step_after_apply(n, dv.ptr(x), dv.ptr(d), dv.ptr(b), dv.ptr(ax), dv.ptr(inv_d), first, th,
                                             cd, cz, mask if fill else None, dv.ptr(ax) if fill else None, _bits(x),
                                             dv.stream()))
            filled = fill
            return
        args = (n, dv.ptr(x), dv.ptr(d), dv.ptr(b), None if zero else dv.ptr(ax), dv.ptr(inv_d), first, th, cd, cz,
                int(zero), None)
        if x.dtype == torch.float32:
            check(L.hf_cheb_step_f32(*args, mask if fill else None, dv.ptr(ax) if fill else None, dv.stream()))
        elif fill:
            check(L.hf_cheb_step_fill(*args, mask, dv.ptr(ax), dv.stream()))
        else:
            check(L.hf_cheb_step(*args, dv.stream()))
        filled = fill

    for step in range(steps):
        zero = x_zero and step == 0
        if not zero:
            _apply_maybe_filled(apply_fn, cur, ax, filled)
        update(1, theta, 0.0, 0.0, zero)
        for cd, cz in coefs:
            _apply_maybe_filled(apply_fn, cur, ax, filled)
            update(0, 0.0, cd, cz, False)
    if cur is not x:  # an odd number of updates left the result in the second buffer
        x.copy_(cur)
    return filled


def chebyshev_apply(apply_fn, inv_diagonal, lam_max: float, b, x, settings: ChebyshevSettings = ChebyshevSettings(),
                    steps: int = 1):
    """Chebyshev semi-iteration targeting [lo, hi] lam_max of D^-1 A (multigrid.py:176-205)."""
    bd = dv.as_dev(b)
    xd = dv.as_dev(x).clone()
    invd = dv.as_dev(inv_diagonal)
    d = torch.empty_like(xd)
    ax = torch.empty_like(xd)
    _chebyshev_into(apply_fn, invd, lam_max, bd, xd, d, ax, settings, steps, False)
    return dv.like_input(xd, x)


def _coarse_kernel_enabled(problem: Problem) -> bool:
    """The one-kernel coarse solve needs the assembled level matrix (element
    matrices are instantiated for 3D Q1-Q2 and 2D Q1-Q4) and a small level.
    HF_COARSE=launches keeps the per-application graph launches."""
    import os

    if os.environ.get("HF_COARSE", "kernel") == "launches":
        return False
    n1 = problem.degree + 1
    ok = (problem.dim == 3 and n1 <= 3) or (problem.dim == 2 and n1 <= 5)
    return ok and problem.n_dofs <= 200_000


class _CoarseHandle:
    """Owns one hf_coarse handle."""

    def __init__(self, h):
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().hf_coarse_destroy(self._h)
        except Exception:
            pass


class _CoarseMatrix:
    """Assembled coarsest-level tangent for the one-kernel coarse solve.  The
    sparsity pattern (cell DoFs + constraint mask) is built once per problem
    and mask (hf_coarse_create_space, cached on the problem); each level
    operator clones it and refreshes the values on the device from the
    element matrices of a tensor4 tangent at the level's displacement
    (hf_coarse_update) -- the same matrix AssembledTangent forms."""

    def __init__(self, problem: Problem, u_level, op=None):
        key = problem.constraints.mask.tobytes()
        proto = getattr(problem, "_coarse_proto", None)
        if proto is None or proto[0] != key:
            h = ct.c_void_p()
            check(lib().hf_coarse_create_space(problem._space, dv.stream(), ct.byref(h)))
            proto = (key, _CoarseHandle(h))
            problem._coarse_proto = proto
        h = ct.c_void_p()
        check(lib().hf_coarse_clone(proto[1]._h, dv.stream(), ct.byref(h)))
        self._own = _CoarseHandle(h)
        self._h = h
        if op is None or op.strategy != "tensor4" or op.storage != "fp64":
            op = MatrixFreeTangent(problem, u_level, "tensor4")  # NonPositiveJacobian propagates
        check(lib().hf_coarse_update(h, op._op, dv.stream()))


class LevelOperator:
    """Tangent of one level plus its smoother data (multigrid.py:208-252)."""

    def __init__(self, problem: Problem, u_level, strategy: str, seed: int, level: int, is_coarsest: bool = False,
                 precision: str = "fp64"):
        """``precision="fp32"``: the diagonal and the Lanczos range come from the
        fp64 tangent; the smoother then runs on an fp32-storage tangent with fp32
        level vectors (half the bytes per application)."""
        self.level = level
        self.problem = problem
        self.precision = precision
        try:
            self.op = MatrixFreeTangent(problem, u_level, strategy)
        except NonPositiveJacobian as err:
            raise NonPositiveJacobian(f"level {level}: {err}", element=err.element, level=level) from err
        self.diag = self.op.diagonal_dev()
        self.inv_diag = torch.reciprocal(self.diag)
        mask = problem.mask_dev
        if is_coarsest:
            # the 30-iteration run the reference does first is the prefix of the
            # longer run (same RHS, same operations), so one run yields both
            al, be = lanczos_coefficients(self.op, self.diag, seed=seed, iterations=max(min(problem.n_dofs, 120), 30),
                                          constrained=mask)
            self.lam_min, self.lam_max = _ritz_extremes(al[:30], be[:29])
            lo, _ = _ritz_extremes(al[:min(problem.n_dofs, 120)], be[:min(problem.n_dofs, 120) - 1])
            self.lam_min = min(self.lam_min, lo)
        else:
            self.lam_min, self.lam_max = estimate_eigenvalue_range(self.op, self.diag, seed=seed, constrained=mask)
        dtype = torch.float64
        if precision == "fp32":
            self.op = MatrixFreeTangent(problem, u_level, strategy, storage="fp32")
            self.inv_diag = self.inv_diag.float()
            dtype = torch.float32
        elif precision != "fp64":
            raise ValueError(f"unknown precision {precision!r}")
        # smoother sweeps alternate direction: each starts on the cache tiles the
        # previous sweep read last.  Measured (tools/smoother_time.py): -3.5 % per
        # application at 32^3 (258 MB cache, 2x L2), +/-1 % at 64^3 (2.1 GB), so
        # only levels whose cache is within a few L2 capacities alternate.
        alt = os.environ.get("HF_ALTERNATE", "1") != "0" and self.op.storage_bytes() <= 512 * 2**20
        check(lib().hf_tangent_set_alternate(self.op._op, int(alt)))
        self._cap_warned = False
        self.coarse = None
        if is_coarsest and precision == "fp64" and _coarse_kernel_enabled(problem):
            try:
                self.coarse = _CoarseMatrix(problem, u_level, self.op)
            except HfError as err:  # level too large for the shared-memory blocks: per-application launches
                if err.code != HF_ERR_UNSUPPORTED:
                    raise
        n = problem.n_dofs
        # per-level V-cycle buffers
        self.b = torch.zeros(n, dtype=dtype, device="cuda")
        self.x = torch.zeros_like(self.b)
        self.d = torch.zeros_like(self.b)
        self.ax = torch.zeros_like(self.b)
        self.r = torch.zeros_like(self.b)
        self.scal = torch.zeros(4, dtype=torch.float64, device="cuda")
        self.flag = torch.zeros(1, dtype=torch.int32, device="cuda")

    def smooth(self, b, x, steps: int, settings: ChebyshevSettings):
        return chebyshev_apply(self.op, self.inv_diag, self.lam_max, b, x, settings, steps)

    def smooth_into(self, b, x, steps, settings, x_zero=False, fill_last=False):
        """Returns whether self.ax now holds mask ? x : 0 for the next apply."""
        return _chebyshev_into(self.op, self.inv_diag, self.lam_max, b, x, self.d, self.ax, settings, steps, x_zero,
                               mask=self.problem.mask_ptr(), fill_last=fill_last)

    def coarse_settings(self, settings: ChebyshevSettings) -> ChebyshevSettings:
        """Range widened to the estimated smallest eigenvalue (multigrid.py:248-252)."""
        lo = max(0.5 * self.lam_min / self.lam_max, 1e-8)
        return ChebyshevSettings(degree=settings.degree, range_lo=min(lo, settings.range_lo),
                                 range_hi=settings.range_hi)

    def cap_reached(self) -> bool:
        """Whether the last coarse solve hit the application cap (reads the device flag)."""
        return int(self.flag.item()) == 0


def _coarse_solve_into(level: LevelOperator, b, x, rel_target=1e-3, max_applications=100,
                       settings: ChebyshevSettings = ChebyshevSettings()):
    """Graph-capturable continuous Chebyshev coarse solve (multigrid.py:255-306).

    The ||r|| test every ``degree`` applications runs on the device and raises
    ``level.flag``; later kernels see the flag and do nothing, which returns
    the same iterate as the reference's early ``return``."""
    s = level.coarse_settings(settings)
    theta = 0.5 * (s.range_hi + s.range_lo) * level.lam_max
    delta = 0.5 * (s.range_hi - s.range_lo) * level.lam_max
    sigma = theta / delta
    n = b.numel()
    L = lib()
    if level.coarse is not None and x.dtype == torch.float64:
        # the whole iteration as one persistent kernel on the assembled level matrix
        check(L.hf_coarse_cheb_solve(level.coarse._h, dv.ptr(b), dv.ptr(x), dv.ptr(level.d), dv.ptr(level.inv_diag),
                                     theta, delta, sigma, rel_target, max_applications, s.degree,
                                     dv.ptr(level.scal), dv.ptr(level.flag), dv.stream()))
        return x
    ws = dv.Workspace.get().handle
    scal, flag, d, ax = level.scal, level.flag, level.d, level.ax
    f32 = x.dtype == torch.float32

    def cheb(args, fill):
        if f32:
            check(L.hf_cheb_step_f32(*args, mask if fill else None, dv.ptr(ax) if fill else None, dv.stream()))
        elif fill:
            check(L.hf_cheb_step_fill(*args, mask, dv.ptr(ax), dv.stream()))
        else:
            check(L.hf_cheb_step(*args, dv.stream()))

    # scal[0] = ||b||^2, scal[1] = rel_target * ||b||, flag = (||b|| == 0)
    if f32:
        check(L.hf_dot_f32(ws, n, dv.ptr(b), dv.ptr(b), dv.ptr(scal[0:1]), dv.stream()))
    else:
        dv.dot(b, b, scal[0:1])
    check(L.hf_scalar_op(1, dv.ptr(scal), 0, 1, rel_target, dv.ptr(flag), dv.stream()))
    # x = 0 + inv_d b / theta; ax = mask ? x : 0 for the first application
    mask = level.problem.mask_ptr()
    cheb((n, dv.ptr(x), dv.ptr(d), dv.ptr(b), None, dv.ptr(level.inv_diag), 1, theta, 0.0, 0.0, 1, None), True)
    rho_old = 1.0 / sigma
    for step in range(2, max_applications + 1):
        level.op.apply_after_fill(x, ax, flag)
        if step % s.degree == 0:
            rn = L.hf_resnorm_check_f32 if f32 else L.hf_resnorm_check
            check(rn(ws, n, dv.ptr(b), dv.ptr(ax), dv.ptr(scal), 2, 1, dv.ptr(flag), dv.stream()))
        rho = 1.0 / (2.0 * sigma - rho_old)
        args = (n, dv.ptr(x), dv.ptr(d), dv.ptr(b), dv.ptr(ax), dv.ptr(level.inv_diag), 0, 0.0, rho * rho_old,
                2.0 * rho / delta, 0, dv.ptr(flag))
        cheb(args, step < max_applications)  # the update also prepares the next application
        rho_old = rho
    return x


def coarse_solve(level: LevelOperator, b, rel_target: float = 1e-3, max_applications: int = 100,
                 settings: ChebyshevSettings = ChebyshevSettings()):
    """Chebyshev iteration as coarse solver (multigrid.py:255-306)."""
    bd = dv.as_dev(b)
    x = torch.empty_like(bd)
    _coarse_solve_into(level, bd, x, rel_target, max_applications, settings)
    if level.cap_reached() and not level._cap_warned:
        log.warning("coarse solve on level %d reached the application cap (%d); iterates remain usable "
                    "(message shown once per level)", level.level, max_applications)
        level._cap_warned = True
    return dv.like_input(x, b)


def _v_cycle_into(levels, transfers, b, x, lvl, steps, settings):
    if lvl == 0:
        return _coarse_solve_into(levels[0], b, x, settings=settings)
    L = levels[lvl]
    C = levels[lvl - 1]
    filled = L.smooth_into(b, x, steps, settings, x_zero=True, fill_last=True)
    _apply_maybe_filled(L.op, x, L.ax, filled)
    rm = lib().hf_resid_masked_f32 if b.dtype == torch.float32 else lib().hf_resid_masked
    check(rm(b.numel(), dv.ptr(L.r), dv.ptr(b), dv.ptr(L.ax), L.problem.mask_ptr(), dv.stream()))
    transfers[lvl - 1].restrict_into(L.r, C.b, mode=1)
    _v_cycle_into(levels, transfers, C.b, C.x, lvl - 1, steps, settings)
    transfers[lvl - 1].prolong_into(C.x, x, mode=2)
    L.smooth_into(b, x, steps, settings, x_zero=False)
    return x


def v_cycle(levels, transfers, b, lvl=None, smoothing_steps: int = 2,
            settings: ChebyshevSettings = ChebyshevSettings()):
    """One V-cycle (multigrid.py:309-332)."""
    if lvl is None:
        lvl = len(levels) - 1
    bd = dv.as_dev(b)
    x = torch.empty_like(bd)
    _v_cycle_into(levels, transfers, bd, x, lvl, smoothing_steps, settings)
    return dv.like_input(x, b)


class GMGPreconditioner:
    """V-cycle preconditioner (multigrid.py:335-351), replayed as one CUDA graph."""

    def __init__(self, levels, transfers, smoothing_steps: int = 2, settings: ChebyshevSettings = ChebyshevSettings(),
                 use_graph: bool = True):
        self.levels = levels
        self.transfers = transfers
        self.smoothing_steps = smoothing_steps
        self.settings = settings
        self.use_graph = use_graph
        self._graph = None
        fine = levels[-1]
        self._b = fine.b if len(levels) > 1 else torch.zeros_like(fine.b)
        self._x = fine.x if len(levels) > 1 else torch.zeros_like(fine.b)

    def _run(self):
        _v_cycle_into(self.levels, self.transfers, self._b, self._x, len(self.levels) - 1, self.smoothing_steps,
                      self.settings)

    def _record(self):
        """The V-cycle as one graph.  Recorded through libhf, where the executable
        graph of an earlier hierarchy of the same shape (levels, strategies,
        storage, smoothing) is updated in place; HF_GRAPH=torch records with
        torch.cuda.CUDAGraph instead (a new instantiation per hierarchy)."""
        if os.environ.get("HF_GRAPH", "native") == "torch":
            return dv.capture_graph(self._run)
        key = ("vcycle", torch.cuda.current_device(), self.smoothing_steps, self.settings.degree,
               tuple((lv.problem.n_dofs, lv.problem.degree, lv.op.strategy, str(lv.b.dtype)) for lv in self.levels))
        return dv.LaunchGraph(self._run, key)

    def apply_into(self, b: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        self._b.copy_(b)
        if not self.use_graph:
            self._run()
        else:
            if self._graph is None:
                self._run()  # eager warm-up, then record the identical launch sequence
                try:
                    self._graph = self._record()
                except RuntimeError as exc:  # e.g. a device allocation inside the recording
                    log.warning("V-cycle graph recording failed (%s); running the V-cycle eagerly", exc)
                    self.use_graph = False
                    self._b.copy_(b)
                    self._run()
                    out.copy_(self._x)
                    return out
                self._b.copy_(b)
            self._graph.replay()
        out.copy_(self._x)
        return out

    def apply(self, b):
        bd = dv.as_dev(b)
        out = torch.empty_like(bd)
        self.apply_into(bd, out)
        return dv.like_input(out, b)

    def __call__(self, b):
        return self.apply(b)


def build_transfers(problems):
    return [TransferOperator(problems[i], problems[i + 1]) for i in range(len(problems) - 1)]


def build_level_operators(problems, u_fine, strategy: str = "tensor4", seed: int = 0, keep_constrained: bool = False,
                          coarse_precision: str = "fp64"):
    """Linearise every level at the injected fine displacement (multigrid.py:358-369);
    ``coarse_precision="fp32"`` runs the levels between the finest and the
    coarsest in fp32 storage.  The coarsest stays fp64: it is latency bound
    (halving its bytes gains nothing) and runs the one-kernel coarse solve."""
    u_levels = restrict_solution(problems, dv.as_dev(u_fine), keep_constrained)
    top = len(problems) - 1
    return [LevelOperator(p, u, strategy, seed=seed + 7919 * lvl, level=lvl, is_coarsest=(lvl == 0),
                          precision=coarse_precision if 0 < lvl < top else "fp64")
            for lvl, (p, u) in enumerate(zip(problems, u_levels))]


def build_gmg(problems, u_fine, strategy: str = "tensor4", seed: int = 0, transfers=None,
              keep_constrained: bool = False, use_graph: bool = True,
              coarse_precision: str = "fp64") -> GMGPreconditioner:
    """(multigrid.py:372-382); ``coarse_precision="fp32"`` for the levels below the finest."""
    if transfers is None:
        transfers = build_transfers(problems)
    levels = build_level_operators(problems, u_fine, strategy, seed, keep_constrained, coarse_precision)
    return GMGPreconditioner(levels, transfers, use_graph=use_graph)
