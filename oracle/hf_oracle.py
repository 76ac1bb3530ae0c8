"""CPU ORACLE — test infrastructure only, never shipped or measured as the product.

A numpy restatement of the reference `hyperfree` package's hot path
(`/root/reference/pkg/src/hyperfree`, cited below as file:line).  It exists so
that the GPU product (``paper_1904_13131_b200``) can be checked on the GPU box,
where the reference itself is absent.  Only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it.

Parity of this restatement is PINNED against outputs of the unmodified
reference, generated in the build container by ``tests/golden/make_golden.py``
and committed as ``tests/golden/*.npz`` (checked by
``tests/test_oracle_golden.py``).

Generalisations over the reference (needed by the B200 build, all reducing to
the reference on its inputs):
* box lattices with a per-axis cell count (the reference only builds cubes);
  multi-GPU slab partitions are boxes;
* an arbitrary constraint mask per problem (the reference harness overrides
  ``Problem.constraints``);
* ``inject(..., keep_constrained=True)`` for prescribed non-zero Dirichlet
  values.

Layouts follow the reference: lexicographic numbering with x fastest
(mesh.py:1-13), node-blocked vector DoFs ``node*ncomp + comp`` (fespace.py:3-8),
element-local tensors (E, C, i_dim, ..., i_1) (fespace.py:180-184).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

# ----------------------------------------------------------------------------
# 1D tables  (fespace.py:33-102)
# ----------------------------------------------------------------------------


def gauss_legendre(q: int):
    """Gauss-Legendre rule mapped to [0, 1] (fespace.py:33-37)."""
    if not 1 <= q <= 16:
        raise ValueError("number of quadrature points must be in [1, 16]")
    t, w = np.polynomial.legendre.leggauss(q)
    return (t + 1.0) / 2.0, w / 2.0


def lagrange_tables(nodes: np.ndarray, pts: np.ndarray):
    """Values and first derivatives of the Lagrange polynomials through
    ``nodes`` at ``pts``, each shaped (n_nodes, n_pts) (fespace.py:40-62)."""
    n = len(nodes)
    pts = np.asarray(pts, dtype=float)
    val = np.empty((n, len(pts)))
    der = np.zeros((n, len(pts)))
    for i in range(n):
        others = [j for j in range(n) if j != i]
        denom = [nodes[i] - nodes[j] for j in others]
        val[i] = np.prod([(pts - nodes[j]) / d for j, d in zip(others, denom)], axis=0) if others else 1.0
        for k, dk in zip(others, denom):
            term = np.full(len(pts), 1.0 / dk)
            for j, dj in zip(others, denom):
                if j != k:
                    term = term * (pts - nodes[j]) / dj
            der[i] += term
    return val, der


def basis_nodes(degree: int, rule: str = "equispaced") -> np.ndarray:
    """Support points of the 1D Lagrange basis (fespace.py:80-102)."""
    if rule == "equispaced":
        return np.arange(degree + 1) / degree
    if rule == "gauss_lobatto":
        inner = np.sort(np.polynomial.legendre.Legendre.basis(degree).deriv().roots())
        return np.concatenate(([0.0], (inner + 1.0) / 2.0, [1.0]))
    raise ValueError(rule)


# ----------------------------------------------------------------------------
# lattices (mesh.py:30-54, fespace.py:125-151)
# ----------------------------------------------------------------------------


def lex_indices(counts) -> np.ndarray:
    """Multi-indices of a tensor grid, x fastest: (prod(counts), dim)."""
    grids = np.meshgrid(*[np.arange(c) for c in counts], indexing="ij")
    return np.stack([g.transpose(tuple(range(len(counts)))[::-1]).reshape(-1) for g in grids], axis=1)


def uniform_vertices(cells, side=1.0) -> np.ndarray:
    """Vertex coordinates of the structured grid on [0, side]^d (mesh.py:157-167)."""
    sides = side if isinstance(side, (tuple, list)) else (side,) * len(cells)
    axes = [np.linspace(0.0, s, c + 1) for s, c in zip(sides, cells)]
    idx = lex_indices([c + 1 for c in cells])
    return np.stack([axes[a][idx[:, a]] for a in range(len(cells))], axis=1)


@dataclass
class OProblem:
    """One level of the discretisation (operators.py:83-116) on a box lattice.

    ``cells`` is the per-axis cell count; ``vertices`` the (n_vertices, dim)
    coordinates in lexicographic order; ``mu_el``/``lam_el`` per-cell Lame
    data (operators.py:101-103); ``mask`` the constrained-DoF mask.
    """

    dim: int
    degree: int
    cells: tuple
    vertices: np.ndarray
    mu_el: np.ndarray
    lam_el: np.ndarray
    mask: np.ndarray
    nq1: int | None = None
    node_rule: str = "equispaced"
    _geo: tuple | None = field(default=None, repr=False)

    def __post_init__(self):
        self.cells = tuple(int(c) for c in self.cells)
        if self.nq1 is None:
            self.nq1 = self.degree + 1
        self.qpts, self.qw = gauss_legendre(self.nq1)
        self.nodes1d = basis_nodes(self.degree, self.node_rule)
        self.V, self.D = lagrange_tables(self.nodes1d, self.qpts)
        self.mu_el = np.asarray(self.mu_el, dtype=float).reshape(-1)
        self.lam_el = np.asarray(self.lam_el, dtype=float).reshape(-1)
        self.mask = np.asarray(self.mask, dtype=bool).reshape(-1)
        assert self.mask.shape == (self.n_dofs,)

    # --- counts
    @property
    def n1(self):
        return self.degree + 1

    @property
    def nodes_per_axis(self):
        return tuple(c * self.degree + 1 for c in self.cells)

    @property
    def n_nodes(self):
        return int(np.prod(self.nodes_per_axis))

    @property
    def n_dofs(self):
        return self.n_nodes * self.dim

    @property
    def n_el(self):
        return int(np.prod(self.cells))

    @property
    def nq(self):
        return self.nq1**self.dim

    @property
    def nloc(self):
        return self.n1**self.dim

    # --- DoF map (fespace.py:125-139)
    def cell_nodes(self) -> np.ndarray:
        p = self.degree
        npa = self.nodes_per_axis
        strides = np.cumprod((1,) + npa[:-1])
        e = lex_indices(self.cells)
        loc = lex_indices((self.n1,) * self.dim)
        return (e[:, None, :] * p + loc[None, :, :]) @ strides

    def corners(self) -> np.ndarray:
        """(n_el, 2^d, d) corner coordinates, corner bit c1 + 2 c2 + 4 c3 (mesh.py:133-139)."""
        vstrides = np.cumprod((1,) + tuple(c + 1 for c in self.cells[:-1]))
        e = lex_indices(self.cells)
        off = lex_indices((2,) * self.dim)
        vid = (e[:, None, :] + off[None, :, :]) @ vstrides
        return self.vertices[vid]

    # --- geometry cache (mesh.py:290-307)
    def geometry(self):
        if self._geo is None:
            d = self.dim
            pts = lex_indices((self.nq1,) * d)
            xi = self.qpts[pts]  # (nq, d)
            wq = np.prod(self.qw[pts], axis=1)
            off = lex_indices((2,) * d)
            # gradients of the multilinear corner functions at the q-points
            dn = np.ones((2**d, self.nq, d))
            for k in range(d):
                fac = np.where(off[:, k : k + 1] == 1, xi[None, :, k], 1.0 - xi[None, :, k])
                dfac = np.where(off[:, k : k + 1] == 1, 1.0, -1.0)
                for a in range(d):
                    dn[:, :, a] *= dfac if a == k else fac
            jac = np.einsum("eci,cqa->eqia", self.corners(), dn)
            det = np.linalg.det(jac)
            if np.any(det <= 0):
                raise ValueError("non-positive mapping Jacobian")
            self._geo = (np.linalg.inv(jac), det * wq[None, :])
        return self._geo


def face_mask(prob: OProblem, axis: int, side: int, comps=None) -> np.ndarray:
    """Constrained-DoF mask of every node on one lattice face (fespace.py:170-175
    generalised: ``axis``/``side`` pick the face, ``comps`` the components)."""
    idx = lex_indices(prob.nodes_per_axis)
    target = 0 if side == 0 else prob.nodes_per_axis[axis] - 1
    nodes = np.flatnonzero(idx[:, axis] == target)
    comps = range(prob.dim) if comps is None else comps
    m = np.zeros(prob.n_dofs, dtype=bool)
    for c in comps:
        m[nodes * prob.dim + c] = True
    return m


def node_coordinates(prob: OProblem) -> np.ndarray:
    """Physical coordinates of the lattice nodes (fespace.py:142-151)."""
    d = prob.dim
    loc = prob.nodes1d[lex_indices((prob.n1,) * d)]  # (nloc, d)
    off = lex_indices((2,) * d)
    q1 = np.ones((2**d, len(loc)))
    for k in range(d):
        q1 *= np.where(off[:, k : k + 1] == 1, loc[None, :, k], 1.0 - loc[None, :, k])
    per_el = np.einsum("eci,cn->eni", prob.corners(), q1)
    out = np.zeros((prob.n_nodes, d))
    out[prob.cell_nodes().reshape(-1)] = per_el.reshape(-1, d)
    return out


# ----------------------------------------------------------------------------
# sum factorisation (fespace.py:187-324)
# ----------------------------------------------------------------------------


def _along(t: np.ndarray, table: np.ndarray, axis_from_x: int) -> np.ndarray:
    """Contract the spatial axis ``axis_from_x`` (0 = x = last array axis)
    with ``table`` (n_in, n_out) (fespace.py:187-193)."""
    ax = t.ndim - 1 - axis_from_x
    return np.moveaxis(np.moveaxis(t, ax, -1) @ table, -1, ax)


def gather(prob: OProblem, u: np.ndarray, cn=None) -> np.ndarray:
    """(n_el, nloc, ncomp) element vectors (fespace.py:291-293)."""
    cn = prob.cell_nodes() if cn is None else cn
    return u.reshape(prob.n_nodes, prob.dim)[cn]


def unit_gradients(prob: OProblem, xloc: np.ndarray) -> np.ndarray:
    """Unit-cell gradients at the q-points (n_el, nq, ncomp, d)
    (fespace.py:230-239): direction g uses the derivative table on axis g."""
    d, n1 = prob.dim, prob.n1
    E, _, C = xloc.shape
    t0 = np.ascontiguousarray(xloc.transpose(0, 2, 1)).reshape((E, C) + (n1,) * d)
    out = np.empty((E, prob.nq, C, d))
    for g in range(d):
        t = t0
        for a in range(d):
            t = _along(t, prob.D if a == g else prob.V, a)
        out[..., g] = t.reshape(E, C, prob.nq).transpose(0, 2, 1)
    return out


def integrate_gradients(prob: OProblem, grads: np.ndarray, jxw: np.ndarray) -> np.ndarray:
    """Sum_q dN_i/dxi_a G_qa JxW_q -> (n_el, nloc, ncomp) (fespace.py:265-288)."""
    d, q1 = prob.dim, prob.nq1
    E, _, C, _ = grads.shape
    w = grads * jxw[:, :, None, None]
    out = 0.0
    for a in range(d):
        t = np.ascontiguousarray(w[..., a].transpose(0, 2, 1)).reshape((E, C) + (q1,) * d)
        for k in range(d):
            t = _along(t, (prob.D if k == a else prob.V).T, k)
        out = out + t
    return out.reshape(E, C, prob.nloc).transpose(0, 2, 1)


def scatter(prob: OProblem, local: np.ndarray, drop_mask=True, cn=None) -> np.ndarray:
    """Element-order accumulation, constrained rows dropped (fespace.py:296-324)."""
    cn = prob.cell_nodes() if cn is None else cn
    if drop_mask:
        keep = ~prob.mask.reshape(prob.n_nodes, prob.dim)
        local = local * keep[cn]
    out = np.zeros((prob.n_nodes, prob.dim))
    flat = cn.reshape(-1)
    for c in range(prob.dim):
        out[:, c] += np.bincount(flat, weights=local[:, :, c].reshape(-1), minlength=prob.n_nodes)
    return out.reshape(-1)


# ----------------------------------------------------------------------------
# material (material.py:121-230)
# ----------------------------------------------------------------------------

SYM = {2: ((0, 0), (1, 1), (0, 1)), 3: ((0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1))}


class NonPositiveJacobian(RuntimeError):
    """det F <= 0 (material.py:34-40)."""

    def __init__(self, msg, element=None, level=None):
        super().__init__(msg)
        self.element = element
        self.level = level


def voigt_tangent(J, mu, lam, dim):
    """Voigt matrix of J c = 2 c1 S + 2 lam I(x)I, engineering shear (material.py:195-208)."""
    c1 = mu - 2.0 * lam * np.log(J)
    nv = len(SYM[dim])
    m = np.zeros(J.shape + (nv, nv))
    m[..., :dim, :dim] = (2.0 * lam)[..., None, None] * np.ones((dim, dim))
    for a in range(dim):
        m[..., a, a] += 2.0 * c1
    for s in range(dim, nv):
        m[..., s, s] = c1
    return m


def pack_upper(m):
    """Upper triangle, row-major (material.py:218-222)."""
    iu = np.triu_indices(m.shape[-1])
    return m[..., iu[0], iu[1]]


def unpack_upper(v, nv):
    iu = np.triu_indices(nv)
    m = np.zeros(v.shape[:-1] + (nv, nv))
    m[..., iu[0], iu[1]] = v
    m[..., iu[1], iu[0]] = v
    return m


def sym_pack(t):
    return np.stack([t[..., i, j] for i, j in SYM[t.shape[-1]]], axis=-1)


def sym_unpack(v, dim):
    out = np.zeros(v.shape[:-1] + (dim, dim))
    for k, (i, j) in enumerate(SYM[dim]):
        out[..., i, j] = v[..., k]
        out[..., j, i] = v[..., k]
    return out


# ----------------------------------------------------------------------------
# deformation state, caches, apply (operators.py:170-417)
# ----------------------------------------------------------------------------

STRATEGIES = ("scalar", "tensor2", "tensor4")


def grad_u(prob: OProblem, u: np.ndarray) -> np.ndarray:
    """Referential displacement gradients (operators.py:170-176)."""
    jinv, _ = prob.geometry()
    return np.einsum("eqia,eqaA->eqiA", unit_gradients(prob, gather(prob, u)), jinv)


def deformation(prob: OProblem, u: np.ndarray):
    """F, J, F^-1, b; raises on det F <= 0 with the argmin element (operators.py:179-189)."""
    F = grad_u(prob, u) + np.eye(prob.dim)
    J = np.linalg.det(F)
    if np.any(J <= 0.0):
        e, q = np.unravel_index(int(np.argmin(J)), J.shape)
        raise NonPositiveJacobian(f"det F = {J[e, q]:.3e} <= 0 in element {e} (quadrature point {q})", element=int(e))
    return F, J, np.linalg.inv(F), F @ np.swapaxes(F, -1, -2)


def jacobian_range(prob: OProblem, u: np.ndarray):
    """(operators.py:192-196)"""
    J = np.linalg.det(grad_u(prob, u) + np.eye(prob.dim))
    return float(J.min()), float(J.max())


def kirchhoff(prob: OProblem, b, J):
    """tau = mu b - (mu - 2 lam ln J) I (material.py:121-124)."""
    mu = prob.mu_el[:, None, None, None]
    c1 = mu - 2.0 * prob.lam_el[:, None, None, None] * np.log(J)[..., None, None]
    return mu * b - c1 * np.eye(prob.dim)


def build_cache(prob: OProblem, ubar: np.ndarray, strategy: str) -> dict:
    """Per-q-point caches of the three strategies (operators.py:244-311)."""
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    F, J, Finv, b = deformation(prob, ubar)
    c1 = prob.mu_el[:, None] - 2.0 * prob.lam_el[:, None] * np.log(J)
    if strategy == "scalar":
        return {"strategy": strategy, "c1": c1, "ubar": ubar.copy()}
    jinv, _ = prob.geometry()
    s_inv = np.einsum("eqaA,eqAj->eqaj", jinv, Finv)
    tau = sym_pack(kirchhoff(prob, b, J))
    if strategy == "tensor2":
        return {"strategy": strategy, "c1": 2.0 * c1, "c2": np.broadcast_to(2.0 * prob.lam_el[:, None], c1.shape).copy(),
                "tau": tau, "s_inv": s_inv}
    M = voigt_tangent(J, prob.mu_el[:, None], prob.lam_el[:, None], prob.dim)
    return {"strategy": strategy, "tau": tau, "cmat": pack_upper(M), "s_inv": s_inv}


def local_apply(prob: OProblem, cache: dict, xloc: np.ndarray, cn=None) -> np.ndarray:
    """Cell-wise tangent action (operators.py:341-393)."""
    d = prob.dim
    jinv, jxw = prob.geometry()
    g_unit = unit_gradients(prob, xloc)
    st = cache["strategy"]
    if st == "scalar":
        gu = np.einsum("eqia,eqaA->eqiA", unit_gradients(prob, gather(prob, cache["ubar"], cn)), jinv)
        F = gu + np.eye(d)
        b = F @ np.swapaxes(F, -1, -2)
        tau = prob.mu_el[:, None, None, None] * b - cache["c1"][..., None, None] * np.eye(d)
        s_inv = np.einsum("eqaA,eqAj->eqaj", jinv, np.linalg.inv(F))
        a1, a2 = 2.0 * cache["c1"], np.broadcast_to(2.0 * prob.lam_el[:, None], cache["c1"].shape)
    else:
        s_inv = cache["s_inv"]
        tau = sym_unpack(cache["tau"], d)
        if st == "tensor2":
            a1, a2 = cache["c1"], cache["c2"]
    g = np.einsum("eqia,eqaj->eqij", g_unit, s_inv)
    gs = 0.5 * (g + np.swapaxes(g, -1, -2))
    if st == "tensor4":
        nv = len(SYM[d])
        gam = sym_pack(gs)
        gam[..., d:] *= 2.0
        sig = np.einsum("eqkl,eql->eqk", unpack_upper(cache["cmat"], nv), gam)
        cgs = sym_unpack(sig, d)
    else:
        tr = np.trace(gs, axis1=-2, axis2=-1)
        cgs = a1[..., None, None] * gs + (a2 * tr)[..., None, None] * np.eye(d)
    queued = np.einsum("eqij,eqaj->eqia", cgs + g @ tau, s_inv)
    return integrate_gradients(prob, queued, jxw)


class Tangent:
    """MatrixFreeTangent restated (operators.py:319-417)."""

    def __init__(self, prob: OProblem, ubar: np.ndarray, strategy: str = "tensor4"):
        self.prob = prob
        self.strategy = strategy
        self.cache = build_cache(prob, ubar, strategy)
        self._cn = prob.cell_nodes()

    @property
    def n_dofs(self):
        return self.prob.n_dofs

    def apply(self, x: np.ndarray) -> np.ndarray:
        """Zero-in / identity-out on the constrained subspace (operators.py:331-339)."""
        p = self.prob
        xe = np.where(p.mask, 0.0, x)
        y = scatter(p, local_apply(p, self.cache, gather(p, xe, self._cn), self._cn), cn=self._cn)
        y[p.mask] = x[p.mask]
        return y

    def apply_unconstrained_input(self, x: np.ndarray) -> np.ndarray:
        """Rows dropped but constrained inputs kept: K_{free,*} x (lifting helper)."""
        p = self.prob
        return scatter(p, local_apply(p, self.cache, gather(p, x, self._cn), self._cn), cn=self._cn)

    def diagonal(self) -> np.ndarray:
        """Local unit-vector applies, accumulated per node; constrained = 1 (operators.py:395-410)."""
        p = self.prob
        cn = self._cn
        out = np.zeros((p.n_nodes, p.dim))
        for n in range(p.nloc):
            for c in range(p.dim):
                xl = np.zeros((p.n_el, p.nloc, p.dim))
                xl[:, n, c] = 1.0
                yl = local_apply(p, self.cache, xl, cn)
                np.add.at(out[:, c], cn[:, n], yl[:, n, c])
        d = out.reshape(-1)
        d[p.mask] = 1.0
        return d

    def storage_bytes(self) -> int:
        """(operators.py:412-417)"""
        nqp = self.prob.n_el * self.prob.nq
        nv = len(SYM[self.prob.dim])
        d = self.prob.dim
        payload = {"scalar": 1, "tensor2": 2 + nv, "tensor4": nv + nv * (nv + 1) // 2}[self.strategy]
        return 8 * nqp * (payload + d * d + 1)


def surface_weights(prob: OProblem) -> np.ndarray:
    """s_n = int_top N_n dS on the face of maximal last coordinate (operators.py:129-167)."""
    d = prob.dim
    fd = d - 1
    top = np.flatnonzero(lex_indices(prob.cells)[:, d - 1] == prob.cells[d - 1] - 1)
    fpts = lex_indices((prob.nq1,) * fd)
    xi = prob.qpts[fpts]
    wq = np.prod(prob.qw[fpts], axis=1)
    off = lex_indices((2,) * d)
    fc = np.flatnonzero(off[:, d - 1] == 1)
    corners = prob.corners()[top][:, fc]  # (nf, 2^fd, d)
    foff = lex_indices((2,) * fd)
    dn = np.ones((2**fd, len(xi), fd))
    for k in range(fd):
        fac = np.where(foff[:, k : k + 1] == 1, xi[None, :, k], 1.0 - xi[None, :, k])
        dfac = np.where(foff[:, k : k + 1] == 1, 1.0, -1.0)
        for a in range(fd):
            dn[:, :, a] *= dfac if a == k else fac
    tang = np.einsum("fci,cqk->fqik", corners, dn)
    if d == 2:
        ds = np.linalg.norm(tang[..., 0], axis=-1)
    else:
        ds = np.linalg.norm(np.cross(tang[..., 0], tang[..., 1]), axis=-1)
    nidx = lex_indices((prob.n1,) * fd)
    nf = np.ones((prob.n1**fd, len(xi)))
    for k in range(fd):
        nf *= prob.V[nidx[:, k][:, None], fpts[:, k][None, :]]
    local = np.einsum("nq,fq->fn", nf, wq[None, :] * ds)
    grid = prob.cell_nodes()[top].reshape((-1,) + (prob.n1,) * d)
    fnodes = grid[:, -1].reshape(len(top), -1)
    out = np.zeros(prob.n_nodes)
    np.add.at(out, fnodes, local)
    return out


def residual(prob: OProblem, u: np.ndarray, traction=None) -> np.ndarray:
    """Internal Kirchhoff term minus top traction; constrained zeroed (operators.py:205-224)."""
    d = prob.dim
    _, J, Finv, b = deformation(prob, u)
    jinv, jxw = prob.geometry()
    tau = kirchhoff(prob, b, J)
    s_inv = np.einsum("eqaA,eqAj->eqaj", jinv, Finv)
    queued = np.einsum("eqij,eqaj->eqia", tau, s_inv)
    local = integrate_gradients(prob, queued, jxw)
    out = np.zeros((prob.n_nodes, d))
    np.add.at(out, prob.cell_nodes(), local)
    if traction is not None:
        out -= np.asarray(traction)[None, :] * surface_weights(prob)[:, None]
    out = out.reshape(-1)
    out[prob.mask] = 0.0
    return out


def energy(prob: OProblem, u: np.ndarray, traction=None) -> float:
    """Total potential energy (operators.py:227-236, material.py:98-106)."""
    F, J, _, _ = deformation(prob, u)
    _, jxw = prob.geometry()
    C = np.swapaxes(F, -1, -2) @ F
    lnj = np.log(J)
    psi = 0.5 * prob.mu_el[:, None] * (np.trace(C, axis1=-2, axis2=-1) - prob.dim - 2 * lnj) + prob.lam_el[:, None] * lnj**2
    tot = float(np.sum(psi * jxw))
    if traction is not None:
        tot -= float(np.asarray(traction) @ (surface_weights(prob) @ u.reshape(-1, prob.dim)))
    return tot


# ----------------------------------------------------------------------------
# FLOP meter (flops.py:28-47 as counted by operators.py:341-393 / fespace.py)
# ----------------------------------------------------------------------------


def meter_flops(dim: int, degree: int, n_el: int, strategy: str, nq1: int | None = None) -> int:
    """The reference's software FLOP count of ONE MatrixFreeTangent.apply."""
    n = degree + 1
    q = n if nq1 is None else nq1
    C = dim
    nq = q**dim
    nv = dim * (dim + 1) // 2

    def eval_grad():
        tot = 0
        for _g in range(dim):
            for k in range(dim):
                tot += 2 * n_el * C * q ** (k + 1) * n ** (dim - k - 1) * n
        return tot

    qp = n_el * nq
    f = eval_grad()
    if strategy == "scalar":
        f += eval_grad()
        f += 2 * qp * dim * dim * dim  # grad_u map
        f += 2 * qp * dim * dim * dim  # b
        f += 2 * qp * dim * dim  # tau
        f += 2 * qp * dim * dim * dim  # s_inv
    f += 2 * qp * dim * dim * dim  # g
    f += 2 * qp * dim * dim  # g_s
    if strategy == "tensor4":
        f += 2 * qp * nv * nv
    else:
        f += 4 * qp * dim * dim
    f += 2 * qp * dim * dim * dim  # g tau
    f += 2 * qp * dim * dim * dim + qp * dim * dim  # queued
    f += qp * C * dim  # fold weights
    for _a in range(dim):
        for k in range(dim):
            f += 2 * n_el * C * n ** (k + 1) * q ** (dim - k - 1) * q
    f += n_el * n**dim * C  # scatter
    return int(f)


# ----------------------------------------------------------------------------
# multigrid (multigrid.py:27-382)
# ----------------------------------------------------------------------------


def interpolation_1d(degree: int, m_coarse: int, nodes: np.ndarray) -> np.ndarray:
    """Coarse -> 2:1 refined nodal interpolation, (n_fine, n_coarse) (multigrid.py:58-73)."""
    p = degree
    nf, nc = 2 * m_coarse * p + 1, m_coarse * p + 1
    P = np.zeros((nf, nc))
    for f in range(nf):
        c = min(f // (2 * p), m_coarse - 1)
        xi = (f - 2 * p * c) / (2.0 * p)
        vals, _ = lagrange_tables(nodes, np.array([xi]))
        P[f, c * p : c * p + p + 1] = vals[:, 0]
    return P


class Transfer:
    """Tensor-product embedding; restriction is its transpose (multigrid.py:27-55)."""

    def __init__(self, coarse: OProblem, fine: OProblem):
        if any(f != 2 * c for f, c in zip(fine.cells, coarse.cells)):
            raise ValueError("transfer requires a 2:1 refined pair of levels")
        self.coarse, self.fine = coarse, fine
        self.mats = [interpolation_1d(coarse.degree, m, coarse.nodes1d) for m in coarse.cells]

    def prolong(self, xc):
        c = self.coarse
        t = xc.reshape(tuple(reversed(c.nodes_per_axis)) + (c.dim,))
        for a in range(c.dim):  # array axis dim-1-a holds spatial axis a
            t = np.moveaxis(np.tensordot(t, self.mats[a].T, axes=([c.dim - 1 - a], [0])), -1, c.dim - 1 - a)
        return t.reshape(-1)

    def restrict(self, rf):
        f = self.fine
        t = rf.reshape(tuple(reversed(f.nodes_per_axis)) + (f.dim,))
        for a in range(f.dim):
            t = np.moveaxis(np.tensordot(t, self.mats[a], axes=([f.dim - 1 - a], [0])), -1, f.dim - 1 - a)
        return t.reshape(-1)


def inject(problems, u_fine, keep_constrained=False):
    """Nodal injection onto every level (multigrid.py:76-92); constrained level
    DoFs are zeroed unless ``keep_constrained`` (prescribed values)."""
    out = [u_fine]
    for lvl in range(len(problems) - 1, 0, -1):
        fp, cp = problems[lvl], problems[lvl - 1]
        g = out[0].reshape(tuple(reversed(fp.nodes_per_axis)) + (fp.dim,))
        uc = g[(slice(None, None, 2),) * fp.dim].reshape(-1).copy()
        if not keep_constrained:
            uc[cp.mask] = 0.0
        out.insert(0, uc)
    return out


def eigen_range(apply_fn, diag, seed=0, iterations=30, constrained=None, rhs=None):
    """Ritz extremes of D^-1 A from a CG/Lanczos run (multigrid.py:112-166)."""
    n = len(diag)
    if rhs is None:
        rhs = np.random.default_rng(seed).standard_normal(n)
    b = rhs.copy()
    if constrained is not None:
        b[constrained] = 0.0
    inv_d = 1.0 / diag
    r = b.copy()
    z = inv_d * r
    p = z.copy()
    rz = r @ z
    al, be = [], []
    for _ in range(iterations):
        if rz <= 0.0 or not np.isfinite(rz):
            break
        ap = apply_fn(p)
        pap = p @ ap
        if pap <= 0.0:
            break
        a = rz / pap
        r = r - a * ap
        z = inv_d * r
        rzn = r @ z
        if rzn <= 1e-28 * rz or not np.isfinite(rzn):
            al.append(a)
            break
        bt = rzn / rz
        al.append(a)
        be.append(bt)
        p = z + bt * p
        rz = rzn
    if not al:
        return 1.0, 1.0
    k = len(al)
    dg = np.array([1.0 / al[0]] + [1.0 / al[i] + be[i - 1] / al[i - 1] for i in range(1, k)])
    if k == 1:
        return float(dg[0]), float(dg[0])
    off = np.array([math.sqrt(be[i]) / al[i] for i in range(k - 1)])
    ritz = scipy.linalg.eigvalsh_tridiagonal(dg, off)
    return float(ritz[0]), float(ritz[-1])


@dataclass(frozen=True)
class Cheb:
    degree: int = 4
    range_lo: float = 0.6
    range_hi: float = 1.2


def chebyshev(apply_fn, inv_d, lam_max, b, x, s: Cheb = Cheb(), steps=1):
    """Restarted Chebyshev semi-iteration (multigrid.py:176-205)."""
    theta = 0.5 * (s.range_hi + s.range_lo) * lam_max
    delta = 0.5 * (s.range_hi - s.range_lo) * lam_max
    sigma = theta / delta
    x = x.copy()
    for _ in range(steps):
        z = inv_d * (b - apply_fn(x))
        d = z / theta
        x += d
        rho_old = 1.0 / sigma
        for _ in range(s.degree - 1):
            z = inv_d * (b - apply_fn(x))
            rho = 1.0 / (2.0 * sigma - rho_old)
            d = (rho * rho_old) * d + (2.0 * rho / delta) * z
            x += d
            rho_old = rho
    return x


class Level:
    """LevelOperator restated (multigrid.py:208-252)."""

    def __init__(self, prob, u_level, strategy, seed, level, coarsest=False, rhs=None, rhs120=None):
        self.prob, self.level = prob, level
        try:
            self.op = Tangent(prob, u_level, strategy)
        except NonPositiveJacobian as err:
            raise NonPositiveJacobian(f"level {level}: {err}", element=err.element, level=level) from err
        self.diag = self.op.diagonal()
        self.inv_diag = 1.0 / self.diag
        self.lam_min, self.lam_max = eigen_range(self.op.apply, self.diag, seed, constrained=prob.mask, rhs=rhs)
        if coarsest:
            lo, _ = eigen_range(self.op.apply, self.diag, seed, iterations=min(prob.n_dofs, 120),
                                constrained=prob.mask, rhs=rhs)
            self.lam_min = min(self.lam_min, lo)
        self.cap_hits = 0

    def smooth(self, b, x, steps, s):
        return chebyshev(self.op.apply, self.inv_diag, self.lam_max, b, x, s, steps)

    def coarse_settings(self, s: Cheb) -> Cheb:
        lo = max(0.5 * self.lam_min / self.lam_max, 1e-8)
        return Cheb(s.degree, min(lo, s.range_lo), s.range_hi)


def coarse_solve(level: Level, b, rel_target=1e-3, max_applications=100, s: Cheb = Cheb()):
    """Continuous Chebyshev to a relative target, checked every ``degree`` applies (multigrid.py:255-306)."""
    bn = np.linalg.norm(b)
    x = np.zeros_like(b)
    if bn == 0.0:
        return x
    cs = level.coarse_settings(s)
    theta = 0.5 * (cs.range_hi + cs.range_lo) * level.lam_max
    delta = 0.5 * (cs.range_hi - cs.range_lo) * level.lam_max
    sigma = theta / delta
    d = (level.inv_diag * b) / theta
    x = x + d
    rho_old = 1.0 / sigma
    for step in range(2, max_applications + 1):
        r = b - level.op.apply(x)
        if step % cs.degree == 0 and np.linalg.norm(r) <= rel_target * bn:
            return x
        rho = 1.0 / (2.0 * sigma - rho_old)
        d = (rho * rho_old) * d + (2.0 * rho / delta) * (level.inv_diag * r)
        x += d
        rho_old = rho
    level.cap_hits += 1
    return x


def v_cycle(levels, transfers, b, lvl=None, steps=2, s: Cheb = Cheb()):
    """(multigrid.py:309-332)"""
    if lvl is None:
        lvl = len(levels) - 1
    if lvl == 0:
        return coarse_solve(levels[0], b, s=s)
    L = levels[lvl]
    x = L.smooth(b, np.zeros_like(b), steps, s)
    r = b - L.op.apply(x)
    r[L.prob.mask] = 0.0
    rc = transfers[lvl - 1].restrict(r)
    rc[levels[lvl - 1].prob.mask] = 0.0
    xc = v_cycle(levels, transfers, rc, lvl - 1, steps, s)
    corr = transfers[lvl - 1].prolong(xc)
    corr[L.prob.mask] = 0.0
    x += corr
    return L.smooth(b, x, steps, s)


class GMG:
    """build_gmg + GMGPreconditioner restated (multigrid.py:335-382)."""

    def __init__(self, problems, u_fine, strategy="tensor4", seed=0, transfers=None, keep_constrained=False):
        self.transfers = transfers or [Transfer(problems[i], problems[i + 1]) for i in range(len(problems) - 1)]
        ul = inject(problems, u_fine, keep_constrained)
        self.levels = [Level(p, u, strategy, seed + 7919 * l, l, l == 0) for l, (p, u) in enumerate(zip(problems, ul))]

    def apply(self, b):
        return v_cycle(self.levels, self.transfers, b)


# ----------------------------------------------------------------------------
# CG and Newton (solver.py:34-201)
# ----------------------------------------------------------------------------


class IndefiniteOperator(RuntimeError):
    pass


def cg(apply_fn, b, x0=None, rel_tol=1e-6, preconditioner=None, max_iterations=None):
    """PCG with recursive residual; returns (x, iterations, history) (solver.py:34-76)."""
    n = len(b)
    max_iterations = 10 * n if max_iterations is None else max_iterations
    x = np.zeros(n) if x0 is None else x0.copy()
    r = b - apply_fn(x) if np.any(x) else b.copy()
    bn = np.linalg.norm(b)
    hist = [np.linalg.norm(r)]
    if bn == 0.0 or hist[0] <= rel_tol * bn:
        return x, 0, hist
    z = preconditioner(r) if preconditioner else r.copy()
    p = z.copy()
    rz = r @ z
    it = 0
    while it < max_iterations:
        ap = apply_fn(p)
        pap = p @ ap
        if pap <= 0.0:
            raise IndefiniteOperator(f"p.Ap = {pap:.3e} <= 0 at iteration {it}")
        a = rz / pap
        x += a * p
        r -= a * ap
        it += 1
        hist.append(np.linalg.norm(r))
        if hist[-1] <= rel_tol * bn:
            return x, it, hist
        z = preconditioner(r) if preconditioner else r
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
    return x, it, hist


def newton_prescribed(problems, target, n_steps=5, strategy="tensor4", seed=0,
                      update_tol=1e-5, res_rel=1e-8, res_abs=1e-8, lin_tol=1e-6, max_it=30, log=None):
    """Incremental Newton with a prescribed displacement on constrained DoFs
    (SURVEY H5 restatement of solver.py:143-201).

    Each load step lifts the previous equilibrium smoothly: the prescribed
    increment ``dg`` is spread over the z component of every node in
    proportion to its height (so bottom stays 0, the top reaches the target
    exactly), then runs full Newton steps with the tangent + GMG rebuilt at
    the current state, CG from zero to ``lin_tol``, and the reference's
    convergence test.  Level displacements keep prescribed values.
    Returns (u, records) with records (step, it, ||R||, ||du||, cg_its).
    """
    fine = problems[-1]
    d = fine.dim
    X = node_coordinates(fine)
    height = X[:, d - 1] / X[:, d - 1].max()
    u = np.zeros(fine.n_dofs)
    recs = []
    transfers = [Transfer(problems[i], problems[i + 1]) for i in range(len(problems) - 1)]
    for step in range(1, n_steps + 1):
        dg = target / n_steps
        u = u.copy()
        u.reshape(-1, d)[:, d - 1] += dg * height
        R = residual(fine, u)
        r0 = np.linalg.norm(R)
        rt = max(res_rel * r0, res_abs)
        for it in range(1, max_it + 1):
            op = Tangent(fine, u, strategy)
            gmg = GMG(problems, u, strategy, seed, transfers, keep_constrained=True)
            du, its, _ = cg(op.apply, -R, rel_tol=lin_tol, preconditioner=gmg.apply)
            u = u + du
            R = residual(fine, u)
            rn, dn = float(np.linalg.norm(R)), float(np.linalg.norm(du))
            recs.append((step, it, rn, dn, its))
            if log:
                log(recs[-1])
            if dn <= update_tol and rn <= rt:
                break
        else:
            raise RuntimeError("Newton did not converge")
    return u, recs
