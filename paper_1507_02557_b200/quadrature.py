"""Host-side quadrature on the bi-unit reference domains (setup only).

Restates the rules the reference discretization is defined by, so that
the device operators built from them reproduce the reference's discrete
operators:

* Gauss-Jacobi / Gauss-Legendre / Gauss-Lobatto 1-D rules by Golub-Welsch
  (reference: hybridwave/quadrature.py:67-130).
* The conical triangle rule GL(N+1) x GJ(1,0)(N+1) and its six-fold
  symmetrised version (quadrature.py:133-182).  The symmetrised rule stores
  every point twice; ``symmetric_triangle_rule``
  keeps the reference's stored layout for the oracle, and
  ``unique_triangle_rule`` merges the coincident pairs (weights summed).
* Volume rules hex / wedge / pyramid / tet (quadrature.py:185-235).
"""

from dataclasses import dataclass, field
from math import gamma

import numpy as np
from scipy.linalg import eigh_tridiagonal

__all__ = [
    "QuadratureRule", "gauss_jacobi_1d", "gauss_legendre_1d",
    "gauss_lobatto_1d", "triangle_rule", "symmetric_triangle_rule",
    "unique_triangle_rule", "element_rule", "TRI_SYMMETRIES",
    "tri_barycentric",
]


@dataclass(frozen=True)
class QuadratureRule:
    points: np.ndarray
    weights: np.ndarray
    exactness_degree: int
    domain: str
    collapsed: np.ndarray | None = field(default=None, compare=False)

    @property
    def n(self):
        return len(self.weights)


def gauss_jacobi_1d(alpha, beta, n):
    """n-point Gauss-Jacobi rule for (1-x)^alpha (1+x)^beta on [-1, 1].

    Golub-Welsch on the symmetric Jacobi matrix of the monic recurrence
    (same construction as hybridwave/quadrature.py:67-102)."""
    if alpha <= -1.0 or beta <= -1.0:
        raise ValueError("Jacobi exponents must exceed -1")
    if n < 1:
        raise ValueError("need at least one point")
    s = alpha + beta
    mu0 = 2.0 ** (s + 1.0) * gamma(alpha + 1.0) * gamma(beta + 1.0) / gamma(s + 2.0)
    k = np.arange(n, dtype=float)
    diag = np.empty(n)
    diag[0] = (beta - alpha) / (s + 2.0)
    if n > 1:
        kk = k[1:]
        diag[1:] = (beta * beta - alpha * alpha) / ((2 * kk + s) * (2 * kk + s + 2))
    if n == 1:
        return QuadratureRule(diag.copy(), np.array([mu0]), 1, "interval")
    kk = k[1:]
    off2 = (4.0 * kk * (kk + alpha) * (kk + beta) * (kk + s)
            / ((2 * kk + s) ** 2 * (2 * kk + s + 1) * (2 * kk + s - 1)))
    x, vec = eigh_tridiagonal(diag, np.sqrt(off2))
    return QuadratureRule(x, mu0 * vec[0, :] ** 2, 2 * n - 1, "interval")


def gauss_legendre_1d(n):
    return gauss_jacobi_1d(0.0, 0.0, n)


def gauss_lobatto_1d(n):
    """n-point Gauss-Lobatto-Legendre rule (endpoints included), weights
    2 / (n (n-1) P_{n-1}(x)^2) (hybridwave/quadrature.py:112-130)."""
    if n < 2:
        raise ValueError("Lobatto rules need n >= 2")
    x = np.empty(n)
    x[0], x[-1] = -1.0, 1.0
    if n > 2:
        x[1:-1] = gauss_jacobi_1d(1.0, 1.0, n - 2).points
    p_prev, p = np.ones_like(x), x.copy()
    for k in range(1, n - 1):
        p_prev, p = p, ((2 * k + 1) * x * p - k * p_prev) / (k + 1)
    return QuadratureRule(x, 2.0 / (n * (n - 1) * p * p), 2 * n - 3, "interval")


def triangle_rule(N):
    """Collapsed GL(N+1) x GJ(1,0)(N+1) rule on the bi-unit triangle."""
    ga = gauss_legendre_1d(N + 1)
    gb = gauss_jacobi_1d(1.0, 0.0, N + 1)
    a = np.repeat(ga.points, N + 1)
    b = np.tile(gb.points, N + 1)
    r = 0.5 * (1.0 + a) * (1.0 - b) - 1.0
    w = np.outer(ga.weights, 0.5 * gb.weights).ravel()
    return QuadratureRule(np.column_stack([r, b]), w, 2 * N + 1, "triangle",
                          collapsed=np.column_stack([a, b]))


_TRI_CORNERS = np.array([[-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0]])
# the six vertex relabelings of the triangle, in the reference's order
# (hybridwave/quadrature.py:157, mesh.py:40)
TRI_SYMMETRIES = [(0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2)]


def tri_barycentric(p):
    p = np.atleast_2d(p)
    return np.column_stack([-(p[:, 0] + p[:, 1]) / 2.0, (1.0 + p[:, 0]) / 2.0,
                            (1.0 + p[:, 1]) / 2.0])


def symmetric_triangle_rule(N):
    """Reference layout: the conical rule averaged over the six relabelings,
    all 6 (N+1)^2 points stored (hybridwave/quadrature.py:165-182)."""
    base = triangle_rule(N)
    lam = tri_barycentric(base.points)
    pts = np.vstack([lam[:, list(s)] @ _TRI_CORNERS for s in TRI_SYMMETRIES])
    wts = np.concatenate([base.weights / 6.0] * 6)
    return QuadratureRule(pts, wts, 2 * N + 1, "triangle")


def unique_triangle_rule(N, tol=1e-12):
    """The symmetric rule with coincident stored points merged (weights
    summed).  Returns (rule, owner) where owner[i] is the unique index of
    stored point i."""
    full = symmetric_triangle_rule(N)
    key = np.round(full.points / tol).astype(np.int64)
    _, first, owner = np.unique(key, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first)            # keep first-appearance order
    remap = np.empty_like(order)
    remap[order] = np.arange(len(order))
    owner = remap[owner.ravel()]
    pts = full.points[np.sort(first)]
    w = np.zeros(len(pts))
    np.add.at(w, owner, full.weights)
    return QuadratureRule(pts, w, 2 * N + 1, "triangle"), owner


def _duffy(elem_type, abc):
    a, b, c = abc[:, 0], abc[:, 1], abc[:, 2]
    if elem_type == "tet":
        return np.column_stack([(1 + a) * (1 - b) * (1 - c) / 4.0 - 1.0,
                                (1 + b) * (1 - c) / 2.0 - 1.0, c])
    if elem_type == "pyramid":
        return np.column_stack([(1 + a) * (1 - c) / 2.0 - 1.0,
                                (1 + b) * (1 - c) / 2.0 - 1.0, c])
    raise ValueError(elem_type)


def element_rule(elem_type, N):
    """Volume rules of hybridwave/quadrature.py:185-235 (same point order:
    first collapsed coordinate slowest)."""
    if elem_type == "hex":
        g = gauss_legendre_1d(N + 1)
        a, b, c = np.meshgrid(g.points, g.points, g.points, indexing="ij")
        abc = np.column_stack([a.ravel(), b.ravel(), c.ravel()])
        w = np.einsum("i,j,k->ijk", g.weights, g.weights, g.weights).ravel()
        return QuadratureRule(abc, w, 2 * N + 1, "hex", collapsed=abc)
    if elem_type == "wedge":
        tri = triangle_rule(N)
        gs = gauss_legendre_1d(N + 1)
        nt, ns = tri.n, gs.n
        r = np.repeat(tri.points[:, 0], ns)
        t = np.repeat(tri.points[:, 1], ns)
        s = np.tile(gs.points, nt)
        w = np.outer(tri.weights, gs.weights).ravel()
        a = np.repeat(tri.collapsed[:, 0], ns)
        c = np.repeat(tri.collapsed[:, 1], ns)
        return QuadratureRule(np.column_stack([r, s, t]), w, 2 * N + 1, "wedge",
                              collapsed=np.column_stack([a, s, c]))
    if elem_type == "pyramid":
        g = gauss_legendre_1d(N + 1)
        gc = gauss_jacobi_1d(2.0, 0.0, N + 1)
        a, b, c = np.meshgrid(g.points, g.points, gc.points, indexing="ij")
        abc = np.column_stack([a.ravel(), b.ravel(), c.ravel()])
        w = np.einsum("i,j,k->ijk", g.weights, g.weights, gc.weights / 4.0).ravel()
        return QuadratureRule(_duffy("pyramid", abc), w, 2 * N + 1, "pyramid",
                              collapsed=abc)
    if elem_type == "tet":
        ga = gauss_legendre_1d(N + 1)
        gb = gauss_jacobi_1d(1.0, 0.0, N + 1)
        gc = gauss_jacobi_1d(2.0, 0.0, N + 1)
        a, b, c = np.meshgrid(ga.points, gb.points, gc.points, indexing="ij")
        abc = np.column_stack([a.ravel(), b.ravel(), c.ravel()])
        w = np.einsum("i,j,k->ijk", ga.weights, gb.weights / 2.0,
                      gc.weights / 4.0).ravel()
        return QuadratureRule(_duffy("tet", abc), w, 2 * N + 1, "tet",
                              collapsed=abc)
    raise ValueError(f"unknown element type {elem_type!r}")
