"""Host-side element bases (setup only).

The state coefficients exchanged through the drop-in API are coefficients
in the reference's bases, so the bases here must be the same functions:

* hex: tensor Lagrange on GL (GL formulation) or GLL (SEM) nodes, node
  order t-fastest (hybridwave/basis.py:135-165);
* tet: nodal on the Hesthaven-Warburton warp-and-blend nodes, equidistant
  ordering r-fastest (basis.py:237-337);
* wedge: orthonormal triangle(r,t) x Legendre(s) modes, triangle-mode
  major (basis.py:344-407);
* pyramid: the semi-nodal rational basis, level k outer, Lagrange at the
  (k+1)-point GL nodes in (a, b), weighted Jacobi in c (basis.py:423-492).

Only values needed to build the device operators are produced here; the
construction follows the published formulas (Hesthaven & Warburton 2008,
Chan & Warburton 2015), written independently of the reference code.
"""

from dataclasses import dataclass
from math import gamma, sqrt

import numpy as np

from .quadrature import gauss_legendre_1d, gauss_lobatto_1d

__all__ = [
    "Vandermonde", "basis_dimension", "jacobi_p", "grad_jacobi_p",
    "lagrange_matrices_1d", "hex_nodes_1d", "hex_nodal_eval",
    "tet_orthobasis_eval", "tet_nodal_points", "wedge_tri_mode_ids",
    "wedge_mode_ids", "wedge_tri_basis_eval", "wedge_orthobasis_eval",
    "pyramid_mode_ids", "pyramid_level_rules", "pyramid_seminodal_eval",
]


@dataclass
class Vandermonde:
    V: np.ndarray
    Vr: np.ndarray
    Vs: np.ndarray
    Vt: np.ndarray


def basis_dimension(elem_type, N):
    return {"hex": (N + 1) ** 3,
            "tet": (N + 1) * (N + 2) * (N + 3) // 6,
            "wedge": (N + 1) ** 2 * (N + 2) // 2,
            "pyramid": (N + 1) * (N + 2) * (2 * N + 3) // 6}[elem_type]


def jacobi_p(x, alpha, beta, n):
    """Jacobi polynomial of degree n normalised to unit L2 norm against
    (1-x)^alpha (1+x)^beta (three-term recurrence of the normalised
    family)."""
    x = np.asarray(x, dtype=float)
    s = alpha + beta
    h0 = 2.0 ** (s + 1) / (s + 1.0) * gamma(alpha + 1) * gamma(beta + 1) / gamma(s + 1)
    pm = np.full_like(x, 1.0 / sqrt(h0))
    if n == 0:
        return pm
    h1 = (alpha + 1.0) * (beta + 1.0) / (s + 3.0) * h0
    p = ((s + 2.0) * x / 2.0 + (alpha - beta) / 2.0) / sqrt(h1)
    a_prev = 2.0 / (2.0 + s) * sqrt((alpha + 1.0) * (beta + 1.0) / (s + 3.0))
    for i in range(1, n):
        h = 2.0 * i + s
        a_next = 2.0 / (h + 2.0) * sqrt((i + 1.0) * (i + 1.0 + s) * (i + 1.0 + alpha)
                                        * (i + 1.0 + beta) / (h + 1.0) / (h + 3.0))
        b_next = -(alpha * alpha - beta * beta) / (h * (h + 2.0))
        pm, p = p, ((x - b_next) * p - a_prev * pm) / a_next
        a_prev = a_next
    return p


def grad_jacobi_p(x, alpha, beta, n):
    x = np.asarray(x, dtype=float)
    if n == 0:
        return np.zeros_like(x)
    return sqrt(n * (n + alpha + beta + 1.0)) * jacobi_p(x, alpha + 1, beta + 1, n - 1)


def _legendre_vdm(x, N, deriv=False):
    f = grad_jacobi_p if deriv else jacobi_p
    return np.column_stack([f(x, 0.0, 0.0, j) for j in range(N + 1)])


def lagrange_matrices_1d(nodes, x):
    """Lagrange basis on `nodes` evaluated at `x`: (values, derivatives),
    shape (len(x), len(nodes)), through the Legendre Vandermonde."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    N = len(nodes) - 1
    inv = np.linalg.inv(_legendre_vdm(nodes, N))
    return _legendre_vdm(x, N) @ inv, _legendre_vdm(x, N, True) @ inv


# ---------------------------------------------------------------- hex

def hex_nodes_1d(N, flavor):
    if flavor == "GL":
        return gauss_legendre_1d(N + 1)
    if flavor == "SEM":
        return gauss_lobatto_1d(N + 1)
    raise ValueError(f"unknown hex flavor {flavor!r}")


def hex_nodal_eval(N, flavor, rst):
    """Tensor Lagrange Vandermonde; node (i, j, k) at flat (i(N+1)+j)(N+1)+k."""
    nodes = hex_nodes_1d(N, flavor).points
    Lr, dLr = lagrange_matrices_1d(nodes, rst[:, 0])
    Ls, dLs = lagrange_matrices_1d(nodes, rst[:, 1])
    Lt, dLt = lagrange_matrices_1d(nodes, rst[:, 2])
    n = N + 1

    def outer(A, B, C):
        return np.einsum("pi,pj,pk->pijk", A, B, C).reshape(len(rst), n ** 3)

    return Vandermonde(outer(Lr, Ls, Lt), outer(dLr, Ls, Lt),
                       outer(Lr, dLs, Lt), outer(Lr, Ls, dLt))


# ---------------------------------------------------------------- tet

def _half_pow(v, p):
    return np.ones_like(v) if p == 0 else (0.5 * (1.0 - v)) ** p


def tet_orthobasis_eval(N, abc):
    """Orthonormal Dubiner basis on the bi-unit tet at collapsed points;
    derivatives by the collapsed chain rule, written so that every term is
    polynomial (safe on the collapsed edges)."""
    abc = np.atleast_2d(np.asarray(abc, dtype=float))
    a, b, c = abc.T
    cols = {k: [] for k in "VRST"}
    for i in range(N + 1):
        fa, dfa = jacobi_p(a, 0, 0, i), grad_jacobi_p(a, 0, 0, i)
        for j in range(N + 1 - i):
            gb, dgb = jacobi_p(b, 2 * i + 1, 0, j), grad_jacobi_p(b, 2 * i + 1, 0, j)
            for k in range(N + 1 - i - j):
                hc = jacobi_p(c, 2 * (i + j) + 2, 0, k)
                dhc = grad_jacobi_p(c, 2 * (i + j) + 2, 0, k)
                sc = 2.0 ** (2 * i + j + 1.5)
                bi, cij = _half_pow(b, i), _half_pow(c, i + j)
                cols["V"].append(sc * fa * gb * bi * hc * cij)
                # d/dr: dfa * (2/(1-b)) * (2/(1-c)) * rest
                dr = dfa * gb * hc * (_half_pow(b, i - 1) if i > 0 else 1.0) \
                    * (_half_pow(c, i + j - 1) if i + j > 0 else 1.0)
                # b-derivative part of d/ds (times 2/(1-c))
                gpart = dgb * bi - (0.5 * i * gb * _half_pow(b, i - 1) if i > 0 else 0.0)
                gpart = gpart * (_half_pow(c, i + j - 1) if i + j > 0 else 1.0)
                gpart = fa * gpart * hc
                cpart = dhc * cij - (0.5 * (i + j) * hc * _half_pow(c, i + j - 1)
                                     if i + j > 0 else 0.0)
                cols["R"].append(sc * dr)
                cols["S"].append(sc * (0.5 * (1 + a) * dr + gpart))
                cols["T"].append(sc * (0.5 * (1 + a) * dr + 0.5 * (1 + b) * gpart
                                       + fa * gb * bi * cpart))
    st = {k: np.column_stack(v) for k, v in cols.items()}
    return Vandermonde(st["V"], st["R"], st["S"], st["T"])


# Warp-and-blend optimised blending parameters (Hesthaven & Warburton,
# "Nodal Discontinuous Galerkin Methods", Nodes3D table), indexed by N.
_ALPHA_OPT_3D = [0.0, 0.0, 0.0, 0.0, 0.1002, 1.1332, 1.5608, 1.3413, 1.2577, 1.1603]


def _warp_deflated(N, x_gll_desc, r):
    """1-D warp (GLL - equidistant) interpolated and divided by (1 - r^2),
    with the division carried out analytically on the Lagrange factors."""
    xe = np.array([-1.0 + 2.0 * (N - i) / N for i in range(N + 1)])
    out = np.zeros_like(r)
    for i in range(1, N):          # endpoint terms vanish (GLL = equidistant there)
        term = np.full_like(r, x_gll_desc[i] - xe[i])
        for j in range(1, N):
            if j != i:
                term = term * (r - xe[j]) / (xe[i] - xe[j])
        out = out + term / (-(xe[i] - xe[0]) * (xe[i] - xe[N]))
    return out


def _face_shift(N, alpha, L1, L2, L3):
    xg = -gauss_lobatto_1d(N + 1).points
    w1 = L2 * L3 * 4.0 * _warp_deflated(N, xg, L3 - L2) * (1 + (alpha * L1) ** 2)
    w2 = L1 * L3 * 4.0 * _warp_deflated(N, xg, L1 - L3) * (1 + (alpha * L2) ** 2)
    w3 = L1 * L2 * 4.0 * _warp_deflated(N, xg, L2 - L1) * (1 + (alpha * L3) ** 2)
    c2, s2 = np.cos(2 * np.pi / 3), np.sin(2 * np.pi / 3)
    c4, s4 = np.cos(4 * np.pi / 3), np.sin(4 * np.pi / 3)
    return w1 + c2 * w2 + c4 * w3, s2 * w2 + s4 * w3


def tet_nodal_points(N, tol=1e-10):
    """Warp-and-blend nodes on the bi-unit tet (Hesthaven-Warburton
    Nodes3D), in the equidistant order t outer, s middle, r inner."""
    if N < 1:
        raise ValueError("nodal sets need N >= 1")
    alpha = _ALPHA_OPT_3D[N] if N < len(_ALPHA_OPT_3D) else 1.0
    rst = np.array([(-1.0 + 2.0 * q / N, -1.0 + 2.0 * m / N, -1.0 + 2.0 * n / N)
                    for n in range(N + 1) for m in range(N + 1 - n)
                    for q in range(N + 1 - n - m)])
    r, s, t = rst.T
    L1, L2, L3, L4 = (1 + t) / 2, (1 + s) / 2, -(1 + r + s + t) / 2, (1 + r) / 2
    v1 = np.array([-1.0, -1 / np.sqrt(3.0), -1 / np.sqrt(6.0)])
    v2 = np.array([1.0, -1 / np.sqrt(3.0), -1 / np.sqrt(6.0)])
    v3 = np.array([0.0, 2 / np.sqrt(3.0), -1 / np.sqrt(6.0)])
    v4 = np.array([0.0, 0.0, 3 / np.sqrt(6.0)])
    X = np.outer(L3, v1) + np.outer(L4, v2) + np.outer(L2, v3) + np.outer(L1, v4)
    t1 = np.array([v2 - v1, v2 - v1, v3 - v2, v3 - v1])
    t2 = np.array([v3 - (v1 + v2) / 2, v4 - (v1 + v2) / 2, v4 - (v2 + v3) / 2,
                   v4 - (v1 + v3) / 2])
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 /= np.linalg.norm(t2, axis=1, keepdims=True)
    shift = np.zeros_like(X)
    for f, (La, Lb, Lc, Ld) in enumerate([(L1, L2, L3, L4), (L2, L1, L3, L4),
                                          (L3, L1, L4, L2), (L4, L1, L3, L2)]):
        wx, wy = _face_shift(N, alpha, Lb, Lc, Ld)
        blend = Lb * Lc * Ld
        den = (Lb + 0.5 * La) * (Lc + 0.5 * La) * (Ld + 0.5 * La)
        ok = den > tol
        blend = np.where(ok, (1 + (alpha * La) ** 2) * blend / np.where(ok, den, 1.0), blend)
        shift += (blend * wx)[:, None] * t1[f] + (blend * wy)[:, None] * t2[f]
        edge = (La < tol) & ((Lb > tol).astype(int) + (Lc > tol) + (Ld > tol) < 3)
        shift[edge] = wx[edge, None] * t1[f] + wy[edge, None] * t2[f]
    X = X + shift
    ref = np.array([[-1.0, -1, -1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]])
    E = np.column_stack([v2 - v1, v3 - v1, v4 - v1])
    R = np.column_stack([ref[1] - ref[0], ref[2] - ref[0], ref[3] - ref[0]])
    return (X - v1) @ (R @ np.linalg.inv(E)).T + ref[0]


# ---------------------------------------------------------------- wedge

def wedge_tri_mode_ids(N):
    return [(i, k) for i in range(N + 1) for k in range(N + 1 - i)]


def wedge_mode_ids(N):
    return [(i, j, k) for (i, k) in wedge_tri_mode_ids(N) for j in range(N + 1)]


def wedge_tri_basis_eval(N, ac):
    """Orthonormal triangle basis in (r, t) at collapsed (a, c)."""
    ac = np.atleast_2d(np.asarray(ac, dtype=float))
    a, c = ac.T
    V, Vr, Vt = [], [], []
    for i, k in wedge_tri_mode_ids(N):
        fa, dfa = jacobi_p(a, 0, 0, i), grad_jacobi_p(a, 0, 0, i)
        hc, dhc = jacobi_p(c, 2 * i + 1, 0, k), grad_jacobi_p(c, 2 * i + 1, 0, k)
        sc = 2.0 ** (i + 0.5)
        V.append(sc * fa * _half_pow(c, i) * hc)
        dr = dfa * hc * (_half_pow(c, i - 1) if i > 0 else 1.0)
        cpart = dhc * _half_pow(c, i) - (0.5 * i * hc * _half_pow(c, i - 1) if i > 0 else 0.0)
        Vr.append(sc * dr)
        Vt.append(sc * (0.5 * (1 + a) * dr + fa * cpart))
    return np.column_stack(V), np.column_stack(Vr), np.column_stack(Vt)


def wedge_orthobasis_eval(N, abc):
    abc = np.atleast_2d(np.asarray(abc, dtype=float))
    T, Tr, Tt = wedge_tri_basis_eval(N, abc[:, [0, 2]])
    P = _legendre_vdm(abc[:, 1], N)
    dP = _legendre_vdm(abc[:, 1], N, True)
    ntri = T.shape[1]
    # mode order (tri mode major, Legendre minor)
    rep = lambda A: np.repeat(A, N + 1, axis=1)
    til = lambda B: np.tile(B, (1, ntri))
    return Vandermonde(rep(T) * til(P), rep(Tr) * til(P), rep(T) * til(dP),
                       rep(Tt) * til(P))


# ---------------------------------------------------------------- pyramid

def pyramid_mode_ids(N):
    return [(k, i, j) for k in range(N + 1) for i in range(k + 1) for j in range(k + 1)]


def pyramid_level_rules(N):
    return [gauss_legendre_1d(k + 1) for k in range(N + 1)]


def _pyramid_gammas(N):
    q = gauss_legendre_1d(N + 2)
    out = np.empty(N + 1)
    for k in range(N + 1):
        f = _half_pow(q.points, k) * jacobi_p(q.points, 2 * k + 3, 0, N - k)
        out[k] = 1.0 / sqrt(np.sum(q.weights * f * f * (0.5 * (1 - q.points)) ** 2))
    return out


def pyramid_seminodal_eval(N, abc):
    """Semi-nodal pyramid basis (values and rst-derivatives) at collapsed
    points.  Mode (k, i, j): w-normalised Lagrange_i(a) Lagrange_j(b) at the
    (k+1) GL points times C_k(c) = g_k ((1-c)/2)^k P_{N-k}^{(2k+3,0)}(c)."""
    abc = np.atleast_2d(np.asarray(abc, dtype=float))
    a, b, c = abc.T
    rules = pyramid_level_rules(N)
    gam = _pyramid_gammas(N)
    V, Vr, Vs, Vt = [], [], [], []
    for k in range(N + 1):
        La, dLa = lagrange_matrices_1d(rules[k].points, a)
        Lb, dLb = lagrange_matrices_1d(rules[k].points, b)
        pk = jacobi_p(c, 2 * k + 3, 0, N - k)
        dpk = grad_jacobi_p(c, 2 * k + 3, 0, N - k)
        Ck = gam[k] * _half_pow(c, k) * pk
        if k > 0:
            Ckm = gam[k] * _half_pow(c, k - 1) * pk
            dCk = gam[k] * _half_pow(c, k) * dpk - 0.5 * k * Ckm
        else:
            Ckm = None
            dCk = gam[k] * dpk
        w = rules[k].weights
        for i in range(k + 1):
            for j in range(k + 1):
                nrm = 1.0 / sqrt(w[i] * w[j])
                AB = La[:, i] * Lb[:, j]
                V.append(nrm * AB * Ck)
                if k > 0:
                    vr = nrm * dLa[:, i] * Lb[:, j] * Ckm
                    vs = nrm * La[:, i] * dLb[:, j] * Ckm
                else:
                    vr = np.zeros_like(a)
                    vs = np.zeros_like(a)
                Vr.append(vr)
                Vs.append(vs)
                Vt.append(0.5 * (1 + a) * vr + 0.5 * (1 + b) * vs + nrm * AB * dCk)
    return Vandermonde(*(np.column_stack(x) for x in (V, Vr, Vs, Vt)))
