"""Per-element-type operator bundles (host setup, run once per (type, N,
formulation)).

Two products:

``build_operators`` restates the reference's constant operators
(hybridwave/operators.py:37-305): the fields the RHS consumes, in the
reference's layouts (face points stored as the reference stores them).  The
test oracle consumes these; ``tests/test_setup_golden.py`` pins them against
fixtures generated from the reference itself.

``device_operators`` derives the compact operators the sm_100a kernels read:

* quad faces keep the reference's (N+1)^2 GL/GLL points;
* triangle faces are represented by the (N+1)(N+2)/2 tet face nodes.  On
  affine elements every trace on a planar triangle face is a degree-N
  polynomial (tet, wedge and pyramid alike) and the flux is linear in the
  traces with per-face constant coefficients, so evaluating the flux at the
  face nodes and integrating against the reference's symmetric rule through
  the nodal interpolant (the ``LIFT`` matrices below) reproduces the
  reference's 6(N+1)^2-point surface integral up to rounding;
* the mass inverses that cancel against the reference's volume weights
  ("algebraic cancellations") are folded out.
"""

import numpy as np

from . import basis as bas
from .quadrature import (element_rule, gauss_legendre_1d, gauss_lobatto_1d,
                         symmetric_triangle_rule)
from .refelem import FACES, face_quadrature_points, inverse_duffy_map

__all__ = ["ElementOperators", "face_rule_2d", "build_operators",
           "tri_face_nodes_2d", "quad_face_points_2d", "device_operators",
           "face_symmetry_perms", "TYPE_ID"]

TYPE_ID = {"hex": 0, "wedge": 1, "pyramid": 2, "tet": 3}


def face_rule_2d(face_type, N, formulation):
    """Reference face cubature (hybridwave/operators.py:37-51)."""
    if face_type == "tri":
        r = symmetric_triangle_rule(N)
        return r.points, r.weights
    g = gauss_legendre_1d(N + 1) if formulation == "GL" else gauss_lobatto_1d(N + 1)
    xi, eta = np.meshgrid(g.points, g.points, indexing="ij")
    return np.column_stack([xi.ravel(), eta.ravel()]), np.outer(g.weights, g.weights).ravel()


class ElementOperators:
    def __init__(self, elem_type, N, formulation, **fields):
        self.elem_type = elem_type
        self.N = N
        self.formulation = formulation
        self.Np = bas.basis_dimension(elem_type, N)
        self.__dict__.update(fields)


def _basis_at(elem_type, N, formulation, rst, extra=None):
    """Basis values (npts, Np) at reference points, in the state basis."""
    if elem_type == "hex":
        return bas.hex_nodal_eval(N, "GL" if formulation == "GL" else "SEM", rst).V
    abc = inverse_duffy_map(elem_type, rst)
    if elem_type == "tet":
        return bas.tet_orthobasis_eval(N, abc).V @ extra
    if elem_type == "wedge":
        return bas.wedge_orthobasis_eval(N, abc).V
    if elem_type == "pyramid":
        return bas.pyramid_seminodal_eval(N, abc).V
    raise ValueError(elem_type)


def _face_data(elem_type, N, formulation, evalf):
    mats, offs, p2s, ws, rsts = [], [0], [], [], []
    for f, (ftype, _) in enumerate(FACES[elem_type]):
        p2, w2 = face_rule_2d(ftype, N, formulation)
        rst = face_quadrature_points(elem_type, f, p2)
        mats.append(evalf(rst))
        offs.append(offs[-1] + len(w2))
        p2s.append(p2)
        ws.append(w2)
        rsts.append(rst)
    return dict(Vf=np.vstack(mats), face_offsets=np.array(offs), face_pts2d=p2s,
                face_wts=ws, face_rst=np.vstack(rsts))


def build_operators(elem_type, N, formulation):
    """Reference-equivalent operator bundle (operators.py:86-305)."""
    if N < 1:
        raise ValueError(f"{elem_type} operators need N >= 1")
    if formulation not in ("GL", "SEM"):
        raise ValueError(f"formulation must be 'SEM' or 'GL', got {formulation!r}")
    if elem_type == "hex":
        flavor = "GL" if formulation == "GL" else "SEM"
        rule = bas.hex_nodes_1d(N, flavor)
        _, D1 = bas.lagrange_matrices_1d(rule.points, rule.points)
        end, _ = bas.lagrange_matrices_1d(rule.points, np.array([-1.0, 1.0]))
        fd = _face_data("hex", N, formulation,
                        lambda rst: _basis_at("hex", N, formulation, rst))
        return ElementOperators("hex", N, formulation, nodes1d=rule.points,
                                weights1d=rule.weights, D1=D1, Vf_end=end, **fd)
    if elem_type == "tet":
        nodes = bas.tet_nodal_points(N)
        vd = bas.tet_orthobasis_eval(N, inverse_duffy_map("tet", nodes))
        Vinv = np.linalg.inv(vd.V)
        fd = _face_data("tet", N, formulation,
                        lambda rst: _basis_at("tet", N, formulation, rst, Vinv))
        return ElementOperators(
            "tet", N, formulation, nodes=nodes, V=vd.V, Vinv=Vinv,
            Dr=vd.Vr @ Vinv, Ds=vd.Vs @ Vinv, Dt=vd.Vt @ Vinv,
            invM_ref=vd.V @ vd.V.T, M_ref=Vinv.T @ Vinv,
            cub=element_rule("tet", N), **fd)
    if elem_type == "wedge":
        cub = element_rule("wedge", N)
        vd = bas.wedge_orthobasis_eval(N, cub.collapsed)
        fd = _face_data("wedge", N, formulation,
                        lambda rst: _basis_at("wedge", N, formulation, rst))
        return ElementOperators("wedge", N, formulation, cub=cub, V=vd.V,
                                Dr3=vd.Vr, Ds3=vd.Vs, Dt3=vd.Vt, **fd)
    if elem_type == "pyramid":
        # quadrature-free weak derivatives: (D_c)[m, n] = int phi_m d(phi_n)/dc
        # over the reference pyramid, exact with the degree-(2N+7) rule
        # (the reference assembles the same integrals from cross-level
        # Lagrange evaluations, operators.py:216-277)
        big = element_rule("pyramid", N + 3)
        vd = bas.pyramid_seminodal_eval(N, big.collapsed)
        Wv = vd.V * big.weights[:, None]
        ids = bas.pyramid_mode_ids(N)
        rules = bas.pyramid_level_rules(N)
        level_abc = np.array([[rules[k].points[i], rules[k].points[j], 0.0]
                              for (k, i, j) in ids])
        fd = _face_data("pyramid", N, formulation,
                        lambda rst: _basis_at("pyramid", N, formulation, rst))
        return ElementOperators("pyramid", N, formulation, Dr=Wv.T @ vd.Vr,
                                Ds=Wv.T @ vd.Vs, Dt=Wv.T @ vd.Vt, level_abc=level_abc,
                                mode_ids=ids, cub=element_rule("pyramid", N), **fd)
    raise ValueError(f"unknown element type {elem_type!r}")


# ---------------------------------------------------------------- device side

def tri_face_nodes_2d(N):
    """The tet's face-node set as 2-D points of the bi-unit face triangle.

    Tet face 0 = vertices (0, 2, 1): face coordinate xi runs along s and eta
    along r, so a node (r, s, -1) sits at (xi, eta) = (s, r).  The set is
    invariant under the six triangle relabelings (checked in tests)."""
    nodes = bas.tet_nodal_points(N)
    on = np.abs(nodes[:, 2] + 1.0) < 1e-10
    return np.column_stack([nodes[on, 1], nodes[on, 0]])


def quad_face_points_2d(N, formulation):
    return face_rule_2d("quad", N, formulation)[0]


def _tri_lagrange(nodes2d, pts2d, N):
    """2-D Lagrange basis of `nodes2d` (P^N) evaluated at `pts2d`."""
    def coll(p):
        xi, eta = p.T
        den = 1.0 - eta
        a = np.where(np.abs(den) > 1e-13, 2 * (1 + xi) / np.where(den == 0, 1, den) - 1, -1.0)
        return np.column_stack([a, eta])
    Vn, _, _ = bas.wedge_tri_basis_eval(N, coll(nodes2d))
    Vp, _, _ = bas.wedge_tri_basis_eval(N, coll(pts2d))
    return Vp @ np.linalg.inv(Vn)


_QUAD_CORNERS = np.array([[-1.0, -1.0], [1.0, -1.0], [1.0, 1.0], [-1.0, 1.0]])
_TRI_CORNERS = np.array([[-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0]])
# vertex permutations that can relate the two sides' face tuples
# (hybridwave/mesh.py:35-42)
TRI_PERMS = [(0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2)]
QUAD_PERMS = [(0, 1, 2, 3), (1, 2, 3, 0), (2, 3, 0, 1), (3, 0, 1, 2),
              (0, 3, 2, 1), (3, 2, 1, 0), (2, 1, 0, 3), (1, 0, 3, 2)]


def face_symmetry_perms(face_type, pts2d, tol=1e-10):
    """For each orientation code c (vertex tuple relation my[i] ==
    nbr[perm_c[i]]), the index map j -> p such that my face point j and the
    neighbour's face point p coincide.  (ncodes, npts) int32.

    My point with face shape-function weights N_i(xi) sits at
    sum_i N_i X_my[i] = sum_i N_i X_nbr[perm_c[i]]; in the neighbour's
    parametrisation that is the point whose weight on vertex perm_c[i] is
    N_i(xi), i.e. the image of xi under the affine map taking corner i to
    corner perm_c[i]."""
    from .refelem import face_shape2d
    corners = _TRI_CORNERS if face_type == "tri" else _QUAD_CORNERS
    perms = TRI_PERMS if face_type == "tri" else QUAD_PERMS
    w = face_shape2d(face_type, pts2d)                 # (P, nv)
    out = np.empty((len(perms), len(pts2d)), dtype=np.int32)
    for c, perm in enumerate(perms):
        img = w @ corners[list(perm)]
        d = np.linalg.norm(img[:, None, :] - pts2d[None, :, :], axis=2)
        idx = np.argmin(d, axis=1)
        if d[np.arange(len(pts2d)), idx].max() > tol:
            raise ValueError("face point set is not symmetric")
        out[c] = idx
    return out


def device_operators(elem_type, N, formulation, ops=None):
    """Compact constant operators for the kernels (fp64 numpy arrays).

    Returns a dict; every matrix is stored so that consecutive threads
    (consecutive output rows) read consecutive addresses."""
    ops = ops or build_operators(elem_type, N, formulation)
    Np = ops.Np
    tri2d = tri_face_nodes_2d(N)
    quad2d = quad_face_points_2d(N, formulation)
    out = {"Np": Np, "tri2d": tri2d, "quad2d": quad2d}
    nf = len(FACES[elem_type])
    # device face point sets and their reference-coordinate positions
    fpts, foffs = [], [0]
    for f, (ftype, _) in enumerate(FACES[elem_type]):
        p2 = tri2d if ftype == "tri" else quad2d
        fpts.append(p2)
        foffs.append(foffs[-1] + len(p2))
    out["face_offsets"] = np.array(foffs, dtype=np.int32)

    if elem_type == "hex":
        n1 = N + 1
        nodes = ops.nodes1d
        out["D1"] = ops.D1                      # (n1, n1), D1[i, l]
        out["Vend"] = ops.Vf_end                # (2, n1)
        out["w1"] = ops.weights1d
        # per face point: (base node, stride along the face normal, end)
        tab = np.empty((foffs[-1], 3), dtype=np.int32)
        strides = (n1 * n1, n1, 1)
        for f in range(nf):
            rst = face_quadrature_points("hex", f, fpts[f])
            fixed = (np.all(np.abs(rst - rst[0]) < 1e-12, axis=0)
                     & (np.abs(np.abs(rst[0]) - 1) < 1e-12))
            axis = int(np.flatnonzero(fixed)[0])
            end = 0 if rst[0, axis] < 0 else 1
            for j, p in enumerate(rst):
                idx = [int(np.argmin(np.abs(nodes - p[d]))) if d != axis else 0
                       for d in range(3)]
                for d in range(3):
                    if d != axis:
                        assert abs(nodes[idx[d]] - p[d]) < 1e-12
                base = (idx[0] * n1 + idx[1]) * n1 + idx[2]
                tab[foffs[f] + j] = (base, strides[axis], end)
        out["face_tab"] = tab
        out["w2"] = np.concatenate([face_rule_2d("quad", N, formulation)[1]] * nf)
        return out

    # dense types: own-trace operator E (Nfp_dev, Np) and lift (Np, Nfp_dev)
    Vf = ops.Vf
    E, LIFT = [], []
    for f, (ftype, _) in enumerate(FACES[elem_type]):
        sl = slice(ops.face_offsets[f], ops.face_offsets[f + 1])
        Vq = Vf[sl]                                   # stored cubature points
        wq = ops.face_wts[f]
        if ftype == "tri":
            rst_dev = face_quadrature_points(elem_type, f, tri2d)
            Ef = (_basis_at(elem_type, N, formulation, rst_dev, getattr(ops, "Vinv", None)))
            Lq = _tri_lagrange(tri2d, ops.face_pts2d[f], N)   # (nq, nfn)
        else:
            Ef = Vq
            Lq = np.eye(len(wq))
        E.append(Ef)
        Lf = Vq.T @ (wq[:, None] * Lq)                # (Np, nfp_dev)
        if elem_type == "tet":
            Lf = ops.invM_ref @ Lf
        LIFT.append(Lf)
    out["E"] = np.vstack(E)                            # (Nfp, Np)
    out["LIFT"] = np.hstack(LIFT)                      # (Np, Nfp)
    if elem_type == "tet":
        out["Dr"], out["Ds"], out["Dt"] = ops.Dr, ops.Ds, ops.Dt
        # face node -> volume node index
        fidx = []
        for f in range(nf):
            rst_dev = face_quadrature_points("tet", f, tri2d)
            d = np.linalg.norm(rst_dev[:, None, :] - ops.nodes[None], axis=2)
            idx = np.argmin(d, axis=1)
            assert d[np.arange(len(idx)), idx].max() < 1e-10
            fidx.append(idx)
        out["face_nodes"] = np.concatenate(fidx).astype(np.int32)
    elif elem_type == "wedge":
        out["V"], out["Dr3"], out["Ds3"], out["Dt3"] = ops.V, ops.Dr3, ops.Ds3, ops.Dt3
        out["wq"] = ops.cub.weights
        # affine LSC wedge: the two cubature passes collapse to
        # S_c = V^T W D3_c (test mode x trial mode), hybridwave/dg.py:423-444
        W = ops.cub.weights[:, None]
        out["S"] = np.stack([ops.V.T @ (W * D) for D in (ops.Dr3, ops.Ds3, ops.Dt3)])
    elif elem_type == "pyramid":
        out["Dr"], out["Ds"], out["Dt"] = ops.Dr, ops.Ds, ops.Dt
    return out
