"""Reference elements, collapse maps and vertex-mapped geometry (host setup).

Conventions are those of the reference package (hybridwave/refelem.py:69-112):
bi-unit elements, face vertex tuples counter-clockwise seen from outside,
faces ordered as listed there.  Geometry is evaluated in batches over
elements; the pyramid's rational vertex map is evaluated in collapsed
coordinates (refelem.py:198-367).
"""

import numpy as np

__all__ = [
    "ELEMENT_TYPES", "FACES", "REF_VERTS", "N_VERTS", "InvalidElementError",
    "duffy_map", "inverse_duffy_map", "shape_functions_abc",
    "shape_gradients_rst", "geometric_factors_batch",
    "face_quadrature_points", "face_geometry_batch", "face_shape2d",
    "map_points", "jacobian_det", "jacobian_det_fast", "affine_mask",
]

ELEMENT_TYPES = ("hex", "wedge", "pyramid", "tet")
N_VERTS = {"hex": 8, "wedge": 6, "pyramid": 5, "tet": 4}

REF_VERTS = {
    "hex": np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                     [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], float),
    "tet": np.array([[-1, -1, -1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], float),
    "wedge": np.array([[-1, -1, -1], [1, -1, -1], [-1, -1, 1],
                       [-1, 1, -1], [1, 1, -1], [-1, 1, 1]], float),
    "pyramid": np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                         [-1, -1, 1]], float),
}

# (face type, vertex tuple) per face, same order as the reference
FACES = {
    "hex": [("quad", (0, 4, 7, 3)), ("quad", (1, 2, 6, 5)), ("quad", (0, 1, 5, 4)),
            ("quad", (2, 3, 7, 6)), ("quad", (0, 3, 2, 1)), ("quad", (4, 5, 6, 7))],
    "tet": [("tri", (0, 2, 1)), ("tri", (0, 1, 3)), ("tri", (1, 2, 3)), ("tri", (0, 3, 2))],
    "wedge": [("tri", (0, 1, 2)), ("tri", (3, 5, 4)), ("quad", (0, 3, 4, 1)),
              ("quad", (0, 2, 5, 3)), ("quad", (1, 4, 5, 2))],
    "pyramid": [("quad", (0, 3, 2, 1)), ("tri", (0, 1, 4)), ("tri", (1, 2, 4)),
                ("tri", (2, 3, 4)), ("tri", (3, 0, 4))],
}


class InvalidElementError(ValueError):
    """Non-positive Jacobian of a vertex map."""


def duffy_map(elem_type, abc):
    abc = np.atleast_2d(np.asarray(abc, dtype=float))
    a, b, c = abc.T
    if elem_type == "hex":
        return abc.copy()
    if elem_type == "tet":
        return np.column_stack([(1 + a) * (1 - b) * (1 - c) / 4 - 1,
                                (1 + b) * (1 - c) / 2 - 1, c])
    if elem_type == "wedge":
        return np.column_stack([(1 + a) * (1 - c) / 2 - 1, b, c])
    if elem_type == "pyramid":
        return np.column_stack([(1 + a) * (1 - c) / 2 - 1, (1 + b) * (1 - c) / 2 - 1, c])
    raise ValueError(elem_type)


def inverse_duffy_map(elem_type, rst, tol=1e-13):
    """Collapsed preimages; singular sets get the limit value -1
    (hybridwave/refelem.py:145-172)."""
    rst = np.atleast_2d(np.asarray(rst, dtype=float))
    r, s, t = rst.T

    def coll(num, den):
        safe = np.where(den == 0, 1.0, den)
        return np.where(np.abs(den) > tol, 2 * (1 + num) / safe - 1, -1.0)

    if elem_type == "hex":
        return rst.copy()
    if elem_type == "tet":
        return np.column_stack([coll(r, -(s + t)), coll(s, 1.0 - t), t])
    if elem_type == "wedge":
        return np.column_stack([coll(r, 1.0 - t), s, t])
    if elem_type == "pyramid":
        return np.column_stack([coll(r, 1.0 - t), coll(s, 1.0 - t), t])
    raise ValueError(elem_type)


def shape_functions_abc(elem_type, abc):
    """Vertex shape functions at collapsed points, (npts, nv)."""
    a, b, c = np.atleast_2d(abc).T
    if elem_type == "hex":
        sg = REF_VERTS["hex"]
        return np.prod(1 + np.atleast_2d(abc)[:, None, :] * sg[None], axis=2) / 8
    if elem_type == "tet":
        l1 = (1 + a) * (1 - b) * (1 - c) / 8
        l2 = (1 + b) * (1 - c) / 4
        l3 = (1 + c) / 2
        return np.column_stack([1 - l1 - l2 - l3, l1, l2, l3])
    if elem_type == "wedge":
        m1 = (1 + a) * (1 - c) / 4
        m2 = (1 + c) / 2
        m0 = 1 - m1 - m2
        lo, hi = (1 - b) / 2, (1 + b) / 2
        return np.column_stack([m0 * lo, m1 * lo, m2 * lo, m0 * hi, m1 * hi, m2 * hi])
    if elem_type == "pyramid":
        am, ap, bm, bp = (1 - a) / 2, (1 + a) / 2, (1 - b) / 2, (1 + b) / 2
        cm = (1 - c) / 2
        return np.column_stack([am * bm * cm, ap * bm * cm, ap * bp * cm, am * bp * cm,
                                (1 + c) / 2])
    raise ValueError(elem_type)


def shape_gradients_rst(elem_type, abc):
    """d(shape)/d(r,s,t) at collapsed points, (npts, nv, 3)."""
    abc = np.atleast_2d(np.asarray(abc, dtype=float))
    n = len(abc)
    if elem_type == "hex":
        sg = REF_VERTS["hex"]
        fac = (1 + abc[:, None, :] * sg[None]) / 2
        out = np.empty((n, 8, 3))
        for d in range(3):
            o1, o2 = [e for e in range(3) if e != d]
            out[:, :, d] = sg[None, :, d] / 2 * fac[:, :, o1] * fac[:, :, o2]
        return out
    if elem_type == "tet":
        g = np.array([[-0.5, -0.5, -0.5], [0.5, 0, 0], [0, 0.5, 0], [0, 0, 0.5]])
        return np.broadcast_to(g, (n, 4, 3)).copy()
    if elem_type == "wedge":
        rst = duffy_map("wedge", abc)
        r, s, t = rst.T
        mu = np.column_stack([-(r + t) / 2, (1 + r) / 2, (1 + t) / 2])
        dmu = np.array([[-0.5, -0.5], [0.5, 0.0], [0.0, 0.5]])
        out = np.zeros((n, 6, 3))
        for i in range(3):
            for half, sgn, off in (((1 - s) / 2, -1.0, 0), ((1 + s) / 2, 1.0, 3)):
                out[:, i + off, 0] = dmu[i, 0] * half
                out[:, i + off, 2] = dmu[i, 1] * half
                out[:, i + off, 1] = sgn * mu[:, i] / 2
        return out
    if elem_type == "pyramid":
        a, b, c = abc.T
        am, ap, bm, bp = (1 - a) / 2, (1 + a) / 2, (1 - b) / 2, (1 + b) / 2
        cm = (1 - c) / 2
        g = np.zeros((n, 5, 3))  # d/d(a,b,c)
        for i, (fa, fb, da, db) in enumerate([(am, bm, -.5, -.5), (ap, bm, .5, -.5),
                                              (ap, bp, .5, .5), (am, bp, -.5, .5)]):
            g[:, i, 0] = da * fb * cm
            g[:, i, 1] = fa * db * cm
            g[:, i, 2] = -fa * fb / 2
        g[:, 4, 2] = 0.5
        # chain rule: d(abc)/d(rst) of the pyramid collapse
        inv = np.zeros((n, 3, 3))
        inv[:, 0, 0] = 2 / (1 - c)
        inv[:, 0, 2] = (1 + a) / (1 - c)
        inv[:, 1, 1] = 2 / (1 - c)
        inv[:, 1, 2] = (1 + b) / (1 - c)
        inv[:, 2, 2] = 1.0
        return np.einsum("pva,par->pvr", g, inv)
    raise ValueError(elem_type)


def _wedge_shape_hessians():
    """Constant second derivatives of the wedge vertex functions
    (only mixed (r,s) and (t,s) terms), (6, 3, 3)."""
    H = np.zeros((6, 3, 3))
    dmu = np.array([[-0.5, -0.5], [0.5, 0.0], [0.0, 0.5]])
    for i in range(3):
        for d, md in ((0, dmu[i, 0]), (2, dmu[i, 1])):
            H[i, d, 1] = H[i, 1, d] = -md / 2
            H[i + 3, d, 1] = H[i + 3, 1, d] = md / 2
    return H


def geometric_factors_batch(elem_type, verts, abc, label="element"):
    """x (K,P,3), J (K,P), G (K,P,3,3) with G[k,p,c,x] = d r_c / d x_x, and for
    wedges grad J (K,P,3) by Jacobi's formula (hybridwave/refelem.py:444-472)."""
    verts = np.asarray(verts, dtype=float)
    shape = shape_functions_abc(elem_type, abc)
    x = np.einsum("kvx,pv->kpx", verts, shape)
    F = np.einsum("kvx,pvr->kpxr", verts, shape_gradients_rst(elem_type, abc))
    J = np.linalg.det(F)
    if np.any(J <= 0):
        k = int(np.argwhere(J <= 0)[0, 0])
        raise InvalidElementError(
            f"nonpositive Jacobian in {elem_type} {label} {k} (min J = {J.min():.3e})")
    G = np.linalg.inv(F)
    gradJ = None
    if elem_type == "wedge":
        dF = np.einsum("kvx,vrc->kxrc", verts, _wedge_shape_hessians())
        dJ = J[..., None] * np.einsum("kprx,kxrc->kpc", G, dF)
        gradJ = np.einsum("kpc,kpcx->kpx", dJ, G)
    return x, J, G, gradJ


def map_points(elem_type, verts, abc):
    """Physical positions (K, P, 3) of collapsed points (no metric work;
    batched GEMM instead of einsum)."""
    verts = np.asarray(verts, dtype=float)
    return np.matmul(shape_functions_abc(elem_type, abc)[None], verts)


def affine_mask(elem_type, verts, tol=1e-12):
    """(K,) bool: the vertex map is affine (tets always; parallelepiped hexes,
    prism wedges with a translated top triangle, parallelogram-based
    pyramids)."""
    X = np.asarray(verts, dtype=float)
    scale = np.abs(X).max(axis=(1, 2)) + 1e-300
    if elem_type == "tet":
        return np.ones(len(X), dtype=bool)
    if elem_type == "hex":
        e = [X[:, 1] - X[:, 0] - (X[:, 2] - X[:, 3]), X[:, 1] - X[:, 0] - (X[:, 5] - X[:, 4]),
             X[:, 1] - X[:, 0] - (X[:, 6] - X[:, 7]), X[:, 4] - X[:, 0] - (X[:, 7] - X[:, 3])]
    elif elem_type == "wedge":
        e = [X[:, 3] - X[:, 0] - (X[:, 4] - X[:, 1]), X[:, 3] - X[:, 0] - (X[:, 5] - X[:, 2])]
    elif elem_type == "pyramid":
        e = [X[:, 1] - X[:, 0] - (X[:, 2] - X[:, 3])]
    else:
        raise ValueError(elem_type)
    err = np.max([np.abs(v).max(axis=1) for v in e], axis=0)
    return err <= tol * scale


def jacobian_det(elem_type, verts, abc):
    """det(dx/dr) (K, P) without forming the inverse (batched GEMMs)."""
    verts = np.asarray(verts, dtype=float)
    g = shape_gradients_rst(elem_type, abc)                  # (P, nv, 3)
    Fc = [np.matmul(g[None, :, :, r], verts) for r in range(3)]   # (K, P, 3) = dx/dr_r
    a, b, c = Fc
    J = (a[..., 0] * (b[..., 1] * c[..., 2] - b[..., 2] * c[..., 1])
         - b[..., 0] * (a[..., 1] * c[..., 2] - a[..., 2] * c[..., 1])
         + c[..., 0] * (a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1]))
    if np.any(J <= 0):
        raise InvalidElementError(f"nonpositive Jacobian in {elem_type} (min J = {J.min():.3e})")
    return J


def jacobian_det_fast(elem_type, verts, abc):
    """jacobian_det, evaluated once per affine element and broadcast."""
    verts = np.asarray(verts, dtype=float)
    aff = affine_mask(elem_type, verts)
    P = len(np.atleast_2d(abc))
    out = np.empty((len(verts), P))
    if aff.any():
        interior = np.atleast_2d(abc)[:1]
        out[aff] = jacobian_det(elem_type, verts[aff], interior)
    if (~aff).any():
        out[~aff] = jacobian_det(elem_type, verts[~aff], abc)
    return out


def face_shape2d(face_type, p):
    xi, eta = np.atleast_2d(p).T
    if face_type == "tri":
        return np.column_stack([-(xi + eta) / 2, (1 + xi) / 2, (1 + eta) / 2])
    return np.column_stack([(1 - xi) * (1 - eta), (1 + xi) * (1 - eta),
                            (1 + xi) * (1 + eta), (1 - xi) * (1 + eta)]) / 4


def _face_shape2d_grad(face_type, p):
    xi, eta = np.atleast_2d(p).T
    n = len(xi)
    if face_type == "tri":
        return np.broadcast_to(np.array([[-.5, -.5], [.5, 0], [0, .5]]), (n, 3, 2))
    g = np.empty((n, 4, 2))
    g[:, 0] = np.column_stack([-(1 - eta), -(1 - xi)]) / 4
    g[:, 1] = np.column_stack([(1 - eta), -(1 + xi)]) / 4
    g[:, 2] = np.column_stack([(1 + eta), (1 + xi)]) / 4
    g[:, 3] = np.column_stack([-(1 + eta), (1 - xi)]) / 4
    return g


def face_quadrature_points(elem_type, face, p2d):
    ftype, ix = FACES[elem_type][face]
    return face_shape2d(ftype, p2d) @ REF_VERTS[elem_type][list(ix)]


def face_geometry_batch(elem_type, verts, face, p2d):
    """Physical face points, surface Jacobians and outward unit normals,
    (K,P,3), (K,P), (K,P,3) (hybridwave/refelem.py:520-538)."""
    ftype, ix = FACES[elem_type][face]
    fv = np.asarray(verts, dtype=float)[:, list(ix), :]
    x = np.einsum("kvx,pv->kpx", fv, face_shape2d(ftype, p2d))
    g = _face_shape2d_grad(ftype, p2d)
    t1 = np.einsum("kvx,pv->kpx", fv, g[:, :, 0])
    t2 = np.einsum("kvx,pv->kpx", fv, g[:, :, 1])
    nv = np.cross(t1, t2)
    Js = np.linalg.norm(nv, axis=2)
    return x, Js, nv / Js[..., None]
