"""Local timesteps and multi-rate level assignment (host setup feeding the
hot loop; hybridwave/stability.py:48-460 restricted to what the solver
path consumes).  Per-element quantities are computed face by face so the
2M-element meshes never materialise per-point face arrays."""

from functools import lru_cache

import numpy as np
import scipy.linalg as la

from . import basis as bas
from .operators import face_rule_2d
from .quadrature import element_rule, gauss_lobatto_1d
from .refelem import (FACES, REF_VERTS, face_geometry_batch, face_quadrature_points,
                      inverse_duffy_map, jacobian_det, jacobian_det_fast)

__all__ = ["computed_trace_constant", "analytic_trace_constant", "local_timesteps",
           "material_constant", "TimestepPlan", "assign_mrab_levels"]

SQRT2, SQRT3 = np.sqrt(2.0), np.sqrt(3.0)


def analytic_trace_constant(elem_type, N):
    """Table 2 closed forms (hybridwave/stability.py:48-58)."""
    return {"hex": 4.0 * (N + 1) ** 2, "wedge": (SQRT2 + 3.0) * (N + 1) * (N + 2),
            "pyramid": (SQRT2 + 2.0) * (N + 1) * (N + 3),
            "tet": (SQRT3 + 3.0) * (N + 1) * (N + 3) / 2.0}[elem_type]


def _ortho_vdm(t, N, abc):
    if t == "hex":
        P = [np.column_stack([bas.jacobi_p(abc[:, d], 0, 0, j) for j in range(N + 1)])
             for d in range(3)]
        return np.einsum("pi,pj,pk->pijk", *P).reshape(len(abc), -1)
    if t == "tet":
        return bas.tet_orthobasis_eval(N, abc).V
    if t == "wedge":
        return bas.wedge_orthobasis_eval(N, abc).V
    return bas.pyramid_seminodal_eval(N, abc).V


@lru_cache(maxsize=None)
def computed_trace_constant(elem_type, N, quad_mode="full"):
    """Largest eigenvalue of the reference surface mass against the volume
    mass in an orthonormal basis (hybridwave/stability.py:114-155)."""
    if not 1 <= N <= 9:
        raise ValueError("computed constants cover N in 1..9")
    verts = REF_VERTS[elem_type][None]
    form = "GL" if quad_mode == "full" else "SEM"
    Ms = 0.0
    for f, (ftype, _) in enumerate(FACES[elem_type]):
        p2, w2 = face_rule_2d(ftype, N, form)
        rst = face_quadrature_points(elem_type, f, p2)
        _, Js, _ = face_geometry_batch(elem_type, verts, f, p2)
        V = _ortho_vdm(elem_type, N, inverse_duffy_map(elem_type, rst))
        Ms = Ms + V.T @ ((w2 * Js[0])[:, None] * V)
    if elem_type == "hex" and quad_mode == "SEM":
        g = gauss_lobatto_1d(N + 1)
        a, b, c = np.meshgrid(g.points, g.points, g.points, indexing="ij")
        abc = np.column_stack([a.ravel(), b.ravel(), c.ravel()])
        w3 = np.einsum("i,j,k->ijk", g.weights, g.weights, g.weights).ravel()
        V = _ortho_vdm("hex", N, abc)
        M = V.T @ (w3[:, None] * V)
    else:
        M = np.eye(Ms.shape[0])
    return float(la.eigh(Ms, M, eigvals_only=True)[-1])


def _impedances(mesh, t):
    mat = np.asarray(mesh.materials[t], dtype=float)
    return mat[:, 0] * np.sqrt(mat[:, 1] / mat[:, 0])


def material_constant(disc, t):
    """max over faces of max(tau_p kappa, tau_u / rho) (stability.py:237-244)."""
    mesh = disc.mesh
    z = _impedances(mesh, t)
    nbr = mesh.nbr[t]
    zp = np.repeat(z[:, None], nbr.shape[1], axis=1)
    for t2 in disc.types:
        sel = nbr[:, :, 0] == ["hex", "wedge", "pyramid", "tet"].index(t2)
        zp[sel] = _impedances(mesh, t2)[nbr[:, :, 1][sel]]
    avg = 0.5 * (z[:, None] + zp)
    tp = (1.0 / avg).max(axis=1)
    tu = avg.max(axis=1)
    mat = np.asarray(mesh.materials[t], dtype=float)
    return np.maximum(tp * mat[:, 1], tu / mat[:, 0])


def _jacobian_norms(disc, t):
    """Maxima of J, 1/J, Js (and Js/J_face for wedges) over the quadrature
    points (hybridwave/stability.py:215-226).  Triangle faces are planar, so
    Js is evaluated once per face; J at wedge face points only when the
    wedge is not affine."""
    verts = disc.mesh.element_vertices(t)
    cub = element_rule(t, disc.N)
    cJ = jacobian_det_fast(t, verts, cub.collapsed)
    Jmax, Jinv = cJ.max(axis=1), (1.0 / cJ).max(axis=1)
    affine = np.all((cJ.max(axis=1) - cJ.min(axis=1)) <= 1e-13 * cJ.max(axis=1))
    op = disc.ops[t]
    Jsmax = np.zeros(len(verts))
    JsoJ = np.zeros(len(verts)) if t == "wedge" else None
    for f, (ftype, _) in enumerate(FACES[t]):
        p2 = op.face_pts2d[f]
        if ftype == "tri":
            p2 = p2[:1]
        _, Js, _ = face_geometry_batch(t, verts, f, p2)
        Jsmax = np.maximum(Jsmax, Js.max(axis=1))
        if t == "wedge":
            if affine:
                JsoJ = np.maximum(JsoJ, Js.max(axis=1) / cJ[:, 0])
            else:
                sl = slice(op.face_offsets[f], op.face_offsets[f + 1])
                _, Js_all, _ = face_geometry_batch(t, verts, f, op.face_pts2d[f])
                Jf = jacobian_det(t, verts, inverse_duffy_map(t, op.face_rst[sl]))
                JsoJ = np.maximum(JsoJ, (Js_all / Jf).max(axis=1))
    return Jmax, Jinv, Jsmax, JsoJ


def local_timesteps(disc, cfl=0.5):
    """Per-element stable timesteps cfl / (C_rk C_T(N) C_J)
    (hybridwave/stability.py:247-258)."""
    mode = "SEM" if disc.formulation.kind == "SEM" else "full"
    out = {}
    for t in disc.types:
        CT = computed_trace_constant(t, disc.N, mode)
        _, Jinv, Jsmax, JsoJ = _jacobian_norms(disc, t)
        CJ = JsoJ if t == "wedge" else Jsmax * Jinv
        out[t] = cfl / (material_constant(disc, t) * CT * CJ)
    return out


class TimestepPlan:
    """Levels 1 (coarsest) .. n_levels; dt_lev = 2^(n_levels-lev) dt_min
    (hybridwave/stability.py:389-426)."""

    def __init__(self, dt_local, levels, n_levels, cfl, order):
        self.dt_local = dt_local
        self.levels = levels
        self.n_levels = n_levels
        self.cfl = cfl
        self.order = order
        self.dt_min = min(float(v.min()) for v in dt_local.values())
        self.level_dts = np.array([2.0 ** (n_levels - lev) * self.dt_min
                                   for lev in range(1, n_levels + 1)])

    def levels_of(self, mesh, t):
        return self.levels[t]

    def dt_of(self, t):
        return self.level_dts[self.levels[t] - 1]

    def validate_neighbor_levels(self, mesh):
        names = ["hex", "wedge", "pyramid", "tet"]
        for t in self.levels:
            nbr = mesh.nbr[t]
            for t2 in self.levels:
                sel = nbr[:, :, 0] == names.index(t2)
                if not sel.any():
                    continue
                mine = np.broadcast_to(self.levels[t][:, None], sel.shape)[sel]
                theirs = self.levels[t2][nbr[:, :, 1][sel]]
                if np.any(np.abs(mine.astype(int) - theirs.astype(int)) > 1):
                    raise ValueError("neighboring elements differ by more than one timestep level")

    def check(self):
        for t, lv in self.levels.items():
            if np.any(self.level_dts[lv - 1] > self.dt_local[t] * (1 + 1e-12)):
                raise AssertionError("element assigned a timestep above its local limit")


def assign_mrab_levels(dt_local, n_levels, mesh, cfl=0.5, order=None):
    """Power-of-two binning then the neighbour sweep to |level difference|
    <= 1, moving elements to finer levels only (stability.py:429-460).  The
    sweep is iterated to its least fixed point with whole-array updates."""
    if n_levels < 1:
        raise ValueError("need at least one level")
    dt_min = min(float(v.min()) for v in dt_local.values())
    levels = {}
    for t, v in dt_local.items():
        ratio = np.maximum(v / dt_min, 1.0)
        levels[t] = np.clip(n_levels - np.floor(np.log2(ratio) + 1e-12).astype(int), 1, n_levels)
    names = ["hex", "wedge", "pyramid", "tet"]
    while True:
        changed = False
        for t in levels:
            nbr = mesh.nbr[t]
            need = levels[t].copy()
            for t2 in levels:
                sel = nbr[:, :, 0] == names.index(t2)
                if not sel.any():
                    continue
                lv = np.full(sel.shape, -10**9)
                lv[sel] = levels[t2][nbr[:, :, 1][sel]] - 1
                need = np.maximum(need, lv.max(axis=1))
            if np.any(need != levels[t]):
                levels[t] = need
                changed = True
        if not changed:
            break
    plan = TimestepPlan(dt_local, levels, n_levels, cfl, order or list(dt_local))
    plan.check()
    return plan
