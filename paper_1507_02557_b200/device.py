"""Device-resident mesh: the HBM layout the sm_100a kernels read.

Per element type (K elements):
  state            (K, 4, Np)  element-major, reference node/mode order
  geometry record  hex: 8 vertices (24); tet/pyramid/wedge (affine): G,
                   per-face normal and Js/J (wedge: 1/sqrt(J), Js/sqrt(J))
  mat              (K, 4): kappa, 1/rho, rho*c, 0
  nbr_elem/code    (K, nfaces) int32: neighbour index and packed
                   type | face << 2 | orientation << 5 | boundary bit
  operators        constant matrices (device_operators), a few KB-100 KB
  face gather index per element: the source offset of every face point's
                   neighbour value, in this element's point order
  face traces      (K, 4, Nfp) ping-pong buffers for the publishing types
                   (wedge, pyramid, GL hex): each stage writes the traces of
                   its output state; tets and SEM hexes are read by their
                   neighbours straight from the state (selection traces)
Per-point geometry exists only where the geometry is non-affine (pyramid
base faces, cubature wedges); affine elements carry per-face records.
"""

import numpy as np
import torch

from . import _native as nat
from .operators import TYPE_ID, device_operators, face_symmetry_perms
from .refelem import FACES, face_geometry_batch, geometric_factors_batch

_CENTROID2D = {"tri": np.array([[-1.0 / 3.0, -1.0 / 3.0]]), "quad": np.array([[0.0, 0.0]])}
_INTERIOR_ABC = {"tet": np.array([[-0.5, -0.5, -0.5]]), "wedge": np.array([[0.0, 0.0, 0.0]]),
                 "pyramid": np.array([[0.0, 0.0, 0.0]])}


def _affine_check(disc, t, verts):
    """Non-affine wedges run the cubature form of the scalar kernel
    (wedge_cubature_ops); their triangle faces are integrated at the
    reference's face cubature.  A tet or pyramid across such a triangle gets
    the matching correction of its nodal lift (wedge_face_corrections)."""
    from .refelem import affine_mask
    if t != "wedge" or len(verts) == 0 or affine_mask(t, verts, tol=1e-10).all():
        return False
    return True


def wedge_cubature_ops(disc, dops):
    """op[8] / op[9] of the non-affine wedge path (layout: Naw in
    csrc/hw_kernels.cuh), from the reference-layout geometry
    (hybridwave/dg.py:139-192): volume cubature G and gJfac premultiplied by
    the weights, per-point quad-face n, Js/sqrt(J), 1/sqrt(J), and at the
    triangle-face cubature points the own and the neighbour's 1/sqrt(J)
    (through the reference gather index, dg.py:284-298) and w Js/sqrt(J)."""
    from .operators import _tri_lagrange
    ops = disc.ops["wedge"]
    d = disc.data["wedge"]
    K, Np = disc.n_elems["wedge"], ops.Np
    w = ops.cub.weights
    nq = len(w)
    vol = np.concatenate([(w[None, :, None, None] * d.G).reshape(K, nq, 9),
                          w[None, :, None] * d.gJfac], axis=2)
    roffs = np.asarray(ops.face_offsets)
    doffs = dops["face_offsets"]
    tot = int(roffs[-1])
    quad = np.zeros((K, int(doffs[-1]), 5))
    for f in range(2, 5):
        rs, ds = slice(roffs[f], roffs[f + 1]), slice(doffs[f], doffs[f + 1])
        quad[:, ds, :3] = d.normals[:, rs]
        quad[:, ds, 3] = d.wJs[:, rs] / ops.face_wts[f][None, :] * d.invsqrtJ_face[:, rs]
        quad[:, ds, 4] = d.invsqrtJ_face[:, rs]
    # the symmetric triangle rule stores each point twice with equal
    # weights: keep one of each pair with the summed
    # weight (identical integrand at both: <= 1e-15 relative)
    nqt = int(roffs[1] - roffs[0])
    uniq, pair = [], []
    for f in range(2):
        key = np.round(ops.face_pts2d[f], 11)
        _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
        inv = inv.ravel()
        partner = np.array([np.flatnonzero(inv == g) for g in range(len(first))])
        if partner.shape[1:] != (2,):
            raise ValueError("triangle face rule is not pairwise duplicated")
        uniq.append(partner[:, 0])
        pair.append(partner)
    nqu = len(uniq[0])
    tri = np.zeros((K, 2, nqu, 3))
    base = disc.trace_bases["wedge"]
    gidx = np.asarray(disc.gather_idx)
    bnd = np.asarray(disc.bnd_mask)
    for f in range(2):
        rs = slice(roffs[f], roffs[f + 1])
        flat = base + np.arange(K)[:, None] * tot + np.arange(roffs[f], roffs[f + 1])[None, :]
        g = gidx[flat] - base
        ok = ~bnd[flat] & (g >= 0) & (g < K * tot)
        gc = np.where(ok, g, 0)
        u = uniq[f]
        tri[:, f, :, 0] = d.invsqrtJ_face[:, rs][:, u]
        # the neighbour's 1/sqrt(J): a wedge's at the coincident point; a tet
        # or pyramid trace carries no sqrt(J) factor
        other = ~bnd[flat] & ~ok
        nb = np.where(ok, d.invsqrtJ_face[gc // tot, gc % tot], np.where(other, 1.0, 0.0))
        tri[:, f, :, 1] = nb[:, u]
        wsc = d.wJs[:, rs] * d.invsqrtJ_face[:, rs]
        tri[:, f, :, 2] = wsc[:, pair[f][:, 0]] + wsc[:, pair[f][:, 1]]
    geo = np.concatenate([vol.reshape(K, -1), quad.reshape(K, -1), tri.reshape(K, -1)], axis=1)
    mats = [ops.V, ops.Dr3, ops.Ds3, ops.Dt3]
    Lq = np.stack([_tri_lagrange(dops["tri2d"], ops.face_pts2d[f][uniq[f]], disc.N)
                   for f in range(2)])
    Vf = np.stack([ops.Vf[roffs[f]:roffs[f + 1]][uniq[f]] for f in range(2)])
    const = np.concatenate([np.stack([m.T for m in mats]).ravel(), np.stack(mats).ravel(),
                            Lq.ravel(), Vf.ravel()])
    return {8: geo, 9: const}


def wedge_face_corrections(disc, pack):
    """Tets and pyramids across a triangle face of a non-affine wedge: the
    wedge trace there is q_w / sqrt(J_w), not a polynomial, so the nodal
    face lift of the tet / pyramid kernels (exact for polynomial fluxes) is
    replaced by the reference's face cubature (hybridwave/dg.py:326-354 at
    the stored 6(N+1)^2 points).  The flux is linear in the neighbour trace,
    so the correction is the lift of the flux of
        delta = (L nb) * (s - 1),   s = the wedge's 1/sqrt(J) at the point,
    nb = the wedge's published (unscaled) triangle trace at my face nodes,
    L = my nodal-to-cubature interpolant:
        dfp = tau_p/2 delta_p - n.delta_u / 2,  dfu = tau_u/2 n.delta_u - delta_p / 2,
        drhs = nodefac * Js * P_f [dfp, n dfu]   (kappa, 1/rho in the kernel),
    P_f = [invM_ref] Vf_f^T diag(w_f).  Returns {t: arrays} for the
    hw_wedge_face_correction kernel, empty when no such face exists."""
    from .operators import _tri_lagrange
    out = {}
    if "wedge" not in disc.types or 8 not in pack["types"]["wedge"]["op"]:
        return out
    N = disc.N
    wd = disc.data["wedge"]
    wops = disc.ops["wedge"]
    wtot = int(wops.face_offsets[-1])
    wbase = disc.trace_bases["wedge"]
    gidx = np.asarray(disc.gather_idx)
    nfp_w = pack["types"]["wedge"]["nfp"]
    for t, tid_faces in (("tet", range(4)), ("pyramid", range(1, 5))):
        if t not in disc.types:
            continue
        nbr = disc.mesh.nbr[t]
        P_ = pack["types"][t]
        dops = P_["dops"]
        ops = disc.ops[t]
        d = disc.data[t]
        K, Np = disc.n_elems[t], ops.Np
        nfn = len(dops["tri2d"])
        roffs = np.asarray(ops.face_offsets)
        tot = int(roffs[-1])
        base = disc.trace_bases[t]
        gi = P_["iop"][1].reshape(K, -1)
        doffs = np.asarray(dops["face_offsets"])
        rows_i, rows_f = [], []
        nq = None
        Ls, Ps = [], []
        for f in range(nbr.shape[1]):
            if f not in tid_faces:
                Ls.append(None)
                Ps.append(None)
                continue
            pts = ops.face_pts2d[f]
            nq = len(pts)
            Ls.append(_tri_lagrange(dops["tri2d"], pts, N))
            Pf = ops.Vf[roffs[f]:roffs[f + 1]].T * ops.face_wts[f][None, :]
            if t == "tet":
                Pf = ops.invM_ref @ Pf
            Ps.append(Pf)
            sel = np.flatnonzero(nbr[:, f, 0] == 1)          # wedge neighbours
            if len(sel) == 0:
                continue
            flat = base + sel[:, None] * tot + np.arange(roffs[f], roffs[f + 1])[None, :]
            g = gidx[flat] - wbase
            s_ = wd.invsqrtJ_face[g // wtot, g % wtot]          # (n, nq)
            if np.abs(s_ - 1.0).max() == 0.0:
                continue
            gv = gi[sel][:, doffs[f]:doffs[f] + nfn] if t == "pyramid" else \
                gi[sel].reshape(len(sel), 4, nfn)[:, f, :]
            nb_off = (-gv.astype(np.int64) - 4) // 2 if t == "tet" else gv.astype(np.int64)
            rec = P_["geo"][sel]
            fb = 9 + 6 * f
            js = d.wJs[sel, roffs[f]] / ops.face_wts[f][0]
            nodefac = (np.repeat(1.0 / d.J[sel, :1], Np, axis=1) if t == "tet"
                       else 1.0 / d.J[sel])
            rows_i.append(np.column_stack([sel, np.full(len(sel), f), nb_off]))
            rows_f.append(np.column_stack([rec[:, fb + 4], rec[:, fb + 5], rec[:, fb:fb + 3],
                                           js, s_ - 1.0, nodefac]))
        if not rows_i:
            continue
        if int(np.max(np.concatenate(rows_i)[:, 2:])) >= 2 ** 31:
            raise ValueError("wedge trace offsets exceed int32")
        zL = np.zeros((nq, nfn))
        zP = np.zeros((Np, nq))
        out[t] = {"idata": np.concatenate(rows_i).astype(np.int32),
                  "fdata": np.concatenate(rows_f).astype(np.float64),
                  "L": np.stack([x if x is not None else zL for x in Ls]),
                  "P": np.stack([x if x is not None else zP for x in Ps]),
                  "nq": nq, "nfn": nfn, "nfp_w": nfp_w}
    return out


def face_impedance_avg(mesh, t):
    """avg(rho c) of the two sides of every face of type t, (K, nfaces); the
    own side twice on the boundary (hybridwave/dg.py:249-276)."""
    def z(tt):
        m = np.asarray(mesh.materials[tt], dtype=float)
        return m[:, 0] * np.sqrt(m[:, 1] / m[:, 0])
    names = ["hex", "wedge", "pyramid", "tet"]
    nbr = mesh.nbr[t]
    zm = z(t)
    zp = np.repeat(zm[:, None], nbr.shape[1], axis=1)
    for tid, t2 in enumerate(names):
        sel = nbr[:, :, 0] == tid
        if sel.any():
            zp[sel] = z(t2)[nbr[:, :, 1][sel]]
    return 0.5 * (zm[:, None] + zp)


def geometry_records(t, verts, zavg):
    """Per-element geometry record (float64 numpy), layouts in the header:
    dense types G(9) [, 1/sqrt(J)] then per face (n, Js-scale, avg(rho c),
    1/avg(rho c)); hex: 8 vertices, per face (avg, 1/avg), affine flag, and
    for affine hexes G(9), J, per face (n, Js), 1/J."""
    K = len(verts)
    if t == "hex":
        out = np.zeros((K, 72))
        out[:, :24] = verts.reshape(K, 24)
        out[:, 24:36:2] = zavg
        out[:, 25:36:2] = 1.0 / zavg
        # affine hexes (parallelepipeds): constant metric and face geometry
        from .refelem import affine_mask
        _, J, G, _ = geometric_factors_batch("hex", verts, np.zeros((1, 3)), label=t)
        out[:, 36] = affine_mask("hex", verts).astype(float)
        out[:, 37:46] = G[:, 0].reshape(K, 9)
        out[:, 46] = J[:, 0]
        out[:, 71] = 1.0 / J[:, 0]
        for f in range(6):
            _, Js, nrm = face_geometry_batch("hex", verts, f, _CENTROID2D["quad"])
            out[:, 47 + 4 * f: 50 + 4 * f] = nrm[:, 0]
            out[:, 50 + 4 * f] = Js[:, 0]
        return out
    _, J, G, _ = geometric_factors_batch(t, verts, _INTERIOR_ABC[t], label=t)
    J, G = J[:, 0], G[:, 0]
    cols = [G.reshape(K, 9)]
    naff = None
    if t == "wedge":
        isj = 1.0 / np.sqrt(J)
        cols.append(isj[:, None])
        scale = isj
    else:
        scale = 1.0 / J
        if t == "pyramid":
            # non-affine pyramids: face scale Js only (the kernel divides the
            # lift by J at each node); flag in the last word
            from .refelem import affine_mask
            naff = ~affine_mask(t, verts, tol=1e-10)
            scale = np.where(naff, 1.0, scale)
    for f, (ftype, _) in enumerate(FACES[t]):
        _, Js, nrm = face_geometry_batch(t, verts, f, _CENTROID2D[ftype])
        cols.append(nrm[:, 0, :])
        cols.append((Js[:, 0] * scale)[:, None])
        cols.append(zavg[:, f:f + 1])
        cols.append(1.0 / zavg[:, f:f + 1])
    if naff is not None:
        cols.append(naff.astype(float)[:, None])
    return np.hstack(cols)


def material_records(mat):
    rho, kappa = mat[:, 0], mat[:, 1]
    if np.any(rho <= 0) or np.any(kappa <= 0):
        raise ValueError("material parameters must be positive")
    z = rho * np.sqrt(kappa / rho)
    return np.column_stack([kappa, 1.0 / rho, z, np.zeros_like(z)])


def neighbour_codes(mesh, t):
    nbr = mesh.nbr[t]
    code = mesh.face_code[t].astype(np.int64)
    K, nf = nbr.shape[:2]
    bnd = nbr[:, :, 0] < 0
    packed = (np.where(bnd, 0, nbr[:, :, 0]) | (np.where(bnd, 0, nbr[:, :, 2]) << 2)
              | (np.where(bnd, 0, code) << 5) | np.where(bnd, nat.HW_NBR_BOUNDARY, 0))
    elem = np.where(bnd, np.arange(K)[:, None], nbr[:, :, 1])
    if elem.max(initial=0) >= 2 ** 31:
        raise ValueError("element index exceeds int32")
    return elem.astype(np.int32), packed.astype(np.int32)


def hex_node_face_points(dops, N):
    """(6, Np): for node n and face f, the face point on the node's line
    normal to f."""
    n1 = N + 1
    Np = n1 ** 3
    nfq = n1 * n1
    tab = dops["face_tab"]
    out = np.empty((6, Np), dtype=np.int32)
    strides = (n1 * n1, n1, 1)
    for f in range(6):
        axis = f >> 1
        lut = {int(tab[f * nfq + j, 0]): j for j in range(nfq)}
        for n in range(Np):
            idx = (n // (n1 * n1), (n // n1) % n1, n % n1)
            out[f, n] = lut[n - idx[axis] * strides[axis]]
    return out


def pyramid_node_geometry(verts, ops, dops):
    """Non-affine pyramids (hybridwave/dg.py:135-152, 446-463): op[8] =
    (K, Np, 10) G[c][x] and J at the level nodes, op[9] = (K, NFQ, 4) unit
    normal and Js at the bilinear base face's points (the device face order)."""
    _, J, G, _ = geometric_factors_batch("pyramid", verts, ops.level_abc, label="pyramid")
    K, Np = J.shape
    node = np.concatenate([G.reshape(K, Np, 9), J[..., None]], axis=2)
    _, Js, nrm = face_geometry_batch("pyramid", verts, 0, dops["quad2d"])
    base = np.concatenate([nrm, Js[..., None]], axis=2)
    return node, base


def hex_face_point_coefficients(dops, N):
    """(6, 4) int32: node (i, j, k) -> its face point on face f is
    c[f] . (i, j, k, 1) (the face rules enumerate points on the tensor grid,
    so the map is affine; checked exactly against hex_node_face_points)."""
    tab = hex_node_face_points(dops, N)
    n1 = N + 1
    n = np.arange(n1 ** 3)
    I = np.stack([n // (n1 * n1), (n // n1) % n1, n % n1, np.ones_like(n)], axis=1)
    out = np.zeros((6, 4), dtype=np.int32)
    for f in range(6):
        c = np.rint(np.linalg.lstsq(I.astype(float), tab[f].astype(float), rcond=None)[0])
        if not np.array_equal(I @ c.astype(np.int64), tab[f]):
            raise ValueError("hex face-point map is not affine in the node indices")
        out[f] = c
    return out


def pack_mesh(disc):
    """Host (numpy) image of everything the kernels read: per type
    {geo, mat, nbr_elem, nbr_code, op{slot}, iop{slot}, form, K} plus the
    face-point permutation tables.  DeviceMesh uploads it verbatim."""
    mesh = disc.mesh
    pack = {"types": {}}
    dops_any = None
    dops_all = {t: device_operators(t, disc.N, disc.formulation.kind, disc.ops[t])
                for t in disc.types}
    face_offsets = {t: (d["face_offsets"], int(d["face_offsets"][-1])) for t, d in dops_all.items()}
    for t in disc.types:
        form = disc.forms[t]
        verts = mesh.element_vertices(t)
        naw = _affine_check(disc, t, verts)
        dops = dops_all[t]
        dops_any = dops
        perm_tri = face_symmetry_perms("tri", dops["tri2d"])
        perm_quad = face_symmetry_perms("quad", dops["quad2d"])
        elem, code = neighbour_codes(mesh, t)
        pack["types"][t] = {
            "K": disc.n_elems[t], "form": form, "dops": dops,
            "geo": geometry_records(t, verts, face_impedance_avg(mesh, t)),
            "mat": material_records(np.asarray(mesh.materials[t], dtype=float)),
            "nbr_elem": elem, "nbr_code": code,
            "op": {**_pack_ops(t, dops), **(_tet_extra_ops(disc.ops[t], dops) if t == "tet" else {}),
                   **(_pyramid_extra_ops(verts, disc.ops[t], dops) if t == "pyramid" else {}),
                   **(wedge_cubature_ops(disc, dops) if naw else {})},
            "iop": _pack_iops(t, dops, disc.N, mesh, perm_tri, face_offsets, dops_all,
                              perm_quad, disc.formulation.kind == "SEM"),
            "nfp": int(dops["face_offsets"][-1]),
            "publishes": t in ("wedge", "pyramid") or (t == "hex"
                                                       and disc.formulation.kind == "GL")}
    pack["perm_tri"] = face_symmetry_perms("tri", dops_any["tri2d"])
    pack["perm_quad"] = face_symmetry_perms("quad", dops_any["quad2d"])
    return pack


# operator slots read as fp64 DMMA fragments by the tensor-core kernels
MMA_SLOTS = {"hex": (), "tet": (2, 3, 5), "wedge": (2, 3, 4, 7), "pyramid": (2, 3, 4, 7)}


def _pyramid_extra_ops(verts, ops, dops):
    """op[8], op[9] only when the mesh has non-affine pyramids (their
    presence routes the pyramids to the per-node-geometry scalar kernel)."""
    from .refelem import affine_mask
    if len(verts) == 0 or affine_mask("pyramid", verts, tol=1e-10).all():
        return {}
    node, base = pyramid_node_geometry(verts, ops, dops)
    return {8: node, 9: base}


def _tet_extra_ops(ops, d):
    """tet op[4] = M_ref (hw_energy); op[5] = the skew-form volume operators
    B_c = invM_ref D_c^T M_ref (rhs_p = sum_c B_c v_c after the mass inverse,
    hybridwave/dg.py:413-416) as padded DMMA fragments."""
    Np = d["Np"]
    rt8, npk = -(-Np // 8) * 8, -(-Np // 4) * 4
    B = np.zeros((3, rt8, npk))
    for c, Dc in enumerate((d["Dr"], d["Ds"], d["Dt"])):
        B[c, :Np, :Np] = ops.invM_ref @ Dc.T @ ops.M_ref
    return {4: ops.M_ref, 5: mma_fragments(B)}


def mma_fragments(A):
    """(..., 8*RT, 4*KS) row-major padded matrix -> (..., RT, KS, 32): the
    mma.m8n8k4 A fragment of row tile rt and k-step ks in lane order
    (lane = 4*row + k), so a warp reads each fragment as 256 contiguous
    bytes instead of 8 rows of 32 bytes."""
    *lead, r8, k4 = A.shape
    B = A.reshape(*lead, r8 // 8, 8, k4 // 4, 4)
    B = np.moveaxis(B, -3, -2)                     # (..., RT, KS, 8, 4)
    return np.ascontiguousarray(B.reshape(*lead, r8 // 8, k4 // 4, 32))


def mma_fragment_pairs(A):
    """mma_fragments with consecutive k-steps paired per lane,
    (..., RT, ceil(KS/2), 32, 2) (odd KS zero padded): one 16-byte load
    feeds two MMAs."""
    F = mma_fragments(A)
    *lead, rt, ks, _ = F.shape
    if ks % 2:
        F = np.concatenate([F, np.zeros((*lead, rt, 1, 32))], axis=-2)
        ks += 1
    F = F.reshape(*lead, rt, ks // 2, 2, 32)
    return np.ascontiguousarray(np.swapaxes(F, -1, -2))


def _pack_ops(t, d):
    if t == "hex":
        return {0: d["D1"], 1: d["Vend"], 2: d["w1"], 4: _hex_nodes(d)}
    if t == "tet":
        Np = d["Np"]
        nfn = len(d["tri2d"])
        rt8, npk, nfk = -(-Np // 8) * 8, -(-Np // 4) * 4, -(-nfn // 4) * 4
        Dpad = np.zeros((3, rt8, npk))
        for c, Dc in enumerate((d["Dr"], d["Ds"], d["Dt"])):
            Dpad[c, :Np, :Np] = Dc
        Lpad = np.zeros((4, rt8, nfk))
        for f in range(4):
            Lpad[f, :Np, :nfn] = d["LIFT"][:, f * nfn:(f + 1) * nfn]
        # 0, 1: scalar kernel (transposed); 2, 3: DMMA kernel (padded, fragment order)
        return {0: np.stack([d["Dr"].T, d["Ds"].T, d["Dt"].T]), 1: d["LIFT"].T,
                2: mma_fragments(Dpad), 3: mma_fragments(Lpad)}
    if t in ("wedge", "pyramid"):
        A = d["S"] if t == "wedge" else np.stack([d["Dr"], d["Ds"], d["Dt"]])
        # scalar kernel: op[0][c][m][n] = A_c[n][m], op[1][c][m][n] = A_c[m][n]
        ops = {0: np.stack([a.T for a in A]), 1: A, 5: d["E"].T, 6: d["LIFT"].T}
        ops.update(_mma_ops(t, d, A))
        return ops
    raise ValueError(t)


def _mma_ops(t, d, A):
    """Zero-padded operands of the DMMA kernels (hw_dense_mma.cuh), stored in
    A-fragment order (mma_fragments): op[2] A_c, op[3] A_c^T (3, RT8, NPK);
    op[4] LIFT with each face's K block padded to a multiple of 4
    (RT8, NFKT); op[7] E (RTF8, NPK)."""
    Np = d["Np"]
    rt8, npk = -(-Np // 8) * 8, -(-Np // 4) * 4
    Ap = np.zeros((3, rt8, npk))
    ATp = np.zeros((3, rt8, npk))
    for c in range(3):
        Ap[c, :Np, :Np] = A[c]
        ATp[c, :Np, :Np] = A[c].T
    offs = d["face_offsets"]
    cnts = np.diff(offs)
    kf = [-(-int(c) // 4) * 4 for c in cnts]
    L = np.zeros((rt8, sum(kf)))
    k0 = 0
    for f, c in enumerate(cnts):
        L[:Np, k0:k0 + c] = d["LIFT"][:, offs[f]:offs[f + 1]]
        k0 += kf[f]
    nfp = int(offs[-1])
    Ep = np.zeros((-(-nfp // 8) * 8, npk))
    Ep[:nfp, :Np] = d["E"]
    return {2: mma_fragment_pairs(Ap), 3: mma_fragment_pairs(ATp), 4: mma_fragment_pairs(L),
            7: mma_fragment_pairs(Ep)}


def tet_gather_index(mesh, dops, perm_tri, face_offsets):
    """(K, 4, NFN) int32: for each tet face node in my face-point order where
    the neighbour's value comes from: >= 0 the flat offset in the tet state
    (element-major (K,4,Np), field 0) of the coincident neighbour node; -1
    on the boundary; <= -3 a published pyramid/wedge trace,
    -3 - (2*offset + is_wedge) with offset into that type's trace buffer
    (K2, 4, Nfp2), field 0."""
    nbr = mesh.nbr["tet"]
    code = mesh.face_code["tet"]
    K = len(nbr)
    Np = dops["Np"]
    nfn = len(dops["tri2d"])
    fn = dops["face_nodes"].reshape(4, nfn)
    out = np.full((K, 4, nfn), -1, dtype=np.int64)
    for f in range(4):
        for tid, name in ((3, "tet"), (1, "wedge"), (2, "pyramid")):
            sel = nbr[:, f, 0] == tid
            if not sel.any():
                continue
            k2, f2, pc = nbr[sel, f, 1], nbr[sel, f, 2], code[sel, f]
            p = perm_tri[pc]
            if name == "tet":
                out[sel, f, :] = k2[:, None] * 4 * Np + fn[f2[:, None], p]
            else:
                offs, nfp2 = face_offsets[name]
                off = k2[:, None] * 4 * nfp2 + offs[f2][:, None] + p
                out[sel, f, :] = -3 - (2 * off + (1 if name == "wedge" else 0))
    if np.abs(out).max(initial=0) >= 2 ** 31:
        raise ValueError("tet gather offsets exceed int32")
    return out.astype(np.int32)


def face_gather_index(mesh, t, dops_all, perm_tri, perm_quad, face_offsets, N, sem):
    """(K, Nfp) int32 for the hex / wedge / pyramid kernels: for each of my face
    points (device order, hybridwave/dg.py:258-300 neighbour trace, already
    permuted into my point order) the field-0 offset of the coincident
    neighbour value in its source array; the source (and its field stride)
    follows from the face's neighbour code: a publishing type's trace buffer
    (K2, 4, Nfp2), else the tet / SEM-hex state (K2, 4, Np2).  -1 on the
    boundary."""
    nbr = mesh.nbr[t]
    code = mesh.face_code[t]
    offs, nfp = face_offsets[t]
    K = len(nbr)
    nfn = (N + 1) * (N + 2) // 2
    out = np.full((K, nfp), -1, dtype=np.int64)
    names = ("hex", "wedge", "pyramid", "tet")
    for f in range(len(offs) - 1):
        a, b = int(offs[f]), int(offs[f + 1])
        perm = perm_tri if b - a == nfn else perm_quad
        for tid2, t2 in enumerate(names):
            sel = nbr[:, f, 0] == tid2
            if not sel.any():
                continue
            k2, f2, pc = nbr[sel, f, 1], nbr[sel, f, 2], code[sel, f]
            p = perm[pc]                                   # (n, cnt) neighbour face point
            if t2 in ("wedge", "pyramid") or (t2 == "hex" and not sem):
                offs2, nfp2 = face_offsets[t2]
                val = k2[:, None] * 4 * nfp2 + offs2[f2][:, None] + p
            elif t2 == "tet":
                d2 = dops_all["tet"]
                fn = d2["face_nodes"].reshape(4, nfn)
                val = k2[:, None] * 4 * d2["Np"] + fn[f2[:, None], p]
            else:                                          # SEM hex: face node of the point
                d2 = dops_all["hex"]
                nfq = (N + 1) ** 2
                tab = d2["face_tab"]
                row = f2[:, None] * nfq + p
                node = tab[row, 0] + np.where(tab[row, 2] != 0, N, 0) * tab[row, 1]
                val = k2[:, None] * 4 * d2["Np"] + node
            out[sel, a:b] = val
    if out.max(initial=0) >= 2 ** 31:
        raise ValueError("face gather offsets exceed int32")
    return out.astype(np.int32)


def _pack_iops(t, d, N, mesh=None, perm_tri=None, face_offsets=None, dops_all=None,
               perm_quad=None, sem=False):
    if t == "hex":
        return {0: d["face_tab"], 1: hex_node_face_points(d, N),
                3: hex_face_point_coefficients(d, N),
                2: face_gather_index(mesh, t, dops_all, perm_tri, perm_quad, face_offsets, N, sem)}
    if t == "tet":
        return {0: d["face_nodes"], 1: tet_gather_index(mesh, d, perm_tri, face_offsets)}
    return {1: face_gather_index(mesh, t, dops_all, perm_tri, perm_quad, face_offsets, N, sem)}


class DeviceMesh:
    """Owns every device tensor the kernels read and the C struct pointing
    at them."""

    def __init__(self, disc, device, dtype=torch.float64):
        if dtype not in (torch.float64, torch.float32):
            raise ValueError("dtype must be float64 or float32")
        self.device = torch.device(device)
        self.dtype = dtype
        self.N = disc.N
        self._keep = []
        self.pack = pack = pack_mesh(disc)
        S = nat.HWMesh()
        S.N = disc.N
        S.dtype = nat.HW_F64 if dtype == torch.float64 else nat.HW_F32
        S.formulation = nat.HW_GL if disc.formulation.kind == "GL" else nat.HW_SEM
        S.penalty_scale = float(disc.penalty_scale)
        S.device = (self.device.index if self.device.index is not None
                    else torch.cuda.current_device())
        for t, P in pack["types"].items():
            T = S.t[TYPE_ID[t]]
            T.K = P["K"]
            T.form = nat.HW_FORM_SKEW if P["form"] == "skew" else nat.HW_FORM_STRONG
            T.geo = self._put(P["geo"])
            T.mat = self._put(P["mat"])
            T.nbr_elem = self._put(P["nbr_elem"], torch.int32)
            T.nbr_code = self._put(P["nbr_code"], torch.int32)
            for slot, arr in P["op"].items():
                # DMMA operand fragments are fp64 for both storage precisions
                T.op[slot] = self._put(arr, torch.float64 if slot in MMA_SLOTS[t] else None)
            for slot, arr in P["iop"].items():
                T.iop[slot] = self._put(arr, torch.int32)
        S.perm_tri = self._put(pack["perm_tri"], torch.int32)
        S.perm_quad = self._put(pack["perm_quad"], torch.int32)
        # face-trace buffers (ping-pong) of the publishing types
        self.traces = [[None] * 4, [None] * 4]
        for t, P in pack["types"].items():
            if P["publishes"]:
                for b in range(2):
                    self.traces[b][TYPE_ID[t]] = torch.zeros((P["K"], 4, P["nfp"]),
                                                             dtype=dtype, device=self.device)
        self.struct = S
        self.set_traces(0, None)
        # tet / pyramid faces across non-affine wedge triangles (face-cubature correction)
        self.corr = {}
        for t, c in wedge_face_corrections(disc, pack).items():
            self.corr[t] = {"n": int(len(c["idata"])), "nq": c["nq"], "nfn": c["nfn"],
                            "idata": torch.as_tensor(c["idata"], device=self.device),
                            "fdata": torch.as_tensor(c["fdata"], device=self.device),
                            "L": torch.as_tensor(c["L"], device=self.device),
                            "P": torch.as_tensor(c["P"], device=self.device),
                            "elems": torch.as_tensor(np.unique(c["idata"][:, 0]).astype(np.int64),
                                                     device=self.device)}
        orders = nat.lib().hw_supported_orders()
        if not (orders >> disc.N) & 1:
            raise ValueError(f"order N={disc.N} not compiled into {nat.LIB_NAME}")
        nat.check(nat.lib().hw_prepare(self.struct))

    def set_traces(self, tin, tout):
        """Point the struct's tr_in / tr_out at trace buffer sets (0/1/None)."""
        for i in range(4):
            a = self.traces[tin][i] if tin is not None else None
            b = self.traces[tout][i] if tout is not None else None
            self.struct.tr_in[i] = a.data_ptr() if a is not None else None
            self.struct.tr_out[i] = b.data_ptr() if b is not None else None

    def compute_traces(self, q_fields, buf, stream, subset=None):
        """hw_traces: face traces of q (HWFields) into trace set `buf`
        (optionally only for the elements of an HWSubset)."""
        nat.check(nat.lib().hw_traces(self.struct, q_fields, nat.fields(self.traces[buf]), subset,
                                      stream))

    def _put(self, arr, dtype=None):
        t = torch.as_tensor(np.ascontiguousarray(arr), dtype=dtype or self.dtype).to(self.device)
        self._keep.append(t)
        return t.data_ptr()


def _hex_nodes(d):
    # 1-D node coordinates: the quad face rule's 1-D points (GL or GLL)
    n1 = len(d["w1"])
    return d["quad2d"][::n1, 0].copy()
