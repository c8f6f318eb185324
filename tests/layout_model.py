"""Numpy model of the device kernels over the exact packed layout
(device.pack_mesh): same tables, same index arithmetic, vectorised over
elements.  Lets the CPU suite check the compact HBM layout, the face
permutations and the nodal-face lifts against the oracle without a GPU."""

import numpy as np

NAMES = ["hex", "wedge", "pyramid", "tet"]
BND = 0x200


def _dims(N):
    n1 = N + 1
    return dict(N1=n1, NFQ=n1 * n1, NFN=(N + 1) * (N + 2) // 2)


def face_layout(t, N):
    """[(face type, offset, count)] of the device face-point ordering."""
    d = _dims(N)
    if t == "hex":
        return [("quad", f * d["NFQ"], d["NFQ"]) for f in range(6)]
    if t == "tet":
        return [("tri", f * d["NFN"], d["NFN"]) for f in range(4)]
    if t == "wedge":
        return ([("tri", f * d["NFN"], d["NFN"]) for f in range(2)]
                + [("quad", 2 * d["NFN"] + f * d["NFQ"], d["NFQ"]) for f in range(3)])
    return ([("quad", 0, d["NFQ"])]
            + [("tri", d["NFQ"] + f * d["NFN"], d["NFN"]) for f in range(4)])


def own_traces(pack, t, q, N, sem):
    """(K, 4, Nfp) traces at the device face points, as the kernels form them."""
    P = pack["types"][t]
    if t == "tet":
        return q[:, :, P["iop"][0]]
    if t == "hex":
        tab = P["iop"][0]
        base, stride, end = tab[:, 0], tab[:, 1], tab[:, 2]
        if sem:
            return q[:, :, base + np.where(end == 1, N, 0) * stride]
        Vend = P["op"][1]
        out = 0.0
        for l in range(N + 1):
            out = out + Vend[end, l][None, None, :] * q[:, :, base + l * stride]
        return out
    ET = P["op"][5]                                    # (Np, Nfp)
    tr = q @ ET
    if t == "wedge":
        tr = tr * P["geo"][:, 9][:, None, None]
    return tr


def _hex_metric(X, r, s, t):
    """X (K, 8, 3) -> G (K, 3, 3) [c][x], J (K,) at one reference point."""
    sg = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                   [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], float)
    p = np.array([r, s, t])
    fac = 0.5 * (1 + sg * p)
    g = np.empty((8, 3))
    g[:, 0] = 0.5 * sg[:, 0] * fac[:, 1] * fac[:, 2]
    g[:, 1] = 0.5 * sg[:, 1] * fac[:, 0] * fac[:, 2]
    g[:, 2] = 0.5 * sg[:, 2] * fac[:, 0] * fac[:, 1]
    F = np.einsum("kvx,vc->kxc", X, g)
    return np.linalg.inv(F), np.linalg.det(F)


_HEX_FV = [(0, 4, 7, 3), (1, 2, 6, 5), (0, 1, 5, 4), (2, 3, 7, 6), (0, 3, 2, 1), (4, 5, 6, 7)]


def rhs(pack, disc, state, traces=None):
    """dU/dtau of every type from the packed layout (fp64).  traces: optional
    dict t -> (K, 4, Nfp) replacing the traces formed from the state (the
    partitioned path delivers ghost traces through the face halo)."""
    N = disc.N
    sem = disc.formulation.kind == "SEM"
    d = _dims(N)
    q = {t: np.asarray(state[t], dtype=float) for t in disc.types}
    own = {t: own_traces(pack, t, q[t], N, sem) for t in disc.types}
    traces = {t: (traces[t] if traces is not None and t in traces else own[t])
              for t in disc.types}
    out = {}
    for t in disc.types:
        P = pack["types"][t]
        K = P["K"]
        Np = q[t].shape[2]
        geo, mat = P["geo"], P["mat"]
        acc = np.zeros((K, 4, Np))
        # ---------------- volume
        if t == "tet" or t == "pyramid":
            G = geo[:, :9].reshape(K, 3, 3)
            v = np.einsum("kcx,kxn->kcn", G, q[t][:, 1:])
            DT = P["op"][0]                     # [c][m][n] = D_c[n][m]
            dp = np.einsum("cmn,km->kcn", DT, q[t][:, 0])
            if t == "pyramid" and P["form"] == "skew":
                acc[:, 0] = np.einsum("cmn,kcm->kn", P["op"][1], v)
            else:
                acc[:, 0] = -np.einsum("cmn,kcm->kn", DT, v)
            acc[:, 1:] = -np.einsum("kcx,kcn->kxn", G, dp)
        elif t == "wedge":
            # affine LSC wedge: S_c = V^T W D3_c, same data flow as the skew pyramid
            G = geo[:, :9].reshape(K, 3, 3)
            v = np.einsum("kcx,kxn->kcn", G, q[t][:, 1:])
            dp = np.einsum("cmn,km->kcn", P["op"][0], q[t][:, 0])
            acc[:, 0] = np.einsum("cmn,kcm->kn", P["op"][1], v)
            acc[:, 1:] = -np.einsum("kcx,kcn->kxn", G, dp)
        else:  # hex
            n1 = d["N1"]
            X = geo[:, :24].reshape(K, 8, 3)
            x1 = P["op"][4]
            D1 = P["op"][0]
            u = q[t].reshape(K, 4, n1, n1, n1)
            der = [np.einsum("il,kflmn->kfimn", D1, u), np.einsum("jl,kfiln->kfijn", D1, u),
                   np.einsum("ml,kfijl->kfijm", D1, u)]
            minv = np.empty((K, Np))
            for n in range(Np):
                i, j, k = n // (n1 * n1), (n // n1) % n1, n % n1
                G, J = _hex_metric(X, x1[i], x1[j], x1[k])
                dd = np.stack([der[c][:, :, i, j, k] for c in range(3)], axis=2)  # (K,4,3)
                acc[:, 1:, n] = -np.einsum("kcx,kc->kx", G, dd[:, 0])
                acc[:, 0, n] = -np.einsum("kcx,kxc->k", G, dd[:, 1:])
                w1 = P["op"][2]
                minv[:, n] = 1.0 / (w1[i] * w1[j] * w1[k] * J)
        # ---------------- surface
        lay = face_layout(t, N)
        nfp = lay[-1][1] + lay[-1][2]
        flux = np.zeros((K, 4 if t == "hex" else 2, nfp))
        zm = mat[:, 2]
        for f, (ft, off, cnt) in enumerate(lay):
            own = traces[t][:, :, off:off + cnt]
            code = P["nbr_code"][:, f]
            k2 = P["nbr_elem"][:, f]
            oth = np.empty_like(own)
            b = (code & BND) != 0
            oth[b, 0] = -own[b, 0]
            oth[b, 1:] = own[b, 1:]
            for tid2, t2 in enumerate(NAMES):
                sel = (~b) & ((code & 3) == tid2)
                if not sel.any():
                    continue
                f2 = (code[sel] >> 2) & 7
                pc = (code[sel] >> 5) & 15
                perm = (pack["perm_tri"] if ft == "tri" else pack["perm_quad"])[pc]   # (n, cnt)
                lay2 = face_layout(t2, N)
                off2 = np.array([lay2[x][1] for x in f2])
                cols = off2[:, None] + perm
                tr2 = traces[t2][k2[sel]]                                      # (n,4,nfp2)
                oth[sel] = np.take_along_axis(tr2, np.repeat(cols[:, None, :], 4, axis=1), axis=2)
                if t in ("wedge", "pyramid", "hex"):
                    # the kernels' path: host gather index into the source array
                    direct = t2 in ("hex", "tet") and (t2 == "tet" or sem)
                    src = q[t2] if direct else traces[t2]
                    g = P["iop"][2 if t == "hex" else 1][sel, off:off + cnt]
                    got = np.stack([src.reshape(-1)[g + c * src.shape[2]] for c in range(4)],
                                   axis=1)
                    assert np.array_equal(got, oth[sel]), (t, f, t2)
            if t == "hex":
                avg, inv = geo[:, 24 + 2 * f], geo[:, 25 + 2 * f]
            else:
                b0 = (10 if t == "wedge" else 9) + 6 * f
                avg, inv = geo[:, b0 + 4], geo[:, b0 + 5]
            tp = disc.penalty_scale * inv
            tu = disc.penalty_scale * avg
            if t == "hex":
                # per-point normal and Js from the face vertices
                X = geo[:, :24].reshape(K, 8, 3)[:, list(_HEX_FV[f])]
                x1 = P["op"][4]
                n1 = d["N1"]
                jj = np.arange(cnt)
                xi, eta = x1[jj // n1], x1[jj % n1]
                g1 = np.stack([-(1 - eta), (1 - eta), (1 + eta), -(1 + eta)]) * 0.25
                g2 = np.stack([-(1 - xi), -(1 + xi), (1 + xi), (1 - xi)]) * 0.25
                t1 = np.einsum("kvx,vp->kpx", X, g1)
                t2_ = np.einsum("kvx,vp->kpx", X, g2)
                nv = np.cross(t1, t2_)
                Js = np.linalg.norm(nv, axis=2)
                nrm = nv / Js[..., None]                                     # (K,cnt,3)
                w1 = P["op"][2]
                scale = w1[jj // n1] * w1[jj % n1] * Js
            else:
                base = 10 if t == "wedge" else 9
                nrm = np.repeat(geo[:, base + 6 * f: base + 6 * f + 3][:, None, :], cnt, axis=1)
                scale = np.repeat(geo[:, base + 6 * f + 3][:, None], cnt, axis=1)
            unm = np.einsum("kpx,kxp->kp", nrm, own[:, 1:])
            unp = np.einsum("kpx,kxp->kp", nrm, oth[:, 1:])
            dp_ = oth[:, 0] - own[:, 0]
            dun = unp - unm
            skew = P["form"] == "skew"
            fp = (0.5 * tp[:, None] * dp_ - 0.5 * (unp + unm)) if skew else \
                0.5 * (tp[:, None] * dp_ - dun)
            fu = 0.5 * (tu[:, None] * dun - dp_)
            if t == "hex":
                flux[:, 0, off:off + cnt] = fp * scale
                flux[:, 1:, off:off + cnt] = np.moveaxis(nrm, 2, 1) * (fu * scale)[:, None, :]
            else:
                flux[:, 0, off:off + cnt] = fp * scale
                flux[:, 1, off:off + cnt] = fu * scale
        # ---------------- lift
        if t == "hex":
            n1 = d["N1"]
            Vend = P["op"][1]
            nfp_tab = P["iop"][1]
            lift = np.zeros_like(acc)
            for n in range(Np):
                idx = (n // (n1 * n1), (n // n1) % n1, n % n1)
                for f in range(6):
                    axis, end = f >> 1, f & 1
                    l = idx[axis]
                    if sem:
                        if l != (N if end else 0):
                            continue
                        w = 1.0
                    else:
                        w = Vend[end, l]
                    pt = nfp_tab[f, n]
                    lift[:, :, n] += w * flux[:, :, f * d["NFQ"] + pt]
            acc += lift * minv[:, None, :]
        else:
            LT = P["op"][1] if t == "tet" else P["op"][6]          # (Nfp, Np)
            base = 10 if t == "wedge" else 9
            for f, (ft, off, cnt) in enumerate(lay):
                tp_ = flux[:, 0, off:off + cnt] @ LT[off:off + cnt]
                tu_ = flux[:, 1, off:off + cnt] @ LT[off:off + cnt]
                acc[:, 0] += tp_
                acc[:, 1:] += geo[:, base + 6 * f: base + 6 * f + 3][:, :, None] * tu_[:, None, :]
        acc[:, 0] *= mat[:, 0][:, None]
        acc[:, 1:] *= mat[:, 1][:, None, None]
        out[t] = acc
    return out


def naw_rhs(pack, disc, state):
    """Model of the non-affine wedge path (Naw in csrc/hw_kernels.cuh) for
    all-wedge meshes: cubature volume passes, per-point quad faces, triangle
    faces at the reference's cubature through the nodal polynomial traces."""
    N = disc.N
    d = _dims(N)
    P = pack["types"]["wedge"]
    K = P["K"]
    q = np.asarray(state["wedge"], dtype=float)
    Np = q.shape[2]
    nq, nqt, nfn = (N + 1) ** 3, 3 * (N + 1) ** 2, d["NFN"]   # deduplicated triangle rule
    lay = face_layout("wedge", N)
    nfp = lay[-1][1] + lay[-1][2]
    GF, GT = nq * 12, nq * 12 + nfp * 5
    g8, cst = P["op"][8], P["op"][9]
    o = np.cumsum([0, 4 * Np * nq, 4 * Np * nq, 2 * nqt * nfn])
    VT = cst[o[0]:o[1]].reshape(4, Np, nq)
    VN = cst[o[1]:o[2]].reshape(4, nq, Np)
    LQ = cst[o[2]:o[3]].reshape(2, nqt, nfn)
    VF = cst[o[3]:].reshape(2, nqt, Np)
    vol = g8[:, :GF].reshape(K, nq, 12)
    fq = g8[:, GF:GT].reshape(K, nfp, 5)
    tb = g8[:, GT:].reshape(K, 2, nqt, 3)
    geo, mat = P["geo"], P["mat"]
    acc = np.zeros((K, 4, Np))
    U = np.einsum("mq,kfm->kfq", VT[0], q)
    dc = np.einsum("cmq,km->kcq", VT[1:], q[:, 0])
    wG = vol[..., :9].reshape(K, nq, 3, 3)
    wgJ = vol[..., 9:]
    gp = np.einsum("kqcx,kcq->kxq", wG, dc) + wgJ.transpose(0, 2, 1) * U[:, 0][:, None, :]
    up = np.einsum("kqcx,kxq->kcq", wG, U[:, 1:])
    uj = np.einsum("kqx,kxq->kq", wgJ, U[:, 1:])
    acc[:, 1:] = -np.einsum("qn,kxq->kxn", VN[0], gp)
    acc[:, 0] = np.einsum("cqn,kcq->kn", VN[1:], up) + uj @ VN[0]
    # published traces: quad points x 1/sqrt(J), triangle points polynomial
    tr = q @ P["op"][5]
    isj = np.ones((K, nfp))
    isj[:, 2 * nfn:] = fq[:, 2 * nfn:, 4]
    tr = tr * isj[:, None, :]
    LT = P["op"][6]
    for f, (ft, off, cnt) in enumerate(lay):
        own = tr[:, :, off:off + cnt]
        code = P["nbr_code"][:, f]
        k2 = P["nbr_elem"][:, f]
        b = (code & BND) != 0
        oth = np.zeros_like(own)
        sel = ~b
        if sel.any():
            f2 = (code[sel] >> 2) & 7
            pc = (code[sel] >> 5) & 15
            perm = (pack["perm_tri"] if ft == "tri" else pack["perm_quad"])[pc]
            off2 = np.array([lay[x][1] for x in f2])
            cols = off2[:, None] + perm
            oth[sel] = np.take_along_axis(tr[k2[sel]], np.repeat(cols[:, None, :], 4, axis=1),
                                          axis=2)
        if ft == "tri":
            own = np.einsum("qj,kcj->kcq", LQ[f], own) * tb[:, f, None, :, 0]
            oth = np.einsum("qj,kcj->kcq", LQ[f], oth) * tb[:, f, None, :, 1]
            npts = nqt
            nrm = np.repeat(geo[:, 10 + 6 * f:13 + 6 * f][:, None, :], npts, axis=1)
            scale = tb[:, f, :, 2]
        else:
            npts = cnt
            nrm = fq[:, off:off + cnt, :3]
            scale = fq[:, off:off + cnt, 3]
        oth[b, 0] = -own[b, 0]
        oth[b, 1:] = own[b, 1:]
        avg, inv = geo[:, 10 + 6 * f + 4], geo[:, 10 + 6 * f + 5]
        tp = disc.penalty_scale * inv
        tu = disc.penalty_scale * avg
        unm = np.einsum("kpx,kxp->kp", nrm, own[:, 1:])
        unp = np.einsum("kpx,kxp->kp", nrm, oth[:, 1:])
        dp_ = oth[:, 0] - own[:, 0]
        dun = unp - unm
        skew = P["form"] == "skew"
        fp = (0.5 * tp[:, None] * dp_ - 0.5 * (unp + unm)) if skew else \
            0.5 * (tp[:, None] * dp_ - dun)
        fu = 0.5 * (tu[:, None] * dun - dp_)
        L = VF[f] if ft == "tri" else LT[off:off + cnt]
        acc[:, 0] += (fp * scale) @ L
        acc[:, 1:] += np.einsum("kpx,kp,pn->kxn", nrm, fu * scale, L)
    acc[:, 0] *= mat[:, 0][:, None]
    acc[:, 1:] *= mat[:, 1][:, None, None]
    return {"wedge": acc}
