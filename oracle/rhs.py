"""TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference RHS.

Works on a discretization bundle exposing the reference layouts:
``types, n_elems, ops[t], data[t], gather_idx, bnd_mask, trace_bases,
trace_size, forms, penalty_scale, mesh.materials`` (the product's
``Discretization`` provides them, built on the host and pinned against the
reference by tests/test_setup_golden.py).  Arithmetic follows the reference
line by line (fp64 numpy).
"""

import numpy as np

NF = 4  # p, u1, u2, u3


def compute_traces(b, state):
    """hybridwave/dg.py:299-316: traces = state @ Vf^T, wedge x 1/sqrt(J)."""
    out = np.empty((NF, b.trace_size))
    for t in b.types:
        op, d = b.ops[t], b.data[t]
        tr = np.asarray(state[t]) @ op.Vf.T
        if t == "wedge":
            tr = tr * d.invsqrtJ_face[:, None, :]
        n = b.n_elems[t] * op.face_offsets[-1]
        base = b.trace_bases[t]
        out[:, base:base + n] = np.moveaxis(tr, 1, 0).reshape(NF, n)
    return out


def exterior_traces(b, traces):
    """hybridwave/dg.py:318-324: mapP gather, mirror ghost p+=-p-, u+=u-."""
    ext = traces[:, b.gather_idx]
    m = b.bnd_mask
    ext[0, m] = -traces[0, m]
    ext[1:, m] = traces[1:, m]
    return ext


def surface_residual(b, t, traces, ext):
    """hybridwave/dg.py:326-354."""
    op, d = b.ops[t], b.data[t]
    K = b.n_elems[t]
    tot = op.face_offsets[-1]
    base = b.trace_bases[t]
    own = np.moveaxis(traces[:, base:base + K * tot].reshape(NF, K, tot), 0, 1)
    oth = np.moveaxis(ext[:, base:base + K * tot].reshape(NF, K, tot), 0, 1)
    n = d.normals                                  # (K, tot, 3)
    jump_p = oth[:, 0] - own[:, 0]
    un_m = np.einsum("kqd,kdq->kq", n, own[:, 1:])
    un_p = np.einsum("kqd,kdq->kq", n, oth[:, 1:])
    jump_un = un_p - un_m
    tp = b.penalty_scale * d.tau_p
    tu = b.penalty_scale * d.tau_u
    if b.forms[t] == "skew":
        fp = 0.5 * tp * jump_p - 0.5 * (un_p + un_m)
    else:
        fp = 0.5 * (tp * jump_p - jump_un)
    fun = 0.5 * (tu * jump_un - jump_p)
    flux = np.empty((K, NF, tot))
    flux[:, 0] = fp
    flux[:, 1:] = np.moveaxis(n, 2, 1) * fun[:, None, :]
    flux *= d.wJs[:, None, :]
    if t == "wedge":
        flux *= d.invsqrtJ_face[:, None, :]
    return flux @ op.Vf


def _vol_hex(b, q):
    """hybridwave/dg.py:371-399."""
    op, d = b.ops["hex"], b.data["hex"]
    K = q.shape[0]
    n1 = b.N + 1
    u = q.reshape(K, NF, n1, n1, n1)
    D = op.D1
    der = np.stack([np.einsum("il,kflmn->kfimn", D, u).reshape(K, NF, -1),
                    np.einsum("jl,kfiln->kfijn", D, u).reshape(K, NF, -1),
                    np.einsum("ml,kfijl->kfijm", D, u).reshape(K, NF, -1)], axis=2)
    G = d.G
    wJ = d.w3[None, :] * d.J
    R = np.zeros_like(q)
    R[:, 1:] = -wJ[:, None, :] * np.einsum("kqcx,kcq->kxq", G, der[:, 0])
    if b.forms["hex"] == "strong":
        R[:, 0] = -wJ * np.einsum("kqcx,kxcq->kq", G, der[:, 1:])
    else:
        pre = np.einsum("kqcx,kxq,kq->kcq", G, q[:, 1:], wJ).reshape(K, 3, n1, n1, n1)
        R[:, 0] = (np.einsum("li,klmn->kimn", D, pre[:, 0]).reshape(K, -1)
                   + np.einsum("lj,kilm->kijm", D, pre[:, 1]).reshape(K, -1)
                   + np.einsum("lm,kijl->kijm", D, pre[:, 2]).reshape(K, -1))
    return R


def _vol_tet(b, q):
    """hybridwave/dg.py:401-421."""
    op, d = b.ops["tet"], b.data["tet"]
    G, J = d.G[:, 0], d.J[:, 0]
    der = np.stack([q @ op.Dr.T, q @ op.Ds.T, q @ op.Dt.T], axis=2)
    R = np.zeros_like(q)
    if b.forms["tet"] == "strong":
        R[:, 0] = -J[:, None] * (np.einsum("kcx,kxcq->kq", G, der[:, 1:]) @ op.M_ref.T)
    else:
        tmp = np.einsum("kcx,kxq->kcq", G, q[:, 1:] @ op.M_ref.T)
        R[:, 0] = J[:, None] * (tmp[:, 0] @ op.Dr + tmp[:, 1] @ op.Ds + tmp[:, 2] @ op.Dt)
    R[:, 1:] = -J[:, None, None] * (np.einsum("kcx,kcq->kxq", G, der[:, 0]) @ op.M_ref.T)
    return R


def _vol_wedge(b, q):
    """hybridwave/dg.py:423-444 (two-pass skew LSC-DG)."""
    op, d = b.ops["wedge"], b.data["wedge"]
    w = op.cub.weights
    U = q @ op.V.T
    der = np.stack([q @ op.Dr3.T, q @ op.Ds3.T, q @ op.Dt3.T], axis=2)
    gp = (np.einsum("kqcx,kcq->kxq", d.G, der[:, 0])
          + np.moveaxis(d.gJfac, 2, 1) * U[:, 0][:, None, :])
    R = np.zeros_like(q)
    R[:, 1:] = -(gp * w[None, None, :]) @ op.V
    pre = np.einsum("kqcx,kxq->kcq", d.G, U[:, 1:]) * w[None, None, :]
    uj = np.einsum("kqx,kxq->kq", d.gJfac, U[:, 1:]) * w[None, :]
    R[:, 0] = pre[:, 0] @ op.Dr3 + pre[:, 1] @ op.Ds3 + pre[:, 2] @ op.Dt3 + uj @ op.V
    return R


def _vol_pyramid(b, q):
    """hybridwave/dg.py:446-463 (quadrature-free semi-nodal)."""
    op, d = b.ops["pyramid"], b.data["pyramid"]
    G, J = d.G, d.J
    der = np.stack([q @ op.Dr.T, q @ op.Ds.T, q @ op.Dt.T], axis=2)
    R = np.zeros_like(q)
    R[:, 1:] = -J[:, None, :] * np.einsum("kqcx,kcq->kxq", G, der[:, 0])
    if b.forms["pyramid"] == "strong":
        R[:, 0] = -J * np.einsum("kqcx,kxcq->kq", G, der[:, 1:])
    else:
        pre = np.einsum("kqcx,kxq->kcq", G, q[:, 1:]) * J[:, None, :]
        R[:, 0] = pre[:, 0] @ op.Dr + pre[:, 1] @ op.Ds + pre[:, 2] @ op.Dt
    return R


_VOL = {"hex": _vol_hex, "tet": _vol_tet, "wedge": _vol_wedge, "pyramid": _vol_pyramid}


def volume_residual(b, t, q):
    return _VOL[t](b, np.asarray(q))


def apply_A(b, state):
    """hybridwave/dg.py:469-477."""
    tr = compute_traces(b, state)
    ext = exterior_traces(b, tr)
    return {t: volume_residual(b, t, state[t]) + surface_residual(b, t, tr, ext)
            for t in b.types}


def mass_inverse(b, t, R):
    """hybridwave/dg.py:479-490."""
    op, d = b.ops[t], b.data[t]
    if t == "hex":
        return R / (d.w3[None, None, :] * d.J[:, None, :])
    if t == "tet":
        return (R @ op.invM_ref.T) / d.J[:, 0][:, None, None]
    if t == "wedge":
        return R
    return R / d.J[:, None, :]


def compute_rhs(b, state, time=0.0):
    """hybridwave/dg.py:492-506 (forcing = None)."""
    res = apply_A(b, state)
    out = {}
    for t in b.types:
        dm = mass_inverse(b, t, res[t])
        mat = b.mesh.materials[t]
        dm[:, 0] *= mat[:, 1][:, None]
        dm[:, 1:] *= (1.0 / mat[:, 0])[:, None, None]
        out[t] = dm
    return out
