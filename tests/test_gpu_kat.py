"""The reference specification's known-answer tests for the hot path
(SPEC.md:479-518), run on the device kernels through the C ABI."""
import numpy as np
import pytest
import torch

import oracle
from conftest import build_mesh, rel_err

pytestmark = pytest.mark.gpu


def _disc(spec, N, form, **kw):
    from paper_1507_02557_b200.dg import Discretization
    return Discretization(build_mesh(spec), N, form, **kw)


def _interior(d, t):
    """Elements of type t with no boundary face."""
    return np.flatnonzero(np.all(d.mesh.nbr[t][:, :, 0] >= 0, axis=1))


def _const(p, u):
    def f(x, tau):
        out = np.empty(x.shape[:-1] + (4,))
        out[..., 0] = p
        out[..., 1:] = u
        return out
    return f


@pytest.mark.parametrize("N,form", [(1, "GL"), (2, "SEM"), (3, "GL"), (4, "SEM"), (5, "GL")])
def test_constant_state_interior_rhs_is_zero(N, form, native_lib):
    """constant p, constant u -> zero jumps, zero gradients:
    the RHS of every interior element vanishes (here: |rhs| <= 1e-11 x the
    RHS scale of a unit random state)."""
    d = _disc("hybrid:4", N, form)
    st = d.project(_const(1.7, (0.3, -0.8, 0.5)), 0.0)
    r = d.compute_rhs(st)
    rng = np.random.default_rng(0)
    scale = max(np.abs(v).max() for v in d.compute_rhs(
        {t: rng.standard_normal(st[t].shape) for t in d.types}).values())
    for t in d.types:
        ids = _interior(d, t)
        if len(ids):
            assert np.abs(r[t][ids]).max() <= 1e-11 * scale, t


@pytest.mark.parametrize("N,form", [(2, "GL"), (3, "SEM"), (4, "GL")])
def test_unit_pressure_traces(N, form, native_lib):
    """p = 1 -> every p-trace equals 1 within 1e-13 (device
    compute_traces at the reference's stored face points)."""
    d = _disc("hybrid:3", N, form)
    st = d.project(_const(1.0, (0.0, 0.0, 0.0)), 0.0)
    tr = d.compute_traces(d.to_device(st))
    assert isinstance(tr, torch.Tensor) and tr.is_cuda
    tr = tr.cpu().numpy()
    assert np.abs(tr[0] - 1.0).max() < 1e-13
    assert np.abs(tr[1:]).max() < 1e-13


def test_gl_hex_trace_of_r(native_lib):
    """GL hex, u = r -> the trace at the r = +1 face is 1
    (endpoint extrapolation of the 1-D GL interpolant)."""
    from paper_1507_02557_b200.refelem import FACES
    d = _disc("hex:1", 3, "GL")
    n1 = d.ops["hex"].nodes1d
    r = np.repeat(n1, len(n1) ** 2)                       # node order: t fastest, r slowest
    st = {"hex": np.zeros((1, 4, len(r)))}
    st["hex"][0, 1] = r
    tr = d.compute_traces(d.to_device(st)).cpu().numpy()
    op = d.ops["hex"]
    # the face whose reference normal is +r: evaluate r there
    for f, (_, ix) in enumerate(FACES["hex"]):
        sl = slice(op.face_offsets[f], op.face_offsets[f + 1])
        rv = op.face_rst[sl, 0]
        np.testing.assert_allclose(tr[1, sl], rv, atol=1e-12)


@pytest.mark.parametrize("spec,N,form", [("hybrid:2", 3, "GL"), ("hybrid:3", 2, "SEM"),
                                          ("tet:2", 4, "GL"), ("hex:2", 5, "GL")])
def test_energy_of_unit_pressure_is_volume(spec, N, form, native_lib):
    """p = 1, u = 0, kappa = 1 on the unit cube -> U^T M U = 1
    (device hw_energy)."""
    d = _disc(spec, N, form)
    st = d.project(_const(1.0, (0.0, 0.0, 0.0)), 0.0)
    assert abs(float(d.energy_device(d.to_device(st))) - 1.0) < 1e-12
    zero = {t: np.zeros_like(v) for t, v in st.items()}
    assert float(d.energy_device(d.to_device(zero))) == 0.0


@pytest.mark.parametrize("spec,N,over", [("tet:2", 3, {"tet": "skew"}),
                                          ("hex:2", 4, {"hex": "skew"}),
                                          ("pyramid:2", 3, {"pyramid": "skew"}),
                                          ("hybrid:3", 3, {"tet": "skew", "hex": "skew",
                                                           "pyramid": "skew"})])
def test_strong_equals_skew(spec, N, over, native_lib):
    """strong and skew forms agree for planar tets, GL hexes
    and GL pyramids (the device RHS of both forms on random states, 1e-10;
    A is linear, so agreement on random vectors is agreement of A)."""
    strong = _disc(spec, N, "GL")
    skew = _disc(spec, N, "GL", forms_override=over)
    rng = np.random.default_rng(5)
    for _ in range(3):
        st = {t: rng.standard_normal((strong.n_elems[t], 4, strong.ops[t].Np))
              for t in strong.types}
        a, b = strong.compute_rhs(st), skew.compute_rhs(st)
        num = np.sqrt(sum(float(np.sum((a[t] - b[t]) ** 2)) for t in a))
        den = np.sqrt(sum(float(np.sum(a[t] ** 2)) for t in a))
        assert num <= 1e-10 * den


def _poly(deg):
    """A global polynomial field of total degree deg and its exact RHS
    (-div u, -grad p) for rho = kappa = 1."""
    c = np.random.default_rng(deg).uniform(-1, 1, (4, 3))

    def mono(x, k):        # sum_i c_k,i x_i^deg + x0 x1 x2 products for deg >= 3
        v = sum(c[k, i] * x[..., i] ** deg for i in range(3))
        if deg >= 3:
            v = v + c[k, 0] * x[..., 0] * x[..., 1] * x[..., 2] ** (deg - 2)
        return v

    def dmono(x, k, j):
        v = c[k, j] * deg * x[..., j] ** (deg - 1)
        if deg >= 3:
            x0, x1, x2 = x[..., 0], x[..., 1], x[..., 2]
            v = v + c[k, 0] * ([x1 * x2 ** (deg - 2), x0 * x2 ** (deg - 2),
                                (deg - 2) * x0 * x1 * x2 ** (deg - 3)][j])
        return v

    def fields(x, tau):
        return np.stack([mono(x, k) for k in range(4)], axis=-1)

    def rhs(x, tau):
        out = np.empty(x.shape[:-1] + (4,))
        out[..., 0] = -(dmono(x, 1, 0) + dmono(x, 2, 1) + dmono(x, 3, 2))
        for j in range(3):
            out[..., 1 + j] = -dmono(x, 0, j)
        return out
    return fields, rhs


@pytest.mark.parametrize("N,form", [(2, "GL"), (3, "GL"), (3, "SEM"), (4, "GL")])
def test_polynomial_preservation(N, form, native_lib):
    """a state in the approximation space with a continuous
    global trace has zero jumps, so on interior elements the RHS is the
    exact derivative (-div u, -grad p) of the polynomial (1e-11)."""
    d = _disc("hybrid:3", N, form)
    fields, rhs = _poly(N)
    st = d.project(fields, 0.0)
    got = d.compute_rhs(st)
    assert rel_err(got, oracle.compute_rhs(d, st)) < 1e-12
    exp = d.project(rhs, 0.0)
    for t in d.types:
        ids = _interior(d, t)
        # SEM integrates quad faces with the (N+1)-point GLL rule (exact to
        # degree 2N-1); the skew forms' average-flux term on them (wedge,
        # SEM pyramid) is degree 2N, so the reference itself does not
        # preserve polynomials there (its RHS = the oracle's, asserted above)
        if form == "SEM" and d.forms[t] == "skew":
            continue
        if len(ids):
            scale = np.abs(exp[t][ids]).max()
            assert np.abs(got[t][ids] - exp[t][ids]).max() <= 1e-11 * max(scale, 1.0), t


@pytest.mark.parametrize("case", [0, 6, 10, 15])
def test_apply_A_and_mass_inverse_on_device(case, native_lib):
    """Public per-operation methods on the device: apply_A = A U (no mass
    inverse, no materials) and apply_mass_inverse reproduce the oracle
    (hybridwave/dg.py:469-490), and M^-1 diag(kappa, 1/rho) A U = RHS."""
    from conftest import make_case
    d, st = make_case(case)
    q = d.to_device(st)
    A = d.apply_A(q)
    assert all(v.is_cuda for v in A.values())
    ref = oracle.apply_A(d, st)
    assert rel_err({t: v.cpu().numpy() for t, v in A.items()}, ref) < 1e-12
    for t in d.types:
        mi = d.apply_mass_inverse(t, A[t])
        assert mi.is_cuda
        exp = oracle.mass_inverse(d, t, ref[t])
        assert np.abs(mi.cpu().numpy() - exp).max() <= 1e-12 * np.abs(exp).max()
    host = d.apply_A(st)
    assert isinstance(next(iter(host.values())), np.ndarray)
    assert rel_err(host, ref) < 1e-12


@pytest.mark.parametrize("case", [2, 10, 13])
def test_compute_traces_matches_oracle(case, native_lib):
    """Device compute_traces (4, trace_size) in the reference's flat layout
    (hybridwave/dg.py:299-316) against the oracle."""
    from conftest import make_case
    d, st = make_case(case)
    got = d.compute_traces(d.to_device(st)).cpu().numpy()
    ref = oracle.compute_traces(d, st)
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    host = d.compute_traces(st)
    assert isinstance(host, np.ndarray)
    assert np.abs(host - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs a second GPU")
def test_second_device(native_lib):
    """A Discretization on cuda:1 launches on cuda:1 while cuda:0 is current
    (the mesh's ordinal is made current inside every ABI call)."""
    from conftest import make_case
    d, st = make_case(6, device="cuda:1")
    with torch.cuda.device(0):
        r = d.compute_rhs(st)
    assert rel_err(r, oracle.compute_rhs(d, st)) < 1e-12


def _host_l2(d, state, exact_fn, time):
    """hybridwave/dg.py:558-572 in numpy (the check for the device version)."""
    tot = {"p": 0.0, "u": 0.0}
    for t in d.types:
        w, V, x, J = d._cubature(t, "over")
        num = np.asarray(state[t]) @ V.T
        if t == "wedge":
            num = num / np.sqrt(J)[:, None, :]
        ex = np.moveaxis(np.asarray(exact_fn(x, time)), -1, 1)
        d2 = (num - ex) ** 2
        wJ = w[None, :] * J
        tot["p"] += float(np.sum(d2[:, 0] * wJ))
        tot["u"] += float(np.sum(d2[:, 1:] * wJ[:, None, :]))
    return {"p": np.sqrt(tot["p"]), "u": np.sqrt(tot["u"]),
            "total": np.sqrt(tot["p"] + tot["u"])}


def test_l2_error_on_device(native_lib):
    """Device l2_error (host or device exact solution) = the host formula."""
    import math
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.timeint import lsrk_run
    d = _disc("hybrid:3", 3, "GL")
    st = d.project(cavity_fields, 0.0)
    q = lsrk_run(d, d.to_device(st), 1e-3, 5e-3)
    host = {t: v.cpu().numpy() for t, v in q.items()}
    ref = _host_l2(d, host, cavity_fields, 5e-3)

    def cav_dev(x, tau):
        w = math.sqrt(3.0) * math.pi
        s = [torch.sin(math.pi * x[..., i]) for i in range(3)]
        c = [torch.cos(math.pi * x[..., i]) for i in range(3)]
        g = -math.pi * math.sin(w * tau) / w
        return torch.stack([s[0] * s[1] * s[2] * math.cos(w * tau), g * c[0] * s[1] * s[2],
                            g * s[0] * c[1] * s[2], g * s[0] * s[1] * c[2]], dim=-1)
    cav_dev.on_device = True
    for got in (d.l2_error(q, cavity_fields, 5e-3), d.l2_error(q, cav_dev, 5e-3),
                d.l2_error(host, cavity_fields, 5e-3)):
        for k in ("p", "u", "total"):
            assert abs(got[k] - ref[k]) <= 1e-12 * ref[k], (k, got[k], ref[k])


def _assemble_rhs_operator(d):
    """L with rhs = L U, assembled column by column from the device RHS of
    unit vectors (the matrix-free operator of SPEC.md:499-502), batched:
    one compute_rhs per unit vector of the global DOF vector."""
    n = d.n_dof
    L = np.empty((n, n))
    base = np.zeros(n)
    for i in range(n):
        base[i] = 1.0
        r = d.compute_rhs(d.vector_to_state(base))
        L[:, i] = d.state_to_vector(r)
        base[i] = 0.0
    return L


def _energy_weights(d):
    """W with U^T W U = discrete_energy(U) (hybridwave/dg.py:655-674)."""
    blocks = []
    for t in d.types:
        dd = d.data[t]
        mat = d.mesh.materials[t]
        Np = d.ops[t].Np
        for k in range(d.n_elems[t]):
            if t == "hex":
                Mk = np.diag(dd.w3 * dd.J[k])
            elif t == "tet":
                Mk = d.ops[t].M_ref * dd.J[k, 0]
            elif t == "wedge":
                Mk = np.eye(Np)
            else:
                Mk = np.diag(dd.J[k])
            blocks += [Mk / mat[k, 1]] + [Mk * mat[k, 0]] * 3
    from scipy.linalg import block_diag
    return block_diag(*blocks)


@pytest.mark.parametrize("spec,N,form", [("hybrid:2", 1, "GL"), ("hybrid:2", 1, "SEM"),
                                          ("tet:1", 2, "GL"), ("pyramid:1", 2, "SEM")])
def test_energy_stability_of_assembled_operator(spec, N, form, native_lib):
    """SPEC.md:500-502, 516 on the device operator: with zero penalty the
    RHS operator is skew in the energy inner product (W L + L^T W = 0,
    1e-10); with the upwind penalty its symmetric part is negative
    semidefinite (1e-10) and max Re eig(L) <= 1e-8 (energy stability)."""
    from conftest import set_random_materials
    m = build_mesh(spec)
    set_random_materials(m, 13)
    from paper_1507_02557_b200.dg import Discretization
    for pen in (0.0, 1.0):
        d = Discretization(m, N, form, penalty_scale=pen)
        if d.n_dof > 2500:
            pytest.skip("mesh too large for dense assembly")
        L = _assemble_rhs_operator(d)
        W = _energy_weights(d)
        S = W @ L
        sym = 0.5 * (S + S.T)
        scale = np.abs(S).max()
        if pen == 0.0:
            assert np.abs(sym).max() <= 1e-10 * scale
        else:
            assert np.linalg.eigvalsh(sym).max() <= 1e-10 * scale
            ev = np.linalg.eigvals(L)
            assert ev.real.max() <= 1e-8 * np.abs(ev).max()
