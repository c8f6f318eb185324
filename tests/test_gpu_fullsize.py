"""Parity at the benchmark sizes (BASELINE configs C2, C3, C4).

The device RHS runs on the whole mesh (full E-element blocks, every side
stream, the largest int32 offsets); the oracle checks a sample of elements
per type (first / last blocks + random) on the neighbour-closed sub-mesh
(tests/sampled.py), 1e-12 max-norm relative in fp64.  tet:20 is small enough
for the whole-mesh oracle.  Size-independent properties (linearity, energy
decay) cover every element at full size."""
import numpy as np
import pytest
import torch

import oracle
from sampled import default_sample, sampled_oracle_rhs

pytestmark = pytest.mark.gpu


def _random_device_state(d, seed):
    g = torch.Generator(device=d.device)
    g.manual_seed(seed)
    return {t: torch.randn((d.n_elems[t], 4, d.ops[t].Np), generator=g, device=d.device,
                           dtype=torch.float64) for t in d.types}


def _rows(q):
    return lambda t, ids: q[t][torch.as_tensor(ids, device=q[t].device)].cpu().numpy()


def _check_sampled(d, q64, got, seed=0, tol=1e-12):
    sample = default_sample(d.mesh, seed=seed)
    ref = sampled_oracle_rhs(d, _rows(q64), sample)
    for t, ids in sample.items():
        g = got[t][torch.as_tensor(ids, device=got[t].device)].double().cpu().numpy()
        err = np.abs(g - ref[t]).max() / np.abs(ref[t]).max()
        assert err < tol, (t, err)


@pytest.fixture(scope="module")
def hyb38():
    from paper_1507_02557_b200.mesh import structured_hybrid_mesh
    m = structured_hybrid_mesh(38)
    assert m.n_elements == 206_492
    return m


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("form", ["GL", "SEM"])
def test_hybrid38_rhs_sampled(hyb38, N, form, native_lib):
    """C3 (hybrid:38, 206,492 elements) single RHS at N = 1..5, GL and SEM."""
    from paper_1507_02557_b200.dg import Discretization
    d = Discretization(hyb38, N, form)
    q = _random_device_state(d, 100 + N)
    _check_sampled(d, q, d.compute_rhs(q), seed=N)


def test_hybrid38_random_materials_sampled(native_lib):
    """C3 N=3 GL with random rho, kappa per element (tau != 1 everywhere)."""
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import structured_hybrid_mesh
    m = structured_hybrid_mesh(38)
    rng = np.random.default_rng(7)
    for t in m.elem_types:
        m.materials[t] = rng.uniform(0.5, 2.0, (len(m.blocks[t]), 2))
    d = Discretization(m, 3, "GL")
    q = _random_device_state(d, 9)
    _check_sampled(d, q, d.compute_rhs(q), seed=3)


def test_hybrid38_fp32_sampled(hyb38, native_lib):
    """C3 N=3 fp32 storage against the fp64 oracle: within the north star's
    1e-4 (max-norm relative on the sample)."""
    from paper_1507_02557_b200.dg import Discretization
    d32 = Discretization(hyb38, 3, "GL", dtype=torch.float32)
    q64 = _random_device_state(d32, 5)
    q64 = {t: v.float().double() for t, v in q64.items()}     # the fp32-representable state
    got = d32.compute_rhs({t: v.float() for t, v in q64.items()})
    _check_sampled(d32, q64, got, tol=1e-4)


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-12), (torch.float32, 1e-4)])
def test_tet20_whole_mesh(dtype, tol, native_lib):
    """C2 (tet:20, 48,000 tets, N=3): every element against the oracle."""
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import uniform_cube_mesh
    d = Discretization(uniform_cube_mesh("tet", 20), 3, "GL", dtype=dtype)
    assert d.n_elems["tet"] == 48_000
    rng = np.random.default_rng(20)
    st = {"tet": rng.standard_normal((48_000, 4, 20))}
    if dtype == torch.float32:
        st = {"tet": st["tet"].astype(np.float32).astype(np.float64)}
    got = d.compute_rhs(st)["tet"].astype(np.float64)
    ref = oracle.compute_rhs(d, st)["tet"]
    if dtype == torch.float64:
        assert np.abs(got - ref).max() / np.abs(ref).max() < tol
    else:
        assert np.sqrt(np.sum((got - ref) ** 2) / np.sum(ref ** 2)) < tol


def test_hexdom120_rhs_sampled(native_lib):
    """C4 (hexdom:120, 2,232,000 elements, 907 M DOF, N=4 GL) single RHS on
    the whole mesh, sampled oracle."""
    from paper_1507_02557_b200.app import build_mesh
    from paper_1507_02557_b200.dg import Discretization
    m = build_mesh("hexdom:120")
    assert m.n_elements == 2_232_000
    d = Discretization(m, 4, "GL")
    q = _random_device_state(d, 44)
    out = d.rhs_device(q)
    _check_sampled(d, q, out, seed=4)


def test_hexdom120_fp32_sampled(native_lib):
    """C4 with fp32 storage against the fp64 oracle on the sample (1e-4)."""
    from paper_1507_02557_b200.app import build_mesh
    from paper_1507_02557_b200.dg import Discretization
    d = Discretization(build_mesh("hexdom:120"), 4, "GL", dtype=torch.float32)
    q64 = _random_device_state(d, 45)
    q64 = {t: v.float().double() for t, v in q64.items()}
    out = d.rhs_device({t: v.float() for t, v in q64.items()})
    _check_sampled(d, q64, out, seed=5, tol=1e-4)


def test_hybrid38_linearity(hyb38, native_lib):
    """RHS(a x + b y) = a RHS(x) + b RHS(y) on every element of C3 (N=3 GL)."""
    from paper_1507_02557_b200.dg import Discretization
    d = Discretization(hyb38, 3, "GL")
    x, y = _random_device_state(d, 1), _random_device_state(d, 2)
    a, b = 0.7, -1.3
    lhs = d.rhs_device({t: a * x[t] + b * y[t] for t in d.types})
    rx, ry = d.rhs_device(x), d.rhs_device(y)
    for t in d.types:
        rhs = a * rx[t] + b * ry[t]
        err = float((lhs[t] - rhs).abs().max() / rhs.abs().max())
        assert err < 1e-13, (t, err)


def test_hybrid38_lsrk_energy_decays(hyb38, native_lib):
    """10 LSRK-45 steps of the cavity mode on all of C3: the discrete energy
    (device) never increases (upwind flux) and the L2 error of
    the standing wave stays at discretisation level."""
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.stability import local_timesteps
    from paper_1507_02557_b200.timeint import lsrk_run
    d = Discretization(hyb38, 3, "GL")
    st = d.project(cavity_fields, 0.0)
    dt = min(float(v.min()) for v in local_timesteps(d, 0.5).values())
    en = []
    q = lsrk_run(d, d.to_device(st), dt, 10 * dt,
                 callback=lambda tau, s: en.append(d.energy_device(s)))
    e = np.array([float(d.energy_device(d.to_device(st)))] + [float(v) for v in en])
    assert np.all(np.diff(e) <= 1e-12 * e[0])
    err = d.l2_error({t: v.cpu().numpy() for t, v in q.items()}, cavity_fields, 10 * dt)
    assert err["total"] < 1e-5
