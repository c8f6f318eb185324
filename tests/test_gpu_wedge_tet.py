"""Non-affine LSC-DG wedges whose triangle faces meet tets (the reference
integrates every such face at its stored 6(N+1)^2 cubature points,
hybridwave/dg.py:217-354, 423-444): the wedge side runs the cubature path,
the tet side gets hw_wedge_face_correction rows in the stage epilogue.
Against the reference's own RHS and 10 LSRK-45 steps (tests/golden/
wedge_tet.npz, make_golden.py wedge_tet) and the oracle."""
import numpy as np
import pytest
import torch

import oracle
from conftest import load_golden, rel_err, set_random_materials

pytestmark = pytest.mark.gpu
G = load_golden("wedge_tet")
CASES = [("n1_gl", 1, "GL"), ("n2_gl", 2, "GL"), ("n3_sem", 3, "SEM"), ("n3_gl", 3, "GL")]


def _l2rel(a, b):
    num = sum(float(np.sum((np.asarray(a[t]) - np.asarray(b[t])) ** 2)) for t in b)
    den = sum(float(np.sum(np.asarray(b[t]) ** 2)) for t in b)
    return np.sqrt(num / den)


def _disc(N, form, **kw):
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import HybridMesh, wedge_tet_columns_mesh
    g = wedge_tet_columns_mesh(4, 2, 2)
    m = HybridMesh(G["X"], g.blocks)
    set_random_materials(m, 4)
    return Discretization(m, N, form, **kw)


@pytest.mark.parametrize("tag,N,form", CASES)
def test_wedge_tet_rhs_matches_reference(tag, N, form, native_lib):
    d = _disc(N, form)
    assert d.has_corrections
    rng = np.random.default_rng(N + 30)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    r = d.compute_rhs(st)
    assert rel_err(r, {t: G[f"{tag}/rhs/{t}"] for t in d.types}) < 1e-11
    assert rel_err(r, oracle.compute_rhs(d, st)) < 1e-11


@pytest.mark.parametrize("tag,N,form", CASES)
def test_wedge_tet_lsrk_matches_reference(tag, N, form, native_lib):
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.timeint import lsrk_run
    d = _disc(N, form)
    st = d.project(cavity_fields, 0.0)
    dt = float(G[f"{tag}/dt"])
    s = lsrk_run(d, st, dt, 10 * dt)
    assert _l2rel(s, {t: G[f"{tag}/lsrk/{t}"] for t in d.types}) < 1e-10


def test_wedge_tet_ab3_and_mrab_vs_oracle(native_lib):
    """AB3 (fused, corrections in the epilogue) and multi-rate AB3 (the
    corrections recomputed every tick from the effective state's traces)
    against the oracle's integrators."""
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.stability import TimestepPlan
    from paper_1507_02557_b200.timeint import mrab_run, single_rate_run
    d = _disc(2, "GL")
    st = d.project(cavity_fields, 0.0)
    dt = float(G["n2_gl/dt"])
    ab = single_rate_run(d, st, dt, 8 * dt)
    ref = oracle.single_rate_run(lambda q, tau: oracle.compute_rhs(d, q), st, dt, 8 * dt)
    assert _l2rel(ab, ref) < 1e-10
    levels = {"wedge": np.full(d.n_elems["wedge"], 1), "tet": np.full(d.n_elems["tet"], 2)}
    plan = TimestepPlan({t: np.ones(d.n_elems[t]) for t in d.types}, levels, 2, 0.5,
                        list(d.types))
    plan.dt_min = dt
    T = 6 * 2 * dt
    s, drv = mrab_run(d, plan, {t: v.copy() for t, v in st.items()}, T)
    ref, _ = oracle.mrab_run(lambda q, tau: oracle.compute_rhs(d, q), levels, 2, dt,
                             {t: v.copy() for t, v in st.items()}, T)
    assert _l2rel(s, ref) < 1e-10


def test_wedge_tet_fp32(native_lib):
    d = _disc(3, "GL", dtype=torch.float32)
    rng = np.random.default_rng(33)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    r = d.compute_rhs(st)
    assert _l2rel(r, {t: G[f"n3_gl/rhs/{t}"] for t in d.types}) < 1e-4
