"""Non-affine LSC-DG wedges whose triangle faces meet (affine) pyramids:
the wedge side runs the cubature path, the pyramid side gets
hw_wedge_face_correction rows (the reference's face cubature,
hybridwave/dg.py:326-354, minus the pyramid kernel's nodal lift) in the
stage epilogue.  Against the reference's own RHS and 10 LSRK-45 steps
(tests/golden/wedge_pyramid.npz, make_golden.py wedge_pyramid) and the
oracle."""
import numpy as np
import pytest
import torch

import oracle
from conftest import load_golden, rel_err, set_random_materials

pytestmark = pytest.mark.gpu
G = load_golden("wedge_pyramid")
CASES = [("n1_gl", 1, "GL"), ("n2_gl", 2, "GL"), ("n3_sem", 3, "SEM"), ("n3_gl", 3, "GL")]


def _l2rel(a, b):
    num = sum(float(np.sum((np.asarray(a[t]) - np.asarray(b[t])) ** 2)) for t in b)
    den = sum(float(np.sum(np.asarray(b[t]) ** 2)) for t in b)
    return np.sqrt(num / den)


def _disc(N, form, **kw):
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import HybridMesh, wedge_pyramid_columns_mesh
    g = wedge_pyramid_columns_mesh(2, 0.3, 1)
    m = HybridMesh(G["X"], g.blocks)
    set_random_materials(m, 5)
    return Discretization(m, N, form, **kw)


@pytest.mark.parametrize("tag,N,form", CASES)
def test_wedge_pyramid_rhs_matches_reference(tag, N, form, native_lib):
    d = _disc(N, form)
    assert set(d.device_mesh.corr) == {"pyramid"}
    rng = np.random.default_rng(N + 40)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    r = d.compute_rhs(st)
    assert rel_err(r, {t: G[f"{tag}/rhs/{t}"] for t in d.types}) < 1e-11
    assert rel_err(r, oracle.compute_rhs(d, st)) < 1e-11


@pytest.mark.parametrize("tag,N,form", CASES)
def test_wedge_pyramid_lsrk_matches_reference(tag, N, form, native_lib):
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.timeint import lsrk_run
    d = _disc(N, form)
    st = d.project(cavity_fields, 0.0)
    dt = float(G[f"{tag}/dt"])
    s = lsrk_run(d, st, dt, 10 * dt)
    assert _l2rel(s, {t: G[f"{tag}/lsrk/{t}"] for t in d.types}) < 1e-10


def test_wedge_pyramid_ab3_vs_oracle(native_lib):
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.timeint import single_rate_run
    d = _disc(2, "GL")
    st = d.project(cavity_fields, 0.0)
    dt = float(G["n2_gl/dt"])
    ab = single_rate_run(d, st, dt, 8 * dt)
    ref = oracle.single_rate_run(lambda q, tau: oracle.compute_rhs(d, q), st, dt, 8 * dt)
    assert _l2rel(ab, ref) < 1e-10


def test_wedge_pyramid_fp32(native_lib):
    d = _disc(3, "GL", dtype=torch.float32)
    rng = np.random.default_rng(43)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    r = d.compute_rhs(st)
    assert _l2rel(r, {t: G[f"n3_gl/rhs/{t}"] for t in d.types}) < 1e-4
