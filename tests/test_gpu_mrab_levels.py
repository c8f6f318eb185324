"""Multi-rate AB3 with 3 and 5 rate levels against the reference's own
mrab_run (hybridwave/timeint.py:75-181) on a graded mesh, plus the SPEC's
MRAB known answers: uniform levels reproduce single-rate
AB3, step counting, energy stability.  Fixtures: tests/golden/mrab_levels.npz
(make_golden.py mrab_levels)."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

G = load_golden("mrab_levels")
CASES = [("g6_n2_gl_l3", 2, "GL", 3), ("g6_n3_gl_l3", 3, "GL", 3),
         ("g6_n2_sem_l3", 2, "SEM", 3), ("g6_n2_gl_l5", 2, "GL", 5)]


def _l2rel(a, b):
    num = sum(float(np.sum((np.asarray(a[t]) - np.asarray(b[t])) ** 2)) for t in b)
    den = sum(float(np.sum(np.asarray(b[t]) ** 2)) for t in b)
    return np.sqrt(num / den)


def _setup(tag, N, form, n_levels):
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import graded_hybrid_mesh
    from paper_1507_02557_b200.stability import TimestepPlan
    d = Discretization(graded_hybrid_mesh(6), N, form)
    st0 = d.project(cavity_fields, 0.0)
    levels = {t: G[f"{tag}/levels/{t}"] for t in d.types}
    plan = TimestepPlan({t: np.ones(d.n_elems[t]) for t in d.types}, levels, n_levels, 0.5,
                        list(d.types))
    plan.dt_min = float(G[f"{tag}/dt_min"])
    return d, st0, plan


@pytest.mark.parametrize("tag,N,form,n_levels", CASES)
def test_mrab_levels_match_reference(tag, N, form, n_levels, native_lib):
    """Active-levels-only launches (subset RHS + fused AB update, dense-output
    state only where a stepping element reads it, CUDA-graph replay of the
    3-macro-step period) reproduce the reference trajectory (1e-10) and its
    per-element RHS evaluation counts exactly."""
    from paper_1507_02557_b200.timeint import mrab_run
    d, st0, plan = _setup(tag, N, form, n_levels)
    occupied = sorted({int(x) for v in plan.levels.values() for x in np.unique(v)})
    assert occupied == list(G[f"{tag}/occupied"]) and len(occupied) >= 3
    s, drv = mrab_run(d, plan, st0, float(G[f"{tag}/T"]))
    assert drv.macro_steps == int(G[f"{tag}/macro_steps"])
    for t in d.types:
        np.testing.assert_array_equal(drv.rhs_evals[t], G[f"{tag}/evals/{t}"])
    assert _l2rel(s, {t: G[f"{tag}/{t}"] for t in d.types}) < 1e-10


@pytest.mark.parametrize("tag,N,form,n_levels", [CASES[0], CASES[3]])
def test_mrab_levels_energy(tag, N, form, n_levels, native_lib):
    """Per-macro-step discrete energy (device hw_energy through the live
    callback state) equals the reference's and never increases once every
    level has its AB3 history (cavity run at CFL 0.5; the
    AB1/AB2 warm-up macro step raises it, in the reference too)."""
    from paper_1507_02557_b200.timeint import mrab_run
    d, st0, plan = _setup(tag, N, form, n_levels)
    st = d.to_device(st0)
    en = []
    mrab_run(d, plan, st, float(G[f"{tag}/T"]),
             callback=lambda tau, s: en.append(d.energy_device(s)))
    en = np.array([float(e) for e in en])
    ref = G[f"{tag}/energy"]
    np.testing.assert_allclose(en, ref, rtol=1e-10)
    e0 = float(G[f"{tag}/energy0"])
    assert np.all(np.diff(en) <= 1e-10 * e0)
    assert np.all(np.diff(ref) <= 1e-10 * e0)


def test_mrab_step_counting(native_lib):
    """total RHS evaluations of a level = 2^(lev-1) x macro
    steps x elements at that level."""
    from paper_1507_02557_b200.timeint import mrab_run
    tag, N, form, L = CASES[3]
    d, st0, plan = _setup(tag, N, form, L)
    _, drv = mrab_run(d, plan, st0, float(G[f"{tag}/T"]))
    for t in d.types:
        lev = plan.levels[t]
        np.testing.assert_array_equal(drv.rhs_evals[t], 2 ** (lev - 1) * drv.macro_steps)


@pytest.mark.parametrize("n_levels", [1, 3])
def test_uniform_levels_equal_ab3(n_levels, native_lib):
    """every element on one level -> the single-rate AB3
    trajectory (device MRAB against the device AB3 run to 1e-12, and against
    the reference's AB3 to 1e-10)."""
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import graded_hybrid_mesh
    from paper_1507_02557_b200.stability import TimestepPlan
    from paper_1507_02557_b200.timeint import mrab_run, single_rate_run
    d = Discretization(graded_hybrid_mesh(6), 2, "GL")
    st0 = d.project(cavity_fields, 0.0)
    dt = float(G["uniform/dt"])
    levels = {t: np.full(d.n_elems[t], n_levels) for t in d.types}
    plan = TimestepPlan({t: np.full(d.n_elems[t], dt) for t in d.types}, levels, n_levels,
                        0.5, list(d.types))
    T = 12 * dt                                   # 12 fine steps = 3 macro steps at 3 levels
    ab = single_rate_run(d, st0, dt, T)
    s, drv = mrab_run(d, plan, {t: v.copy() for t, v in st0.items()}, T)
    assert _l2rel(s, ab) < 1e-12
    assert _l2rel(s, {t: G[f"uniform/ab3/{t}"] for t in d.types}) < 1e-10
    for t in d.types:
        assert np.all(drv.rhs_evals[t] == 12)
