"""The CPU oracle (oracle/) against the reference's own outputs."""
import numpy as np
import pytest

import oracle
from conftest import RHS_CASES, build_mesh, load_golden, make_case, rel_err

RHS = load_golden("rhs")
TRAJ = load_golden("trajectories")


@pytest.mark.parametrize("case", range(len(RHS_CASES)))
def test_oracle_rhs_matches_reference(case):
    d, st = make_case(case)
    r = oracle.compute_rhs(d, st)
    ref = {t: RHS[f"{case}/{t}"] for t in d.types}
    assert rel_err(r, ref) < 1e-12


def _cavity_setup(spec, N, form):
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    d = Discretization(build_mesh(spec), N, form)
    return d, d.project(cavity_fields, 0.0)


@pytest.mark.parametrize("tag,spec,N,form", [("c1_sem", "hex:4", 2, "SEM"),
                                             ("c1_gl", "hex:4", 2, "GL")])
def test_oracle_ab3_trajectory(tag, spec, N, form):
    d, st0 = _cavity_setup(spec, N, form)
    dt = float(TRAJ[f"{tag}/dt"])
    s = oracle.single_rate_run(lambda s, tau: oracle.compute_rhs(d, s), st0, dt, 100 * dt)
    ref = {t: TRAJ[f"{tag}/ab3/{t}"] for t in d.types}
    num = sum(np.sum((s[t] - ref[t]) ** 2) for t in d.types)
    den = sum(np.sum(ref[t] ** 2) for t in d.types)
    assert np.sqrt(num / den) < 1e-12


@pytest.mark.parametrize("tag,spec,N,form", [("c1_sem", "hex:4", 2, "SEM"),
                                             ("hyb4_gl", "hybrid:4", 3, "GL")])
def test_oracle_lsrk_trajectory(tag, spec, N, form):
    from paper_1507_02557_b200.app import cavity_fields
    d, st0 = _cavity_setup(spec, N, form)
    dt = float(TRAJ[f"{tag}/dt"])
    s = oracle.lsrk_run(lambda s, tau: oracle.compute_rhs(d, s), st0, dt, 100 * dt)
    ref = {t: TRAJ[f"{tag}/lsrk/{t}"] for t in d.types}
    num = sum(np.sum((s[t] - ref[t]) ** 2) for t in d.types)
    den = sum(np.sum(ref[t] ** 2) for t in d.types)
    assert np.sqrt(num / den) < 1e-12
    err = d.l2_error(s, cavity_fields, 100 * dt)
    np.testing.assert_allclose([err["p"], err["u"], err["total"]], TRAJ[f"{tag}/lsrk/err"],
                               rtol=1e-9)


def test_oracle_mrab_trajectory():
    d, st0 = _cavity_setup("hybrid:2", 2, "GL")
    levels = {t: TRAJ[f"mrab/levels/{t}"] for t in d.types}
    s, evals = oracle.mrab_run(lambda s, tau: oracle.compute_rhs(d, s), levels, 3,
                               float(TRAJ["mrab/dt_min"]), st0, float(TRAJ["mrab/T"]))
    for t in d.types:
        np.testing.assert_array_equal(evals[t], TRAJ[f"mrab/evals/{t}"])
    ref = {t: TRAJ[f"mrab/{t}"] for t in d.types}
    assert rel_err(s, ref) < 1e-11


def test_lsrk_coefficients_order_conditions():
    """Carpenter-Kennedy (4,5): the 2N-storage scheme has classical order 4
    (checked on y' = lambda y: amplification = exp(z) to O(z^5))."""
    A, B = oracle.LSRK_A, oracle.LSRK_B
    for z in (1e-2, 2e-2):
        y, r = 1.0, 0.0
        for a, b in zip(A, B):
            r = a * r + z * y
            y = y + b * r
        assert abs(y - np.exp(z)) < 5 * z ** 5
