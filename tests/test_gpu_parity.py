"""Device kernels (through the C ABI) against the reference's outputs and
the CPU oracle.  Tolerances: fp64 1e-12 per RHS (max-norm, relative), 1e-10
relative L2 after 100 steps (north star); fp32 1e-4."""
import numpy as np
import pytest
import torch

import oracle
from conftest import RHS_CASES, build_mesh, load_golden, make_case, rel_err

pytestmark = pytest.mark.gpu

RHS = load_golden("rhs")
TRAJ = load_golden("trajectories")


def _l2rel(a, b):
    num = sum(float(np.sum((np.asarray(a[t]) - np.asarray(b[t])) ** 2)) for t in b)
    den = sum(float(np.sum(np.asarray(b[t]) ** 2)) for t in b)
    return np.sqrt(num / den)


@pytest.mark.parametrize("case", range(len(RHS_CASES)))
def test_rhs_fp64_matches_reference(case, native_lib):
    d, st = make_case(case)
    r = d.compute_rhs(st)                      # host arrays in/out: the e2e path
    ref = {t: RHS[f"{case}/{t}"] for t in d.types}
    assert rel_err(r, ref) < 1e-12


@pytest.mark.parametrize("case", range(len(RHS_CASES)))
def test_rhs_fp32(case, native_lib):
    """fp32 storage (fp64 arithmetic in the kernels) on every reference case:
    within the north star's fp32 bound (1e-4), in practice ~1e-7."""
    d, st = make_case(case, dtype=torch.float32)
    r = d.compute_rhs(st)
    ref = {t: RHS[f"{case}/{t}"] for t in d.types}
    assert _l2rel(r, ref) < 1e-4


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("form", ["GL", "SEM"])
def test_rhs_all_orders_vs_oracle(N, form, native_lib):
    from paper_1507_02557_b200.dg import Discretization
    from conftest import set_random_materials
    m = build_mesh("hybrid:2")
    set_random_materials(m, 11)
    d = Discretization(m, N, form)
    rng = np.random.default_rng(100 + N)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    assert rel_err(d.compute_rhs(st), oracle.compute_rhs(d, st)) < 1e-11


def test_device_tensors_stay_resident(native_lib):
    d, st = make_case(6)
    q = d.to_device(st)
    out = d.compute_rhs(q)
    assert all(v.is_cuda for v in out.values())
    ref = {t: RHS[f"6/{t}"] for t in d.types}
    assert rel_err({t: v.cpu().numpy() for t, v in out.items()}, ref) < 1e-12


def test_subset_launch_equals_full(native_lib):
    d, st = make_case(6)
    q = d.to_device(st)
    full = d.rhs_device(q)
    part = d.zeros_state()
    lists = [None] * 4
    from paper_1507_02557_b200.operators import TYPE_ID
    for t in d.types:
        lists[TYPE_ID[t]] = torch.arange(0, d.n_elems[t], 2, dtype=torch.int32, device=d.device)
    d.rhs_device(q, out=part, subset=lists)
    for t in d.types:
        assert torch.equal(part[t][::2], full[t][::2])
        assert torch.count_nonzero(part[t][1::2]) == 0


def _cavity(spec, N, form, **kw):
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    d = Discretization(build_mesh(spec), N, form, **kw)
    return d, d.project(cavity_fields, 0.0)


@pytest.mark.parametrize("tag,spec,N,form", [("c1_sem", "hex:4", 2, "SEM"),
                                             ("c1_gl", "hex:4", 2, "GL")])
def test_ab3_100_steps(tag, spec, N, form, native_lib):
    from paper_1507_02557_b200.timeint import single_rate_run
    d, st0 = _cavity(spec, N, form)
    dt = float(TRAJ[f"{tag}/dt"])
    s = single_rate_run(d, st0, dt, 100 * dt)
    ref = {t: TRAJ[f"{tag}/ab3/{t}"] for t in d.types}
    assert _l2rel(s, ref) < 1e-10


@pytest.mark.parametrize("tag,spec,N,form", [("c1_sem", "hex:4", 2, "SEM"),
                                             ("c1_gl", "hex:4", 2, "GL"),
                                             ("hyb4_gl", "hybrid:4", 3, "GL")])
def test_lsrk_100_steps(tag, spec, N, form, native_lib):
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.timeint import lsrk_run
    d, st0 = _cavity(spec, N, form)
    dt = float(TRAJ[f"{tag}/dt"])
    s = lsrk_run(d, st0, dt, 100 * dt)
    ref = {t: TRAJ[f"{tag}/lsrk/{t}"] for t in d.types}
    assert _l2rel(s, ref) < 1e-10
    err = d.l2_error(s, cavity_fields, 100 * dt)
    np.testing.assert_allclose(err["total"], TRAJ[f"{tag}/lsrk/err"][2], rtol=1e-8)


def test_lsrk_fp32_100_steps(native_lib):
    from paper_1507_02557_b200.timeint import lsrk_run
    d, st0 = _cavity("hybrid:4", 3, "GL", dtype=torch.float32)
    dt = float(TRAJ["hyb4_gl/dt"])
    s = lsrk_run(d, st0, dt, 100 * dt)
    ref = {t: TRAJ[f"hyb4_gl/lsrk/{t}"] for t in d.types}
    assert _l2rel(s, ref) < 1e-4


def test_mrab_matches_reference(native_lib):
    from paper_1507_02557_b200.stability import TimestepPlan
    from paper_1507_02557_b200.timeint import mrab_run
    d, st0 = _cavity("hybrid:2", 2, "GL")
    levels = {t: TRAJ[f"mrab/levels/{t}"] for t in d.types}
    dtl = {t: np.full(d.n_elems[t], 1.0) for t in d.types}
    plan = TimestepPlan(dtl, levels, 3, 0.5, list(d.types))
    plan.dt_min = float(TRAJ["mrab/dt_min"])
    s, drv = mrab_run(d, plan, st0, float(TRAJ["mrab/T"]))
    for t in d.types:
        np.testing.assert_array_equal(drv.rhs_evals[t], TRAJ[f"mrab/evals/{t}"])
    ref = {t: TRAJ[f"mrab/{t}"] for t in d.types}
    assert _l2rel(s, ref) < 1e-10


@pytest.mark.parametrize("spec,N,form", [("hybrid:2", 3, "GL"), ("hybrid:2", 2, "SEM"),
                                          ("hex:2", 3, "GL"), ("tet:2", 4, "GL")])
def test_energy_matches_host(native_lib, spec, N, form):
    """hw_energy (device, per type, atomics) = discrete_energy (host)."""
    from paper_1507_02557_b200.dg import discrete_energy
    d, st = _cavity(spec, N, form)
    rng = np.random.default_rng(3)
    st = {t: v + 0.1 * rng.standard_normal(v.shape) for t, v in st.items()}
    ref = discrete_energy(st, d)
    got = float(d.energy_device(d.to_device(st)))
    assert abs(got - ref) <= 1e-12 * abs(ref)


def test_skew_nonaffine_hex(native_lib):
    from paper_1507_02557_b200.dg import Discretization
    d = Discretization(_perturbed("hex:3", 0.04, 5), 3, "GL", forms_override={"hex": "skew"})
    rng = np.random.default_rng(6)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    assert rel_err(d.compute_rhs(st), oracle.compute_rhs(d, st)) < 1e-11


def test_energy_nonaffine_hex(native_lib):
    from paper_1507_02557_b200.dg import Discretization, discrete_energy
    d = Discretization(_perturbed("hex:3", 0.04, 7), 3, "GL")
    rng = np.random.default_rng(4)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    ref = discrete_energy(st, d)
    assert abs(float(d.energy_device(d.to_device(st))) - ref) <= 1e-12 * abs(ref)


def test_mrab_graph_replay_matches_eager(native_lib):
    """The CUDA-graph replay of the 3-macro-step launch period reproduces the
    eager launches bit for bit (same kernels, same arguments), counters too."""
    from paper_1507_02557_b200.stability import TimestepPlan
    from paper_1507_02557_b200.timeint import MRABDriver
    d, st0 = _cavity("hybrid:2", 2, "GL")
    levels = {t: TRAJ[f"mrab/levels/{t}"] for t in d.types}
    dtl = {t: np.full(d.n_elems[t], 1.0) for t in d.types}
    plan = TimestepPlan(dtl, levels, 3, 0.5, list(d.types))
    plan.dt_min = float(TRAJ["mrab/dt_min"])
    T = 11 * 4 * plan.dt_min                      # 11 macro steps: eager, 3 replays, tail
    outs, evals = [], []
    for graph in (False, True):
        drv = MRABDriver(d, plan)
        st = {t: v.copy() for t, v in st0.items()}
        drv.run(st, T, graph=graph)
        outs.append(st)
        evals.append(drv.rhs_evals)
        assert drv.macro_steps == 11
    for t in d.types:
        np.testing.assert_array_equal(outs[0][t], outs[1][t])
        np.testing.assert_array_equal(evals[0][t], evals[1][t])


@pytest.mark.parametrize("nparts", [2, 3])
def test_partitioned_mrab_loopback(nparts, native_lib):
    """Element-partitioned multi-rate AB3 (per-tick exchange of the
    boundary elements' effective state, emulated in one process) equals the
    single-GPU MRABDriver to rounding, levels spanning the partition cuts."""
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.parallel import LoopbackTransport, PartMRAB, make_parts
    from paper_1507_02557_b200.stability import assign_mrab_levels, local_timesteps
    from paper_1507_02557_b200.timeint import MRABDriver
    from paper_1507_02557_b200.app import build_mesh as app_mesh
    m = app_mesh("graded:6")
    N = 2
    d = Discretization(m, N, "GL")
    plan = assign_mrab_levels(local_timesteps(d, 0.5), 3, m)
    assert len({int(x) for v in plan.levels.values() for x in np.unique(v)}) == 3
    st = d.project(cavity_fields, 0.0)
    n_macro, dt_min = 5, plan.dt_min
    drv = MRABDriver(d, plan)
    ref = {t: v.copy() for t, v in st.items()}
    drv.run(ref, n_macro * 4 * dt_min, graph=False)
    parts = make_parts(m, nparts, "xslab", N=N)
    T = LoopbackTransport()
    ps = [PartMRAB(p, N, "GL", {t: st[t][p.global_ids[t]] for t in p.types},
                   {t: plan.levels[t][p.global_ids[t]] for t in p.types}, 3, T) for p in parts]
    for _ in range(n_macro):
        for tick in range(4):
            for p in ps:
                p.tick_effective(tick, dt_min)
            hs = [p.tick_exchange() for p in ps]
            for p, h in zip(ps, hs):
                p.tick_step(tick, dt_min, h)
    for p in ps:
        own = p.owned_state()
        for t in p.disc.types:
            g = p.part.global_ids[t][:p.part.n_owned[t]]
            r_ = ref[t][g]
            assert np.abs(own[t].cpu().numpy() - r_).max() <= 1e-12 * np.abs(r_).max()


def _forcing_fn(x, time):
    return (np.sin(np.pi * x[..., 0]) * np.cos(np.pi * x[..., 1]) * (1.0 + x[..., 2])
            * np.cos(3.0 * time))


@pytest.mark.parametrize("tag,spec,N,form", [("hyb2_gl", "hybrid:2", 2, "GL"),
                                             ("hyb2_sem", "hybrid:2", 2, "SEM"),
                                             ("tet2_gl", "tet:2", 3, "GL")])
def test_forcing_matches_reference(tag, spec, N, form, native_lib):
    """compute_rhs with a forcing callback and 10 AB3 / LSRK-45 steps with it
    against the reference's own outputs (tests/golden/forcing.npz)."""
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.timeint import lsrk_run, single_rate_run
    from conftest import set_random_materials
    G = load_golden("forcing")
    m = build_mesh(spec)
    set_random_materials(m, 5)
    d = Discretization(m, N, form, forcing=_forcing_fn)
    st = d.project(cavity_fields, 0.0)
    dt = float(G[f"{tag}/dt"])
    rhs = d.compute_rhs(st, 0.37)
    assert rel_err(rhs, {t: G[f"{tag}/rhs/{t}"] for t in d.types}) < 1e-12
    ab = single_rate_run(d, st, dt, 10 * dt)
    assert _l2rel(ab, {t: G[f"{tag}/ab3/{t}"] for t in d.types}) < 1e-10
    lk = lsrk_run(d, st, dt, 10 * dt)
    assert _l2rel(lk, {t: G[f"{tag}/lsrk/{t}"] for t in d.types}) < 1e-10


def test_mrab_forcing_matches_reference(native_lib):
    """Multi-rate AB3 with a forcing callback (unfused path) against the
    reference's mrab_run with the same forcing (tests/golden/forcing.npz)."""
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.stability import TimestepPlan
    from paper_1507_02557_b200.timeint import mrab_run
    G = load_golden("forcing")
    d = Discretization(build_mesh("hybrid:2"), 2, "GL", forcing=_forcing_fn)
    st0 = d.project(cavity_fields, 0.0)
    levels = {t: G[f"mrab/levels/{t}"] for t in d.types}
    dtl = {t: np.full(d.n_elems[t], 1.0) for t in d.types}
    plan = TimestepPlan(dtl, levels, 3, 0.5, list(d.types))
    plan.dt_min = float(G["mrab/dt_min"])
    s, _ = mrab_run(d, plan, st0, float(G["mrab/T"]))
    assert _l2rel(s, {t: G[f"mrab/{t}"] for t in d.types}) < 1e-10


@pytest.mark.parametrize("tag,spec,N,form,over", [
    ("hyb2_skew", "hybrid:2", 2, "GL", {"hex": "skew", "tet": "skew"}),
    ("hyb3_skew", "hybrid:2", 3, "SEM", {"hex": "skew", "tet": "skew"}),
    ("hex2_skew", "hex:2", 3, "GL", {"hex": "skew"}),
    ("tet2_skew", "tet:2", 3, "GL", {"tet": "skew"}),
    ("hyb2_wstrong", "hybrid:2", 2, "GL", {"wedge": "strong", "pyramid": "skew"}),
    ("hyb2_pstrong", "hybrid:2", 2, "SEM", {"pyramid": "strong"})])
def test_skew_forms_match_reference(tag, spec, N, form, over, native_lib):
    """forms_override (the reference's testing hook): skew hex and tet
    volume + flux on the device against the reference's own RHS."""
    from paper_1507_02557_b200.dg import Discretization
    from conftest import set_random_materials
    G = load_golden("forms")
    m = build_mesh(spec)
    set_random_materials(m, 9)
    d = Discretization(m, N, form, forms_override=over)
    rng = np.random.default_rng(11)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    assert rel_err(d.compute_rhs(st), {t: G[f"{tag}/rhs/{t}"] for t in d.types}) < 1e-12
    assert rel_err(d.compute_rhs(st), oracle.compute_rhs(d, st)) < 1e-12


@pytest.mark.parametrize("scheme,levels", [("lsrk", 1), ("ab3", 1), ("ab3", 3)])
def test_solve_run_cavity(scheme, levels, native_lib):
    """app.solve_run (the reference's cavity driver) on the device: L2 error
    of the standing wave small, discrete energy (tracked on the device every
    step) non-increasing under the upwind flux and equal to the host value."""
    from paper_1507_02557_b200.app import RunConfig, cavity_fields, solve_run
    from paper_1507_02557_b200.dg import discrete_energy
    cfg = RunConfig(mesh="hybrid:3", N=3, formulation="GL", cfl=0.3, n_levels=levels,
                    T_final=0.05, scheme=scheme)
    out = solve_run(cfg, verbose=False)
    assert out["errors"]["total"] < 5e-3
    en = [e for _, e in out["energies"]]
    assert len(en) >= 2 and all(b <= a * (1 + 1e-12) for a, b in zip(en, en[1:]))
    d = out["disc"]
    assert abs(en[-1] - discrete_energy(out["state"], d)) <= 1e-10 * en[-1]


@pytest.mark.parametrize("N,form", [(1, "GL"), (2, "GL"), (3, "GL"), (2, "SEM"), (3, "SEM")])
def test_convergence_matches_reference(N, form, native_lib):
    """app.convergence_study on the device reproduces the reference's own
    cavity errors and h-convergence rate (hybrid:2,3,4, AB3, T = 0.1)."""
    from paper_1507_02557_b200.app import RunConfig, convergence_study
    G = load_golden("convergence")
    cfg = RunConfig(mesh="hybrid:2", N=N, formulation=form, cfl=0.5, T_final=0.1)
    errs, rate = convergence_study(cfg, [2, 3, 4], verbose=False)
    ref = G[f"N{N}_{form}/errs"]
    assert np.abs(errs - ref).max() <= 1e-8 * ref.max()
    assert abs(rate - float(G[f"N{N}_{form}/rate"])) < 1e-6


def _perturbed(spec, amp, seed):
    from paper_1507_02557_b200.mesh import HybridMesh
    m = build_mesh(spec)
    rng = np.random.default_rng(seed)
    X = m.vertices.copy()
    inner = np.all((X > 1e-9) & (X < 1 - 1e-9), axis=1)
    X[inner] += amp * rng.uniform(-1, 1, (inner.sum(), 3))
    return HybridMesh(X, m.blocks)


@pytest.mark.parametrize("tag,spec,N,form,seed", [("pyr3_gl2", "pyramid:3", 2, "GL", 3),
                                                  ("pyr3_sem3", "pyramid:3", 3, "SEM", 4),
                                                  ("pyr2_gl4", "pyramid:2", 4, "GL", 5)])
def test_nonaffine_pyramids_match_reference(tag, spec, N, form, seed, native_lib):
    """Jittered pyramids (non-planar bilinear bases): per-node G and J,
    per-point base-face geometry, against the reference's own RHS and the
    oracle."""
    from paper_1507_02557_b200.dg import Discretization
    G = load_golden("nonaffine")
    d = Discretization(_perturbed(spec, 0.04, seed), N, form)
    rng = np.random.default_rng(seed + 10)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    r = d.compute_rhs(st)
    assert rel_err(r, {t: G[f"{tag}/rhs/{t}"] for t in d.types}) < 1e-11
    assert rel_err(r, oracle.compute_rhs(d, st)) < 1e-11


@pytest.mark.parametrize("form", ["GL", "SEM"])
def test_nonaffine_pyramid_lsrk(form, native_lib):
    """20 LSRK-45 steps on jittered pyramids + a hex band (the published
    pyramid traces of the non-affine path) against the oracle."""
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.stability import local_timesteps
    from paper_1507_02557_b200.timeint import lsrk_run
    d = Discretization(_perturbed("pyramid:3", 0.04, 8), 2, form)
    st = d.project(cavity_fields, 0.0)
    dt = 0.5 * min(float(v.min()) for v in local_timesteps(d, 0.5).values())
    s = lsrk_run(d, st, dt, 20 * dt)
    ref = oracle.lsrk_run(lambda q, tau: oracle.compute_rhs(d, q), st, dt, 20 * dt)
    assert _l2rel(s, ref) < 1e-10


@pytest.mark.parametrize("spec,form", [("hex:3", "GL"), ("hex:3", "SEM"), ("tet:2", "GL")])
def test_rhs_non_affine_vs_oracle(spec, form, native_lib):
    """Trilinear (non-affine) hexes take the per-node metric path."""
    from paper_1507_02557_b200.dg import Discretization
    d = Discretization(_perturbed(spec, 0.04, 5), 3, form)
    rng = np.random.default_rng(9)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    assert rel_err(d.compute_rhs(st), oracle.compute_rhs(d, st)) < 1e-11


@pytest.mark.parametrize("form,nparts,method", [("GL", 2, "xslab"), ("SEM", 3, "rcb")])
def test_partitioned_lsrk_loopback(form, nparts, method, native_lib):
    """Element-partitioned LSRK (ghost elements, halo exchange emulated in
    one process on one GPU) equals the single-GPU run to rounding."""
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.parallel import LoopbackTransport, PartStepper, make_parts
    from paper_1507_02557_b200.timeint import LSRK_A, LSRK_B, Stepper
    from conftest import set_random_materials
    m = build_mesh("hybrid:4")
    set_random_materials(m, 3)
    N, h = 2, 2e-4
    d = Discretization(m, N, form)
    rng = np.random.default_rng(2)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    S = Stepper(d, st, "lsrk")
    for _ in range(3):
        S.lsrk_step(h)
    ref = {t: S.q[t].cpu().numpy() for t in d.types}
    parts = make_parts(m, nparts, method, N=N)
    T = LoopbackTransport()
    ps = [PartStepper(p, N, form, {t: st[t][p.global_ids[t]] for t in p.types}, T)
          for p in parts]
    for _ in range(3):
        for a, b in zip(LSRK_A, LSRK_B):
            for p in ps:
                p.begin()
            for p in ps:
                p.finish(a, b, h)
            for p in ps:
                p.swap()
    for p in ps:
        own = p.owned_state()
        for t in p.disc.types:
            g = p.part.global_ids[t][:p.part.n_owned[t]]
            r_ = ref[t][g]
            assert np.abs(own[t].cpu().numpy() - r_).max() <= 1e-12 * np.abs(r_).max()


NAW_CASES = [("wed2_gl1", "wedge:2", 1, "GL", 6), ("wed3_gl2", "wedge:3", 2, "GL", 7),
             ("wed3_sem3", "wedge:3", 3, "SEM", 8), ("wed2_gl5", "wedge:2", 5, "GL", 9)]


@pytest.mark.parametrize("tag,spec,N,form,seed", NAW_CASES)
def test_nonaffine_wedges_match_reference(tag, spec, N, form, seed, native_lib):
    """Jittered (non-affine) LSC-DG wedges: the cubature path of the scalar
    kernel (volume G / grad J at the cubature points, triangle faces at the
    reference's face cubature) against the reference's own RHS."""
    from paper_1507_02557_b200.dg import Discretization
    G = load_golden("nonaffine")
    d = Discretization(_perturbed(spec, 0.04, seed), N, form)
    rng = np.random.default_rng(seed + 10)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    r = d.compute_rhs(st)
    assert rel_err(r, {"wedge": G[f"{tag}/rhs/wedge"]}) < 1e-11
    assert rel_err(r, oracle.compute_rhs(d, st)) < 1e-11


def test_nonaffine_wedges_fp32(native_lib):
    from paper_1507_02557_b200.dg import Discretization
    G = load_golden("nonaffine")
    d = Discretization(_perturbed("wedge:3", 0.04, 8), 3, "SEM", dtype=torch.float32)
    rng = np.random.default_rng(18)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    assert _l2rel(d.compute_rhs(st), {"wedge": G["wed3_sem3/rhs/wedge"]}) < 1e-4


@pytest.mark.parametrize("spec,N,form,steps", [("wedge:3", 2, "GL", 20), ("wedge:3", 3, "SEM", 20),
                                               ("hybrid:2", 2, "GL", 10),
                                               ("hybrid:2", 3, "SEM", 10)])
def test_nonaffine_wedge_lsrk(spec, N, form, steps, native_lib):
    """LSRK-45 on jittered meshes (hybrid: non-affine wedges next to
    non-affine pyramids and trilinear hexes on their quad faces) against the
    oracle: the per-point published wedge traces of the cubature path."""
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.stability import local_timesteps
    from paper_1507_02557_b200.timeint import lsrk_run
    d = Discretization(_perturbed(spec, 0.04, 11), N, form)
    st = d.project(cavity_fields, 0.0)
    dt = 0.5 * min(float(v.min()) for v in local_timesteps(d, 0.5).values())
    s = lsrk_run(d, st, dt, steps * dt)
    ref = oracle.lsrk_run(lambda q, tau: oracle.compute_rhs(d, q), st, dt, steps * dt)
    assert _l2rel(s, ref) < 1e-10


@pytest.mark.parametrize("mesh_name,nparts,method", [("wedge_tet", 2, "xslab"),
                                                     ("wedge_tet", 3, "rcb"),
                                                     ("wedge_pyramid", 2, "rcb")])
def test_partitioned_lsrk_loopback_face_corrections(mesh_name, nparts, method, native_lib):
    """Partitioned LSRK on meshes whose tets / pyramids meet non-affine wedge
    triangles: the correction rows of ghost wedges run after the halo
    exchange; equal to the single-GPU run to rounding."""
    from paper_1507_02557_b200 import mesh as M
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.parallel import LoopbackTransport, PartStepper, make_parts
    from paper_1507_02557_b200.timeint import LSRK_A, LSRK_B, Stepper
    from conftest import load_golden, set_random_materials
    g = (M.wedge_tet_columns_mesh(4, 2, 2) if mesh_name == "wedge_tet"
         else M.wedge_pyramid_columns_mesh(2, 0.3, 1))
    m = M.HybridMesh(load_golden(mesh_name)["X"], g.blocks)
    set_random_materials(m, 4)
    N, h = 2, 1e-3
    d = Discretization(m, N, "GL")
    assert d.has_corrections
    rng = np.random.default_rng(3)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    S = Stepper(d, st, "lsrk")
    for _ in range(3):
        S.lsrk_step(h)
    ref = {t: S.q[t].cpu().numpy() for t in d.types}
    parts = make_parts(m, nparts, method, N=N)
    T = LoopbackTransport()
    ps = [PartStepper(p, N, "GL", {t: st[t][p.global_ids[t]] for t in p.types}, T)
          for p in parts]
    n_ghost_rows = sum(c["n"] for p in ps if p.corr_rows for c in p.corr_rows[1].values())
    if mesh_name == "wedge_tet" and method == "xslab":
        assert n_ghost_rows > 0            # the cut runs between a tet and a wedge column
    for _ in range(3):
        for a, b in zip(LSRK_A, LSRK_B):
            for p in ps:
                p.begin()
            for p in ps:
                p.finish(a, b, h)
            for p in ps:
                p.swap()
    for p in ps:
        own = p.owned_state()
        for t in p.disc.types:
            g_ = p.part.global_ids[t][:p.part.n_owned[t]]
            r_ = ref[t][g_]
            if r_.size:
                assert np.abs(own[t].cpu().numpy() - r_).max() <= 1e-12 * np.abs(r_).max()


@pytest.mark.parametrize("nparts", [2, 3])
def test_partitioned_mrab_loopback_face_corrections(nparts, native_lib):
    """Partitioned multi-rate AB3 on the wedge/tet mesh (wedges level 1, tets
    level 2; the tets across non-affine wedge triangles get their correction
    rows every tick) equals the single-GPU MRABDriver to rounding."""
    from paper_1507_02557_b200 import mesh as M
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.parallel import LoopbackTransport, PartMRAB, make_parts
    from paper_1507_02557_b200.stability import TimestepPlan
    from paper_1507_02557_b200.timeint import MRABDriver
    from conftest import load_golden, set_random_materials
    g = M.wedge_tet_columns_mesh(4, 2, 2)
    m = M.HybridMesh(load_golden("wedge_tet")["X"], g.blocks)
    set_random_materials(m, 4)
    N = 2
    d = Discretization(m, N, "GL")
    assert d.has_corrections
    levels = {"wedge": np.full(d.n_elems["wedge"], 1), "tet": np.full(d.n_elems["tet"], 2)}
    plan = TimestepPlan({t: np.ones(d.n_elems[t]) for t in d.types}, levels, 2, 0.5,
                        list(d.types))
    dt_min = plan.dt_min = 2e-3
    st = d.project(cavity_fields, 0.0)
    n_macro = 5
    ref = {t: v.copy() for t, v in st.items()}
    MRABDriver(d, plan).run(ref, n_macro * 2 * dt_min, graph=False)
    parts = make_parts(m, nparts, "xslab", N=N)
    T = LoopbackTransport()
    ps = [PartMRAB(p, N, "GL", {t: st[t][p.global_ids[t]] for t in p.types},
                   {t: levels[t][p.global_ids[t]] for t in p.types}, 2, T) for p in parts]
    for _ in range(n_macro):
        for tick in range(2):
            for p in ps:
                p.tick_effective(tick, dt_min)
            hs = [p.tick_exchange() for p in ps]
            for p, h in zip(ps, hs):
                p.tick_step(tick, dt_min, h)
    for p in ps:
        own = p.owned_state()
        for t in p.disc.types:
            g_ = p.part.global_ids[t][:p.part.n_owned[t]]
            r_ = ref[t][g_]
            if r_.size:
                assert np.abs(own[t].cpu().numpy() - r_).max() <= 1e-12 * np.abs(r_).max()
