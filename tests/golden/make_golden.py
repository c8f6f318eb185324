"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is not on the GPU box):
    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz (`make_golden.py forcing`: only forcing.npz).  States are regenerated in the tests from the
recorded seeds (np.random.default_rng(seed).standard_normal(shape)), so
only reference outputs are stored.
"""

import os
import sys

import numpy as np

import hybridwave
from hybridwave import operators as ops_mod
from hybridwave.app import cavity_fields
from hybridwave.dg import Discretization, discrete_energy
from hybridwave.mesh import structured_hybrid_mesh, uniform_cube_mesh
from hybridwave.stability import assign_mrab_levels, local_timesteps
from hybridwave.timeint import mrab_run, single_rate_run

HERE = os.path.dirname(os.path.abspath(__file__))

# LSRK(4,5) 2N-storage, Carpenter & Kennedy 1994 (the reference has none)
A = [0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
     -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0]
B = [1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
     1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
     2277821191437.0 / 14882151754819.0]
C = [0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
     2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0]


def build_mesh(spec):
    kind, n = spec.split(":")
    n = int(n)
    return structured_hybrid_mesh(n) if kind == "hybrid" else uniform_cube_mesh(kind, n)


def set_random_materials(mesh, seed):
    rng = np.random.default_rng(seed)
    for t in mesh.elem_types:
        mesh.materials[t] = rng.uniform(0.5, 2.0, (len(mesh.blocks[t]), 2))


def lsrk_run_ref(disc, state, dt, T_final):
    q = {t: v.copy() for t, v in state.items()}
    res = {t: np.zeros_like(v) for t, v in q.items()}
    time = 0.0
    while time < T_final - 1e-14:
        h = min(dt, T_final - time)
        for a, b, c in zip(A, B, C):
            k = disc.compute_rhs(q, time + c * h)
            for t in q:
                res[t] = a * res[t] + h * k[t]
                q[t] = q[t] + b * res[t]
        time += h
    return q


RHS_CASES = [
    # (mesh, N, formulation, materials seed or None, penalty_scale, state seed)
    ("hybrid:2", 1, "GL", None, 1.0, 0),
    ("hybrid:2", 2, "GL", None, 1.0, 1),
    ("hybrid:2", 3, "GL", 7, 1.0, 2),
    ("hybrid:2", 1, "SEM", None, 1.0, 3),
    ("hybrid:2", 2, "SEM", 7, 1.0, 4),
    ("hybrid:2", 3, "SEM", None, 1.0, 5),
    ("hybrid:3", 2, "GL", 7, 1.0, 6),
    ("hybrid:2", 2, "GL", None, 0.0, 7),
    ("hex:2", 2, "SEM", None, 1.0, 8),
    ("hex:2", 3, "GL", 7, 1.0, 9),
    ("tet:2", 3, "GL", None, 1.0, 10),
    ("wedge:2", 2, "SEM", None, 1.0, 11),
    ("pyramid:2", 2, "SEM", None, 1.0, 12),
    ("pyramid:2", 2, "GL", 7, 1.0, 13),
    ("hybrid:2", 4, "GL", None, 1.0, 14),
    ("hybrid:2", 5, "SEM", None, 1.0, 15),
]


def main():
    out = {"reference_version": hybridwave.__version__, "numpy": np.__version__}
    # ---- operators
    opsd = {}
    for t in ("hex", "wedge", "pyramid", "tet"):
        for N in (1, 2, 3):
            for form in ("GL", "SEM"):
                o = ops_mod.build_operators(t, N, form)
                for f in ("Vf", "D1", "Vf_end", "Dr", "Ds", "Dt", "M_ref", "invM_ref", "V",
                          "Dr3", "Ds3", "Dt3", "nodes", "level_abc"):
                    if hasattr(o, f):
                        opsd[f"{t}/{N}/{form}/{f}"] = np.asarray(getattr(o, f))
    np.savez_compressed(os.path.join(HERE, "operators.npz"), **opsd)

    # ---- meshes and connectivity
    md = {}
    for spec in ("hybrid:3", "hex:2", "tet:2", "wedge:2", "pyramid:2"):
        m = build_mesh(spec)
        md[f"{spec}/vertices"] = m.vertices
        for t in m.elem_types:
            md[f"{spec}/{t}/blocks"] = m.blocks[t]
            nb = np.full((len(m.blocks[t]), len(m.face_links[t][0]), 4), -1)
            tid = {"hex": 0, "wedge": 1, "pyramid": 2, "tet": 3}
            for k, row in enumerate(m.face_links[t]):
                for f, l in enumerate(row):
                    if not l.is_boundary:
                        t2, k2, f2 = l.neighbor
                        nb[k, f] = (tid[t2], k2, f2, l.orientation)
            md[f"{spec}/{t}/links"] = nb
    np.savez_compressed(os.path.join(HERE, "meshes.npz"), **md)

    # ---- single-RHS parity
    rd = {}
    for i, (spec, N, form, mseed, pen, sseed) in enumerate(RHS_CASES):
        m = build_mesh(spec)
        if mseed is not None:
            set_random_materials(m, mseed)
        d = Discretization(m, N, form, penalty_scale=pen)
        rng = np.random.default_rng(sseed)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        r = d.compute_rhs(st)
        for t in d.types:
            rd[f"{i}/{t}"] = r[t]
        # geometry / coupling arrays of the first cases
        if i < 2:
            for t in d.types:
                for f in ("J", "G", "wJs", "normals", "tau_p", "tau_u", "gJfac",
                          "invsqrtJ_face"):
                    v = getattr(d.data[t], f)
                    if v is not None:
                        rd[f"{i}/{t}/data/{f}"] = v
            rd[f"{i}/gather"] = d.gather_idx
            rd[f"{i}/bnd"] = d.bnd_mask
    np.savez_compressed(os.path.join(HERE, "rhs.npz"), **rd)

    # ---- trajectories (100 steps)
    td = {}
    for tag, spec, N, form in (("c1_sem", "hex:4", 2, "SEM"), ("c1_gl", "hex:4", 2, "GL"),
                               ("hyb4_gl", "hybrid:4", 3, "GL")):
        m = build_mesh(spec)
        d = Discretization(m, N, form)
        st0 = d.project(cavity_fields, 0.0)
        dt = min(float(v.min()) for v in local_timesteps(d, 0.5).values())
        T = 100 * dt
        if tag != "hyb4_gl":
            en = []
            sab = single_rate_run(d, st0, dt, T, callback=lambda tau, s: en.append(
                discrete_energy(s, d)))
            err = d.l2_error(sab, cavity_fields, T)
            for t in d.types:
                td[f"{tag}/ab3/{t}"] = sab[t]
            td[f"{tag}/ab3/err"] = np.array([err["p"], err["u"], err["total"]])
            td[f"{tag}/ab3/energy"] = np.array(en)
        slr = lsrk_run_ref(d, st0, dt, T)
        err = d.l2_error(slr, cavity_fields, T)
        for t in d.types:
            td[f"{tag}/lsrk/{t}"] = slr[t]
        td[f"{tag}/lsrk/err"] = np.array([err["p"], err["u"], err["total"]])
        td[f"{tag}/dt"] = np.array(dt)
        td[f"{tag}/energy0"] = np.array(discrete_energy(st0, d))
    # MRAB on the reference hybrid mesh (2 occupied levels) and uniform-level check
    m = build_mesh("hybrid:2")
    d = Discretization(m, 2, "GL")
    st0 = d.project(cavity_fields, 0.0)
    dtl = local_timesteps(d, 0.5)
    plan = assign_mrab_levels(dtl, 3, m, cfl=0.5)
    T = 8 * 4 * plan.dt_min
    s, drv = mrab_run(d, plan, {t: v.copy() for t, v in st0.items()}, T)
    for t in d.types:
        td[f"mrab/{t}"] = s[t]
        td[f"mrab/levels/{t}"] = plan.levels[t]
        td[f"mrab/evals/{t}"] = drv.rhs_evals[t]
    td["mrab/dt_min"] = np.array(plan.dt_min)
    td["mrab/T"] = np.array(T)
    np.savez_compressed(os.path.join(HERE, "trajectories.npz"), **td)
    np.savez_compressed(os.path.join(HERE, "meta.npz"), **{k: np.array(v) for k, v in out.items()})
    print("golden fixtures written to", HERE)


def forcing_fn(x, time):
    """Smooth volume source f(x, t) for the forcing fixtures (K, nq, 3) -> (K, nq)."""
    return (np.sin(np.pi * x[..., 0]) * np.cos(np.pi * x[..., 1]) * (1.0 + x[..., 2])
            * np.cos(3.0 * time))


def forcing_fixtures():
    """compute_rhs with a forcing callback, and 10 AB3 / LSRK steps with it."""
    fd = {}
    for tag, spec, N, form in [("hyb2_gl", "hybrid:2", 2, "GL"), ("hyb2_sem", "hybrid:2", 2, "SEM"),
                               ("tet2_gl", "tet:2", 3, "GL")]:
        mesh = build_mesh(spec)
        set_random_materials(mesh, 5)
        d = Discretization(mesh, N, form, forcing=forcing_fn)
        st = d.project(cavity_fields, 0.0)
        rhs = d.compute_rhs(st, 0.37)
        dt = 0.5 * min(float(v.min()) for v in local_timesteps(d, 0.5).values())
        ab = single_rate_run(d, st, dt, 10 * dt)
        lk = lsrk_run_ref(d, st, dt, 10 * dt)
        for t in d.types:
            fd[f"{tag}/rhs/{t}"] = rhs[t]
            fd[f"{tag}/ab3/{t}"] = ab[t]
            fd[f"{tag}/lsrk/{t}"] = lk[t]
        fd[f"{tag}/dt"] = np.array(dt)
    # multi-rate AB3 with forcing (hybrid:2, the trajectories.npz MRAB setup)
    m = build_mesh("hybrid:2")
    d = Discretization(m, 2, "GL", forcing=forcing_fn)
    st0 = d.project(cavity_fields, 0.0)
    plan = assign_mrab_levels(local_timesteps(d, 0.5), 3, m, cfl=0.5)
    T = 6 * 4 * plan.dt_min
    s, drv = mrab_run(d, plan, {t: v.copy() for t, v in st0.items()}, T)
    for t in d.types:
        fd[f"mrab/{t}"] = s[t]
        fd[f"mrab/levels/{t}"] = plan.levels[t]
    fd["mrab/dt_min"] = np.array(plan.dt_min)
    fd["mrab/T"] = np.array(T)
    np.savez_compressed(os.path.join(HERE, "forcing.npz"), **fd)
    print("forcing fixtures written")


def forms_fixtures():
    """compute_rhs with the forms_override testing hook (skew hex / tet,
    strong pyramid SEM) on random states."""
    fd = {}
    cases = [("hyb2_skew", "hybrid:2", 2, "GL", {"hex": "skew", "tet": "skew"}),
             ("hyb3_skew", "hybrid:2", 3, "SEM", {"hex": "skew", "tet": "skew"}),
             ("hex2_skew", "hex:2", 3, "GL", {"hex": "skew"}),
             ("tet2_skew", "tet:2", 3, "GL", {"tet": "skew"}),
             ("hyb2_wstrong", "hybrid:2", 2, "GL", {"wedge": "strong", "pyramid": "skew"}),
             ("hyb2_pstrong", "hybrid:2", 2, "SEM", {"pyramid": "strong"})]
    for tag, spec, N, form, over in cases:
        mesh = build_mesh(spec)
        set_random_materials(mesh, 9)
        d = Discretization(mesh, N, form, forms_override=over)
        rng = np.random.default_rng(11)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        rhs = d.compute_rhs(st, 0.0)
        for t in d.types:
            fd[f"{tag}/rhs/{t}"] = rhs[t]
    np.savez_compressed(os.path.join(HERE, "forms.npz"), **fd)
    print("forms fixtures written")


def convergence_fixtures():
    """The reference's own h-convergence studies of the cavity mode (AB3,
    cfl 0.5, T = 0.1): errors and least-squares rates."""
    from hybridwave.app import RunConfig, convergence_study
    fd = {}
    for N, form in [(1, "GL"), (2, "GL"), (3, "GL"), (2, "SEM"), (3, "SEM")]:
        cfg = RunConfig(mesh="hybrid:2", N=N, formulation=form, cfl=0.5, T_final=0.1)
        errs, rate = convergence_study(cfg, [2, 3, 4], verbose=False)
        fd[f"N{N}_{form}/errs"] = np.asarray(errs)
        fd[f"N{N}_{form}/rate"] = np.array(rate)
    np.savez_compressed(os.path.join(HERE, "convergence.npz"), **fd)
    print("convergence fixtures written")


def nonaffine_fixtures():
    """compute_rhs on jittered (non-affine) pyramid and wedge meshes, random
    states; same perturbation as tests/test_gpu_parity.py::_perturbed."""
    from hybridwave.mesh import HybridMesh
    fd = {}
    for tag, spec, N, form, seed in [("pyr3_gl2", "pyramid:3", 2, "GL", 3),
                                     ("pyr3_sem3", "pyramid:3", 3, "SEM", 4),
                                     ("pyr2_gl4", "pyramid:2", 4, "GL", 5),
                                     ("wed2_gl1", "wedge:2", 1, "GL", 6),
                                     ("wed3_gl2", "wedge:3", 2, "GL", 7),
                                     ("wed3_sem3", "wedge:3", 3, "SEM", 8),
                                     ("wed2_gl5", "wedge:2", 5, "GL", 9)]:
        m = build_mesh(spec)
        rng = np.random.default_rng(seed)
        X = m.vertices.copy()
        inner = np.all((X > 1e-9) & (X < 1 - 1e-9), axis=1)
        X[inner] += 0.04 * rng.uniform(-1, 1, (inner.sum(), 3))
        m = HybridMesh(X, m.blocks)
        d = Discretization(m, N, form)
        rng = np.random.default_rng(seed + 10)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        rhs = d.compute_rhs(st, 0.0)
        for t in d.types:
            fd[f"{tag}/rhs/{t}"] = rhs[t]
    np.savez_compressed(os.path.join(HERE, "nonaffine.npz"), **fd)
    print("non-affine fixtures written")


def mrab_multilevel_fixtures():
    """Reference mrab_run on a graded mesh where 3 (and, with n_levels=5,
    more) rate levels are occupied.  The graded generator is the repo's own
    (the reference has none); its vertices / blocks are wrapped in the
    reference's HybridMesh so every number below comes from the reference."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1507_02557_b200.mesh import graded_hybrid_mesh
    from hybridwave.mesh import HybridMesh
    fd = {}
    g = graded_hybrid_mesh(6)
    for tag, N, form, n_levels, n_macro in [("g6_n2_gl_l3", 2, "GL", 3, 7),
                                            ("g6_n3_gl_l3", 3, "GL", 3, 6),
                                            ("g6_n2_sem_l3", 2, "SEM", 3, 6),
                                            ("g6_n2_gl_l5", 2, "GL", 5, 3)]:
        m = HybridMesh(g.vertices.copy(), {t: g.blocks[t].copy() for t in g.elem_types})
        d = Discretization(m, N, form)
        st0 = d.project(cavity_fields, 0.0)
        plan = assign_mrab_levels(local_timesteps(d, 0.5), n_levels, m, cfl=0.5)
        occupied = sorted({int(x) for v in plan.levels.values() for x in np.unique(v)})
        T = n_macro * 2 ** (n_levels - 1) * plan.dt_min
        en = []
        s, drv = mrab_run(d, plan, {t: v.copy() for t, v in st0.items()}, T,
                          callback=lambda tau, st: en.append(discrete_energy(st, d)))
        for t in d.types:
            fd[f"{tag}/{t}"] = s[t]
            fd[f"{tag}/levels/{t}"] = plan.levels[t]
            fd[f"{tag}/evals/{t}"] = drv.rhs_evals[t]
        fd[f"{tag}/dt_min"] = np.array(plan.dt_min)
        fd[f"{tag}/T"] = np.array(T)
        fd[f"{tag}/occupied"] = np.array(occupied)
        fd[f"{tag}/macro_steps"] = np.array(drv.macro_steps)
        fd[f"{tag}/energy"] = np.array(en)
        fd[f"{tag}/energy0"] = np.array(discrete_energy(st0, d))
        print(tag, "levels", occupied, "macro", drv.macro_steps,
              "elements", {t: d.n_elems[t] for t in d.types})
    # uniform levels: one occupied level must reproduce single-rate AB3
    m = HybridMesh(g.vertices.copy(), {t: g.blocks[t].copy() for t in g.elem_types})
    d = Discretization(m, 2, "GL")
    st0 = d.project(cavity_fields, 0.0)
    dt = min(float(v.min()) for v in local_timesteps(d, 0.5).values())
    sab = single_rate_run(d, {t: v.copy() for t, v in st0.items()}, dt, 12 * dt)
    for t in d.types:
        fd[f"uniform/ab3/{t}"] = sab[t]
    fd["uniform/dt"] = np.array(dt)
    np.savez_compressed(os.path.join(HERE, "mrab_levels.npz"), **fd)
    print("multi-level MRAB fixtures written")


def wedge_tet_fixtures():
    """Non-affine (jittered) wedges whose triangle faces meet tets: the
    reference's RHS (face cubature on both sides) and 10 LSRK-45 steps.  The
    mesh generator is the repo's (wedge_tet_columns_mesh); every number
    below comes from the reference's HybridMesh / Discretization."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1507_02557_b200.mesh import wedge_tet_columns_mesh
    from hybridwave.mesh import HybridMesh
    fd = {}
    g = wedge_tet_columns_mesh(4, 2, 2)
    rng = np.random.default_rng(21)
    X = g.vertices.copy()
    inner = np.all((X > 1e-9) & (X < 1 - 1e-9), axis=1)
    X[inner] += 0.04 * rng.uniform(-1, 1, (inner.sum(), 3))
    fd["X"] = X
    for tag, N, form in [("n1_gl", 1, "GL"), ("n2_gl", 2, "GL"), ("n3_sem", 3, "SEM"),
                         ("n3_gl", 3, "GL")]:
        m = HybridMesh(X, {t: g.blocks[t].copy() for t in g.elem_types})
        set_random_materials(m, 4)
        d = Discretization(m, N, form)
        rng = np.random.default_rng(N + 30)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        rhs = d.compute_rhs(st, 0.0)
        for t in d.types:
            fd[f"{tag}/rhs/{t}"] = rhs[t]
        st0 = d.project(cavity_fields, 0.0)
        dt = 0.5 * min(float(v.min()) for v in local_timesteps(d, 0.5).values())
        lk = lsrk_run_ref(d, st0, dt, 10 * dt)
        for t in d.types:
            fd[f"{tag}/lsrk/{t}"] = lk[t]
        fd[f"{tag}/dt"] = np.array(dt)
    np.savez_compressed(os.path.join(HERE, "wedge_tet.npz"), **fd)
    print("wedge/tet fixtures written")


def wedge_pyramid_fixtures():
    """Non-affine (jittered) wedges whose triangle faces meet affine
    pyramids: the reference's RHS and 10 LSRK-45 steps on the repo's
    wedge_pyramid_columns_mesh (every number from the reference)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1507_02557_b200.mesh import wedge_pyramid_columns_mesh
    from hybridwave.mesh import HybridMesh
    fd = {}
    g = wedge_pyramid_columns_mesh(2, 0.3, 1)
    fd["X"] = g.vertices.copy()
    for tag, N, form in [("n1_gl", 1, "GL"), ("n2_gl", 2, "GL"), ("n3_sem", 3, "SEM"),
                         ("n3_gl", 3, "GL")]:
        m = HybridMesh(g.vertices.copy(), {t: g.blocks[t].copy() for t in g.elem_types})
        set_random_materials(m, 5)
        d = Discretization(m, N, form)
        rng = np.random.default_rng(N + 40)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        rhs = d.compute_rhs(st, 0.0)
        for t in d.types:
            fd[f"{tag}/rhs/{t}"] = rhs[t]
        st0 = d.project(cavity_fields, 0.0)
        dt = 0.5 * min(float(v.min()) for v in local_timesteps(d, 0.5).values())
        lk = lsrk_run_ref(d, st0, dt, 10 * dt)
        for t in d.types:
            fd[f"{tag}/lsrk/{t}"] = lk[t]
        fd[f"{tag}/dt"] = np.array(dt)
    np.savez_compressed(os.path.join(HERE, "wedge_pyramid.npz"), **fd)
    print("wedge/pyramid fixtures written")


if __name__ == "__main__":
    if sys.argv[1:] == ["wedge_pyramid"]:
        sys.exit(wedge_pyramid_fixtures())
    if sys.argv[1:] == ["wedge_tet"]:
        sys.exit(wedge_tet_fixtures())
    if sys.argv[1:] == ["mrab_levels"]:
        sys.exit(mrab_multilevel_fixtures())
    if sys.argv[1:] == ["nonaffine"]:
        sys.exit(nonaffine_fixtures())
    if sys.argv[1:] == ["convergence"]:
        sys.exit(convergence_fixtures())
    if sys.argv[1:] == ["forcing"]:
        sys.exit(forcing_fixtures())
    if sys.argv[1:] == ["forms"]:
        sys.exit(forms_fixtures())
    sys.exit(main())
