"""Host setup (operators, meshes, reference-layout geometry) against
fixtures generated from the reference package (tests/golden/make_golden.py)."""
import numpy as np
import pytest

from conftest import RHS_CASES, build_mesh, load_golden, make_case
from paper_1507_02557_b200 import operators as ops_mod

OPS = load_golden("operators")


@pytest.mark.parametrize("t", ["hex", "wedge", "pyramid", "tet"])
@pytest.mark.parametrize("N", [1, 2, 3])
@pytest.mark.parametrize("form", ["GL", "SEM"])
def test_operators_match_reference(t, N, form):
    o = ops_mod.build_operators(t, N, form)
    keys = [k for k in OPS.files if k.startswith(f"{t}/{N}/{form}/")]
    assert keys
    for k in keys:
        ref = OPS[k]
        mine = np.asarray(getattr(o, k.split("/")[-1]))
        assert mine.shape == ref.shape, k
        assert np.abs(mine - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), k


MESH = load_golden("meshes")


@pytest.mark.parametrize("spec", ["hybrid:3", "hex:2", "tet:2", "wedge:2", "pyramid:2"])
def test_mesh_numbering_and_links(spec):
    m = build_mesh(spec)
    np.testing.assert_allclose(m.vertices, MESH[f"{spec}/vertices"], atol=1e-14)
    tid = {"hex": 0, "wedge": 1, "pyramid": 2, "tet": 3}
    for t in m.elem_types:
        np.testing.assert_array_equal(m.blocks[t], MESH[f"{spec}/{t}/blocks"])
        ref = MESH[f"{spec}/{t}/links"]
        nb = m.nbr[t]
        np.testing.assert_array_equal(nb[:, :, 0], np.where(ref[:, :, 0] >= 0, ref[:, :, 0], -1))
        inner = ref[:, :, 0] >= 0
        np.testing.assert_array_equal(nb[:, :, 1][inner], ref[:, :, 1][inner])
        np.testing.assert_array_equal(nb[:, :, 2][inner], ref[:, :, 2][inner])
        np.testing.assert_array_equal(m._ref_code[t][inner], ref[:, :, 3][inner])


RHS = load_golden("rhs")


@pytest.mark.parametrize("case", [0, 1])
def test_reference_layout_geometry(case):
    d, _ = make_case(case)
    for t in d.types:
        for f in ("J", "G", "wJs", "normals", "tau_p", "tau_u", "gJfac", "invsqrtJ_face"):
            key = f"{case}/{t}/data/{f}"
            mine = getattr(d.data[t], f)
            if key not in RHS.files:
                assert mine is None
                continue
            ref = RHS[key]
            assert np.abs(mine - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), (t, f)
    assert np.array_equal(d.bnd_mask, RHS[f"{case}/bnd"])
    # gathers may pick either copy of a duplicated triangle point: compare positions
    g_ref = RHS[f"{case}/gather"]
    pos = np.concatenate([d.data[t].x_face.reshape(-1, 3) for t in d.types])
    assert np.abs(pos[d.gather_idx] - pos[g_ref]).max() < 1e-12


def test_tri_face_nodes_symmetric():
    for N in range(1, 8):
        p = ops_mod.tri_face_nodes_2d(N)
        assert len(p) == (N + 1) * (N + 2) // 2
        perms = ops_mod.face_symmetry_perms("tri", p)
        for row in perms:
            assert sorted(row) == list(range(len(p)))


def test_nodal_lift_reproduces_stored_rule():
    """The nodal-face LIFT equals the reference's 6(N+1)^2-point surface
    integral for polynomial face data (SURVEY 0.5 / DESIGN.md)."""
    rng = np.random.default_rng(3)
    for t in ("tet", "wedge", "pyramid"):
        for N in (1, 2, 3, 4):
            o = ops_mod.build_operators(t, N, "GL")
            dops = ops_mod.device_operators(t, N, "GL", o)
            q = rng.standard_normal(o.Np)
            offs = dops["face_offsets"]
            for f, (ft, _) in enumerate(__import__("paper_1507_02557_b200.refelem",
                                                   fromlist=["FACES"]).FACES[t]):
                if ft != "tri":
                    continue
                sl = slice(o.face_offsets[f], o.face_offsets[f + 1])
                ref = o.Vf[sl].T @ (o.face_wts[f] * (o.Vf[sl] @ q))
                if t == "tet":
                    ref = o.invM_ref @ ref
                dv = slice(offs[f], offs[f + 1])
                mine = dops["LIFT"][:, dv] @ (dops["E"][dv] @ q)
                assert np.abs(mine - ref).max() < 1e-12 * max(1, np.abs(ref).max()), (t, N, f)
