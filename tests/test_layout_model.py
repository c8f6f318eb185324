"""The packed device layout (tables, permutations, nodal-face lifts,
geometry records) reproduces the reference RHS, checked on the CPU through a
numpy model of the kernels (tests/layout_model.py)."""
import numpy as np
import pytest

import oracle
from conftest import RHS_CASES, load_golden, make_case, rel_err
from layout_model import rhs as model_rhs
from paper_1507_02557_b200.device import pack_mesh

RHS = load_golden("rhs")


@pytest.mark.parametrize("case", range(len(RHS_CASES)))
def test_layout_model_matches_reference(case):
    d, st = make_case(case)
    got = model_rhs(pack_mesh(d), d, st)
    ref = {t: RHS[f"{case}/{t}"] for t in d.types}
    assert rel_err(got, ref) < 1e-12


def test_mma_fragment_layouts():
    """A-fragment order of the DMMA operands: fragment (rt, ks) lane l holds
    A[8 rt + l // 4, 4 ks + l % 4]; pairs interleave k-steps 2m, 2m+1."""
    from paper_1507_02557_b200.device import mma_fragment_pairs, mma_fragments
    rng = np.random.default_rng(0)
    A = rng.standard_normal((2, 24, 20))
    F = mma_fragments(A)
    assert F.shape == (2, 3, 5, 32)
    for rt in range(3):
        for ks in range(5):
            for lane in range(32):
                assert F[1, rt, ks, lane] == A[1, 8 * rt + lane // 4, 4 * ks + lane % 4]
    P = mma_fragment_pairs(A)
    assert P.shape == (2, 3, 3, 32, 2)
    assert np.array_equal(P[..., :2, :, 0], F[..., 0:4:2, :])
    assert np.array_equal(P[..., :2, :, 1], F[..., 1:4:2, :])
    assert np.array_equal(P[..., 2, :, 0], F[..., 4, :]) and not P[..., 2, :, 1].any()


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("form", ["GL", "SEM"])
def test_hex_face_point_map_is_affine(N, form):
    from paper_1507_02557_b200.device import hex_face_point_coefficients, hex_node_face_points
    from paper_1507_02557_b200.operators import build_operators, device_operators
    d = device_operators("hex", N, form, build_operators("hex", N, form))
    c = hex_face_point_coefficients(d, N)
    tab = hex_node_face_points(d, N)
    n1 = N + 1
    n = np.arange(n1 ** 3)
    I = np.stack([n // (n1 * n1), (n // n1) % n1, n % n1, np.ones_like(n)], axis=1)
    assert np.array_equal(I @ c.T.astype(np.int64), tab.T)


def _perturbed(spec, amp, seed):
    from conftest import build_mesh
    from paper_1507_02557_b200.mesh import HybridMesh
    m = build_mesh(spec)
    rng = np.random.default_rng(seed)
    X = m.vertices.copy()
    inner = np.all((X > 1e-9) & (X < 1 - 1e-9), axis=1)
    X[inner] += amp * rng.uniform(-1, 1, (inner.sum(), 3))
    return HybridMesh(X, m.blocks)


NAW_CASES = [("wed2_gl1", "wedge:2", 1, "GL", 6), ("wed3_gl2", "wedge:3", 2, "GL", 7),
             ("wed3_sem3", "wedge:3", 3, "SEM", 8)]


@pytest.mark.parametrize("tag,spec,N,form,seed", NAW_CASES)
def test_nonaffine_wedge_layout_matches_reference(tag, spec, N, form, seed):
    """Non-affine wedges: the packed cubature data (op[8], op[9]) through the
    model of the kernel's cubature path reproduce the reference's RHS."""
    from layout_model import naw_rhs
    from paper_1507_02557_b200.dg import Discretization
    G = load_golden("nonaffine")
    d = Discretization(_perturbed(spec, 0.04, seed), N, form)
    rng = np.random.default_rng(seed + 10)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    pack = pack_mesh(d)
    assert set(pack["types"]["wedge"]["op"]) >= {8, 9}
    assert rel_err(naw_rhs(pack, d, st), {"wedge": G[f"{tag}/rhs/wedge"]}) < 1e-12
    assert rel_err(oracle.compute_rhs(d, st), {"wedge": G[f"{tag}/rhs/wedge"]}) < 1e-12


def test_nonaffine_wedge_next_to_tets_gets_face_corrections():
    """A non-affine wedge whose triangle face touches a tet: the tet side
    gets the face-cubature correction rows (device.wedge_face_corrections);
    an affine wedge needs none."""
    from paper_1507_02557_b200.device import wedge_face_corrections
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import HybridMesh
    def mesh(x4):
        X = np.array([(0, 0, 0), (0, 1, 1), (0, 1, 0), (1, 0, 0), (x4, 1, 1), (1, 1, 0),
                      (2.0, 0.7, 0.3)])
        return HybridMesh(X, {"wedge": np.array([[0, 1, 2, 3, 4, 5]]),
                              "tet": np.array([[3, 5, 4, 6]])})
    m = mesh(1.2)
    assert 3 in m.nbr["wedge"][0, :2, 0]
    d = Discretization(m, 2, "GL")
    c = wedge_face_corrections(d, pack_mesh(d))
    assert set(c) == {"tet"} and c["tet"]["idata"].shape[0] == 1
    assert np.abs(c["tet"]["fdata"][:, 6:6 + c["tet"]["nq"]]).max() > 0   # s - 1 != 0
    d1 = Discretization(mesh(1.0), 2, "GL")
    assert wedge_face_corrections(d1, pack_mesh(d1)) == {}


def test_wedge_tet_mesh_corrections_cover_every_shared_triangle():
    from paper_1507_02557_b200.device import wedge_face_corrections
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import HybridMesh, wedge_tet_columns_mesh
    g = wedge_tet_columns_mesh(4, 2, 2)
    X = load_golden("wedge_tet")["X"]
    d = Discretization(HybridMesh(X, g.blocks), 2, "GL")
    c = wedge_face_corrections(d, pack_mesh(d))
    shared = int(np.sum(d.mesh.nbr["tet"][:, :, 0] == 1))
    assert c["tet"]["idata"].shape[0] == shared == 24


def test_oracle_on_wedge_tet_mesh_matches_reference():
    """The oracle on the jittered wedge/tet column mesh = the reference's RHS
    (pins the oracle for the device's face-correction path)."""
    from conftest import set_random_materials
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import HybridMesh, wedge_tet_columns_mesh
    Gw = load_golden("wedge_tet")
    g = wedge_tet_columns_mesh(4, 2, 2)
    for tag, N, form in [("n1_gl", 1, "GL"), ("n3_sem", 3, "SEM")]:
        m = HybridMesh(Gw["X"], g.blocks)
        set_random_materials(m, 4)
        d = Discretization(m, N, form, device="cpu")
        rng = np.random.default_rng(N + 30)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        assert rel_err(oracle.compute_rhs(d, st), {t: Gw[f"{tag}/rhs/{t}"] for t in d.types}) < 1e-12


def test_wedge_pyramid_mesh_corrections_cover_every_shared_triangle():
    """Jittered wedges next to affine pyramids (wedge_pyramid_columns_mesh):
    every pyramid triangle shared with a wedge gets a correction row; the
    pyramids stay affine (DMMA kernel), the wedges take the cubature path."""
    from paper_1507_02557_b200.device import wedge_face_corrections
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import HybridMesh, mesh_volume, wedge_pyramid_columns_mesh
    from paper_1507_02557_b200.refelem import affine_mask
    g = wedge_pyramid_columns_mesh(2, 0.3, 1)
    X = load_golden("wedge_pyramid")["X"]
    np.testing.assert_array_equal(g.vertices, X)
    m = HybridMesh(X, g.blocks)
    assert abs(mesh_volume(m) - 0.5) < 1e-12
    assert not affine_mask("wedge", X[m.blocks["wedge"]], tol=1e-10).any()
    assert affine_mask("pyramid", X[m.blocks["pyramid"]], tol=1e-10).all()
    d = Discretization(m, 2, "GL")
    pack = pack_mesh(d)
    assert 8 in pack["types"]["wedge"]["op"] and 8 not in pack["types"]["pyramid"]["op"]
    c = wedge_face_corrections(d, pack)
    shared = int(np.sum(d.mesh.nbr["pyramid"][:, :, 0] == 1))
    assert set(c) == {"pyramid"} and c["pyramid"]["idata"].shape[0] == shared == 8
    assert set(c["pyramid"]["idata"][:, 1]) <= {1, 2, 3, 4}          # triangle faces only


def test_oracle_on_wedge_pyramid_mesh_matches_reference():
    from conftest import set_random_materials
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import HybridMesh, wedge_pyramid_columns_mesh
    Gw = load_golden("wedge_pyramid")
    g = wedge_pyramid_columns_mesh(2, 0.3, 1)
    for tag, N, form in [("n1_gl", 1, "GL"), ("n3_sem", 3, "SEM")]:
        m = HybridMesh(Gw["X"], g.blocks)
        set_random_materials(m, 5)
        d = Discretization(m, N, form, device="cpu")
        rng = np.random.default_rng(N + 40)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        assert rel_err(oracle.compute_rhs(d, st), {t: Gw[f"{tag}/rhs/{t}"] for t in d.types}) < 1e-12
