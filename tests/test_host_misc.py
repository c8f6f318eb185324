"""Host-side pieces on CPU: the sampled sub-mesh oracle used by the
full-size GPU parity tests, the GMSH reader, mesh_volume, the app config."""
import os

import numpy as np
import pytest

import oracle
from conftest import build_mesh, set_random_materials
from sampled import default_sample, neighbour_closure, sampled_oracle_rhs


@pytest.mark.parametrize("spec,N,form", [("hybrid:4", 2, "GL"), ("hybrid:3", 3, "SEM")])
def test_sampled_oracle_equals_whole_mesh_oracle(spec, N, form):
    """The oracle on the neighbour-closed sub-mesh reproduces the whole-mesh
    oracle on the sampled rows (the basis of the full-size GPU parity)."""
    from paper_1507_02557_b200.dg import Discretization
    m = build_mesh(spec)
    set_random_materials(m, 2)
    d = Discretization(m, N, form, device="cpu")
    rng = np.random.default_rng(1)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    full = oracle.compute_rhs(d, st)
    sample = default_sample(m, n_random=20, n_edge=5, seed=3)
    keep = neighbour_closure(m, sample)
    assert sum(len(v) for v in keep.values()) < m.n_elements
    got = sampled_oracle_rhs(d, lambda t, ids: st[t][ids], sample)
    for t, ids in sample.items():
        assert np.abs(got[t] - full[t][ids]).max() <= 1e-13 * np.abs(full[t]).max()


def _write_msh(path, mesh, extra_lines=()):
    """GMSH 2.2 writer for the test (prism corners in gmsh order)."""
    code = {"tet": 4, "hex": 5, "wedge": 6, "pyramid": 7}
    to_gmsh = {"wedge": [0, 2, 1, 3, 5, 4]}
    lines = ["$MeshFormat", "2.2 0 8", "$EndMeshFormat", "$Nodes", str(len(mesh.vertices))]
    lines += [f"{i + 11} {x:.17g} {y:.17g} {z:.17g}" for i, (x, y, z) in enumerate(mesh.vertices)]
    lines += ["$EndNodes", "$Elements"]
    rows = list(extra_lines)
    e = 1
    for t in mesh.elem_types:
        for k, c in enumerate(mesh.blocks[t]):
            c = c[to_gmsh[t]] if t in to_gmsh else c
            rows.append(f"{e} {code[t]} 2 {k % 3 + 1} 0 " + " ".join(str(v + 11) for v in c))
            e += 1
    lines += [str(len(rows))] + rows + ["$EndElements"]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def test_gmsh_round_trip(tmp_path):
    from paper_1507_02557_b200.mesh import mesh_volume, read_gmsh
    m = build_mesh("hybrid:3")
    p = tmp_path / "h.msh"
    _write_msh(p, m, extra_lines=["900 2 2 1 1 11 12 13", "901 15 1 4 11"])
    r = read_gmsh(str(p))
    assert r.elem_types == m.elem_types
    np.testing.assert_array_equal(r.vertices, m.vertices)
    for t in m.elem_types:
        np.testing.assert_array_equal(r.blocks[t], m.blocks[t])
        np.testing.assert_array_equal(r.nbr[t], m.nbr[t])
        np.testing.assert_array_equal(r.physical[t], np.arange(len(m.blocks[t])) % 3 + 1)
    assert abs(mesh_volume(r) - 1.0) < 1e-12


@pytest.mark.parametrize("edit,msg,line", [
    (lambda L: L.__setitem__(1, "4.1 0 8"), "only msh format 2.2", 2),
    (lambda L: L.__setitem__(4, "x"), "bad node count", 5),
    (lambda L: L.__setitem__(5, "11 0.0 0.0"), "bad node line", 6),
    (lambda L: L.__setitem__(0, "$Mesh"), "expected $MeshFormat", 1),
])
def test_gmsh_errors_name_the_line(tmp_path, edit, msg, line):
    from paper_1507_02557_b200.mesh import GmshParseError, read_gmsh
    m = build_mesh("tet:1")
    p = tmp_path / "t.msh"
    _write_msh(p, m)
    L = p.read_text().splitlines()
    edit(L)
    p.write_text("\n".join(L) + "\n")
    with pytest.raises(GmshParseError) as e:
        read_gmsh(str(p))
    assert msg in str(e.value) and f":{line}:" in str(e.value)


def test_gmsh_bad_elements(tmp_path):
    from paper_1507_02557_b200.mesh import GmshParseError, read_gmsh
    m = build_mesh("tet:1")
    for bad, msg in [("99 9 2 1 1 11 12 13", "unsupported element code 9"),
                     ("99 4 2 1 1 11 12 13", "tet element needs 4 nodes, got 3"),
                     ("99 4 2 1 1 11 12 13 999", "unknown node id 999")]:
        p = tmp_path / "b.msh"
        _write_msh(p, m, extra_lines=[bad])
        with pytest.raises(GmshParseError, match=msg):
            read_gmsh(str(p))


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference absent")
def test_gmsh_reader_matches_reference(tmp_path):
    """Same vertices, blocks and physical groups as the reference's reader."""
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.dont_write_bytecode = True
    try:
        from hybridwave.mesh import read_gmsh as ref_read
    finally:
        sys.path.remove("/root/reference/pkg/src")
    from paper_1507_02557_b200.mesh import read_gmsh
    m = build_mesh("hybrid:2")
    p = tmp_path / "h.msh"
    _write_msh(p, m)
    a, b = read_gmsh(str(p)), ref_read(str(p))
    np.testing.assert_array_equal(a.vertices, b.vertices)
    for t in b.elem_types:
        np.testing.assert_array_equal(a.blocks[t], b.blocks[t])
        np.testing.assert_array_equal(a.physical[t], b.physical[t])


def test_run_config_validation():
    from paper_1507_02557_b200.app import RunConfig, build_mesh as app_mesh
    with pytest.raises(ValueError):
        RunConfig(N=8)
    with pytest.raises(ValueError):
        RunConfig(scheme="rk4")
    assert app_mesh("graded:4").n_elements > 0
    with pytest.raises(ValueError):
        app_mesh("torus:3")


def test_energy_weight_matrix_matches_discrete_energy():
    """The energy inner product the GPU stability test uses (tests/
    test_gpu_kat.py::_energy_weights) is discrete_energy's."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_gpu_kat import _energy_weights
    from paper_1507_02557_b200.dg import Discretization, discrete_energy
    m = build_mesh("hybrid:2")
    set_random_materials(m, 13)
    d = Discretization(m, 1, "GL", device="cpu")
    rng = np.random.default_rng(4)
    u = rng.standard_normal(d.n_dof)
    W = _energy_weights(d)
    assert abs(u @ W @ u - discrete_energy(d.vector_to_state(u), d)) <= 1e-12 * abs(u @ W @ u)
