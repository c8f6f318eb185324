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
