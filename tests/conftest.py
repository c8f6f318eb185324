import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def build_mesh(spec):
    from paper_1507_02557_b200.mesh import structured_hybrid_mesh, uniform_cube_mesh
    kind, n = spec.split(":")
    n = int(n)
    return structured_hybrid_mesh(n) if kind == "hybrid" else uniform_cube_mesh(kind, n)


def set_random_materials(mesh, seed):
    rng = np.random.default_rng(seed)
    for t in mesh.elem_types:
        mesh.materials[t] = rng.uniform(0.5, 2.0, (len(mesh.blocks[t]), 2))


# same list as tests/golden/make_golden.py
RHS_CASES = [
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


def make_case(i, **kw):
    from paper_1507_02557_b200.dg import Discretization
    spec, N, form, mseed, pen, sseed = RHS_CASES[i]
    m = build_mesh(spec)
    if mseed is not None:
        set_random_materials(m, mseed)
    d = Discretization(m, N, form, penalty_scale=pen, **kw)
    rng = np.random.default_rng(sseed)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    return d, st


def rel_err(a, b):
    return max(float(np.abs(np.asarray(a[t]) - np.asarray(b[t])).max()
                     / max(np.abs(np.asarray(b[t])).max(), 1e-300)) for t in b)


@pytest.fixture(scope="session")
def native_lib():
    from paper_1507_02557_b200 import build, _native
    build.build_native()
    return _native.lib()
