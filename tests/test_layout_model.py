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
