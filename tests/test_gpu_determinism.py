"""Race detection without compute-sanitizer (closed on this GPU pool): the
stage kernels alias shared memory across phases and fill it with cp.async
and TMA bulk copies, so a missing barrier or an early reuse shows up as
run-to-run differences.  Every kernel at N = 1..5, fp64 and fp32, GL and
SEM, must be bitwise reproducible, and a subset launch must equal the same
rows of the full launch bit for bit."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("form,dtype", [("GL", torch.float64), ("SEM", torch.float64),
                                        ("GL", torch.float32)])
def test_stage_kernels_bitwise_reproducible(N, form, dtype, native_lib):
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import structured_hybrid_mesh
    from paper_1507_02557_b200.operators import TYPE_ID
    from paper_1507_02557_b200.timeint import Stepper
    d = Discretization(structured_hybrid_mesh(4), N, form, dtype=dtype)
    rng = np.random.default_rng(N)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    q = d.to_device(st)
    ref = d.rhs_device(q)
    for _ in range(4):
        again = d.rhs_device(q)
        for t in d.types:
            assert torch.equal(again[t], ref[t]), t
    lists = [None] * 4
    for t in d.types:
        lists[TYPE_ID[t]] = torch.arange(1, d.n_elems[t], 3, dtype=torch.int32, device=d.device)
    part = d.rhs_device(q, subset=lists)
    for t in d.types:
        assert torch.equal(part[t][1::3], ref[t][1::3]), t
    outs = []
    for _ in range(2):
        S = Stepper(d, st, "lsrk")
        for _ in range(2):
            S.lsrk_step(1e-4)
        outs.append({t: S.q[t].clone() for t in d.types})
    for t in d.types:
        assert torch.equal(outs[0][t], outs[1][t]), t
