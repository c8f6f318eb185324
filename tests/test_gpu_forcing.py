"""Forcing on the device (hybridwave/dg.py:497-515): the callback's values
at the cubature points are integrated by hw_forcing and, in the time loops,
added to dp/dtau inside the fused stage kernels' epilogue.  Against the
reference's own forced RHS and trajectories (tests/golden/forcing.npz),
with the callback evaluated on the host (numpy points, as in the reference)
and on the device (torch points, ``on_device = True``)."""
import math

import numpy as np
import pytest
import torch

from conftest import build_mesh, load_golden, rel_err, set_random_materials

pytestmark = pytest.mark.gpu


def _l2rel(a, b):
    num = sum(float(np.sum((np.asarray(a[t]) - np.asarray(b[t])) ** 2)) for t in b)
    den = sum(float(np.sum(np.asarray(b[t]) ** 2)) for t in b)
    return np.sqrt(num / den)


def _torch_forcing(x, time):
    """tests/golden/make_golden.py:forcing_fn on CUDA tensors."""
    return (torch.sin(math.pi * x[..., 0]) * torch.cos(math.pi * x[..., 1]) * (1.0 + x[..., 2])
            * math.cos(3.0 * time))


_torch_forcing.on_device = True


@pytest.mark.parametrize("tag,spec,N,form", [("hyb2_gl", "hybrid:2", 2, "GL"),
                                             ("hyb2_sem", "hybrid:2", 2, "SEM"),
                                             ("tet2_gl", "tet:2", 3, "GL")])
def test_device_forcing_matches_reference(tag, spec, N, form, native_lib):
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.timeint import lsrk_run, single_rate_run
    G = load_golden("forcing")
    m = build_mesh(spec)
    set_random_materials(m, 5)
    d = Discretization(m, N, form, forcing=_torch_forcing)
    st = d.project(cavity_fields, 0.0)
    dt = float(G[f"{tag}/dt"])
    assert rel_err(d.compute_rhs(st, 0.37), {t: G[f"{tag}/rhs/{t}"] for t in d.types}) < 1e-12
    ab = single_rate_run(d, st, dt, 10 * dt)
    assert _l2rel(ab, {t: G[f"{tag}/ab3/{t}"] for t in d.types}) < 1e-10
    lk = lsrk_run(d, st, dt, 10 * dt)
    assert _l2rel(lk, {t: G[f"{tag}/lsrk/{t}"] for t in d.types}) < 1e-10
    # the forcing pointers are cleared after the forced loops: a plain RHS of
    # an unforced twin discretisation on the same mesh is unaffected
    plain = Discretization(m, N, form)
    r0 = plain.compute_rhs(st)
    r1 = d.compute_rhs(st, 0.37)
    assert max(np.abs(r1[t] - r0[t]).max() for t in d.types) > 0


def test_forced_lsrk_fp32(native_lib):
    """fp32 storage with forcing: within 1e-4 of the reference."""
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.timeint import lsrk_run
    G = load_golden("forcing")
    m = build_mesh("hybrid:2")
    set_random_materials(m, 5)
    d = Discretization(m, 2, "GL", forcing=_torch_forcing, dtype=torch.float32)
    st = d.project(cavity_fields, 0.0)
    dt = float(G["hyb2_gl/dt"])
    lk = lsrk_run(d, st, dt, 10 * dt)
    assert _l2rel(lk, {t: G[f"hyb2_gl/lsrk/{t}"] for t in d.types}) < 1e-4
