"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
every stage kernel at N = 1..5 (GL and SEM hybrid:2, plus a jittered mesh for
the per-point geometry paths) through the C ABI: hw_rhs, hw_traces,
hw_lsrk_stage, hw_ab_step, an MRAB subset tick, hw_energy.
    compute-sanitizer --tool racecheck python tools/sanitize_case.py [N ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1507_02557_b200.dg import Discretization            # noqa: E402
from paper_1507_02557_b200.mesh import HybridMesh, structured_hybrid_mesh  # noqa: E402
from paper_1507_02557_b200.timeint import Stepper               # noqa: E402


def jitter(m, amp=0.04, seed=1):
    rng = np.random.default_rng(seed)
    X = m.vertices.copy()
    inner = np.all((X > 1e-9) & (X < 1 - 1e-9), axis=1)
    X[inner] += amp * rng.uniform(-1, 1, (inner.sum(), 3))
    return HybridMesh(X, m.blocks)


def run(N):
    for mesh, form, dtype in [(structured_hybrid_mesh(2), "GL", torch.float64),
                              (structured_hybrid_mesh(2), "SEM", torch.float64),
                              (structured_hybrid_mesh(3), "GL", torch.float32),
                              (jitter(structured_hybrid_mesh(2)), "GL", torch.float64)]:
        d = Discretization(mesh, N, form, dtype=dtype)
        rng = np.random.default_rng(N)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        q = d.to_device(st)
        d.rhs_device(q)
        sub = [None] * 4
        from paper_1507_02557_b200.operators import TYPE_ID
        for t in d.types:
            sub[TYPE_ID[t]] = torch.arange(0, d.n_elems[t], 3, dtype=torch.int32, device=d.device)
        d.rhs_device(q, subset=sub)
        S = Stepper(d, st, "lsrk")
        S.lsrk_step(1e-4)
        A = Stepper(d, st, "ab")
        for _ in range(3):
            A.ab_step(1e-4)
        float(d.energy_device(S.q))
    torch.cuda.synchronize()
    print(f"N={N} ok", flush=True)


if __name__ == "__main__":
    for n in (sys.argv[1:] or ["1", "2", "3", "4", "5"]):
        run(int(n))
