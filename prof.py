#!/usr/bin/env python
"""Small driver for ncu captures: build one workload, run a few LSRK
stages (no CUDA graph, so every kernel is a separate launch)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mesh", default="hybrid:38")
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--form", default="GL")
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1507_02557_b200.app import build_mesh
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.timeint import Stepper
    dtype = torch.float64 if a.dtype == "f64" else torch.float32
    d = Discretization(build_mesh(a.mesh), a.order, a.form, dtype=dtype)
    rng = np.random.default_rng(0)
    st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
    S = Stepper(d, st, "lsrk")
    for _ in range(a.steps):
        S.lsrk_step(1e-5)
    torch.cuda.synchronize()
    print("ok", {t: float(S.q[t].abs().max()) for t in d.types})


if __name__ == "__main__":
    main()
