"""Kernel launch list of MRAB macro steps (run under ncu --metrics
gpu__time_duration.sum): python tools/mrab_prof.py [mesh] [macro steps]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))


def main(spec="graded:24", n=2):
    import torch
    from paper_1507_02557_b200.app import build_mesh, cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.stability import assign_mrab_levels, local_timesteps
    from paper_1507_02557_b200.timeint import MRABDriver
    mesh = build_mesh(spec)
    d = Discretization(mesh, 3, "GL")
    plan = assign_mrab_levels(local_timesteps(d, 0.5), 3, mesh)
    drv = MRABDriver(d, plan)
    q = d.to_device(d.project(cavity_fields, 0.0))
    macro = 4 * plan.dt_min
    drv.run(q, 4 * macro, graph=False)          # warm (history full)
    torch.cuda.synchronize()
    drv.run(q, int(n) * macro, graph=False)
    torch.cuda.synchronize()
    print({t: int(v.sum()) for t, v in drv.rhs_evals.items()},
          {lev: sum(int((plan.levels[t] == lev).sum()) for t in d.types) for lev in (1, 2, 3)},
          {t: d.n_elems[t] for t in d.types})


if __name__ == "__main__":
    main(*sys.argv[1:])
