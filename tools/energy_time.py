import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_1507_02557_b200.app import build_mesh, cavity_fields
from paper_1507_02557_b200.dg import Discretization
for spec, N in (("hybrid:38", 3), ("hexdom:120", 4)):
    d = Discretization(build_mesh(spec), N, "GL")
    q = d.to_device(d.project(cavity_fields, 0.0))
    for _ in range(3): d.energy_device(q)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): e = d.energy_device(q)
    b.record(); torch.cuda.synchronize()
    print(spec, N, "hw_energy ms", a.elapsed_time(b) / 20, "state MB", sum(v.numel() * 8 for v in q.values()) / 1e6, float(e))
