#!/usr/bin/env python
"""Benchmark: LSRK-45 steps of the DG acoustic RHS + update on B200.

Default workload (BASELINE.json configs[3], the configuration the metric's
1/2/4/8-GPU series is quoted on): the hex-dominant hybrid cube hexdom:120
(1,584,000 hex, 115,200 wedge, 72,000 pyramid, 460,800 tet = 2,232,000
elements, 907 M DOF), N=4, GL, fp64, cavity-mode initial data projected on
the host, dt from the reference's local timestep rule (CFL 0.5).  The SAME
mesh at every GPU count (strong scaling): N=1 runs the whole mesh on one
B200, N>1 element-partitions it (x-slabs).  One step = 5 RHS stages, each
one fused kernel launch per element type; on one GPU the timed loop replays
a CUDA graph of one step.  ``--mesh hybrid:38 --order 3`` is configs[2]
(the reference's own hybrid cube), ``--mesh tet:20`` configs[1].

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                  [--mesh hexdom:120 --order 4 --form GL --dtype f64]

Multi-GPU (torchrun, N > 1): every LSRK stage exchanges the shared-face
values of the partition-boundary elements (face nodes or published face
traces) with NCCL batched P2P while the interior elements compute
(paper_1507_02557_b200/parallel.py); timing is the max over ranks.
hybrid:n meshes are instead extended along x to n*N cells (weak scaling).
"""

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GDOF·stage/s per LSRK step (N=1..5, hybrid mesh, 1/2/4/8 B200); kernel GB/s vs HBM"
UNIT = "GDOF*stage/s"
GEO_WORDS = {"hex": 72, "wedge": 40, "pyramid": 40, "tet": 33}
NFACES = {"hex": 6, "wedge": 5, "pyramid": 5, "tet": 4}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mesh", default="hexdom:120")
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--form", default="GL", choices=["GL", "SEM"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--cpu-mesh", default=None, help="reference-arm sample mesh")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--jitter", type=float, default=0.0,
                    help="perturb interior vertices by this fraction of the mesh spacing "
                         "(non-affine hexes, pyramids and wedges: the per-point geometry paths)")
    ap.add_argument("--scheme", default="lsrk", choices=["lsrk", "mrab"],
                    help="mrab: multi-rate AB3 (active levels only), --levels levels")
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--partitioned", action="store_true",
                    help="use the element-partitioned path even on one rank")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the other BASELINE configurations measured alongside the "
                         "default single-GPU line (other_configs)")
    return ap.parse_args()


def build_mesh(spec):
    from paper_1507_02557_b200.app import build_mesh as bm
    return bm(spec)


def config_index(spec):
    """BASELINE.json config a mesh spec stands for (hex:4 -> configs[0],
    tet:* -> [1], hybrid:* -> [2], hexdom:* -> [3], graded:* -> [4])."""
    kind = spec.split(":")[0]
    idx = {"hex": 0, "tet": 1, "hybrid": 2, "hexdom": 3, "graded": 4}.get(kind)
    return f"configs[{idx}]" if idx is not None else "custom mesh"


def jittered(mesh, amp, seed=0):
    from paper_1507_02557_b200.mesh import HybridMesh
    rng = np.random.default_rng(seed)
    X = mesh.vertices.copy()
    inner = np.all((X > 1e-9) & (X < 1 - 1e-9), axis=1)
    X[inner] += amp * rng.uniform(-1, 1, (inner.sum(), 3))
    return HybridMesh(X, mesh.blocks)


def n_dof(disc):
    return disc.n_dof


# ------------------------------------------------------------------ CPU arm

def cpu_sample_mesh(args):
    """Bounded sample of the workload for the CPU oracle: the same band
    layout, order and formulation on a coarser cube (per-DOF rate):
    hexdom:14 (4 hex / 4 wedge / 1 pyramid / 5 tet layers of 14 x 14 cells)
    for configs[3], hybrid:20 for configs[2]."""
    if args.cpu_mesh:
        return args.cpu_mesh
    kind, n = args.mesh.split(":")
    n = int(n)
    cap = {"hexdom": 14, "hybrid": 20, "tet": 20, "hex": 12, "graded": 12}.get(kind, 10)
    return f"{kind}:{min(n, cap)}"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def run_cpu_oracle(args, steps, warmup):
    """The reference's algorithm (oracle/ numpy port) for LSRK steps on the
    host cores; returns (value GDOF*stage/s, seconds/step, sample, cores)."""
    import oracle
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.stability import local_timesteps
    spec = cpu_sample_mesh(args)
    d = Discretization(build_mesh(spec), args.order, args.form)
    st = d.project(cavity_fields, 0.0)
    dt = min(float(v.min()) for v in local_timesteps(d, 0.5).values())
    d._ensure_reference_layout()
    rhs = lambda s, tau: oracle.compute_rhs(d, s)
    for _ in range(warmup):
        st = oracle.lsrk_run(rhs, st, dt, dt)
    t0 = time.perf_counter()
    for _ in range(steps):
        st = oracle.lsrk_run(rhs, st, dt, dt)
    el = time.perf_counter() - t0
    value = d.n_dof * 5 * steps / el / 1e9
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    sample = (f"{spec} N={args.order} {args.form} fp64 ({sum(d.n_elems.values())} elements, "
              f"{d.n_dof} DOF), {steps} LSRK steps (5 oracle RHS each); "
              f"host CPU: {cpu_model()}, {os.cpu_count()} logical cores")
    return value, el / steps, sample, cores


def scaling_of(spec):
    """hybrid:n is extended along x with the GPU count (weak); every other
    mesh is the same at every GPU count (strong)."""
    return "weak" if spec.split(":")[0] == "hybrid" else "strong"


def workload_label(args):
    return (f"{args.mesh} N={args.order} {args.form} LSRK-45 ({config_index(args.mesh)})"
            + (f", jitter {args.jitter}" if args.jitter else ""))


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps = max(1, min(args.steps, 5))
    warm = 1
    value, sps, sample, cores = run_cpu_oracle(args, steps, warm)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": sps * 1e3,
            "higher_is_better": True, "scaling": scaling_of(args.mesh), "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (cavity eigenmode projected on the mesh)",
            "config": {"workload": workload_label(args), "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clock + throttle reasons sampled with NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ GPU arm

def face_points(t, N):
    nfn, nfq = (N + 1) * (N + 2) // 2, (N + 1) ** 2
    return {"hex": 6 * nfq, "tet": 4 * nfn, "wedge": 2 * nfn + 3 * nfq,
            "pyramid": nfq + 4 * nfn}[t]


def alg_bytes_per_elem(t, Np, s, N, gl=True):
    """Compulsory HBM traffic of one LSRK stage per element in this layout:
    read q, read res, write res, write q_out (4 x 4 Np words), geometry
    record, material record, the neighbour links (tets: the int32 gather
    index per face node; other types: index + code per face), and for the
    trace-publishing types (wedge, pyramid, GL hex) reading the own face
    traces of q_in and writing those of q_out (2 x 4 x Nfp words).
    Neighbour states / traces are re-read from L2 (not counted)."""
    links = 4 * 4 * (N + 1) * (N + 2) // 2 if t == "tet" else 8 * NFACES[t]
    pub = t in ("wedge", "pyramid") or (t == "hex" and gl)
    tr = 2 * 4 * face_points(t, N) * s if pub else 0
    return 4 * 4 * Np * s + GEO_WORDS[t] * s + 4 * s + links + tr


# the other BASELINE configurations, measured by the default N=1 run in
# separate processes (each its own JSON line, summarised in other_configs)
EXTRA_CONFIGS = [
    ("configs[2] hybrid:38 N=3 GL fp64 LSRK-45", ["--mesh", "hybrid:38", "--order", "3"]),
    ("configs[2] hybrid:38 N=3 GL fp32 LSRK-45",
     ["--mesh", "hybrid:38", "--order", "3", "--dtype", "f32"]),
    ("configs[1] tet:20 N=3 GL fp64 LSRK-45", ["--mesh", "tet:20", "--order", "3"]),
    ("configs[4] graded:24 N=3 GL fp64 MRAB-AB3, 3 levels",
     ["--mesh", "graded:24", "--order", "3", "--scheme", "mrab", "--levels", "3"]),
]


def other_configs(args):
    import subprocess
    out = {}
    for label, extra in EXTRA_CONFIGS:
        cmd = [sys.executable, os.path.abspath(__file__), "--no-cpu-baseline", "--no-extra",
               "--steps", str(min(args.steps, 20)), "--warmup", str(args.warmup)] + extra
        try:
            p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
            line = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
        except Exception as e:  # pragma: no cover - reported, not fatal
            out[label] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
            continue
        roof = line.get("roofline") or {}
        out[label] = {"value": line["value"], "unit": line["unit"],
                      "ms_per_step": line["ms_per_step"], "steps": line["steps"],
                      "e2e": (line.get("e2e") or {}).get("value"),
                      "gpu_launches": line.get("gpu_launches"),
                      "roofline_frac": roof.get("frac"), "roofline_kernel": roof.get("kernel"),
                      "per_type_us": {t: v["us_per_launch"]
                                      for t, v in (roof.get("per_type") or {}).items()},
                      "config": line["config"].get("workload")}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    from paper_1507_02557_b200 import _native as nat
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.operators import TYPE_ID
    from paper_1507_02557_b200.stability import local_timesteps
    from paper_1507_02557_b200.timeint import LSRK_A, LSRK_B, Stepper, lsrk_run

    dtype = torch.float64 if args.dtype == "f64" else torch.float32
    s_bytes = 8 if args.dtype == "f64" else 4
    if world > 1 or args.partitioned:
        if world == 1 and not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1)
        if args.scheme == "mrab":
            return partitioned_mrab(args, world, rank, local, dev, dtype, s_bytes)
        return partitioned(args, world, rank, local, dev, dtype, s_bytes)
    t_setup = time.perf_counter()
    mesh = build_mesh(args.mesh)
    if args.jitter > 0:
        mesh = jittered(mesh, args.jitter / int(args.mesh.split(":")[1]))
    disc = Discretization(mesh, args.order, args.form, dtype=dtype, device=dev)
    host_state = disc.project(cavity_fields, 0.0)
    dt = min(float(v.min()) for v in local_timesteps(disc, 0.5).values())
    _ = disc.device_mesh
    setup_s = time.perf_counter() - t_setup
    if args.scheme == "mrab":
        return mrab_bench(args, disc, mesh, host_state, dev, setup_s)
    S = Stepper(disc, host_state, "lsrk")
    stream = torch.cuda.current_stream(dev)

    # CUDA graphs of one step for each buffer parity
    graphs = []
    if not args.no_graph:
        S.lsrk_step(dt)               # warm (sets kernel attributes outside capture)
        S.lsrk_step(dt)
        torch.cuda.synchronize()
        cap = torch.cuda.Stream(dev)
        c0 = nat.lib().hw_launch_count()
        for _ in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                S.lsrk_step(dt)
            graphs.append(g)
        launches_per_step = (nat.lib().hw_launch_count() - c0) / 2   # captured kernel nodes

    def step(i):
        if graphs:
            graphs[i % 2].replay()
        else:
            S.lsrk_step(dt)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        c0 = nat.lib().hw_launch_count()
        e0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if not graphs:
        launches_per_step = (nat.lib().hw_launch_count() - c0) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    total_dof = disc.n_dof * world
    value = total_dof * 5 * args.steps / (ms * 1e-3) / 1e9
    assert all(torch.isfinite(S.q[t]).all() for t in disc.types), "state diverged"

    # ---- per-type kernel time (roofline of the dominant kernel)
    per_type = {}
    L = nat.lib()
    for t in disc.types:
        lists = [torch.zeros(0, dtype=torch.int32, device=dev)] * 4
        lists[TYPE_ID[t]] = None
        sub = nat.subset(lists)
        F = lambda x: nat.fields(disc.slots(x))
        reps = 20
        for _ in range(3):
            nat.check(L.hw_lsrk_stage(disc.device_mesh.struct, F(S.q), F(S.q2), F(S.res),
                                      LSRK_A[1], LSRK_B[1], 0.0, sub, stream.cuda_stream))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            nat.check(L.hw_lsrk_stage(disc.device_mesh.struct, F(S.q), F(S.q2), F(S.res),
                                      LSRK_A[1], LSRK_B[1], 0.0, sub, stream.cuda_stream))
        b.record(stream)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / reps
        Np = disc.ops[t].Np
        nbytes = disc.n_elems[t] * alg_bytes_per_elem(t, Np, s_bytes, args.order,
                                                     args.form == "GL")
        per_type[t] = {"us_per_launch": us, "elements": disc.n_elems[t],
                       "alg_bytes": nbytes, "GBps": nbytes / (us * 1e-6) / 1e9}
    dom = max(per_type, key=lambda t: per_type[t]["us_per_launch"])
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    prof = {}
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        pass
    # (jittered meshes run other kernels than the captured ones: no traffic)
    tr_ent = None if args.jitter else prof.get(f"{args.mesh}/N{args.order}/{args.form}/{args.dtype}/{dom}")
    traffic = tr_ent["bytes"] if isinstance(tr_ent, dict) else tr_ent
    kname = {"hex": f"hex_kernel<{args.order},{'double' if s_bytes == 8 else 'float'}>",
             "wedge": f"dense_mma_kernel<{args.order},1>", "pyramid": f"dense_mma_kernel<{args.order},2>",
             "tet": f"tet_mma_kernel<{args.order}>"}[dom] if s_bytes == 8 else \
        f"{dom}_kernel<{args.order},float>"
    if args.jitter and dom in ("wedge", "pyramid"):   # non-affine: the scalar per-point kernel
        kname = f"dense_kernel<{args.order},{1 if dom == 'wedge' else 2}>"
    roof = {"bound": "hbm", "kernel": kname,
            "achieved": per_type[dom]["GBps"], "peak": hbm, "unit": "GB/s",
            "frac": per_type[dom]["GBps"] / hbm, "traffic": traffic,
            "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks
            else "fallback 6650 GB/s",
            "per_type": per_type,
            "step_share": {t: per_type[t]["us_per_launch"] * 5 / (ms * 1e3 / args.steps)
                           for t in per_type}}

    # ---- end-to-end through the public API: host state in (pinned numpy
    # arrays), host state out (written into pinned numpy arrays)
    e2e_steps = max(2, min(args.steps, 100))   # the timed device run's step count
    np_dt = np.float64 if s_bytes == 8 else np.float32

    def pinned_like(a):
        buf = torch.empty(a.shape, dtype=torch.float64 if s_bytes == 8 else torch.float32,
                          pin_memory=True).numpy()
        buf[...] = a
        return buf
    h_in = {t: pinned_like(np.asarray(v, dtype=np_dt)) for t, v in host_state.items()}
    h_out = {t: pinned_like(np.zeros_like(h_in[t])) for t in h_in}
    lsrk_run(disc, h_in, dt, 2 * dt * (1 - 1e-12), out=h_out)       # warm the path
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = lsrk_run(disc, h_in, dt, e2e_steps * dt * (1 - 1e-12), out=h_out)
    t1 = time.perf_counter()
    state_bytes = sum(v.nbytes for v in out.values()) * s_bytes // 8
    e2e_val = disc.n_dof * world * 5 * e2e_steps / (t1 - t0) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sps, sample, cores = run_cpu_oracle(args, 2, 0)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
               "cpu_model": cpu_model()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": scaling_of(args.mesh), "vs_baseline": None,
                "dtype": args.dtype,
                "data": "synthetic (cavity eigenmode projected on the mesh)",
                "config": {"workload": workload_label(args),
                           "elements": {t: disc.n_elems[t] for t in disc.types},
                           "n_dof_per_rank": disc.n_dof, "dt": dt,
                           "l2_policy": "inputs larger than L2 (state+res+q_out "
                                        f"{3 * disc.n_dof * s_bytes / 1e6:.0f} MB > 126 MB)",
                           "cuda_graph": bool(graphs), "setup_s": setup_s,
                           "parallelism": f"replica x{world}"},
                "gpu_launches": int(round(launches_per_step * args.steps)),
                "clocks": clk.summary(), "roofline": roof,
                "e2e": {"value": e2e_val, "unit": UNIT,
                        "h2d_bytes_per_step": state_bytes / e2e_steps,
                        "d2h_bytes_per_step": state_bytes / e2e_steps,
                        "steps": e2e_steps,
                        "api": "timeint.lsrk_run(disc, host_state, dt, T, out=host_out): pinned numpy in/out"},
                "cpu_baseline": cpu}
        if world == 1 and not args.no_extra and args.scheme == "lsrk":
            line["other_configs"] = other_configs(args)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def mrab_bench(args, disc, mesh, host_state, dev, setup_s):
    """Multi-rate AB3 (config 5): one step = one macro step; the unit of work
    is an element RHS + update, so the metric counts the DOFs of the elements
    that step at each tick (the reference evaluates the whole mesh every tick
    and discards the rest, hybridwave/timeint.py:120)."""
    import torch
    from paper_1507_02557_b200.stability import assign_mrab_levels, local_timesteps
    from paper_1507_02557_b200.timeint import MRABDriver
    L = args.levels
    plan = assign_mrab_levels(local_timesteps(disc, 0.5), L, mesh)
    drv = MRABDriver(disc, plan)
    macro = 2 ** (L - 1) * plan.dt_min
    q = disc.to_device(host_state)
    graph = not args.no_graph
    drv.run(q, macro * args.warmup, graph=graph)
    drv.run(q, macro * args.steps, graph=graph)      # same T: captures the replay graph
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        e0.record(stream)
        drv.run(q, macro * args.steps, graph=graph)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    from paper_1507_02557_b200 import _native as nat
    # end to end: host state (pinned) into HBM, the macro steps, the state
    # back to pinned host memory, on the device clock
    h_in = {t: torch.empty(q[t].shape, dtype=q[t].dtype, pin_memory=True) for t in disc.types}
    for t in disc.types:
        h_in[t].copy_(torch.as_tensor(np.asarray(host_state[t])).to(q[t].dtype))
    h_out = {t: torch.empty_like(h_in[t], pin_memory=True) for t in disc.types}
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    x0.record(stream)
    for t in disc.types:
        q[t].copy_(h_in[t], non_blocking=True)
    drv.run(q, macro * args.steps, graph=graph)
    for t in disc.types:
        h_out[t].copy_(q[t], non_blocking=True)
    x1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = x0.elapsed_time(x1)
    state_bytes = sum(v.numel() * v.element_size() for v in h_in.values())
    # kernel launches per macro step, counted on an eager (uncaptured) run
    c0 = nat.lib().hw_launch_count()
    drv.run(q, macro * 3, graph=False)
    torch.cuda.synchronize()
    launches_per_macro = (nat.lib().hw_launch_count() - c0) / 3
    active = sum(int((plan.levels[t] == lev).sum()) * 4 * disc.ops[t].Np * 2 ** (lev - 1)
                 for t in disc.types for lev in range(1, L + 1))
    full = disc.n_dof * 2 ** (L - 1)
    value = active * args.steps / (ms * 1e-3) / 1e9
    occ = {lev: sum(int((plan.levels[t] == lev).sum()) for t in disc.types)
           for lev in range(1, L + 1)}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (cavity eigenmode projected on the mesh)",
            "config": {"workload": f"{args.mesh} N={args.order} {args.form} MRAB-AB3 "
                                   f"{L} levels (configs[4]); step = macro step",
                       "level_occupancy": occ, "active_dof_per_macro": active,
                       "full_mesh_dof_per_macro": full, "dt_min": plan.dt_min,
                       "setup_s": setup_s},
            "gpu_launches": int(round(launches_per_macro * args.steps)),
            "clocks": clk.summary(), "roofline": None,
            "e2e": {"value": active * args.steps / (ms_e2e * 1e-3) / 1e9, "unit": UNIT,
                    "h2d_bytes_per_step": state_bytes / args.steps,
                    "d2h_bytes_per_step": state_bytes / args.steps, "steps": args.steps,
                    "api": "MRABDriver.run(q, T) with the state copied from / to pinned "
                           "host memory inside the timed region"},
            "cpu_baseline": None}
    print(json.dumps(line), flush=True)
    return 0


def partitioned(args, world, rank, local, dev, dtype, s_bytes):
    """N > 1: element-partitioned LSRK with a per-stage NCCL halo exchange.
    hybrid:n meshes are extended along x to n*N cells (each rank owns one
    x-slab the size of the single-GPU workload: weak scaling); other mesh
    specs are partitioned as given (strong scaling)."""
    import torch
    from paper_1507_02557_b200 import _native as nat
    import torch.distributed as dist
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.mesh import structured_hybrid_mesh
    from paper_1507_02557_b200.parallel import NCCLTransport, PartStepper, make_parts
    from paper_1507_02557_b200.stability import local_timesteps
    t_setup = time.perf_counter()
    kind, n = args.mesh.split(":")
    weak = kind == "hybrid"
    mesh = structured_hybrid_mesh(int(n), nx=int(n) * world) if weak else build_mesh(args.mesh)
    part = make_parts(mesh, world, "xslab", N=args.order, ranks=[rank])[rank]
    del mesh
    from paper_1507_02557_b200.dg import Discretization
    dl = Discretization(part.mesh, args.order, args.form, dtype=dtype, device=dev)
    st = dl.project(cavity_fields, 0.0)
    dtl = local_timesteps(dl, 0.5)
    dt_loc = min(float(v[:part.n_owned[t]].min()) for t, v in dtl.items() if part.n_owned[t])
    t = torch.tensor([dt_loc], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    dt = float(t.item())
    ps = PartStepper(part, args.order, args.form, st, NCCLTransport(), dtype=dtype, device=dev)
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        ps.lsrk_step(dt)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        c0 = nat.lib().hw_launch_count()
        e0.record(stream)
        for _ in range(args.steps):
            ps.lsrk_step(dt)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = nat.lib().hw_launch_count() - c0   # this rank's kernels (rank 0 reports)
    # end to end: this rank's state from pinned host memory into HBM, the
    # steps, the owned state back to pinned host memory (max over ranks)
    h_in = {t_: torch.empty(ps.S.q[t_].shape, dtype=ps.S.q[t_].dtype, pin_memory=True)
            for t_ in dl.types}
    for t_ in dl.types:
        h_in[t_].copy_(ps.S.q[t_])
    h_out = {t_: torch.empty(ps.owned_state()[t_].shape, dtype=ps.S.q[t_].dtype,
                             pin_memory=True) for t_ in dl.types}
    torch.cuda.synchronize()
    dist.barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(2, min(args.steps, 100))   # the timed device run's step count
    x0.record(stream)
    for t_ in dl.types:
        ps.S.q[t_].copy_(h_in[t_], non_blocking=True)
    for _ in range(e2e_steps):
        ps.lsrk_step(dt)
    own = ps.owned_state()
    for t_ in dl.types:
        h_out[t_].copy_(own[t_], non_blocking=True)
    x1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = x0.elapsed_time(x1)
    tt = torch.tensor([ms, float(ps.n_dof_owned), ms_e2e], device=dev, dtype=torch.float64)
    mx = tt.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm_ = tt.clone()
    dist.all_reduce(sm_, op=dist.ReduceOp.SUM)
    ms, total_dof, ms_e2e = float(mx[0]), float(sm_[1]), float(mx[2])
    h2d = sum(v.numel() * v.element_size() for v in h_in.values())
    d2h = sum(v.numel() * v.element_size() for v in h_out.values())
    assert all(torch.isfinite(ps.S.q[t_]).all() for t_ in dl.types), "state diverged"
    value = total_dof * 5 * args.steps / (ms * 1e-3) / 1e9
    halo = ps.halo_bytes
    halo_full = sum(int(b - a) * 4 * dl.ops[t_].Np * s_bytes
                    for per_t in part.recv.values() for t_, (a, b) in per_t.items())
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "weak" if weak else "strong",
                "vs_baseline": None, "dtype": args.dtype,
                "data": "synthetic (cavity eigenmode projected on the mesh)",
                "config": {"workload": workload_label(args),
                           "partition": (f"x-extended x{world}, x-slab" if weak else
                                         f"x-slab x{world}"),
                           "n_dof_total": int(total_dof), "dt": dt, "setup_s": setup_s,
                           "halo_bytes_per_stage_rank0": halo,
                           "halo_bytes_if_whole_ghost_states_rank0": halo_full,
                           "parallelism": f"element partition x{world}, NCCL face halo",
                           "cuda_graph": False,
                           "l2_policy": "inputs larger than L2"},
                "gpu_launches": launches,
                "clocks": clk.summary(), "roofline": None,
                "e2e": {"value": total_dof * 5 * e2e_steps / (ms_e2e * 1e-3) / 1e9, "unit": UNIT,
                        "h2d_bytes_per_step": h2d / e2e_steps,
                        "d2h_bytes_per_step": d2h / e2e_steps, "steps": e2e_steps,
                        "api": "PartStepper.lsrk_step per rank, rank state H2D / owned "
                               "state D2H (pinned) inside the timed region, max over ranks"},
                "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def partitioned_mrab(args, world, rank, local, dev, dtype, s_bytes):
    """N > 1 multi-rate AB3 (config 5 at 1/8 GPUs): graded:n extended along x
    to n*N cells (weak scaling), levels assigned on the global mesh (host,
    identical on every rank), x-slab partition, per-tick NCCL exchange of the
    boundary elements' effective state (parallel.PartMRAB).  One step = one
    macro step; the metric counts the DOFs of the elements that step."""
    import torch
    from paper_1507_02557_b200 import _native as nat
    import torch.distributed as dist
    from paper_1507_02557_b200.app import cavity_fields
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.mesh import graded_hybrid_mesh
    from paper_1507_02557_b200.parallel import NCCLTransport, PartMRAB, make_parts
    from paper_1507_02557_b200.stability import assign_mrab_levels, local_timesteps
    t_setup = time.perf_counter()
    kind, n = args.mesh.split(":")
    weak = kind == "graded"
    mesh = graded_hybrid_mesh(int(n), nx=int(n) * world) if weak else build_mesh(args.mesh)
    L = args.levels
    dg = Discretization(mesh, args.order, args.form, device="cpu")
    plan = assign_mrab_levels(local_timesteps(dg, 0.5), L, mesh)
    del dg
    part = make_parts(mesh, world, "xslab", N=args.order, ranks=[rank])[rank]
    del mesh
    dl = Discretization(part.mesh, args.order, args.form, dtype=dtype, device=dev)
    st = dl.project(cavity_fields, 0.0)
    lev_loc = {t: plan.levels[t][part.global_ids[t]] for t in dl.types}
    pm = PartMRAB(part, args.order, args.form, st, lev_loc, L, NCCLTransport(), dtype=dtype,
                  device=dev)
    dt_min = plan.dt_min
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 3)):          # history warm-up + timing warm-up
        pm.macro_step(dt_min)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        c0 = nat.lib().hw_launch_count()
        e0.record(stream)
        for _ in range(args.steps):
            pm.macro_step(dt_min)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = nat.lib().hw_launch_count() - c0   # this rank's kernels (rank 0 reports)
    active = sum(int(((lev_loc[t] == lev) & (np.arange(dl.n_elems[t]) < part.n_owned[t])).sum())
                 * 4 * dl.ops[t].Np * 2 ** (lev - 1) for t in dl.types for lev in range(1, L + 1))
    tt = torch.tensor([ms, float(active)], device=dev, dtype=torch.float64)
    mx = tt.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm_ = tt.clone()
    dist.all_reduce(sm_, op=dist.ReduceOp.SUM)
    ms, active_total = float(mx[0]), float(sm_[1])
    assert all(torch.isfinite(pm.q[t_]).all() for t_ in dl.types), "state diverged"
    value = active_total * args.steps / (ms * 1e-3) / 1e9
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "weak" if weak else "strong",
                "vs_baseline": None, "dtype": args.dtype,
                "data": "synthetic (cavity eigenmode projected on the mesh)",
                "config": {"workload": f"{args.mesh} N={args.order} {args.form} MRAB-AB3 {L} levels"
                                       f" (configs[4]), x-extended x{world}, x-slab partition; "
                                       "step = macro step" if weak else
                                       f"{args.mesh} N={args.order} {args.form} MRAB-AB3 {L} "
                                       "levels (configs[4]), x-slab partition; step = macro step",
                           "active_dof_per_macro_total": int(active_total), "dt_min": dt_min,
                           "setup_s": setup_s,
                           "parallelism": f"element partition x{world}, NCCL per-tick halo",
                           "cuda_graph": False, "l2_policy": "inputs larger than L2"},
                "gpu_launches": launches,
                "clocks": clk.summary(), "roofline": None, "e2e": None, "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
