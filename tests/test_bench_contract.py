"""bench.py's JSON-line contract (the driver parses it every round).

CPU: the reference arm (oracle port of the reference's CPU path) on a tiny
sample, and the non-zero-rank exit.  GPU: the product arm on a small hybrid
mesh, with the roofline, cpu_baseline, e2e, clocks and gpu_launches keys."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.update(env_extra or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return [json.loads(ln) for ln in lines]


def test_reference_arm_line():
    (line,) = run_bench(["--impl", "reference", "--cpu-mesh", "hybrid:2", "--order", "2",
                         "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"],
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in line["config"] and "sample" in line["config"]


def test_reference_arm_other_ranks_silent():
    assert run_bench(["--impl", "reference", "--cpu-mesh", "hybrid:2", "--steps", "1"],
                     {"RANK": "1", "WORLD_SIZE": "2"}) == []


@pytest.mark.gpu
def test_product_arm_line():
    (line,) = run_bench(["--mesh", "hybrid:8", "--order", "3", "--steps", "3", "--warmup", "3",
                         "--no-cpu-baseline", "--no-extra"])
    assert BASE_KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["warmup"] >= 3 and line["steps"] == 3
    assert line["value"] > 0 and line["dtype"] == "f64"
    # LSRK-45: one fused kernel per element type per stage (hw_launch_count)
    assert line["gpu_launches"] == 3 * 5 * 4
    assert "workload" in line["config"] and "l2_policy" in line["config"]
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s"
    assert r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = line["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)


@pytest.mark.gpu
def test_mrab_line():
    (line,) = run_bench(["--scheme", "mrab", "--mesh", "graded:6", "--order", "2",
                         "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(line)
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.gpu
def test_partitioned_line_one_rank():
    """The element-partitioned (NCCL) stepper at world size 1: same contract;
    with no peers every stage is the interior launch of each type."""
    (line,) = run_bench(["--partitioned", "--mesh", "hybrid:8", "--order", "2", "--steps", "3",
                         "--warmup", "3"])
    assert BASE_KEYS <= set(line)
    assert line["value"] > 0 and line["gpu_launches"] == 3 * 5 * 4
    assert line["e2e"]["value"] > 0


@pytest.mark.gpu
def test_other_configs_summary():
    """The default single-GPU line carries the other BASELINE configurations
    (run as subprocesses with --no-extra), each with its value and workload."""
    import bench
    from types import SimpleNamespace
    saved = bench.EXTRA_CONFIGS
    bench.EXTRA_CONFIGS = [("small", ["--mesh", "hybrid:4", "--order", "2"]),
                           ("small mrab", ["--mesh", "graded:6", "--order", "2",
                                           "--scheme", "mrab"])]
    try:
        out = bench.other_configs(SimpleNamespace(steps=3, warmup=3))
    finally:
        bench.EXTRA_CONFIGS = saved
    assert set(out) == {"small", "small mrab"}
    for v in out.values():
        assert "error" not in v, v
        assert v["value"] > 0 and v["config"]
