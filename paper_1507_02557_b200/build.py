"""Build the in-tree sm_100a shared library (nvcc, no torch JIT cache)."""

import os
import subprocess
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
MAIN = os.path.join(_HERE, "csrc", "hw_abi.cu")


def _sources():
    d = os.path.join(_HERE, "csrc")
    return sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cu", ".cuh")))


HEADER = os.path.join(_ROOT, "include", "hybridwave_b200.h")
OUT = os.path.join(_HERE, "libhybridwave_b200.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def build_native(max_order=7, force=False, verbose=False):
    deps = _sources() + [HEADER]
    if (not force and os.path.exists(OUT)
            and os.path.getmtime(OUT) >= max(os.path.getmtime(p) for p in deps)):
        return OUT
    # HW_NVCC_DEFS: extra -D flags for tuning experiments (e.g. -DHW_TET_MINB=8)
    extra = os.environ.get("HW_NVCC_DEFS", "").split()
    cmd = [nvcc()] + NVCC_FLAGS + extra + [f"-DHW_MAX_ORDER={max_order}", "-o", OUT + ".tmp",
                                           MAIN]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(_HERE, "csrc", "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stderr[-4000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build_native(force="--force" in sys.argv, verbose=True)
