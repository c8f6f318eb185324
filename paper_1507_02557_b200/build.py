"""Build the in-tree sm_100a shared library (nvcc, no torch JIT cache)."""

import hashlib
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


def _stamp(cmd_flags, deps):
    """Content hash of everything that determines the library: the nvcc
    flags (incl. HW_NVCC_DEFS and HW_MAX_ORDER) and every source byte."""
    h = hashlib.sha256()
    h.update("\0".join(cmd_flags).encode())
    for p in deps:
        h.update(os.path.basename(p).encode() + b"\0")
        with open(p, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


STAMP = OUT + ".stamp"


def build_native(max_order=7, force=False, verbose=False, out=None):
    """Compile csrc/hw_abi.cu into the in-tree library unless the stamp next
    to it records the same sources and flags.  HW_NVCC_DEFS adds -D flags
    (tuning experiments); ``out`` builds a variant to another path so the
    default library is never silently replaced by a tuning build."""
    deps = _sources() + [HEADER]
    extra = os.environ.get("HW_NVCC_DEFS", "").split()
    flags = NVCC_FLAGS + extra + [f"-DHW_MAX_ORDER={max_order}"]
    target = out or OUT
    stamp_path = target + ".stamp"
    want = _stamp(flags, deps)
    if not force and os.path.exists(target) and os.path.exists(stamp_path):
        with open(stamp_path) as fh:
            if fh.read().strip() == want:
                return target
    cmd = [nvcc()] + flags + ["-o", target + ".tmp", MAIN]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(_HERE, "csrc", "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stderr[-4000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(target + ".tmp", target)
    with open(stamp_path, "w") as fh:
        fh.write(want + "\n")
    if verbose:
        print(f"built {target}")
    return target


if __name__ == "__main__":
    build_native(force="--force" in sys.argv, verbose=True)
