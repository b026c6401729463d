"""Build libmpm_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_1910_00935_b200.build [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmpm_b200.so")
SOURCES = ["engine.cu", "engine_dd.cu", "kernels_tile.cu", "kernels_misc.cu"]
HEADERS = ["kernels.h", "mpm_device.cuh", "engine.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-shared"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "mpm.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, extra=(), out: str = LIB) -> str:
    """extra: additional nvcc flags (e.g. -D tuning knobs); out: library path (A/B variants)."""
    if not force and out == LIB and not _stale():
        return LIB
    tmp = out + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *ARCH, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log") if out == LIB else out + ".log"
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(res.stderr)
    # every library symbol must resolve inside the library (a shared object links with
    # undefined symbols silently; one would only fail at dlopen on the GPU box)
    und = subprocess.run(["nm", "-uC", tmp], capture_output=True, text=True).stdout
    bad = [l for l in und.splitlines() if "mpm::" in l and l.split()[0] == "U"]  # weak refs are fine
    if bad:
        os.remove(tmp)
        raise RuntimeError("undefined library symbols: " + "; ".join(bad))
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force=True, verbose="--verbose" in sys.argv)
    print(LIB)
