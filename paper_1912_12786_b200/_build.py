"""Build libvsr.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_1912_12786_b200._build [--force]

Flags: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, and the
arithmetic contract of DESIGN.md (A.1-A.3): -fmad=false (no FMA contraction),
IEEE division/sqrt (-prec-div=true -prec-sqrt=true), denormals preserved
(-ftz=false); host code with -ffp-contract=off.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvsr.so")
SOURCES = ["api.cpp", "api_trace.cpp", "api_compound.cpp", "api_wide.cpp", "bvh_build.cpp",
           "bvh8_build.cpp", "trace.cu", "compound.cu", "prims.cu", "lbvh.cu", "wide.cu"]
HEADERS = ["api_internal.hpp", "layout.hpp", "builder.hpp", "trace.hpp", "intersectors.cuh",
           "traverse.cuh", "wide.hpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "vsr.h"))
    deps.append(os.path.abspath(__file__))
    lib_t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > lib_t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Build libvsr.so (or a tuning variant at `out` with extra -D`defines`)."""
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    tmp = target + ".tmp"
    cmd = [nvcc(), "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-Xcompiler",
           "-ffp-contract=off", *ARCH, "-lineinfo", "-fmad=false", "-prec-div=true",
           "-prec-sqrt=true", "-ftz=false", "-Xptxas", "-v", "-Xfatbin", "-compress-all", "-I", os.path.join(ROOT, "include"),
           *[f"-D{d}" for d in defines],
           "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES] + ["-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libvsr.so")
    info = os.path.join(HERE, "ptxas_info.txt" if out is None else
                        os.path.basename(target) + ".ptxas.txt")
    with open(info, "w") as f:
        f.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, target)
    return target


CHECKED = os.path.join(ROOT, "variants", "libvsr_checked.so")


def build_checked(force: bool = False) -> str:
    """The bounds-checked variant (-DVSR_CHECKED=1: device-side index checks that trap;
    tests/test_gpu_checked.py) — the kernels' memory-safety evidence, compute-sanitizer
    being closed on this GPU pool.  Rebuilt when the main library is newer."""
    if (not force and os.path.exists(CHECKED) and os.path.exists(LIB)
            and os.path.getmtime(CHECKED) >= os.path.getmtime(LIB) and not _stale()):
        return CHECKED
    os.makedirs(os.path.dirname(CHECKED), exist_ok=True)
    return build(out=CHECKED, defines=("VSR_CHECKED=1",))


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("-")]
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                out=args[0] if args else None, defines=defs))
