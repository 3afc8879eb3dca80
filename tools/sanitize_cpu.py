"""ASan + UBSan runs of everything that executes on the host: the oracle
(oracle.c, walker.c) and the product's host code (api*.cpp, bvh_build.cpp: scene creation,
validation, SAH build, export/import, instances top level) — each built with
-fsanitize=address,undefined into /tmp and driven by the CPU test suites under LD_PRELOAD.
(compute-sanitizer for the kernels is closed on this GPU pool.)

    python tools/sanitize_cpu.py > profiles/r01_sanitizers_cpu.md
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1912_12786_b200 import _build  # noqa: E402  (source list only; nothing is built)
SAN = ["-fsanitize=address", "-fsanitize=undefined", "-fno-omit-frame-pointer"]


def run(cmd, env=None):
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True)
    return r.returncode, (r.stdout + r.stderr)


def main():
    tmp = tempfile.mkdtemp(prefix="vsr_san_")
    orc = os.path.join(tmp, "liboracle_san.so")
    lib = os.path.join(tmp, "libvsr_san.so")
    rc, out = run(["gcc", "-O1", "-g", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
                   "-fno-fast-math", "-pthread", "-D_GNU_SOURCE", *SAN, "-o", orc,
                   "oracle/oracle.c", "oracle/walker.c", "-lm"])
    assert rc == 0, out
    xc = [a for f in SAN for a in ("-Xcompiler", f)]
    rc, out = run(["/usr/local/cuda/bin/nvcc", "-O1", "-g", "-std=c++17", "-shared", "-Xcompiler",
                   "-fPIC", "-Xcompiler", "-ffp-contract=off", *xc, "-gencode",
                   "arch=compute_100a,code=sm_100a", "-fmad=false", "-prec-div=true",
                   "-prec-sqrt=true", "-ftz=false", "-I", "include", "-o", lib,
                   *[os.path.join("paper_1912_12786_b200/csrc", f) for f in _build.SOURCES],
                   "-lcudart"])
    assert rc == 0, out
    pre = " ".join(subprocess.check_output(["gcc", f"-print-file-name={n}"], text=True).strip()
                   for n in ("libasan.so", "libubsan.so"))
    env = dict(os.environ, LD_PRELOAD=pre, ASAN_OPTIONS="detect_leaks=0:protect_shadow_gap=0",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1", ORACLE_MUTANT_LIB=orc,
               VSR_LIB=lib)
    suites = ["tests/test_oracle_pins.py", "tests/test_oracle_multi.py", "tests/test_oracle_list.py",
              "tests/test_oracle_variants.py", "tests/test_instances_cpu.py", "tests/test_abi_cpu.py",
              "tests/test_multi_rank_cpu.py", "tests/test_c_consumer.py"]
    rc, out = run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *suites], env)
    tail = [ln for ln in out.strip().splitlines() if ln.strip()][-1]
    print("# r01 — ASan + UBSan on the host code (CPU)\n")
    print("Built with `-fsanitize=address,undefined` (oracle with gcc, product host code with nvcc's "
          "host compiler) and run under `LD_PRELOAD=libasan.so libubsan.so`, "
          "`UBSAN_OPTIONS=halt_on_error=1`:\n")
    print("| suites | result |\n|---|---|")
    print(f"| {', '.join(os.path.basename(s) for s in suites)} | {tail} |")
    print(f"\nexit code {rc}; any sanitizer report would have failed the run.")
    return rc


if __name__ == "__main__":
    sys.exit(main())
