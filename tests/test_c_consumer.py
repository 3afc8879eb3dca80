"""The boundary is a plain C ABI: examples/c_host_only.c compiles against include/vsr.h with a C
compiler, links libvsr.so and runs host-only entry points (create, build, stats, export, error
reporting) without Python or a GPU."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_uses_the_library(tmp_path):
    from paper_1912_12786_b200 import _build
    lib = _build.build()
    exe = tmp_path / "vsr_c"
    libdir = os.path.dirname(lib)
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_host_only.c"), "-L", libdir, "-lvsr",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "tris 4 nodes 3 leaves 4" in out.stdout
    assert "cannot be traced" in out.stdout
