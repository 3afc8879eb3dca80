"""Kernel memory safety without compute-sanitizer (closed on this GPU pool:
profiles/r02_compute_sanitizer_closed.log): the bounds-checked build (-DVSR_CHECKED=1) checks
every node, triangle, sidecar, texel, 1-bit-plane word, instance record and stack index on the
device and traps on a violation.  The fuzz sweep (scales 1e-3..1e4, offsets to 1e6, degenerate
directions), soups, C1, the alpha variants, lists, instances (incl. far origins), multi-hit and
the wide BVH run on it in a subprocess; any trap fails the launch and the run."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_runs_clean():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_12786_b200 import _build
    lib = _build.build_checked()
    env = dict(os.environ, VSR_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                        "tests/test_gpu_fuzz.py", "tests/test_gpu_variants.py", "tests/test_gpu_list.py",
                        "tests/test_gpu_instances.py", "tests/test_gpu_multi.py", "tests/test_gpu_wide.py",
                        "tests/test_gpu_alpha_bits.py", "-k", "not c2"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
    assert " passed" in r.stdout
