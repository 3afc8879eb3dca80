"""The real bench launcher at --gpus 2 on one B200: two ranks share
cuda:0 over gloo (no kernel waits on another rank's kernel: the ranks meet only at host
barriers), rank 0 prints one JSON line with n_gpus 2, and the strong-scaling tile frame —
assembled by both ranks' trace kernels storing into rank 0's IPC-mapped buffer — is
bit-identical to one plain launch over the whole frame."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_strong_frame_identical():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, VSR_DIST_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--no-variants", "--no-cpu",
                        "--no-counters", "--strong-config", "C2", "--strong-frames", "4"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    s = d["strong"]
    assert "error" not in s, s
    assert s["frame_bit_identical_to_single_launch"] is True
    assert s["gpu_launches"] >= 4
