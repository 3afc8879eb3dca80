"""bench.py's N-rank launcher, CPU only: `python bench.py --gpus 2`
outside torchrun must re-launch itself as 2 ranks (torch.distributed.run on 127.0.0.1),
and rank 0 alone prints one JSON line with n_gpus = 2.  `--plumbing` exercises the host
side of the multi-rank path — rendezvous, the round-robin 8x8-tile deal, frame assembly
by all-gather, max-over-ranks — without tracing (no GPU here); the assembled frame must
equal the P = 1 frame position for position.  The traced version is
tests/test_gpu_bench_launcher.py."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(gpus):
    env = dict(os.environ, VSR_DIST_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                        "--plumbing"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return lines


def test_launcher_spawns_two_ranks_one_line():
    lines = _run(2)
    assert len(lines) == 1, lines          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["plumbing"] is True and d["value"] is None
    assert d["frame_identical_to_p1"] is True


def test_launcher_single_rank_runs_in_process():
    d = json.loads(_run(1)[0])
    assert d["n_gpus"] == 1 and d["frame_identical_to_p1"] is True
