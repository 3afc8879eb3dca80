"""Concurrency claims of include/vsr.h: a built scene is read-only and may be traced from several
streams — and several host threads — at once; each stream gets its own order-pass scratch, reused
in stream order.  Results must equal a serial trace bit for bit."""
import threading

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def V():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_12786_b200 import _build
    _build.build()
    from paper_1912_12786_b200 import vsr
    return vsr


def test_many_streams_and_threads(V):
    sc, rays = W.config("C2", 480, 272)
    scene = V.Scene.from_workload(sc).build()
    d = torch.from_numpy(rays.data).cuda()
    ref = {}
    for q in (V.CLOSEST, V.ANY):
        h, _ = scene.trace(d, q, V.ALPHA_TEXTURE)
        torch.cuda.synchronize()
        ref[q] = h.clone()
    n_threads, reps = 4, 12
    errors = []

    def worker(i):
        try:
            st = torch.cuda.Stream()
            q = V.CLOSEST if i % 2 == 0 else V.ANY
            # different ray counts per thread: scratch grows per stream
            m = rays.n - 128 * i
            outs = []
            for _ in range(reps):
                h = torch.empty((m, 4), dtype=torch.float32, device="cuda")
                scene.trace(d[:m], q, V.ALPHA_TEXTURE, hits=h, stream=st)
                outs.append(h)
            st.synchronize()
            for h in outs:
                if not torch.equal(h.view(torch.int32), ref[q][:m].view(torch.int32)):
                    errors.append(f"thread {i}: mismatch")
                    break
        except Exception as e:  # pragma: no cover - reported below
            errors.append(f"thread {i}: {e!r}")

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(n_threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_threads_building_alpha_planes(V, monkeypatch):
    """Several threads, each with its own alpha threshold, trace concurrently while the scene
    builds a 1-bit plane per new threshold (under its lock) — every result equals the A8 path's."""
    sc, rays = W.config("C2", 480, 272)
    scene = V.Scene.from_workload(sc).build()
    d = torch.from_numpy(rays.data).cuda()
    thrs = [0.05, 0.2, 0.4, 0.6, 0.8, 0.95]
    monkeypatch.setenv("VSR_ALPHA_BITS", "0")
    ref = {}
    for t in thrs:
        h, _ = scene.trace(d, V.ANY, V.ALPHA_TEXTURE, alpha_threshold=t)
        torch.cuda.synchronize()
        ref[t] = h.clone()
    monkeypatch.setenv("VSR_ALPHA_BITS", "1")
    errors = []

    def worker(t):
        try:
            st = torch.cuda.Stream()
            outs = []
            for _ in range(6):
                h = torch.empty((rays.n, 4), dtype=torch.float32, device="cuda")
                scene.trace(d, V.ANY, V.ALPHA_TEXTURE, hits=h, stream=st, alpha_threshold=t)
                outs.append(h)
            st.synchronize()
            if any(not torch.equal(h.view(torch.int32), ref[t].view(torch.int32)) for h in outs):
                errors.append(f"threshold {t}: mismatch")
        except Exception as e:  # pragma: no cover - reported below
            errors.append(f"threshold {t}: {e!r}")

    ts = [threading.Thread(target=worker, args=(t,)) for t in thrs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
