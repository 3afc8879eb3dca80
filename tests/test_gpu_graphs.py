"""CUDA-graph capture of the trace entry points (include/vsr.h, vsr_trace "CUDA graphs"): the
order pass + trace launches are captured into a torch.cuda.CUDAGraph (its scratch becomes graph
memory nodes) and replayed; every replay equals an eager trace of the rays then in the input
buffer, bit for bit — on fresh ray contents, for plain, pinhole, multi-hit and instance traces."""
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


@pytest.fixture(scope="module")
def forest(V):
    sc, rays = W.config("C2", 480, 272)
    return V.Scene.from_workload(sc).build(), rays


def capture(fn):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()   # warm-up on the capture stream (plane build, scratch, lazy init)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    return g


@pytest.mark.parametrize("q", ["any", "closest"])
@pytest.mark.parametrize("isect", ["ALPHA_TEXTURE", "DEFAULT", "COUNT_ALPHA_TEXTURE"])
def test_trace_graph_replay(V, forest, q, isect):
    s, rays = forest
    query = V.ANY if q == "any" else V.CLOSEST
    k = getattr(V, isect)
    base = torch.from_numpy(rays.data).cuda()
    r = base.clone()
    hits = torch.empty((r.shape[0], 4), dtype=torch.float32, device="cuda")
    counts = torch.empty((r.shape[0], 4), dtype=torch.int32, device="cuda") \
        if isect.startswith("COUNT") else None
    g = capture(lambda: s.trace(r, query, k, hits=hits, counts=counts))
    gen = torch.Generator(device="cpu").manual_seed(7)
    for rep in range(3):
        # new ray contents in the captured buffer: a permutation of the frame's rays
        r.copy_(base[torch.randperm(base.shape[0], generator=gen).cuda()])
        g.replay()
        torch.cuda.synchronize()
        eh, ec = s.trace(r.clone(), query, k)
        torch.cuda.synchronize()
        assert torch.equal(hits.view(torch.int32), eh.view(torch.int32)), (q, isect, rep)
        if counts is not None:
            assert torch.equal(counts, ec)


def test_pinhole_and_multi_graph_replay(V, forest):
    s, rays = forest
    cam = V.pinhole_camera((0.0, 60.0, -1100.0), (0.0, 10.0, 0.0), (0.0, 1.0, 0.0), 45.0, 480,
                           272, 1)
    n = 480 * 272
    ph = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    r = torch.from_numpy(rays.data).cuda()
    mh = torch.empty((r.shape[0], 4, 4), dtype=torch.float32, device="cuda")
    mn = torch.empty((r.shape[0],), dtype=torch.int32, device="cuda")

    def work():
        s.trace_pinhole(cam, V.ANY, V.ALPHA_TEXTURE, hits=ph)
        s.trace_multi(r, 4, V.ALPHA_TEXTURE, hits=mh, num_hits=mn)

    g = capture(work)
    ph.zero_()
    mh.zero_()
    g.replay()
    torch.cuda.synchronize()
    eh, _ = s.trace_pinhole(cam, V.ANY, V.ALPHA_TEXTURE)
    emh, emn, _ = s.trace_multi(r, 4, V.ALPHA_TEXTURE)
    torch.cuda.synchronize()
    assert torch.equal(ph.view(torch.int32), eh.view(torch.int32))
    assert torch.equal(mh.view(torch.int32), emh.view(torch.int32)) and torch.equal(mn, emn)


def test_instances_graph_replay(V):
    models, ibvh, imat = W.instanced_forest(n_instances=500, n_models=2, cards=16)
    scenes = [V.Scene.from_workload(m).build() for m in models]
    inst = V.Instances(scenes, ibvh, imat)
    _, rays = W.config("C2", 240, 136)
    r = torch.from_numpy(rays.data).cuda()
    hits = torch.empty((r.shape[0], 4), dtype=torch.float32, device="cuda")
    which = torch.empty((r.shape[0],), dtype=torch.int32, device="cuda")
    g = capture(lambda: inst.trace(r, V.ANY, V.ALPHA_TEXTURE, hits=hits, inst=which))
    hits.zero_()
    g.replay()
    torch.cuda.synchronize()
    eh, ew, _ = inst.trace(r, V.ANY, V.ALPHA_TEXTURE)
    torch.cuda.synchronize()
    assert torch.equal(hits.view(torch.int32), eh.view(torch.int32)) and torch.equal(which, ew)
