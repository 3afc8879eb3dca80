"""Fused multi-GPU frame assembly (vsr_trace_tiles) on one GPU: every rank's
trace kernel stores its tile shard's hits straight into one frame buffer at frame positions;
the assembled frame equals the single-launch frame bit for bit.  The IPC path (rank 1 maps rank
0's buffer) is exercised by two processes sharing the GPU — no kernel waits on another, the
ranks only meet at a host barrier."""
import os

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


def test_tiles_assemble_the_frame(V):
    from paper_1912_12786_b200 import shard
    sc, rays = W.config("C2", 480, 272)
    scene = V.Scene.from_workload(sc).build()
    full, cfull = scene.trace(torch.from_numpy(rays.data).cuda(), V.ANY, V.COUNT_ALPHA_TEXTURE)
    n = rays.n
    for P in (1, 3, 8):
        frame = torch.full((n, 4), -1.0, device="cuda")
        counts = torch.full((n, 4), -1, dtype=torch.int32, device="cuda")
        for r in range(P):
            idx = shard.rank_ray_indices(n, 64, r, P)
            loc = torch.from_numpy(rays.data[idx]).cuda()
            scene.trace_tiles(loc, 64, r, P, frame.data_ptr(), V.ANY, V.COUNT_ALPHA_TEXTURE,
                              frame_counts_ptr=counts.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(frame.view(torch.int32), full.view(torch.int32)), P
        assert torch.equal(counts, cfull), P
    with pytest.raises(V.VsrError):
        scene.trace_tiles(torch.from_numpy(rays.data[:100]).cuda(), 64, 0, 2, frame.data_ptr())


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1912_12786_b200 import shard, vsr
        torch.cuda.set_device(0)
        sc, rays = W.config("C2", 240, 136)
        scene = vsr.Scene.from_workload(sc).build()
        pf = shard.PeerFrame(rays.n, 0, dist)
        idx = shard.rank_ray_indices(rays.n, 64, rank, world)
        scene.trace_tiles(torch.from_numpy(rays.data[idx]).cuda(), 64, rank, world, pf.ptr, vsr.ANY,
                          vsr.ALPHA_TEXTURE)
        torch.cuda.synchronize()
        dist.barrier()           # every shard's stores are complete
        ok = True
        if rank == 0:
            full, _ = scene.trace(torch.from_numpy(rays.data).cuda(), vsr.ANY, vsr.ALPHA_TEXTURE)
            torch.cuda.synchronize()
            ok = bool(torch.equal(pf.tensor().view(torch.int32), full.view(torch.int32)))
        dist.barrier()           # the owner frees only after the peer has unmapped
        if rank != 0:
            pf.close()
        dist.barrier()
        if rank == 0:
            pf.close()
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_tiles_over_ipc_two_processes(V):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert all(ok for _, ok in res), res
