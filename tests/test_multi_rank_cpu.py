"""World-size-2 gloo tests of the multi-GPU host logic (CPU only):
scene replication (export -> broadcast -> import), the round-robin tile deal,
and the hit all-gather + re-ordering."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workloads as W
        from paper_1912_12786_b200 import shard, vsr

        sc = W.random_soup(500, seed=5)
        base = vsr.Scene.from_workload(sc, device=-1).build() if rank == 0 else None
        scene, arrs = shard.broadcast_scene(base, -1, dist, tensor_device="cpu")
        ex = scene.export()
        ref = vsr.Scene.from_workload(sc, device=-1).build().export()   # deterministic build
        same = all(np.array_equal(ex[k], ref[k]) for k in shard.ARRAY_KEYS)
        same &= ex["root_ref"] == ref["root_ref"]
        # tile deal + gather: 4 tiles of 64 rays per rank
        n, tile = 64 * 8, 64
        idx = shard.rank_ray_indices(n, tile, rank, world)
        local = torch.from_numpy(np.stack([idx.astype(np.float32)] * 4, axis=1))
        full = shard.gather_hits(local, n, tile, dist)
        ordered = np.array_equal(full[:, 0].numpy(), np.arange(n, dtype=np.float32))
        q.put((rank, bool(same), bool(ordered), len(idx)))
    finally:
        dist.destroy_process_group()


def test_broadcast_import_gather_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    for rank, same, ordered, nloc in res:
        assert same, f"rank {rank}: replicated scene differs from rank 0's"
        assert ordered, f"rank {rank}: gathered hits not in tile order"
        assert nloc == 256


def test_rank_indices_partition():
    from paper_1912_12786_b200 import shard

    n, tile = 64 * 32400, 64
    for P in (1, 2, 4, 8):
        parts = [shard.rank_ray_indices(n, tile, r, P) for r in range(P)]
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(n))
        assert len({len(p) for p in parts}) == 1


def test_frame_index_inverts_the_tile_deal():
    """vsr_trace_tiles' store mapping (shard.frame_index) sends local ray i of rank r to the
    frame position rank_ray_indices gave it, for tile counts that do and do not divide P."""
    from paper_1912_12786_b200 import shard

    for n_tiles, tile in ((32400, 64), (37, 256), (5, 64)):
        n = n_tiles * tile
        for P in (1, 2, 3, 8):
            for r in range(P):
                idx = shard.rank_ray_indices(n, tile, r, P)
                assert np.array_equal(shard.frame_index(np.arange(idx.size), tile, r, P), idx)
