"""Multi-GPU host logic: tile sharding and scene replication.

Every ray is independent and traversal has no exchange step, so the path
shards without a data-path collective:

* ``rank_ray_indices`` deals 8×8-pixel tiles (× spp) round-robin, tile k to
  rank k mod P (interleaving balances sky against forest);
* ``broadcast_scene`` replicates a built scene once (untimed setup): rank 0
  exports the flattened arrays (``vsr_bvh_export``), ``torch.distributed``
  broadcasts them (NCCL over NVLink on GPUs, gloo in CPU tests), every other
  rank calls ``vsr_scene_import``;
* ``gather_hits`` is the optional output assembly on rank 0
  (``all_gather_into_tensor`` of equal-size shards, then a scatter into
  image order).

Argument marshalling and torch plumbing only — no ray tracing arithmetic.
"""
from __future__ import annotations

import numpy as np

ARRAY_KEYS = ("nodes", "tris", "sides", "texdescs", "texels")


def rank_ray_indices(n_rays: int, rays_per_tile: int, rank: int, world: int) -> np.ndarray:
    """Indices of the rays of tiles k ≡ rank (mod world), in tile order."""
    assert n_rays % rays_per_tile == 0, "ray count must be a whole number of tiles"
    tiles = n_rays // rays_per_tile
    mine = np.arange(rank, tiles, world, dtype=np.int64)
    return (mine[:, None] * rays_per_tile + np.arange(rays_per_tile, dtype=np.int64)[None, :]).reshape(-1)


def shard_sizes(n_rays: int, rays_per_tile: int, world: int):
    tiles = n_rays // rays_per_tile
    return [len(range(r, tiles, world)) * rays_per_tile for r in range(world)]


def _meta(arrs: dict) -> np.ndarray:
    m = np.zeros(16, np.float64)
    m[0] = arrs["root_ref"]
    m[1:4] = arrs["root_lo"]
    m[4:7] = arrs["root_hi"]
    for k, key in enumerate(ARRAY_KEYS):
        m[7 + k] = arrs[key].shape[0]
    return m


def broadcast_scene(scene_or_none, device, dist, src: int = 0, tensor_device=None):
    """Replicate rank ``src``'s built scene to every rank; returns the local Scene.

    ``tensor_device`` is where the broadcast buffers live ("cuda:i" for NCCL,
    "cpu" for gloo).  ``device`` is the CUDA ordinal for vsr_scene_import
    (-1: host-only import, used by the CPU tests)."""
    import torch

    from .vsr import Scene

    rank = dist.get_rank()
    tdev = tensor_device or ("cpu" if device < 0 else f"cuda:{device}")
    if rank == src:
        arrs = scene_or_none.export()
        meta = torch.from_numpy(_meta(arrs))
    else:
        arrs = None
        meta = torch.zeros(16, dtype=torch.float64)
    meta = meta.to(tdev)
    dist.broadcast(meta, src)
    meta = meta.cpu().numpy()
    widths = {"nodes": 16, "tris": 12, "sides": 8, "texdescs": 4, "texels": 1}
    # 32-bit words everywhere except the A8 alpha plane
    dtypes = {"texels": (np.uint8, torch.uint8)}
    out = {"root_ref": int(meta[0]), "root_lo": meta[1:4].astype(np.float32),
           "root_hi": meta[4:7].astype(np.float32)}
    for k, key in enumerate(ARRAY_KEYS):
        rows = int(meta[7 + k])
        shape = (rows, widths[key]) if widths[key] > 1 else (rows,)
        np_dt, t_dt = dtypes.get(key, (np.int32, torch.int32))
        if rank == src:
            t = torch.from_numpy(np.ascontiguousarray(arrs[key]).view(np_dt).reshape(shape)).to(tdev)
        else:
            t = torch.empty(shape, dtype=t_dt, device=tdev)
        if t.numel():
            dist.broadcast(t, src)
        out[key] = t
    if rank == src and scene_or_none is not None and device >= 0:
        return scene_or_none, out
    host = {k: (v.cpu().numpy().view(np.uint8 if k == "texels" else np.uint32)
                if hasattr(v, "cpu") else v) for k, v in out.items()}
    if device >= 0:
        # import straight from the device buffers the broadcast filled
        dev = {k: v for k, v in out.items()}
        return Scene.import_arrays(dev, device=device), host
    return Scene.import_arrays(host, device=-1), host


def gather_hits(local_hits, n_total: int, rays_per_tile: int, dist, out=None, reorder=True):
    """all_gather_into_tensor equal-size hit shards (and re-order into tile order).

    local_hits: [n_local, 4] float32 tensor.  Every rank's shard has the same size
    (the tile counts divide P).  `out`: optional [world * n_local, 4] gather buffer.
    Returns the full [n_total, 4] tensor on every rank (rank-major if not reorder)."""
    import torch

    world = dist.get_world_size()
    sizes = shard_sizes(n_total, rays_per_tile, world)
    assert len(set(sizes)) == 1, "tile counts must divide the world size"
    gathered = out if out is not None else torch.empty(
        (world * sizes[0], 4), dtype=local_hits.dtype, device=local_hits.device)
    if local_hits.is_cuda or dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(gathered, local_hits.contiguous())
    else:   # gloo (CPU tests): list form
        parts = list(gathered.view(world, sizes[0], 4).unbind(0))
        dist.all_gather(parts, local_hits.contiguous())
    if not reorder:
        return gathered
    # rank r's j-th tile is global tile r + j*world
    g = gathered.view(world, sizes[0] // rays_per_tile, rays_per_tile, 4)
    return g.transpose(0, 1).reshape(n_total, 4)


def frame_index(local_ids, rays_per_tile: int, rank: int, world: int) -> np.ndarray:
    """Frame position of this rank's local ray i (its j-th tile is frame tile j*world + rank):
    the mapping vsr_trace_tiles applies when storing hits; inverse of rank_ray_indices."""
    local_ids = np.asarray(local_ids, dtype=np.int64)
    tile = local_ids // rays_per_tile
    return (tile * world + rank) * rays_per_tile + local_ids % rays_per_tile


class PeerFrame:
    """A frame hit buffer on rank ``owner`` that every rank's trace kernel writes into directly
    (vsr_trace_tiles over CUDA IPC / NVLink): the owner allocates it (vsr_device_alloc) and
    publishes its IPC handle; the other ranks map it (vsr_ipc_open).  ``ptr`` is valid in every
    process; ``tensor()`` (owner only) views it as a [rows, 4] float32 torch tensor."""

    def __init__(self, rows: int, device: int, dist, owner: int = 0):
        from . import vsr
        self.vsr, self.rows, self.device, self.owner = vsr, rows, device, owner
        self.rank = dist.get_rank()
        box = [None]
        if self.rank == owner:
            self.ptr = vsr.device_alloc(rows * 16, device)
            box = [vsr.ipc_handle(self.ptr)]
        dist.broadcast_object_list(box, src=owner)
        if self.rank != owner:
            self.ptr = vsr.ipc_open(box[0], device)

    def tensor(self):
        import torch
        assert self.rank == self.owner, "only the owner reads the frame"
        return torch.as_tensor(self.vsr.DeviceArray(self.ptr, (self.rows, 4), "<f4"),
                               device=f"cuda:{self.device}")

    def release(self, dist):
        """Collective teardown: peers unmap first, then the owner frees."""
        import torch
        torch.cuda.synchronize()
        dist.barrier()
        if self.rank != self.owner:
            self.close()
        dist.barrier()
        if self.rank == self.owner:
            self.close()

    def close(self):
        if self.ptr:
            if self.rank == self.owner:
                self.vsr.device_free(self.ptr, self.device)
            else:
                self.vsr.ipc_close(self.ptr, self.device)
            self.ptr = 0

