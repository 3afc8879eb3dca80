"""Seeded synthetic scenes and rays (inputs only — no method arithmetic).

Array conventions (the input contract both sides consume, byte for byte):

* ``Scene.vertices``   float32 [N, 9]  — v0.xyz, v1.xyz, v2.xyz per triangle
* ``Scene.geom_ids``   uint32  [N]     — mesh group of each triangle (PAPER.md:304 ``hr.geom_id``)
* ``Scene.texcoords``  float32 [N, 6]  — uv0, uv1, uv2 per triangle (PAPER.md:306-308 ``tex_coords[prim_id*3+k]``)
* ``Scene.geom_texture`` uint32 [G]    — geom_id → texture index
* ``Scene.textures``   list of uint8 [H, W, 4] RGBA8, row j = memory row j
* ``Rays.data``        float32 [n, 8]  — ox, oy, oz, tmin, dx, dy, dz, tmax (SURVEY.md §8(b) ``vsr_ray``)

Rays are emitted in 8×8-pixel tile order (tile row-major, then sample, then
y, then x inside the tile), so one warp of 32 consecutive rays covers an 8×4
pixel block (SURVEY.md §8(d) "Configs as concrete synthetic inputs").
All randomness is numpy PCG64 (``default_rng(seed)``) or the integer
``pcg_hash`` below.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

TILE = 8
DEFAULT_TMIN = 1e-4


@dataclass
class Scene:
    name: str
    vertices: np.ndarray
    geom_ids: np.ndarray
    texcoords: np.ndarray
    geom_texture: np.ndarray
    textures: list = field(default_factory=list)
    source_index: np.ndarray | None = None   # split_scene: original triangle indices

    @property
    def num_tris(self) -> int:
        return int(self.vertices.shape[0])

    def tri_texture(self) -> np.ndarray:
        """Texture index of every triangle (geom_texture[geom_ids[i]])."""
        return self.geom_texture[self.geom_ids]


@dataclass
class Rays:
    data: np.ndarray          # float32 [n, 8]
    width: int = 0
    height: int = 0
    spp: int = 1
    pixel: np.ndarray | None = None   # int64 [n] image-order pixel index y*W + x
    sample: np.ndarray | None = None  # int64 [n]

    @property
    def n(self) -> int:
        return int(self.data.shape[0])


def pcg_hash(x):
    """PCG-RXS-M-XS 32-bit hash (integer mixing only), vectorised over uint32."""
    x = np.asarray(x, dtype=np.uint64) & np.uint64(0xFFFFFFFF)
    state = (x * np.uint64(747796405) + np.uint64(2891336453)) & np.uint64(0xFFFFFFFF)
    shift = (state >> np.uint64(28)) + np.uint64(4)
    word = (((state >> shift) ^ state) * np.uint64(277803737)) & np.uint64(0xFFFFFFFF)
    return ((word >> np.uint64(22)) ^ word).astype(np.uint32)


# --------------------------------------------------------------------------
# ray order helpers
# --------------------------------------------------------------------------

def tile_order(width: int, height: int, spp: int = 1):
    """Return (px, py, s) int64 arrays in (tile, sample, y, x) order."""
    assert width % TILE == 0 and height % TILE == 0, "image must tile by 8"
    tx = width // TILE
    ty = height // TILE
    t_idx = np.arange(tx * ty, dtype=np.int64)
    s_idx = np.arange(spp, dtype=np.int64)
    yy, xx = np.meshgrid(np.arange(TILE), np.arange(TILE), indexing="ij")
    yy = yy.reshape(-1).astype(np.int64)
    xx = xx.reshape(-1).astype(np.int64)
    # broadcast to [tiles, spp, 64]
    tile_x = (t_idx % tx)[:, None, None]
    tile_y = (t_idx // tx)[:, None, None]
    px = tile_x * TILE + xx[None, None, :] + 0 * s_idx[None, :, None]
    py = tile_y * TILE + yy[None, None, :] + 0 * s_idx[None, :, None]
    s = np.broadcast_to(s_idx[None, :, None], px.shape)
    return px.reshape(-1), py.reshape(-1), np.ascontiguousarray(s).reshape(-1)


def _pack_rays(org, dirs, tmin=DEFAULT_TMIN, tmax=np.inf) -> np.ndarray:
    n = dirs.shape[0]
    out = np.empty((n, 8), dtype=np.float32)
    out[:, 0:3] = org
    out[:, 3] = np.float32(tmin)
    out[:, 4:7] = dirs
    out[:, 7] = np.float32(tmax)
    return out


# --------------------------------------------------------------------------
# C1 — quad pair
# --------------------------------------------------------------------------

def _quad_tris(corners_xy, z, tc_lo, tc_hi):
    """Axis-aligned quad at depth z split along its (lo,lo)-(hi,hi) diagonal."""
    (x0, y0), (x1, y1) = corners_xy
    (s0, t0), (s1, t1) = tc_lo, tc_hi
    p00, p10, p11, p01 = (x0, y0, z), (x1, y0, z), (x1, y1, z), (x0, y1, z)
    c00, c10, c11, c01 = (s0, t0), (s1, t0), (s1, t1), (s0, t1)
    verts = [p00 + p10 + p11, p00 + p11 + p01]
    tcs = [c00 + c10 + c11, c00 + c11 + c01]
    return verts, tcs


def c1_texture() -> np.ndarray:
    """16×16 RGBA8: alpha 255 on a checker of 4×4-texel blocks, else 0; row 15
    overridden to a8=3 for i<8 and a8=2 for i>=8 (threshold exercise)."""
    tex = np.zeros((16, 16, 4), dtype=np.uint8)
    tex[..., 0] = 40
    tex[..., 1] = 160
    tex[..., 2] = 40
    j, i = np.meshgrid(np.arange(16), np.arange(16), indexing="ij")
    tex[..., 3] = np.where(((i // 4) + (j // 4)) % 2 == 0, 255, 0)
    tex[15, :8, 3] = 3
    tex[15, 8:, 3] = 2
    return tex


def quad_pair_scene() -> Scene:
    va, ta = _quad_tris(((0.0, 0.0), (1.0, 0.75)), 1.0, (0.0, 0.0), (1.0, 1.0))
    vb, tb = _quad_tris(((-0.5, -0.5), (1.5, 1.25)), 2.0, (0.0, 0.0), (2.0, 2.0))
    vertices = np.array(va + vb, dtype=np.float32)
    texcoords = np.array(ta + tb, dtype=np.float32)
    geom_ids = np.array([0, 0, 1, 1], dtype=np.uint32)
    geom_texture = np.array([0, 0], dtype=np.uint32)
    return Scene("C1-quad-pair", vertices, geom_ids, texcoords, geom_texture, [c1_texture()])


def quad_pair_rays(res: int = 64) -> Rays:
    """Orthographic rays o=(x,y,0), d=(0,0,1) on a non-dyadic grid."""
    px, py, s = tile_order(res, res, 1)
    x = -0.6 + 2.2 * (px + 0.5) / res
    y = -0.6 + 2.0 * (py + 0.5) / res
    n = px.shape[0]
    org = np.stack([x, y, np.zeros(n)], axis=1)
    dirs = np.tile(np.array([0.0, 0.0, 1.0]), (n, 1))
    return Rays(_pack_rays(org, dirs), res, res, 1, py * res + px, s)


# --------------------------------------------------------------------------
# textures — K "tree" alpha masks
# --------------------------------------------------------------------------

def tree_textures(k: int = 16, size: int = 1024, seed: int = 2, discs: int = 48) -> list:
    rng = np.random.default_rng(seed)
    out = []
    jj, ii = np.meshgrid(np.arange(size, dtype=np.float32), np.arange(size, dtype=np.float32),
                         indexing="ij")
    for _ in range(k):
        canopy = np.zeros((size, size), dtype=bool)
        cx = rng.uniform(0.12 * size, 0.88 * size, discs)
        cy = rng.uniform(0.25 * size, 0.95 * size, discs)
        rad = rng.uniform(40.0, 160.0, discs) * (size / 1024.0)
        for a, b, r in zip(cx, cy, rad):
            x0, x1 = int(max(0, a - r)), int(min(size, a + r + 1))
            y0, y1 = int(max(0, b - r)), int(min(size, b + r + 1))
            sub_i = ii[y0:y1, x0:x1] + 0.5 - a
            sub_j = jj[y0:y1, x0:x1] + 0.5 - b
            canopy[y0:y1, x0:x1] |= (sub_i * sub_i + sub_j * sub_j) <= r * r
        # leaf gaps: 25 % of the 8×8 blocks that touch the canopy are cleared
        nb = size // 8
        blk = canopy.reshape(nb, 8, nb, 8).any(axis=(1, 3))
        gaps = blk & (rng.random((nb, nb)) < 0.25)
        gap_mask = np.repeat(np.repeat(gaps, 8, axis=0), 8, axis=1)
        opaque = canopy & ~gap_mask
        # trunk rectangle (bottom centre; row 0 is the bottom, t = 0)
        tw = max(1, size // 32)
        opaque[0:int(0.40 * size), size // 2 - tw:size // 2 + tw] = True
        alpha = np.where(opaque, 255, 0).astype(np.uint8)
        # one-texel rim alternating a8 = 3 / a8 = 2 around the opaque set
        nbr = np.zeros_like(opaque)
        nbr[1:, :] |= opaque[:-1, :]
        nbr[:-1, :] |= opaque[1:, :]
        nbr[:, 1:] |= opaque[:, :-1]
        nbr[:, :-1] |= opaque[:, 1:]
        rim = nbr & ~opaque
        parity = ((ii.astype(np.int64) + jj.astype(np.int64)) % 2) == 0
        alpha[rim & parity] = 3
        alpha[rim & ~parity] = 2
        tex = np.empty((size, size, 4), dtype=np.uint8)
        tex[..., 0] = 30 + (rng.integers(0, 40))
        tex[..., 1] = 110 + (rng.integers(0, 80))
        tex[..., 2] = 30
        tex[..., 3] = alpha
        out.append(tex)
    return out


def stress_textures(k: int = 1024, size: int = 1024, seed: int = 2, base: int = 64) -> list:
    """SURVEY.md §8(c) A25 stress variant: K distinct RGBA8 tree masks (K = 1024 at 1024²
    is 4 GiB), so texel reads of C2 reach HBM.  `base` masks come from the C2 recipe; mask i
    is base i mod `base`, rolled sideways by a seeded offset and mirrored when (i // base)
    is odd — the canopy/trunk/rim statistics of C2, every mask distinct."""
    bases = tree_textures(base, size, seed)
    rng = np.random.default_rng(seed + 1000)
    per = -(-k // base)   # variants per base mask, each with its own distinct shift
    shifts = np.stack([rng.permutation(np.arange(1, size))[:per] for _ in range(base)])
    out = []
    for i in range(k):
        t = bases[i % base]
        if i >= base:
            t = np.roll(t, int(shifts[i % base, i // base]), axis=1)
            if (i // base) % 2:
                t = t[:, ::-1]
        out.append(np.ascontiguousarray(t))
    return out


def white_texture() -> np.ndarray:
    return np.full((1, 1, 4), 255, dtype=np.uint8)


# --------------------------------------------------------------------------
# billboards, terrain
# --------------------------------------------------------------------------

def _billboards(n: int, extent: float, seed: int, base_height=None):
    rng = np.random.default_rng(seed)
    cx = rng.uniform(-extent, extent, n)
    cz = rng.uniform(-extent, extent, n)
    yaw = rng.uniform(0.0, math.pi, n)
    width = rng.uniform(3.0, 8.0, n)
    height = width * rng.uniform(1.2, 2.0, n)
    y0 = np.zeros(n) if base_height is None else base_height(cx, cz)
    hx = 0.5 * width * np.cos(yaw)
    hz = 0.5 * width * np.sin(yaw)
    bl = np.stack([cx - hx, y0, cz - hz], axis=1)
    br = np.stack([cx + hx, y0, cz + hz], axis=1)
    tr = np.stack([cx + hx, y0 + height, cz + hz], axis=1)
    tl = np.stack([cx - hx, y0 + height, cz - hz], axis=1)
    verts = np.empty((2 * n, 9), dtype=np.float64)
    verts[0::2] = np.concatenate([bl, br, tr], axis=1)
    verts[1::2] = np.concatenate([bl, tr, tl], axis=1)
    tcs = np.empty((2 * n, 6), dtype=np.float64)
    tcs[0::2] = np.array([0, 0, 1, 0, 1, 1], dtype=np.float64)
    tcs[1::2] = np.array([0, 0, 1, 1, 0, 1], dtype=np.float64)
    gids = np.repeat(np.arange(n, dtype=np.uint32), 2)
    return verts.astype(np.float32), tcs.astype(np.float32), gids


def forest_scene(n_billboards: int = 20000, extent: float = 250.0, seed: int = 1,
                 k_textures: int = 16, tex_size: int = 1024, tex_seed: int = 2,
                 textures=None) -> Scene:
    """C2: 20k vertical alpha-masked billboards (40k triangles), no ground."""
    verts, tcs, gids = _billboards(n_billboards, extent, seed)
    if textures is None:
        textures = tree_textures(k_textures, tex_size, tex_seed)
    gtex = (pcg_hash(np.arange(n_billboards, dtype=np.uint32)) % np.uint32(len(textures))).astype(np.uint32)
    return Scene("C2-forest", verts, gids, tcs, gtex, textures)


def _value_noise(x, z, seed):
    xi = np.floor(x).astype(np.int64)
    zi = np.floor(z).astype(np.int64)
    fx = x - xi
    fz = z - zi
    sx = fx * fx * (3 - 2 * fx)
    sz = fz * fz * (3 - 2 * fz)

    def lat(a, b):
        h = pcg_hash((a * 73856093) ^ (b * 19349663) ^ (seed * 83492791))
        return h.astype(np.float64) / 4294967295.0 * 2.0 - 1.0

    v00 = lat(xi, zi)
    v10 = lat(xi + 1, zi)
    v01 = lat(xi, zi + 1)
    v11 = lat(xi + 1, zi + 1)
    return (v00 * (1 - sx) + v10 * sx) * (1 - sz) + (v01 * (1 - sx) + v11 * sx) * sz


def fbm_height(x, z, seed: int, amplitude: float, wavelength: float = 128.0, octaves: int = 5):
    total = np.zeros(np.broadcast(x, z).shape)
    norm = 0.0
    for o in range(octaves):
        f = (2.0 ** o) / wavelength
        a = 0.5 ** o
        total += a * _value_noise(x * f, z * f, seed * 131 + o)
        norm += a
    return amplitude * total / norm


def heightfield_scene(nx: int, nz: int, extent_x: float, extent_z: float, seed: int,
                      amplitude: float, geom_id: int):
    xs = np.linspace(-extent_x, extent_x, nx + 1)
    zs = np.linspace(-extent_z, extent_z, nz + 1)
    gx, gz = np.meshgrid(xs, zs, indexing="xy")        # [nz+1, nx+1]
    gy = fbm_height(gx, gz, seed, amplitude)
    p = np.stack([gx, gy, gz], axis=-1).astype(np.float32)   # [nz+1, nx+1, 3]
    p00 = p[:-1, :-1].reshape(-1, 3)
    p10 = p[:-1, 1:].reshape(-1, 3)
    p11 = p[1:, 1:].reshape(-1, 3)
    p01 = p[1:, :-1].reshape(-1, 3)
    nq = p00.shape[0]
    verts = np.empty((2 * nq, 9), dtype=np.float32)
    verts[0::2, 0:3] = p00
    verts[0::2, 3:6] = p10
    verts[0::2, 6:9] = p11
    verts[1::2, 0:3] = p00
    verts[1::2, 3:6] = p11
    verts[1::2, 6:9] = p01
    tcs = np.zeros((2 * nq, 6), dtype=np.float32)
    gids = np.full(2 * nq, geom_id, dtype=np.uint32)
    return verts, tcs, gids


def _terrain_plus_billboards(name, tnx, tnz, ext, tseed, amp, nbb, bseed, textures):
    tv, ttc, tg = heightfield_scene(tnx, tnz, ext, ext, tseed, amp, geom_id=nbb)
    bv, btc, bg = _billboards(nbb, ext, bseed,
                              base_height=lambda x, z: fbm_height(x, z, tseed, amp))
    k = len(textures)
    gtex = np.empty(nbb + 1, dtype=np.uint32)
    gtex[:nbb] = pcg_hash(np.arange(nbb, dtype=np.uint32)) % np.uint32(k)
    gtex[nbb] = k          # terrain → 1×1 opaque white
    verts = np.concatenate([tv, bv])
    tcs = np.concatenate([ttc, btc])
    gids = np.concatenate([tg, bg])
    return Scene(name, verts, gids, tcs, gtex, list(textures) + [white_texture()])


def c4_scene(textures=None, terrain=(1000, 500), n_billboards=20000) -> Scene:
    """C4: 1000×500-quad fBm terrain (1M tris) + the C2 billboards on it."""
    if textures is None:
        textures = tree_textures(16, 1024, 2)
    return _terrain_plus_billboards("C4-heatmap-1M", terrain[0], terrain[1], 250.0, 3, 12.0,
                                    n_billboards, 1, textures)


def c5_scene(textures=None, terrain=(2500, 2000), n_billboards=100000) -> Scene:
    """C5: 2500×2000-quad terrain (10M tris) + 100k billboards (10.2M tris)."""
    if textures is None:
        textures = tree_textures(16, 1024, 2)
    return _terrain_plus_billboards("C5-big-4K", terrain[0], terrain[1], 1000.0, 4, 30.0,
                                    n_billboards, 5, textures)


# --------------------------------------------------------------------------
# cameras
# --------------------------------------------------------------------------

def pinhole_rays(eye, look_at, up, vfov_deg: float, width: int, height: int,
                 spp: int = 1, jitter_seed: int = 6, tmin: float = DEFAULT_TMIN) -> Rays:
    """Pinhole primary rays, unnormalised d = W + sx·tan(fov/2)·aspect·U + sy·tan(fov/2)·V.

    spp = 1 samples pixel centres; spp = 4 uses 2×2 strata with a pcg_hash
    jitter per (pixel, sample)."""
    eye = np.asarray(eye, dtype=np.float64)
    w = np.asarray(look_at, dtype=np.float64) - eye
    w /= np.linalg.norm(w)
    u = np.cross(np.asarray(up, dtype=np.float64), w)
    u /= np.linalg.norm(u)
    v = np.cross(w, u)
    px, py, s = tile_order(width, height, spp)
    if spp == 1:
        jx = np.full(px.shape, 0.5)
        jy = np.full(px.shape, 0.5)
    else:
        side = int(round(math.sqrt(spp)))
        assert side * side == spp
        key = (py * width + px) * spp + s
        h1 = pcg_hash((key.astype(np.uint64) * np.uint64(2) + np.uint64(jitter_seed * 7919)) & np.uint64(0xFFFFFFFF))
        h2 = pcg_hash((key.astype(np.uint64) * np.uint64(2) + np.uint64(1 + jitter_seed * 7919)) & np.uint64(0xFFFFFFFF))
        r1 = h1.astype(np.float64) / 4294967296.0
        r2 = h2.astype(np.float64) / 4294967296.0
        jx = ((s % side) + r1) / side
        jy = ((s // side) + r2) / side
    th = math.tan(math.radians(vfov_deg) * 0.5)
    aspect = width / height
    sx = 2.0 * (px + jx) / width - 1.0
    sy = 1.0 - 2.0 * (py + jy) / height
    dirs = w[None, :] + (sx * th * aspect)[:, None] * u[None, :] + (sy * th)[:, None] * v[None, :]
    org = np.broadcast_to(eye, dirs.shape)
    return Rays(_pack_rays(org, dirs, tmin), width, height, spp, py * width + px, s)


# --------------------------------------------------------------------------
# small test workloads
# --------------------------------------------------------------------------

def random_soup(n: int, seed: int, extent: float = 10.0, size: float = 2.0, n_geoms: int = 4,
                n_textures: int = 2, tex_size: int = 8) -> Scene:
    """Random triangles in a cube with random texcoords and small random RGBA8 textures."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(-extent, extent, (n, 1, 3))
    off = rng.uniform(-size, size, (n, 3, 3))
    verts = (c + off).reshape(n, 9).astype(np.float32)
    tcs = rng.uniform(-1.5, 2.5, (n, 6)).astype(np.float32)
    gids = rng.integers(0, n_geoms, n).astype(np.uint32)
    gtex = rng.integers(0, n_textures, n_geoms).astype(np.uint32)
    texs = []
    for _ in range(n_textures):
        t = rng.integers(0, 256, (tex_size, tex_size, 4)).astype(np.uint8)
        texs.append(t)
    return Scene(f"soup-{n}-{seed}", verts, gids, tcs, gtex, texs)


def random_rays(n: int, seed: int, extent: float = 12.0, target: float = 8.0,
                tmin: float = DEFAULT_TMIN) -> Rays:
    """Rays from a shell around the cube aimed at random points inside it."""
    rng = np.random.default_rng(seed)
    o = rng.normal(size=(n, 3))
    o = o / np.linalg.norm(o, axis=1, keepdims=True) * extent * 1.5
    tgt = rng.uniform(-target, target, (n, 3))
    d = (tgt - o) * rng.uniform(0.05, 3.0, (n, 1))
    return Rays(_pack_rays(o, d, tmin), n, 1, 1, np.arange(n), np.zeros(n, dtype=np.int64))


def stacked_quads(k: int = 5, z0: float = 1.0, dz: float = 1.0) -> Scene:
    """k parallel unit quads at z = z0 .. z0+(k-1)·dz."""
    verts, tcs = [], []
    for q in range(k):
        v, t = _quad_tris(((0.0, 0.0), (1.0, 1.0)), z0 + q * dz, (0.0, 0.0), (1.0, 1.0))
        verts += v
        tcs += t
    vertices = np.array(verts, dtype=np.float32)
    texcoords = np.array(tcs, dtype=np.float32)
    gids = np.repeat(np.arange(k, dtype=np.uint32), 2)
    gtex = np.zeros(k, dtype=np.uint32)
    return Scene(f"stack-{k}", vertices, gids, texcoords, gtex, [white_texture()])


# --------------------------------------------------------------------------
# named configs (BASELINE.json "configs")
# --------------------------------------------------------------------------

CONFIGS = {
    "C1": "64×64 primary rays vs 2 alpha-masked billboard quads (4 triangles, 16×16 alpha texture)",
    "C2": "billboard forest: 20k billboards (40k tris), 1024×1024 RGBA alpha textures, 1920×1080 primary rays",
    "C3": "C2 scene, procedural vs default vs no intersector (zero-cost check)",
    "C4": "1M-triangle terrain + 20k billboards, 1920×1080, counting intersector",
    "C5": "10M-triangle terrain + 100k billboards, 3840×2160×4 spp",
    "C2K": "C2 with K = 1024 distinct 1024×1024 RGBA alpha textures (4 GiB; SURVEY A25 HBM-stress "
           "variant), 1920×1080 primary rays",
}


# --------------------------------------------------------------------------
# two-level instancing (NEXT-2; "the BVH will store BVHs as primitives")
# --------------------------------------------------------------------------

def tree_model(seed: int, n_cards: int = 16, textures=None) -> Scene:
    """One tree object in its own space: n_cards vertical alpha cards (the C2 billboard
    recipe) scattered within 4 m of the y axis, base at y = 0."""
    verts, tcs, gids = _billboards(n_cards, 4.0, seed)
    if textures is None:
        textures = tree_textures(4, 256, seed + 100, discs=24)
    gtex = (pcg_hash(np.arange(n_cards, dtype=np.uint32) + np.uint32(seed * 7919))
            % np.uint32(len(textures))).astype(np.uint32)
    return Scene(f"tree{seed}", verts, gids, tcs, gtex, textures)


def object_from_world(yaw, scale, tx, ty, tz, shear=0.0) -> np.ndarray:
    """[A | b] (float32, 12 per instance) of world_from_object = T(t) R_y(yaw) S(scale) K(shear),
    K(shear) = identity + shear in the x-from-y entry; inverted in float64."""
    yaw, scale, tx, ty, tz = (np.atleast_1d(np.asarray(x, np.float64)) for x in (yaw, scale, tx, ty, tz))
    shear = np.broadcast_to(np.asarray(shear, np.float64), yaw.shape)
    n = yaw.shape[0]
    out = np.empty((n, 12), np.float32)
    for k in range(n):
        c, s_ = math.cos(yaw[k]), math.sin(yaw[k])
        R = np.array([[c, 0.0, s_], [0.0, 1.0, 0.0], [-s_, 0.0, c]])
        K = np.eye(3)
        K[0, 1] = shear[k]
        W = R @ (scale[k] * K)
        A = np.linalg.inv(W)
        b = -A @ np.array([tx[k], ty[k], tz[k]])
        out[k] = np.concatenate([A, b[:, None]], axis=1).reshape(12)
    return out


def instanced_forest(n_instances: int = 10000, n_models: int = 4, cards: int = 64,
                     extent: float = 250.0, seed: int = 5, textures=None):
    """NEXT-2 workload: n_models tree models of `cards` alpha cards each, instanced
    n_instances times over the C2 ground square with a random yaw, uniform scale 0.7-1.4
    and a small shear.  Returns (models, bvh uint32[n], object_from_world float32[n, 12])."""
    if textures is None:
        textures = tree_textures(8, 512, seed + 1, discs=32)
    models = [tree_model(seed * 31 + k, cards, textures) for k in range(n_models)]
    rng = np.random.default_rng(seed)
    bvh = rng.integers(0, n_models, n_instances).astype(np.uint32)
    m = object_from_world(rng.uniform(0, 2 * math.pi, n_instances), rng.uniform(0.7, 1.4, n_instances),
                          rng.uniform(-extent, extent, n_instances), np.zeros(n_instances),
                          rng.uniform(-extent, extent, n_instances),
                          rng.uniform(-0.1, 0.1, n_instances))
    return models, bvh, m


def split_scene(scene: Scene, k: int, axis: int = 0) -> list:
    """Partition a scene's triangles into k sub-scenes by centroid slab along `axis`
    (objects for list / compound-BVH queries).  Sub-scenes share the texture list and
    geom -> texture table; each keeps its triangles in caller order."""
    c = scene.vertices.reshape(-1, 3, 3)[:, :, axis].mean(axis=1)
    edges = np.quantile(c, np.linspace(0, 1, k + 1))
    out = []
    for j in range(k):
        m = (c >= edges[j]) & ((c < edges[j + 1]) if j < k - 1 else (c <= edges[j + 1]))
        out.append(Scene(f"{scene.name}-part{j}", scene.vertices[m], scene.geom_ids[m],
                         scene.texcoords[m], scene.geom_texture, scene.textures,
                         np.nonzero(m)[0]))
    return out


def concat_scenes(scenes: list) -> tuple:
    """One scene holding every sub-scene's triangles in list order (for brute force),
    plus the start offset of each sub-scene's triangles."""
    verts, gids, tcs, gtex, texs, offs = [], [], [], [], [], []
    g_off = t_off = n_off = 0
    for s in scenes:
        offs.append(n_off)
        verts.append(s.vertices)
        tcs.append(s.texcoords)
        gids.append(s.geom_ids.astype(np.uint64) + g_off)
        gtex.append(s.geom_texture.astype(np.uint64) + t_off)
        texs += list(s.textures)
        g_off += len(s.geom_texture)
        t_off += len(s.textures)
        n_off += s.num_tris
    sc = Scene("concat", np.concatenate(verts), np.concatenate(gids).astype(np.uint32),
               np.concatenate(tcs), np.concatenate(gtex).astype(np.uint32), texs)
    return sc, np.array(offs, dtype=np.int64)


CAMERAS = {
    # eye, look_at, up, vfov, width, height, spp
    "C2": ((0.0, 4.0, -280.0), (0.0, 4.0, 0.0), (0.0, 1.0, 0.0), 45.0, 1920, 1080, 1),
    "C3": ((0.0, 4.0, -280.0), (0.0, 4.0, 0.0), (0.0, 1.0, 0.0), 45.0, 1920, 1080, 1),
    "C4": ((0.0, 40.0, -300.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 45.0, 1920, 1080, 1),
    "C5": ((0.0, 60.0, -1100.0), (0.0, 10.0, 0.0), (0.0, 1.0, 0.0), 45.0, 3840, 2160, 4),
    "C2K": ((0.0, 4.0, -280.0), (0.0, 4.0, 0.0), (0.0, 1.0, 0.0), 45.0, 1920, 1080, 1),
}


def scene(name: str, textures=None) -> Scene:
    if name == "C1":
        return quad_pair_scene()
    if name in ("C2", "C3"):
        return forest_scene(textures=textures)
    if name == "C2K":
        return forest_scene(textures=textures if textures is not None else stress_textures())
    if name == "C4":
        return c4_scene(textures=textures)
    if name == "C5":
        return c5_scene(textures=textures)
    raise KeyError(name)


def rays_for(name: str, width: int | None = None, height: int | None = None,
             spp: int | None = None, shift_x: float = 0.0) -> Rays:
    """The config's primary rays; `shift_x` moves the camera sideways (per-rank frames)."""
    if name == "C1":
        return quad_pair_rays(width or 64)
    eye, look, up, fov, w, h, s = CAMERAS[name]
    eye = (eye[0] + shift_x, eye[1], eye[2])
    look = (look[0] + shift_x, look[1], look[2])
    return pinhole_rays(eye, look, up, fov, width or w, height or h, spp or s)


def config(name: str, width: int | None = None, height: int | None = None, spp: int | None = None,
           textures=None):
    """Return (scene, rays) for a named config; width/height/spp may be reduced for tests."""
    return scene(name, textures), rays_for(name, width, height, spp)
