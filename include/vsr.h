/*
 * vsr.h — C ABI of the B200-native custom-intersector ray tracing path.
 *
 * What it implements (PAPER.md = arXiv 1912.12786, "custom intersectors"):
 *   per-ray BVH traversal with ray–triangle intersection, where the
 *   intersector — the user code that may veto a hit (PAPER.md:140-184
 *   [§3.1 listings 2-3]) — is injected at COMPILE time into both call sites
 *   of the while-while traversal (PAPER.md:228-252 [§3.2 pseudocode]).
 *   Every (query, intersector) pair is its own kernel instantiation chosen
 *   once on the host, so the default path carries no device-side branch or
 *   function pointer: the paper's zero-cost claim.
 *
 * Conventions for every entry point:
 *   - all functions are extern "C", return a vsr_status, and never throw;
 *   - argument errors are detected synchronously and leave no side effect;
 *   - on error, vsr_last_error() returns a thread-local message that stays
 *     valid until the next vsr_* call on that thread;
 *   - distinct scenes may be used from distinct threads concurrently; a
 *     built scene is read-only and may be traced from several streams at
 *     once; building while tracing the same scene is not allowed.
 *
 * Layouts below are little-endian and part of the ABI (DESIGN.md §"Data
 * layout" documents each byte).
 */
#ifndef VSR_H
#define VSR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VSR_ABI_VERSION 2u   /* 2: slab contract r02, 8-wide BVH entry points */

typedef enum {
  VSR_OK = 0,
  VSR_ERR_INVALID_ARG = 1,  /* NULL handle/pointer, misaligned buffer, bad enum, bad size */
  VSR_ERR_EMPTY_SCENE = 2,  /* zero triangles, or every triangle degenerate */
  VSR_ERR_NONFINITE = 3,    /* NaN/Inf vertex or texcoord                    */
  VSR_ERR_BVH_TOO_DEEP = 4, /* traversal stack would exceed 64 entries      */
  VSR_ERR_NOT_BUILT = 5,    /* vsr_trace before vsr_bvh_build / vsr_scene_import         */
  VSR_ERR_CUDA = 6,         /* a CUDA runtime call failed; message in vsr_last_error()   */
  VSR_ERR_OOM = 7,          /* host or device allocation failed                          */
  VSR_ERR_UNSUPPORTED = 8   /* combination not provided (e.g. > 2^26 triangles)          */
} vsr_status;

/* Visibility queries: closest-hit = min-t accepted hit;
 * any-hit = the first accepted hit encountered during traversal. */
typedef enum { VSR_QUERY_CLOSEST = 0, VSR_QUERY_ANY = 1 } vsr_query;

/* Intersectors.  Each value selects a distinct compile-time instantiation.
 *   NONE              the default overload without an intersector argument
 *                     (PAPER.md:195-205): traversal calls intersect() directly.
 *   DEFAULT           basic_intersector with no override: every
 *                     hook forwards to intersect().  Compiles to the same SASS as NONE.
 *   ALPHA_TEXTURE     §4 alpha-mask listing: on a geometric hit,
 *                     look up textures[geom_texture[geom_id]] at lerp(uv0,uv1,uv2,u,v)
 *                     (nearest, wrap) and keep the hit iff alpha >= alpha_threshold.
 *                     A vetoed hit does not shrink tmax: traversal continues.
 *   ALPHA_PROCEDURAL  procedural mask: keep iff
 *                     floor(u*M) + floor(v*M) is even, M = checker_freq.
 *   COUNT             bvh_costs: ++num_boxes per box hook,
 *                     ++num_tris per triangle hook, default filter; writes d_counts.
 *   COUNT_ALPHA_TEXTURE  bvh_costs stacked on ALPHA_TEXTURE (the cost of the alpha
 *                     intersector's traversal; also counts alpha lookups).
 *   ALPHA_TEXTURE_BILINEAR  NEXT-4 variant (reading A28): as ALPHA_TEXTURE with a
 *                     bilinear filter (texel centres (i+.5)/W, wrap) and the filtered alpha
 *                     compared with alpha_threshold.
 *   ALPHA_PROCEDURAL_UV  NEXT-4 variant: the checker of ALPHA_PROCEDURAL evaluated on the
 *                     interpolated texcoords (s, t) instead of the barycentrics.
 *   RUNTIME_*         measurement controls for the zero-cost claim: the same
 *                     traversal with the filter chosen at RUN time inside the loop,
 *                     the Embree/OptiX style the paper contrasts with.
 *                     100+k: switch on kind k; 200+k: device function pointer with a
 *                     null check (k = DEFAULT means a null pointer). */
typedef enum {
  VSR_ISECT_NONE = 0,
  VSR_ISECT_DEFAULT = 1,
  VSR_ISECT_ALPHA_TEXTURE = 2,
  VSR_ISECT_ALPHA_PROCEDURAL = 3,
  VSR_ISECT_COUNT = 4,
  VSR_ISECT_COUNT_ALPHA_TEXTURE = 5,
  VSR_ISECT_ALPHA_TEXTURE_BILINEAR = 6,
  VSR_ISECT_ALPHA_PROCEDURAL_UV = 7,
  VSR_ISECT_RUNTIME_SWITCH_DEFAULT = 101,
  VSR_ISECT_RUNTIME_SWITCH_ALPHA_TEXTURE = 102,
  VSR_ISECT_RUNTIME_SWITCH_ALPHA_PROCEDURAL = 103,
  VSR_ISECT_RUNTIME_FNPTR_DEFAULT = 201,
  VSR_ISECT_RUNTIME_FNPTR_ALPHA_TEXTURE = 202,
  VSR_ISECT_RUNTIME_FNPTR_ALPHA_PROCEDURAL = 203
} vsr_isect;

/* 32 B, 16-B aligned.  t is in units of d (d need not be normalised);
 * the accepted interval is [tmin, tmax], inclusive. */
typedef struct { float ox, oy, oz, tmin, dx, dy, dz, tmax; } vsr_ray;

/* 16 B.  prim_id is the caller's triangle index (reordering is invisible).
 * Miss: prim_id = 0xFFFFFFFF, t = +inf, u = v = 0 (reading A24).
 * Barycentrics: hit point = v0 + u*(v1-v0) + v*(v2-v0). */
typedef struct { float t, u, v; uint32_t prim_id; } vsr_hit;
#define VSR_MISS 0xFFFFFFFFu

/* 16 B per ray, written by COUNT and COUNT_ALPHA_TEXTURE only. */
typedef struct { uint32_t num_boxes, num_tris, num_alpha, reserved; } vsr_counts;

/* Row-major RGBA8, row j holds texture coordinate t in [j/H, (j+1)/H). */
typedef struct { uint32_t width, height; const uint8_t* rgba8; } vsr_texture_desc;

typedef struct {
  uint32_t num_tris;
  const float* vertices;          /* host, 9 floats per triangle (v0, v1, v2); copied      */
  const uint32_t* geom_ids;       /* host, num_tris; NULL -> all 0                          */
  const float* texcoords;         /* host, 6 floats per triangle (uv0,uv1,uv2); NULL -> 0;
                                     |value| <= 1024                                        */
  uint32_t num_geoms;             /* size of geom_texture (ignored if geom_texture NULL)    */
  const uint32_t* geom_texture;   /* host, geom -> texture index; NULL -> identity          */
  uint32_t num_textures;          /* 0 -> one implicit 1x1 opaque white texture     */
  const vsr_texture_desc* textures; /* host; 1 <= width, height <= 65536                    */
  int device;                     /* CUDA ordinal that owns the device copies               */
} vsr_scene_desc;

/* Binned SAH parameters.  NULL -> {2, 16, 1.0, 1.0} (max_leaf 2 measured
 * fastest on C2 and C5; SPEC's CPU program uses 4; reading A22).
 * 1 <= max_leaf_size <= 32, 2 <= sah_bins <= 256. */
typedef struct {
  uint32_t max_leaf_size, sah_bins;
  float traversal_cost, intersection_cost;
} vsr_build_params;

/* NULL -> {0.01f, 8 (reading A4)}.  checker_freq >= 1. */
typedef struct { float alpha_threshold; uint32_t checker_freq; } vsr_isect_params;

typedef struct vsr_scene vsr_scene;

/* Flattened acceleration structure in the export layout:
 *   nodes    64 B each: float x[4], y[4], z[4]; uint32 ref[2]; uint32 pad[2], where axis
 *            k holds (lo0.k, lo1.k, hi0.k, hi1.k) — child 0 / child 1 slab planes side by
 *            side; every child box must be finite with lo <= hi
 *   tris     48 B each: float v0[3]; uint32 prim_id; float e1[3]; 0; float e2[3]; 0
 *   sides    32 B each: float uv0[2],uv1[2],uv2[2]; uint32 texel_offset (first texel of the
 *            triangle's texture in `texels`); uint32 dims = (W-1) | (H-1) << 16
 *   texdescs 16 B each: uint64 texel_offset; uint32 width, height
 *   texels    1 B each: the textures' alpha channel (A8), row-major, textures back to back;
 *            the mask intersector reads color.w only.  <= 2^32 texels
 * ref encoding: bit31 = leaf; leaf: bits 26..30 = count-1, bits 0..25 = first tri;
 * inner: node index.  root_ref may be a leaf (no nodes). */
typedef struct {
  uint32_t root_ref;
  float root_lo[3], root_hi[3];
  uint32_t num_nodes, num_tris, num_textures;
  uint64_t num_texels;
  void* nodes;
  void* tris;
  void* sides;
  void* texdescs;
  void* texels;
} vsr_bvh_view;

typedef struct {
  uint32_t num_tris_input, num_tris, num_degenerate;
  uint32_t num_nodes, num_leaves, max_depth, num_textures, built;
  uint64_t num_texels, device_bytes;
  double build_ms;
} vsr_stats;

/* Validate and copy a host scene description.  No device work.
 * Errors: INVALID_ARG (NULL desc/out, vertices NULL with num_tris > 0, geom or texture
 * index out of range, bad texture size, |texcoord| > 1024), NONFINITE, OOM. */
vsr_status vsr_scene_create(const vsr_scene_desc* desc, vsr_scene** out);

/* Build the BVH on the host (binned SAH), flatten it to the export
 * layout and upload everything to desc->device.  Synchronous; untimed setup.
 * Degenerate triangles (e1 x e2 == 0) are excluded and never hit.
 * Errors: INVALID_ARG, EMPTY_SCENE, BVH_TOO_DEEP, UNSUPPORTED, CUDA, OOM. */
vsr_status vsr_bvh_build(vsr_scene* scene, const vsr_build_params* params);

/* Build the BVH on the scene's GPU instead: a linear BVH (Karras,
 * HPG 2012 — 63-bit centroid Morton codes, device radix sort, one thread per internal node,
 * bottom-up boxes), subtrees of <= max_leaf_size (1..32) triangles collapsed into leaves.  Same
 * export layout, padding, degenerate rule and depth bound as vsr_bvh_build; lower tree quality
 * than binned SAH (slower traces), a much faster build.  Synchronous; untimed setup.
 * Errors: INVALID_ARG, EMPTY_SCENE, BVH_TOO_DEEP, UNSUPPORTED (host-only scene), CUDA, OOM. */
vsr_status vsr_bvh_build_gpu(vsr_scene* scene, uint32_t max_leaf_size);

/* The same GPU build with PLOC clustering (Meister & Bittner, TVCG 2018) instead of Karras
 * splits: on the Morton-sorted triangles, every cluster pairs with its nearest neighbour
 * (smallest union surface area, ties to the lower position) within +-radius (1..256; 16 is
 * typical) and mutual pairs merge, round after round — trees close to binned SAH in quality at
 * GPU build speed.  Same layout, rules and errors as vsr_bvh_build_gpu. */
vsr_status vsr_bvh_build_ploc(vsr_scene* scene, uint32_t max_leaf_size, uint32_t radius);

/* 8-WIDE COMPRESSED BVH (SURVEY.md §8(f) NEXT-3 "wide / compressed BVH (8-wide quantized
 * nodes)"; Ylitie, Karras & Laine, HPG 2017).  Collapses the scene's built binary BVH (any
 * builder; leaves of at most 4 triangles) into 80-B nodes of up to 8 children whose boxes are
 * quantized to 8 bits per plane on a per-node grid: plane(q) = fma(2^23 + q, 2^(e-127), pm),
 * the codes chosen so every decoded child box contains the binary child box.
 * Children are visited in slot order s ^ octant(ray); the box hook of a wide node counts one box
 * test per valid child (COUNT: num_boxes = 1 root + the valid children of every visited node).
 * The triangles / sidecars are reordered for the wide leaves (prim ids unchanged).  Synchronous,
 * untimed; kept until the binary BVH is rebuilt or the scene destroyed; works for host-only
 * scenes (device -1: exportable, not traceable) and imported scenes.  Errors: INVALID_ARG,
 * NOT_BUILT, UNSUPPORTED (a leaf with > 4 triangles), BVH_TOO_DEEP, CUDA, OOM. */
vsr_status vsr_bvh8_build(vsr_scene* scene);

/* Host copies of the wide BVH.  Two calls: first with NULL arrays (sizes filled), then with
 * caller-owned host arrays of num_nodes x 80 B (wide.hpp WideNode: pm[3] f32, e[3] u8, imask
 * u8, child_base u32, tri_base u32, meta[8] u8, qlo[3][8] u8, qhi[3][8] u8), num_tris x 48 B
 * triangles and num_tris x 32 B sidecars (the binary export layouts, in the wide leaf order).
 * Root box = the binary root box (tested once, counted).  Errors: INVALID_ARG, NOT_BUILT. */
typedef struct {
  uint32_t num_nodes, num_tris, max_depth, pad;
  float root_lo[3], root_hi[3];
  double build_ms;
  void* nodes;
  void* tris;
  void* sides;
} vsr_bvh8_view;
vsr_status vsr_bvh8_export(const vsr_scene* scene, vsr_bvh8_view* out);

/* vsr_trace over the wide BVH: same arguments, semantics, asynchrony and results (hits are
 * those of vsr_trace up to exact-t ties; the BVH only prunes); counts follow the wide
 * traversal.  Intersectors: every kind except the run-time controls (>= 100: UNSUPPORTED).
 * Errors: INVALID_ARG, NOT_BUILT (no wide BVH: call vsr_bvh8_build), UNSUPPORTED, CUDA. */
vsr_status vsr_trace_bvh8(vsr_scene* scene, const vsr_ray* d_rays, uint64_t n, vsr_query query,
                          vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                          vsr_counts* d_counts, void* stream);

/* Enqueue one trace of n rays on `stream` (a cudaStream_t; NULL = legacy default).
 * d_rays / d_hits / d_counts are caller-owned DEVICE buffers on the scene's device,
 * 16-B aligned.  d_counts is required iff isect is COUNT or COUNT_ALPHA_TEXTURE.
 * Asynchronous: results are valid once the stream is synchronised.  n = 0 is a
 * no-op.  Errors: INVALID_ARG, NOT_BUILT, CUDA (launch failure).
 * CUDA graphs: the call may be captured (stream capture) and the graph replayed; a captured
 * call takes its order-pass scratch as graph memory nodes (stream-ordered allocation), and
 * ALPHA_TEXTURE uses the scene's 1-bit alpha plane only if one call with the same threshold ran
 * before capture (otherwise the A8 path is captured; same results).  The same holds for
 * vsr_trace_multi, vsr_trace_pinhole, vsr_trace_tiles and the list / instance traces;
 * vsr_trace_host synchronises and cannot be captured. */
vsr_status vsr_trace(vsr_scene* scene, const vsr_ray* d_rays, uint64_t n, vsr_query query,
                     vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                     vsr_counts* d_counts, void* stream);

/* Query on the scene's triangles as a plain LIST, without the BVH ("the user
 * might decide that a BVH is not required and just pass iterators to a linear list of primitives
 * to the query routines"; the intersector then replaces the primitive test inside the loop).
 * Every ray tests every triangle in caller order (degenerate ones excluded, as by the build):
 * closest keeps the lowest index among equal t, any-hit returns the lowest accepted index — the
 * brute-force definition.  O(rays x triangles): for small scenes and as the BVH's reference.
 * COUNT kinds count triangle tests (num_boxes = 0).  Other arguments as vsr_trace; RUNTIME_*
 * controls: VSR_ERR_UNSUPPORTED. */
vsr_status vsr_trace_primitives(vsr_scene* scene, const vsr_ray* d_rays, uint64_t n,
                                vsr_query query, vsr_isect isect, const vsr_isect_params* params,
                                vsr_hit* d_hits, vsr_counts* d_counts, void* stream);

/* Primary rays generated INSIDE the trace kernel (SURVEY.md §8(f) NEXT-4 "fused camera ray
 * generator": no ray buffer, no 32 B/ray read).  Ray i is the i-th of the input recipe's
 * (8x8 tile, sample, y, x) order and is bit-identical to the host recipe:
 *   px, py = pixel, s = sample; spp = 1: (jx, jy) = (0.5, 0.5); spp = k*k: jx = ((s % k) + r1)/k,
 *   jy = ((s / k) + r2)/k, r1,2 = pcg_hash32((key*2 [+1] + 7919*jitter_seed) mod 2^32) / 2^32,
 *   key = (py*width + px)*spp + s;  sx = 2(px + jx)/width - 1,  sy = 1 - 2(py + jy)/height;
 *   d = fp32((w + (sx*tan_half_vfov*aspect) u) + (sy*tan_half_vfov) v)   [fp64, this order],
 *   o = fp32(eye), [tmin, tmax] as given.
 * w, u, v: the camera's forward / right / up unit vectors in fp64 (vsr.py pinhole_camera).
 * n = width*height*spp rays; d_hits / d_counts in ray order as vsr_trace.  Not provided for the
 * RUNTIME_* controls.  Errors: INVALID_ARG (NULL, width/height not multiples of 8, spp not a
 * square, non-finite camera, more than 2^31 blocks), NOT_BUILT, UNSUPPORTED, CUDA. */
typedef struct {
  double eye[3];
  double w[3], u[3], v[3];
  double tan_half_vfov, aspect;
  uint32_t width, height, spp, jitter_seed;
  float tmin, tmax;
} vsr_pinhole;
vsr_status vsr_trace_pinhole(vsr_scene* scene, const vsr_pinhole* camera, vsr_query query,
                             vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                             vsr_counts* d_counts, void* stream);

/* Multi-hit query ("the first N hit points"): per ray the
 * max_hits (1..16) smallest-t ACCEPTED hits in ascending t (equal t: the order traversal found
 * them).  Once max_hits hits are held, tmax shrinks to the worst kept t.
 * d_hits: n*max_hits vsr_hit, ray-major (ray i's j-th hit at i*max_hits+j); unused slots hold
 * the miss record.  d_num_hits: optional, n uint32 (hits kept).  d_counts as in vsr_trace.
 * The RUNTIME_* controls are not provided for this query (VSR_ERR_UNSUPPORTED). */
vsr_status vsr_trace_multi(vsr_scene* scene, const vsr_ray* d_rays, uint64_t n, uint32_t max_hits,
                           vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                           uint32_t* d_num_hits, vsr_counts* d_counts, void* stream);

/* A LIST of built scenes queried as one (BVHs act as compound primitives,
 * the object hierarchy "may optionally have more than one root node", and the intersector is
 * passed on into every BVH's traversal).  Untransformed (no instance matrices).  All scenes on
 * one device; they must stay alive and unmodified while the group exists.  1 <= count <= 1024.
 * Errors: INVALID_ARG (NULL, count, mixed devices), NOT_BUILT, UNSUPPORTED (host-only), CUDA, OOM. */
typedef struct vsr_group vsr_group;
vsr_status vsr_group_create(vsr_scene* const* scenes, uint32_t count, vsr_group** out);
vsr_status vsr_group_destroy(vsr_group* group);   /* NULL is a no-op */

/* Trace the list in order with one running best_t: closest = the min-t accepted hit over all
 * elements (equal t: the earlier element); any = the first accepted hit (list order).  Each
 * element's root box is tested and counted (counts are summed over the list).
 * prim_id in d_hits is the index within the hit's own scene; d_which (optional, n uint32) gets
 * that scene's list index (0xFFFFFFFF on a miss).  Other arguments as vsr_trace; the
 * RUNTIME_* controls are not provided (VSR_ERR_UNSUPPORTED). */
vsr_status vsr_trace_group(vsr_group* group, const vsr_ray* d_rays, uint64_t n, vsr_query query,
                           vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                           uint32_t* d_which, vsr_counts* d_counts, void* stream);

/* Two-level INSTANCING ("object instancing, where the BVH will store BVHs as
 * primitives"): a top-level BVH (binned SAH, built here, untimed) over instances, each showing
 * one built scene through an affine map.  A ray reaching an instance in the top-level traversal
 * is mapped into the instance's object space and traverses that scene's BVH with the same
 * intersector and the same running best_t (closest: min t over all instances; any: the first
 * accepted hit in traversal order).
 *
 * vsr_instance.object_from_world: row-major 3x4 [A | b] taking WORLD points to OBJECT points,
 * p_obj = A p + b.  The ray maps, in fp32 in exactly this order (reading A27):
 *   o'_i = ((A_i0*o_x + A_i1*o_y) + A_i2*o_z) + b_i,   d'_i = (A_i0*d_x + A_i1*d_y) + A_i2*d_z,
 * tmin and tmax unchanged, so t is the same parameter in both spaces.  A must be finite and
 * invertible (|det A| > 1e-30 in fp64).  Instance world boxes: the scene's padded root box mapped
 * by the fp64 inverse, then padded outward by 2^-10 of (box diagonal + max |coordinate|).
 * That pad covers the fp32 ray map's error for ray origins up to a bound r_safe derived per
 * instance from |A|, |A^-1|, |b| and the box (reading A27; thousands of scene
 * diagonals for well-conditioned maps); a ray with max_k |o_k| > r_safe skips the top-level
 * BVH and visits every instance in leaf order (the definition itself: conservative at any
 * distance, slower only for such rays).  Counts: top root 1, then per instance as below.
 * Scenes: built, one device, alive and unmodified while the object exists; 1..1024 scenes,
 * 1..2^26 instances.  Host-only scenes (device -1) give host-only instances: built and
 * exportable, not traceable.  params: top-level build (NULL = {1, 16, 1, 1}; max_leaf_size
 * 1..32).  Errors: INVALID_ARG (NULL, counts, bvh index, non-finite or singular matrix, mixed
 * devices, bad params), NOT_BUILT, BVH_TOO_DEEP, CUDA, OOM. */
typedef struct {
  uint32_t bvh;                  /* index into the scenes array */
  float object_from_world[12];   /* [A | b], row-major */
} vsr_instance;
typedef struct vsr_instances vsr_instances;
vsr_status vsr_instances_create(vsr_scene* const* scenes, uint32_t num_scenes,
                                const vsr_instance* instances, uint32_t num_instances,
                                const vsr_build_params* params, vsr_instances** out);
vsr_status vsr_instances_destroy(vsr_instances* inst);   /* NULL is a no-op */

/* Trace rays against the instanced hierarchy.  Counting (COUNT*): the top-level root box once,
 * 2 per top-level inner node, then per instance reached its scene's root box (1), 2 per inner
 * node and 1 per triangle, as in vsr_trace.  prim_id in d_hits is the index within the hit's
 * scene; d_inst (optional, n uint32, 4-B aligned) gets the caller's instance index (0xFFFFFFFF
 * on a miss).  Other arguments as vsr_trace; RUNTIME_* controls and host-only instances:
 * VSR_ERR_UNSUPPORTED. */
vsr_status vsr_trace_instances(vsr_instances* inst, const vsr_ray* d_rays, uint64_t n,
                               vsr_query query, vsr_isect isect, const vsr_isect_params* params,
                               vsr_hit* d_hits, uint32_t* d_inst, vsr_counts* d_counts,
                               void* stream);

/* The built top level, for checking (host copies; NULL pointers: sizes only).
 * nodes: num_nodes x 64 B pair nodes (export layout, leaf refs index `records`);
 * records: num_instances x 64 B in leaf order: float object_from_world[12], uint32 bvh,
 * uint32 instance index (the caller's), uint32 pad[2]. */
typedef struct {
  uint32_t root_ref;
  float root_lo[3], root_hi[3];
  uint32_t num_nodes, num_instances, max_depth;
  float r_safe;   /* rays with max_k |o_k| > r_safe skip the top level (see vsr_trace_instances) */
  void* nodes;
  void* records;
} vsr_instances_view;
vsr_status vsr_instances_export(const vsr_instances* inst, vsr_instances_view* view);

/* Multi-GPU frame assembly fused into the trace: this rank traces its
 * round-robin tile shard — its j-th tile is frame tile j*world + rank, tile_rays rays per tile,
 * n = its ray count (a multiple of tile_rays, n < 2^32) — and the kernel stores every hit (and
 * count) straight to that ray's FRAME position in d_frame_hits / d_frame_counts.  Those are
 * normally rank 0's frame buffers opened in this process with vsr_ipc_open, so the stores travel
 * over NVLink / NVSwitch inside the trace kernel and no gather collective runs.  The frame is
 * complete once every rank's stream has passed the call (the caller synchronises: stream sync +
 * barrier).  Other arguments and errors as vsr_trace. */
vsr_status vsr_trace_tiles(vsr_scene* scene, const vsr_ray* d_rays, uint64_t n, uint32_t tile_rays,
                           uint32_t rank, uint32_t world, vsr_query query, vsr_isect isect,
                           const vsr_isect_params* params, vsr_hit* d_frame_hits,
                           vsr_counts* d_frame_counts, void* stream);

/* Device buffers that other processes can map (CUDA IPC).  vsr_device_alloc: cudaMalloc on
 * `device` (the pointer is an allocation base, as IPC requires); vsr_ipc_handle: its 64-byte
 * handle; vsr_ipc_open: map a handle from another process on this process's `device` (peer
 * access enabled lazily); vsr_ipc_close / vsr_device_free undo them.  Errors: INVALID_ARG, CUDA. */
vsr_status vsr_device_alloc(uint64_t bytes, int device, void** d_ptr);
vsr_status vsr_device_free(void* d_ptr, int device);
vsr_status vsr_ipc_handle(const void* d_ptr, void* handle64);
vsr_status vsr_ipc_open(const void* handle64, int device, void** d_ptr);
vsr_status vsr_ipc_close(void* d_ptr, int device);

/* Multi-hit query over a list of BVHs / over instances (closest_hit, any_hit
 * and multi_hit iterate over lists whose elements may be BVHs): one buffer of the max_hits
 * (1..16) smallest-t accepted hits across all elements, in ascending t (equal t: the order
 * traversal found them), with the group's single running best_t (the worst kept t once full).
 * d_hits: n*max_hits ray-major as vsr_trace_multi; d_num_hits (optional): n; d_which / d_inst
 * (optional): n*max_hits, the list index / caller's instance index of each kept hit
 * (0xFFFFFFFF in unused slots).  Counting as vsr_trace_group / vsr_trace_instances.
 * RUNTIME_* controls: VSR_ERR_UNSUPPORTED. */
vsr_status vsr_trace_group_multi(vsr_group* group, const vsr_ray* d_rays, uint64_t n,
                                 uint32_t max_hits, vsr_isect isect,
                                 const vsr_isect_params* params, vsr_hit* d_hits,
                                 uint32_t* d_num_hits, uint32_t* d_which, vsr_counts* d_counts,
                                 void* stream);
vsr_status vsr_trace_instances_multi(vsr_instances* inst, const vsr_ray* d_rays, uint64_t n,
                                     uint32_t max_hits, vsr_isect isect,
                                     const vsr_isect_params* params, vsr_hit* d_hits,
                                     uint32_t* d_num_hits, uint32_t* d_inst,
                                     vsr_counts* d_counts, void* stream);

/* End-to-end variant over HOST buffers (pinned memory recommended): copies rays in,
 * traces, copies hits (and counts) out, all on `stream`, in chunks so that copies
 * overlap the kernel; returns after the stream work completed. */
vsr_status vsr_trace_host(vsr_scene* scene, const vsr_ray* h_rays, uint64_t n,
                          vsr_query query, vsr_isect isect, const vsr_isect_params* params,
                          vsr_hit* h_hits, vsr_counts* h_counts, void* stream);

/* Free a scene and all its device memory.  NULL is a no-op. */
vsr_status vsr_destroy(vsr_scene* scene);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* vsr_last_error(void);

/* Sizes (all pointers NULL in *view) or copies (non-NULL pointers, host or device,
 * cudaMemcpyDefault) of the built structure in the export layout. */
vsr_status vsr_bvh_export(const vsr_scene* scene, vsr_bvh_view* view);

/* Create a built scene on `device` directly from export-layout buffers (host or
 * device pointers), e.g. after a broadcast.  The structure is validated: every
 * ref in range, every triangle referenced by exactly one leaf, depth <= 64,
 * texture indices and texel ranges in bounds.
 * Errors: INVALID_ARG (malformed), BVH_TOO_DEEP, CUDA, OOM. */
vsr_status vsr_scene_import(const vsr_bvh_view* view, int device, vsr_scene** out);

vsr_status vsr_scene_stats(const vsr_scene* scene, vsr_stats* out);

/* Profiling hook: on this thread, subsequent traces record `start` right before and
 * `stop` right after the trace kernel itself (cudaEvent_t handles created by the caller on
 * the scene's device; NULL, NULL disables).  The block-order pass runs before `start`. */
vsr_status vsr_set_kernel_events(void* start, void* stop);

/* Number of kernels this library has launched in this process (all scenes). */
uint64_t vsr_launch_count(void);

uint32_t vsr_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VSR_H */
