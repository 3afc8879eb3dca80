/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU oracle for the custom-intersector
 * hot path of arXiv 1912.12786 (PAPER.md = /root/reference/PAPER.md).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the product (paper_1912_12786_b200/, include/):
 * every struct below is re-declared here from the documented layouts in
 * DESIGN.md, never included from the product.
 *
 * Three parts:
 *   oracle S  (oracle.c)  brute force over every triangle in caller order —
 *             the plain definition the BVH method must reach exactly
 *             (PAPER.md:185-190 queries, :228-252 traversal only prunes).
 *   oracle BVH (walker.c) a simple object-median BVH written in the export
 *             layout, so count parity never needs an input from the product.
 *   walker C  (walker.c)  the traversal contract of DESIGN.md §"Arithmetic
 *             contract" over an exported/imported BVH;
 *             the oracle for the counting intersector.
 *
 * Arithmetic: IEEE fp32 (the paper's listings use basic_triangle<3,float>
 * and the literal .01f), compiled with
 * -ffp-contract=off -fno-fast-math so no FMA contraction happens.
 */
#ifndef VSR_ORACLE_H
#define VSR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* query kinds */
enum { OR_CLOSEST = 0, OR_ANY = 1 };
/* intersector kinds (PAPER.md:195-219 default overload vs intersector;
   §4 listings: alpha texture :296-316, procedural :319-322, bvh_costs :332-366) */
enum { OR_NONE = 0, OR_DEFAULT = 1, OR_ALPHA_TEX = 2, OR_ALPHA_PROC = 3, OR_COUNT = 4,
       /* NEXT-4 sampling variants (reading A28): bilinear alpha, and the
          procedural checker on the interpolated texcoords instead of (u, v) */
       OR_ALPHA_BILIN = 5, OR_ALPHA_PROC_UV = 6 };

/* ambiguity flags (SURVEY.md §8(c) exclusion classes), computed in double */
enum { OR_X1_NEAR_TIE = 1u, OR_X2_EDGE_GRAZE = 2u, OR_X3_TEXEL_EDGE = 4u,
       OR_X4_CHECKER_EDGE = 8u, OR_X5_ALPHA_NEAR = 16u /* bilinear alpha within 1e-4 of thr */ };

typedef struct {
  uint32_t num_tris;
  const float* vertices;       /* 9 floats per triangle: v0, v1, v2          */
  const uint32_t* geom_ids;    /* num_tris                                    */
  const float* texcoords;      /* 6 floats per triangle: uv0, uv1, uv2        */
  uint32_t num_geoms;
  const uint32_t* geom_texture;/* geom_id -> texture index                    */
  uint32_t num_textures;
  const uint32_t* tex_w;       /* per texture width                           */
  const uint32_t* tex_h;       /* per texture height                          */
  const uint8_t* const* tex_rgba; /* per texture row-major RGBA8, row j = t-row j */
} or_scene;

typedef struct { float t, u, v; uint32_t prim; } or_hit;       /* 16 B */
typedef struct { uint32_t boxes, tris, alpha; } or_counts;      /* walker */

/* Brute-force oracle S.  rays: 8 floats each (o.xyz, tmin, d.xyz, tmax).
 * flags may be NULL (no double shadow).  ntie may be NULL; else receives the
 * number of accepted candidates whose t equals the winner's t exactly.
 * Returns 0 on success. */
int oracle_trace(const or_scene* s, const float* rays, uint64_t n, int query, int isect,
                 float alpha_threshold, uint32_t checker_freq, or_hit* hits,
                 uint32_t* flags, uint32_t* ntie, int nthreads);

/* Multi-hit query by brute force: the K smallest-t accepted hits per ray, ascending t,
 * equal t by caller index; hits has n*K records (miss record in unused slots).
 * nhits (optional): hits kept per ray; ncut (optional): number of accepted candidates
 * whose t equals the K-th kept t when more than K were accepted (0 otherwise). */
int oracle_trace_multi(const or_scene* s, const float* rays, uint64_t n, uint32_t K, int isect,
                       float alpha_threshold, uint32_t checker_freq, or_hit* hits,
                       uint32_t* nhits, uint32_t* ncut, int nthreads);

/* One ray against one triangle (caller index) with the intersector's filter.
 * Returns 1 iff accepted (geometric hit and filter); fills *out either way
 * with the geometric t,u,v. */
int oracle_eval_pair(const or_scene* s, const float* ray, uint32_t prim, int isect,
                     float alpha_threshold, uint32_t checker_freq, or_hit* out);
/* Batch form: accepted flags and (t, u, v, prim) of n (ray, caller-indexed prim)
 * pairs; -1 on a NULL argument or a prim out of range. */
int oracle_eval_pairs(const or_scene* s, const float* rays, const uint32_t* prims, uint64_t n,
                      int isect, float thr, uint32_t M, uint8_t* acc, or_hit* out);

/* Individual textbook pieces, exposed for the closed-form pins. */
int oracle_mt(const float* ray, const float* v0, const float* v1, const float* v2,
              float tmax_cur, float* t, float* u, float* v);
float oracle_tex_alpha(uint32_t w, uint32_t h, const uint8_t* rgba, float s, float t);
/* Bilinear tex2D (reading A28): texel centres at (i+.5)/W, wrap; x = s*W - 0.5f,
 * i0 = floor(x), fx = x - i0 (same for y); alpha = ((1-fx)*a00 + fx*a10)*(1-fy) +
 * ((1-fx)*a01 + fx*a11)*fy with a = a8/255.0f, fp32 in exactly this order. */
float oracle_tex_alpha_bilinear(uint32_t w, uint32_t h, const uint8_t* rgba, float s, float t);
void oracle_lerp2(const float* a, const float* b, const float* c, float u, float v,
                  float* out);

/* ---------------- export layout (re-declared from DESIGN.md) -------------- */
typedef struct {          /* 64 B pair node; per axis k: lo0.k, lo1.k, hi0.k, hi1.k */
  float x[4], y[4], z[4];
  uint32_t ref[2];
  uint32_t pad[2];
} or_node;
typedef struct {          /* 48 B triangle: v0, prim_id, e1, 0, e2, 0 */
  float v0[3]; uint32_t prim;
  float e1[3]; uint32_t pad1;
  float e2[3]; uint32_t pad2;
} or_tri;
typedef struct {          /* 32 B sidecar: texcoords, texture's first texel, (W-1)|(H-1)<<16 */
  float uv[6]; uint32_t offset; uint32_t dims;
} or_side;
typedef struct {          /* 16 B texture descriptor */
  uint64_t offset; uint32_t w, h;
} or_texdesc;

typedef struct {
  uint32_t root_ref;
  float root_lo[3], root_hi[3];
  uint32_t num_nodes, num_tris, num_textures;
  const or_node* nodes;
  const or_tri* tris;
  const or_side* sides;
  const or_texdesc* texdescs;
  const uint8_t* texels;    /* alpha plane (A8), textures back to back */
} or_bvh;

/* Oracle-side BVH builder: object-median split on the widest centroid axis,
 * leaves of <= max_leaf triangles, written in the export layout.
 * Output arrays are malloc'd and owned by the caller (or_bvh_free).
 * Degenerate triangles (e1 x e2 == 0 exactly) are left out. */
int oracle_build_bvh(const or_scene* s, uint32_t max_leaf, or_bvh* out);
void oracle_bvh_free(or_bvh* b);

/* Contract walker C: traversal of SURVEY.md App. A.2 over `b`.
 * hits required; counts may be NULL.  Returns 0 on success, -1 on
 * stack overflow (depth > 64) or a malformed reference. */
int walker_trace(const or_bvh* b, const float* rays, uint64_t n, int query, int isect,
                 float alpha_threshold, uint32_t checker_freq, or_hit* hits,
                 or_counts* counts, int nthreads);

/* Walker C for the multi-hit query (GPU acceptance rule: stable insertion by t,
 * a full buffer only takes t < its worst, tmax shrinks to the worst once full). */
int walker_trace_multi(const or_bvh* b, const float* rays, uint64_t n, uint32_t K, int isect,
                       float alpha_threshold, uint32_t checker_freq, or_hit* hits,
                       uint32_t* nhits, or_counts* counts, int nthreads);

/* Walker C for a LIST of BVHs: walked in order with one running best_t;
 * every element's root box is tested and counted; which (optional) gets the list index of
 * the kept hit (0xFFFFFFFF on a miss); prims are indices within their own BVH. */
int walker_trace_list(const or_bvh* list, uint32_t nlist, const float* rays, uint64_t n,
                      int query, int isect, float alpha_threshold, uint32_t checker_freq,
                      or_hit* hits, uint32_t* which, or_counts* counts, int nthreads);

/* Two-level instancing ("the BVH will store BVHs as primitives"):
 * a top-level BVH whose leaves index `recs` (64 B records: float m[12] = [A | b]
 * object_from_world row-major, uint32 bvh, uint32 caller index, 2 x pad).  Walker C
 * for it: the top level is walked like any BVH (root box counted once, 2 box tests per
 * inner node); at a top-level leaf each instance, in stored order, maps the ray to
 * object space (reading A27: o'_i = ((A_i0 o_x + A_i1 o_y) + A_i2 o_z) + b_i, d'_i =
 * (A_i0 d_x + A_i1 d_y) + A_i2 d_z, fp32, no FMA) and walks bottoms[bvh] from its root
 * box (counted) with the one running best_t.  inst (optional) gets the caller index of
 * the kept hit (0xFFFFFFFF on a miss).  top->num_tris = number of records. */
typedef struct {
  float m[12]; uint32_t bvh, index, pad[2];
} or_instance;
/* 8-wide compressed BVH, re-declared from the
 * documented 80-B layout: per axis k a decode origin pm[k] and scale exponent field e[k]
 * (scale = the float with exponent field e[k], mantissa 0); imask bit s = slot s is an inner
 * child; inner children of a node are nodes child_base + (rank of s among the inner slots);
 * meta[s] = 0xFF empty, 0x80 inner, else leaf: triangles tri_base + (meta & 31), count
 * (meta >> 5) + 1; child box planes plane(q) = fmaf(2^23 + q, scale, pm) of the codes
 * qlo[k][s], qhi[k][s]. */
typedef struct {
  float pm[3]; uint8_t e[3]; uint8_t imask;
  uint32_t child_base, tri_base;
  uint8_t meta[8];
  uint8_t qlo[3][8], qhi[3][8];
} or_wnode;

/* Walker over the wide BVH: the root box of `b` (tested once, counted), then from node 0:
 * test every valid child (counted, one box each), the triangles of hit leaf children in key
 * order (key of slot s = s XOR the ray octant, ascending; octant bit k = sign bit of inv_k),
 * then descend into the hit inner child of smallest key and keep the rest as a pending group;
 * when a group member is popped, a closest-hit query re-tests its decoded box against the
 * current best_t (one counted box test) and skips it on a miss — an any-hit query (best_t never
 * shrinks before it ends) visits it directly.  b->tris /
 * b->sides must be the wide leaf order; b->nodes is unused.  Closest / any only. */
int walker_trace_wide(const or_bvh* b, const or_wnode* nodes, uint32_t num_nodes,
                      const float* rays, uint64_t n, int query, int isect, float alpha_threshold,
                      uint32_t checker_freq, or_hit* hits, or_counts* counts, int nthreads);

/* r_safe (reading A27, round 2): a ray whose origin has max_k |o_k| > r_safe (fp32
 * compare) tests the top root box (counted) and then visits EVERY instance record in leaf
 * order instead of walking the top level — the product exports the bound it traces with
 * (vsr_instances_view.r_safe); INFINITY = always the top level. */
int walker_trace_instances(const or_bvh* top, const or_instance* recs, const or_bvh* bottoms,
                           uint32_t nbottoms, const float* rays, uint64_t n, int query,
                           int isect, float alpha_threshold, uint32_t checker_freq,
                           or_hit* hits, uint32_t* inst, or_counts* counts, float r_safe,
                           int nthreads);

/* Multi-hit over a list of BVHs / over instances: one K-entry buffer across
 * all elements (walk_one's acceptance rule), which / inst get K entries per ray: the list index /
 * caller instance index of each kept hit (0xFFFFFFFF in unused slots); nhits may be NULL. */
int walker_trace_list_multi(const or_bvh* list, uint32_t nlist, const float* rays, uint64_t n,
                            uint32_t K, int isect, float alpha_threshold, uint32_t checker_freq,
                            or_hit* hits, uint32_t* nhits, uint32_t* which, or_counts* counts,
                            int nthreads);
int walker_trace_instances_multi(const or_bvh* top, const or_instance* recs,
                                 const or_bvh* bottoms, uint32_t nbottoms, const float* rays,
                                 uint64_t n, int query, uint32_t K, int isect,
                                 float alpha_threshold, uint32_t checker_freq, or_hit* hits,
                                 uint32_t* nhits, uint32_t* inst, or_counts* counts, float r_safe,
                                 int nthreads);

/* The ray map of reading A27 on its own (pins): out = 8 floats (o', tmin, d', tmax). */
void oracle_ray_to_object(const float* m, const float* ray, float* out);

/* Slab test of the walker (exposed for pins). Returns box hit; *tn entry
 * clipped to tmin, *tf exit times (1+2*gamma_3) before the best_t clip. */
int walker_slab(const float* lo, const float* hi, const float* ray, float best_t, float* tn,
                float* tf);

#ifdef __cplusplus
}
#endif
#endif
