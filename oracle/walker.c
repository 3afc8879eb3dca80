/*
 * walker.c — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * (1) oracle_build_bvh: a deliberately simple object-median BVH, written in
 *     the documented export layout (DESIGN.md §"Data layout"), so that the
 *     GPU's counting intersector can be checked on a tree the product did not
 *     build.  Any valid BVH prunes exactly: the tree shape
 *     changes counts, never accepted hits.
 * (2) walker_trace: contract walker C — the while-while traversal of
 *     PAPER.md:228-247 [§3.2 pseudocode] with both `intersect` call sites
 *     (box and primitive) routed through the intersector,
 *     under the pinned arithmetic of DESIGN.md §"Arithmetic contract"
 *     (SURVEY.md App. A.2).  It is the oracle for the bvh_costs counting
 *     intersector ("++num_boxes", "++num_tris").
 *
 * Counting rule (reading A11/A12 in DESIGN.md): the root
 * box is tested once before the loop and counted; each inner node visited
 * costs 2 box tests (both children); every triangle hook call counts 1.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define LEAF_BIT 0x80000000u
#define MAX_STACK 64

/* ====================== oracle BVH builder ================================ */
typedef struct {
  const or_scene* s;
  uint32_t max_leaf;
  uint32_t* idx;       /* triangle indices being partitioned */
  float* cen;          /* 3 centroids per triangle (double-free: float) */
  or_node* nodes;
  uint32_t num_nodes, cap_nodes;
  uint32_t* leaf_order; /* output triangle order */
  uint32_t num_out;
  int axis_sort;
  int depth_max;
} bld_t;

static bld_t* g_bld; /* qsort context (builder is single-threaded) */

static int cmp_axis(const void* a, const void* b) {
  uint32_t ia = *(const uint32_t*)a, ib = *(const uint32_t*)b;
  float ca = g_bld->cen[ia * 3 + g_bld->axis_sort], cb = g_bld->cen[ib * 3 + g_bld->axis_sort];
  if (ca < cb) return -1;
  if (ca > cb) return 1;
  return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

static void tri_bounds(const float* vt, float* lo, float* hi) {
  for (int k = 0; k < 3; ++k) {
    float a = vt[k], b = vt[3 + k], c = vt[6 + k];
    float mn = a < b ? a : b; mn = mn < c ? mn : c;
    float mx = a > b ? a : b; mx = mx > c ? mx : c;
    lo[k] = mn; hi[k] = mx;
  }
}

static void range_bounds(const bld_t* b, uint32_t beg, uint32_t end, float* lo, float* hi) {
  lo[0] = lo[1] = lo[2] = INFINITY;
  hi[0] = hi[1] = hi[2] = -INFINITY;
  for (uint32_t k = beg; k < end; ++k) {
    float tl[3], th[3];
    tri_bounds(b->s->vertices + (size_t)b->idx[k] * 9, tl, th);
    for (int a = 0; a < 3; ++a) {
      if (tl[a] < lo[a]) lo[a] = tl[a];
      if (th[a] > hi[a]) hi[a] = th[a];
    }
  }
}

/* outward padding 2^-20 * max(1,|x|), rounded outward to float */
static void pad_box(float* lo, float* hi) {
  for (int a = 0; a < 3; ++a) {
    double l = lo[a], h = hi[a];
    double pl = ldexp(fabs(l) > 1.0 ? fabs(l) : 1.0, -20);
    double ph = ldexp(fabs(h) > 1.0 ? fabs(h) : 1.0, -20);
    double ld = l - pl, hd = h + ph;
    float lf = (float)ld, hf = (float)hd;
    if ((double)lf > ld) lf = nextafterf(lf, -INFINITY);
    if ((double)hf < hd) hf = nextafterf(hf, INFINITY);
    lo[a] = lf; hi[a] = hf;
  }
}

/* export layout: per axis k the node stores (lo0.k, lo1.k, hi0.k, hi1.k) */
static void put_child_box(or_node* nd, int c, const float* lo, const float* hi) {
  float* ax[3] = {nd->x, nd->y, nd->z};
  for (int a = 0; a < 3; ++a) {
    ax[a][c] = lo[a];
    ax[a][2 + c] = hi[a];
  }
}
static void get_child_box(const or_node* nd, int c, float* lo, float* hi) {
  const float* ax[3] = {nd->x, nd->y, nd->z};
  for (int a = 0; a < 3; ++a) {
    lo[a] = ax[a][c];
    hi[a] = ax[a][2 + c];
  }
}

static uint32_t emit_leaf(bld_t* b, uint32_t beg, uint32_t end) {
  uint32_t first = b->num_out;
  for (uint32_t k = beg; k < end; ++k) b->leaf_order[b->num_out++] = b->idx[k];
  return LEAF_BIT | ((end - beg - 1u) << 26) | first;
}

/* returns the ref of the subtree over idx[beg,end) */
static uint32_t build_rec(bld_t* b, uint32_t beg, uint32_t end, int depth) {
  if (depth > b->depth_max) b->depth_max = depth;
  uint32_t n = end - beg;
  if (n <= b->max_leaf) return emit_leaf(b, beg, end);
  /* widest centroid axis, median split in sorted order */
  float clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (uint32_t k = beg; k < end; ++k)
    for (int a = 0; a < 3; ++a) {
      float c = b->cen[b->idx[k] * 3 + a];
      if (c < clo[a]) clo[a] = c;
      if (c > chi[a]) chi[a] = c;
    }
  int axis = 0;
  float ext = chi[0] - clo[0];
  for (int a = 1; a < 3; ++a)
    if (chi[a] - clo[a] > ext) { ext = chi[a] - clo[a]; axis = a; }
  b->axis_sort = axis;
  qsort(b->idx + beg, n, sizeof(uint32_t), cmp_axis);
  uint32_t mid = beg + n / 2;
  uint32_t me = b->num_nodes++;
  if (me >= b->cap_nodes) return 0xFFFFFFFFu;
  or_node* nd = &b->nodes[me];
  memset(nd, 0, sizeof *nd);
  for (int c = 0; c < 2; ++c) {
    float lo[3], hi[3];
    if (c == 0) range_bounds(b, beg, mid, lo, hi);
    else range_bounds(b, mid, end, lo, hi);
    pad_box(lo, hi);
    put_child_box(&b->nodes[me], c, lo, hi);
  }
  uint32_t r0 = build_rec(b, beg, mid, depth + 1);
  uint32_t r1 = build_rec(b, mid, end, depth + 1);
  b->nodes[me].ref[0] = r0;
  b->nodes[me].ref[1] = r1;
  return me;
}

static int degenerate9(const float* vt) {
  float e1[3] = {vt[3] - vt[0], vt[4] - vt[1], vt[5] - vt[2]};
  float e2[3] = {vt[6] - vt[0], vt[7] - vt[1], vt[8] - vt[2]};
  double cx = (double)e1[1] * e2[2] - (double)e1[2] * e2[1];
  double cy = (double)e1[2] * e2[0] - (double)e1[0] * e2[2];
  double cz = (double)e1[0] * e2[1] - (double)e1[1] * e2[0];
  return cx == 0.0 && cy == 0.0 && cz == 0.0;
}

int oracle_build_bvh(const or_scene* s, uint32_t max_leaf, or_bvh* out) {
  memset(out, 0, sizeof *out);
  if (!s || max_leaf < 1 || max_leaf > 32) return -1;
  bld_t b;
  memset(&b, 0, sizeof b);
  b.s = s;
  b.max_leaf = max_leaf;
  b.idx = (uint32_t*)malloc(sizeof(uint32_t) * (s->num_tris + 1));
  b.cen = (float*)malloc(sizeof(float) * 3 * (s->num_tris + 1));
  uint32_t m = 0;
  for (uint32_t i = 0; i < s->num_tris; ++i) {
    const float* vt = s->vertices + (size_t)i * 9;
    if (degenerate9(vt)) continue;
    b.idx[m++] = i;
    float lo[3], hi[3];
    tri_bounds(vt, lo, hi);
    for (int a = 0; a < 3; ++a) b.cen[i * 3 + a] = 0.5f * lo[a] + 0.5f * hi[a];
  }
  if (m == 0) { free(b.idx); free(b.cen); return -2; }
  b.cap_nodes = m;
  b.nodes = (or_node*)calloc(m, sizeof(or_node));
  b.leaf_order = (uint32_t*)malloc(sizeof(uint32_t) * m);
  g_bld = &b;
  uint32_t root = build_rec(&b, 0, m, 0);
  g_bld = NULL;
  float lo[3], hi[3];
  range_bounds(&b, 0, m, lo, hi);
  pad_box(lo, hi);

  /* textures: descriptors and the alpha plane (A8, textures back to back) */
  uint32_t nt = s->num_textures;
  or_texdesc* td = (or_texdesc*)calloc(nt ? nt : 1, sizeof(or_texdesc));
  uint64_t total = 0;
  for (uint32_t k = 0; k < nt; ++k) {
    td[k].offset = total; td[k].w = s->tex_w[k]; td[k].h = s->tex_h[k];
    total += (uint64_t)s->tex_w[k] * s->tex_h[k];
  }
  uint8_t* texels = (uint8_t*)malloc(total ? total : 1);
  for (uint32_t k = 0; k < nt; ++k) {
    const uint8_t* p = s->tex_rgba[k];
    uint64_t cnt = (uint64_t)s->tex_w[k] * s->tex_h[k];
    for (uint64_t q = 0; q < cnt; ++q) texels[td[k].offset + q] = p[4 * q + 3];
  }
  or_tri* tris = (or_tri*)calloc(m, sizeof(or_tri));
  or_side* sides = (or_side*)calloc(m, sizeof(or_side));
  for (uint32_t k = 0; k < m; ++k) {
    uint32_t i = b.leaf_order[k];
    const float* vt = s->vertices + (size_t)i * 9;
    for (int a = 0; a < 3; ++a) {
      tris[k].v0[a] = vt[a];
      tris[k].e1[a] = vt[3 + a] - vt[a];
      tris[k].e2[a] = vt[6 + a] - vt[a];
    }
    tris[k].prim = i;
    memcpy(sides[k].uv, s->texcoords ? s->texcoords + (size_t)i * 6 : (const float[6]){0}, 24);
    uint32_t g = s->geom_ids ? s->geom_ids[i] : 0u;
    uint32_t tex = s->geom_texture ? s->geom_texture[g] : g;
    sides[k].offset = (uint32_t)td[tex].offset;
    sides[k].dims = (td[tex].w - 1u) | ((td[tex].h - 1u) << 16);
  }
  out->root_ref = root;
  memcpy(out->root_lo, lo, sizeof lo);
  memcpy(out->root_hi, hi, sizeof hi);
  out->num_nodes = b.num_nodes;
  out->num_tris = m;
  out->num_textures = nt;
  out->nodes = b.nodes;
  out->tris = tris;
  out->sides = sides;
  out->texdescs = td;
  out->texels = texels;
  free(b.idx);
  free(b.cen);
  free(b.leaf_order);
  return b.depth_max > MAX_STACK ? -3 : 0;
}

void oracle_bvh_free(or_bvh* b) {
  if (!b) return;
  free((void*)b->nodes);
  free((void*)b->tris);
  free((void*)b->sides);
  free((void*)b->texdescs);
  free((void*)b->texels);
  memset(b, 0, sizeof *b);
}

/* ====================== contract walker C ================================== */

/* Slab test of App. A.2, contract r02 (DESIGN.md §3 A.2): each plane crossing is
 * ONE explicit fused multiply-add t = fmaf(plane, inv, noi) with noi = -(o*inv)
 * (rounded once, clamped to +-FLT_MAX); tf is widened by (1 + 2 gamma_3) and by
 * pad = 4 max_k |e_k|, e_k = fmaf(o_k, inv_k, noi_k) being noi_k's exact rounding
 * error (the fma form's absolute error allowance), and tn is compared against
 * best_t + pad.  No implicit contraction (-ffp-contract=off): every fma here is
 * written out.  Box hook default. */
static float clamp_noi(float x) { return fminf(fmaxf(x, -3.40282347e38f), 3.40282347e38f); }

static void slab_consts(const float* o, const float* inv, float* noi, float* pad) {
  float e[3];
  for (int a = 0; a < 3; ++a) noi[a] = clamp_noi(-(o[a] * inv[a]));
  for (int a = 0; a < 3; ++a) e[a] = fmaf(o[a], inv[a], noi[a]);
  *pad = fmaxf(fmaxf(fabsf(e[0]), fabsf(e[1])), fabsf(e[2])) * 4.0f;
}

/* the culling bound of the box test and of the pop skip: best_t + pad */
static float cull_bound(const float* o, const float* inv, float best_t) {
  float noi[3], pad;
  slab_consts(o, inv, noi, &pad);
  return best_t + pad;
}

static int slab(const float* lo, const float* hi, const float* o, const float* inv, float tmin,
                float best_t, float* tn_out) {
  float noi[3], pad;
  slab_consts(o, inv, noi, &pad);
  float t0x = fmaf(lo[0], inv[0], noi[0]), t1x = fmaf(hi[0], inv[0], noi[0]);
  float t0y = fmaf(lo[1], inv[1], noi[1]), t1y = fmaf(hi[1], inv[1], noi[1]);
  float t0z = fmaf(lo[2], inv[2], noi[2]), t1z = fmaf(hi[2], inv[2], noi[2]);
  float tn = fmaxf(fmaxf(fminf(t0x, t1x), fminf(t0y, t1y)), fmaxf(fminf(t0z, t1z), tmin));
  float tf = fmaf(fminf(fminf(fmaxf(t0x, t1x), fmaxf(t0y, t1y)), fmaxf(t0z, t1z)), 1.0000003576f,
                  pad);
  tf = fminf(tf, best_t + pad);
  *tn_out = tn;
  return tn <= tf;
}

/* Exposed for the closed-form pins: guarded reciprocal of
 * App. A.2 followed by the slab test; tf returned before the best_t clip. */
int walker_slab(const float* lo, const float* hi, const float* ray, float best_t, float* tn,
                float* tf) {
  float inv[3];
  for (int a = 0; a < 3; ++a) {
    float dk = ray[4 + a];
    inv[a] = 1.0f / (fabsf(dk) > 0x1p-80f ? dk : copysignf(0x1p-80f, dk));
  }
  float noi[3], pad;
  slab_consts(ray, inv, noi, &pad);
  float t0x = fmaf(lo[0], inv[0], noi[0]), t1x = fmaf(hi[0], inv[0], noi[0]);
  float t0y = fmaf(lo[1], inv[1], noi[1]), t1y = fmaf(hi[1], inv[1], noi[1]);
  float t0z = fmaf(lo[2], inv[2], noi[2]), t1z = fmaf(hi[2], inv[2], noi[2]);
  *tf = fmaf(fminf(fminf(fmaxf(t0x, t1x), fmaxf(t0y, t1y)), fmaxf(t0z, t1z)), 1.0000003576f, pad);
  return slab(lo, hi, ray, inv, ray[3], best_t, tn);
}

/* Möller–Trumbore on the stored (v0, e1, e2), App. A.1 order. */
static int mt_tri(const or_tri* tr, const float* o, const float* d, float tmin, float tmax_cur,
                  float* t, float* u, float* v) {
  const float* e1 = tr->e1;
  const float* e2 = tr->e2;
  float p[3] = {d[1] * e2[2] - d[2] * e2[1], d[2] * e2[0] - d[0] * e2[2],
                d[0] * e2[1] - d[1] * e2[0]};
  float det = (e1[0] * p[0] + e1[1] * p[1]) + e1[2] * p[2];
  if (!(fabsf(det) >= 1e-12f)) return 0;
  float inv = 1.0f / det;
  float s[3] = {o[0] - tr->v0[0], o[1] - tr->v0[1], o[2] - tr->v0[2]};
  *u = ((s[0] * p[0] + s[1] * p[1]) + s[2] * p[2]) * inv;
  float q[3] = {s[1] * e1[2] - s[2] * e1[1], s[2] * e1[0] - s[0] * e1[2],
                s[0] * e1[1] - s[1] * e1[0]};
  *v = ((d[0] * q[0] + d[1] * q[1]) + d[2] * q[2]) * inv;
  *t = ((e2[0] * q[0] + e2[1] * q[1]) + e2[2] * q[2]) * inv;
  return (*u >= 0.0f) && (*u <= 1.0f) && (*v >= 0.0f) && (*u + *v <= 1.0f) && (*t >= tmin) &&
         (*t <= tmax_cur);
}

static long wrapi(float x, uint32_t n) {
  long i = (long)floorf(x * (float)n);
  long m = (long)n;
  return ((i % m) + m) % m;
}

static int walk_filter(const or_bvh* b, uint32_t k, int isect, float u, float v, float thr,
                       uint32_t M) {
  if (isect == OR_ALPHA_TEX) {
    const or_side* sd = &b->sides[k];
    float w = (1.0f - u) - v;
    float s = (w * sd->uv[0] + u * sd->uv[2]) + v * sd->uv[4];
    float t = (w * sd->uv[1] + u * sd->uv[3]) + v * sd->uv[5];
    uint32_t w_tex = (sd->dims & 0xFFFFu) + 1u, h_tex = (sd->dims >> 16) + 1u;
    long i = wrapi(s, w_tex), j = wrapi(t, h_tex);
    uint8_t a8 = b->texels[(uint64_t)sd->offset + (uint64_t)j * w_tex + (uint64_t)i];
    float a = (float)a8 / 255.0f;
    return a >= thr;
  }
  if (isect == OR_ALPHA_PROC) {
    float fm = (float)M;
    int cu = (int)floorf(u * fm), cv = (int)floorf(v * fm);
    return ((cu + cv) % 2) == 0;
  }
  if (isect == OR_ALPHA_BILIN || isect == OR_ALPHA_PROC_UV) {
    /* reading A28 on the A8 plane through the sidecar */
    const or_side* sd = &b->sides[k];
    float w = (1.0f - u) - v;
    float s = (w * sd->uv[0] + u * sd->uv[2]) + v * sd->uv[4];
    float t = (w * sd->uv[1] + u * sd->uv[3]) + v * sd->uv[5];
    if (isect == OR_ALPHA_PROC_UV) {
      float fm = (float)M;
      long cs = (long)floorf(s * fm), ct = (long)floorf(t * fm);
      return ((cs + ct) & 1L) == 0;
    }
    long W = (long)(sd->dims & 0xFFFFu) + 1, H = (long)(sd->dims >> 16) + 1;
    float x = s * (float)W - 0.5f, y = t * (float)H - 0.5f;
    float x0 = floorf(x), y0 = floorf(y);
    float fx = x - x0, fy = y - y0;
    long i0 = (((long)x0 % W) + W) % W, i1 = ((((long)x0 + 1) % W) + W) % W;
    long j0 = (((long)y0 % H) + H) % H, j1 = ((((long)y0 + 1) % H) + H) % H;
    const uint8_t* p = b->texels + sd->offset;
    float a00 = (float)p[j0 * W + i0] / 255.0f, a10 = (float)p[j0 * W + i1] / 255.0f;
    float a01 = (float)p[j1 * W + i0] / 255.0f, a11 = (float)p[j1 * W + i1] / 255.0f;
    float a = ((1.0f - fx) * a00 + fx * a10) * (1.0f - fy) + ((1.0f - fx) * a01 + fx * a11) * fy;
    return a >= thr;
  }
  return 1;
}

typedef struct {
  const or_bvh* b;
  const float* rays;
  uint64_t n;
  int query, isect;
  float thr;
  uint32_t M;
  or_hit* hits;     /* K == 0: one per ray; K > 0: K per ray (multi-hit) */
  or_counts* counts;
  uint32_t K;       /* multi-hit query: hits kept per ray (0 = closest/any) */
  uint32_t* nhits;  /* multi-hit: hits kept per ray (may be NULL) */
  const or_bvh* list; /* list query: nlist BVHs walked in order (else b alone) */
  uint32_t nlist;
  uint32_t* which;  /* list query: list index of the kept hit (may be NULL) */
  uint64_t next;
  int err;
} wjob_t;

#define MAX_MULTI 64

static int walk_one(const wjob_t* jb, uint64_t r) {
  const or_bvh* b = jb->nlist ? jb->list : jb->b;
  const float* ray = jb->rays + r * 8;
  const float* o = ray;
  const float* d = ray + 4;
  float tmin = ray[3];
  float inv[3];
  for (int a = 0; a < 3; ++a) {
    float dk = d[a];
    inv[a] = 1.0f / (fabsf(dk) > 0x1p-80f ? dk : copysignf(0x1p-80f, dk));
  }
  or_hit best = {INFINITY, 0.0f, 0.0f, 0xFFFFFFFFu};
  float best_t = ray[7];
  int have = 0;
  or_counts c = {0, 0, 0};
  uint32_t st_ref[MAX_STACK];
  float st_tn[MAX_STACK];
  int sp = 0;
  int bad = 0;
  float tn;
  /* multi-hit buffer: ascending t, equal t in the order found; a full buffer
     drops its worst and tmax shrinks to its last entry */
  or_hit mb[MAX_MULTI];
  uint32_t mbw[MAX_MULTI]; /* list index of each kept hit (lists + multi-hit) */
  uint32_t nk = 0;
  const uint32_t K = jb->K;

  /* list query: the BVHs in order, one running best_t */
  const uint32_t nb = jb->nlist ? jb->nlist : 1u;
  uint32_t which = 0xFFFFFFFFu;
  for (uint32_t li = 0; li < nb; ++li) {
  if (jb->nlist) b = &jb->list[li];
  sp = 0;
  c.boxes++;
  if (!slab(b->root_lo, b->root_hi, o, inv, tmin, best_t, &tn)) continue;
  uint32_t cur = b->root_ref;
  for (;;) {
    /* inner-node loop */
    while (!(cur & LEAF_BIT)) {
      if (cur >= b->num_nodes) { bad = 1; goto done; }
      const or_node* nd = &b->nodes[cur];
      float tn0, tn1;
      c.boxes += 2;
      float lo0[3], hi0[3], lo1[3], hi1[3];
      get_child_box(nd, 0, lo0, hi0);
      get_child_box(nd, 1, lo1, hi1);
      int h0 = slab(lo0, hi0, o, inv, tmin, best_t, &tn0);
      int h1 = slab(lo1, hi1, o, inv, tmin, best_t, &tn1);
      if (h0 && h1) {
        uint32_t nearr, farr;
        float ftn;
        if (tn1 < tn0) { nearr = nd->ref[1]; farr = nd->ref[0]; ftn = tn0; }
        else { nearr = nd->ref[0]; farr = nd->ref[1]; ftn = tn1; }
        if (sp >= MAX_STACK) { bad = 1; goto done; }
        st_ref[sp] = farr; st_tn[sp] = ftn; sp++;
        cur = nearr;
      } else if (h0) {
        cur = nd->ref[0];
      } else if (h1) {
        cur = nd->ref[1];
      } else {
        goto pop;
      }
    }
    /* leaf loop */
    {
      uint32_t first = cur & 0x03FFFFFFu;
      uint32_t cnt = ((cur >> 26) & 31u) + 1u;
      if ((uint64_t)first + cnt > b->num_tris) { bad = 1; goto done; }
      for (uint32_t k = first; k < first + cnt; ++k) {
        const or_tri* tr = &b->tris[k];
        float t, u, v;
        c.tris++;
        if (!mt_tri(tr, o, d, tmin, best_t, &t, &u, &v)) continue;
        if (jb->isect == OR_ALPHA_TEX) c.alpha++;
        if (!walk_filter(b, k, jb->isect, u, v, jb->thr, jb->M)) continue;
        if (K) {
          if (nk < K || t < best_t) {
            uint32_t pos = nk < K ? nk : K - 1;
            while (pos > 0 && mb[pos - 1].t > t) {
              mb[pos] = mb[pos - 1];
              mbw[pos] = mbw[pos - 1];
              pos--;
            }
            mb[pos].t = t; mb[pos].u = u; mb[pos].v = v; mb[pos].prim = tr->prim;
            mbw[pos] = li;
            if (nk < K) nk++;
            if (nk == K) best_t = mb[K - 1].t;
          }
          continue;
        }
        if (jb->query == OR_ANY) {
          best.t = t; best.u = u; best.v = v; best.prim = tr->prim;
          which = li;
          goto done;
        }
        if (!have || t < best_t) {
          best.t = t; best.u = u; best.v = v; best.prim = tr->prim;
          best_t = t;
          have = 1;
          which = li;
        }
      }
    }
  pop:
    for (;;) {
      if (sp == 0) goto next_bvh;
      sp--;
      if (st_tn[sp] > cull_bound(o, inv, best_t)) continue;
      cur = st_ref[sp];
      break;
    }
  }
  next_bvh:;
  }
done:
  if (K) {
    const or_hit miss = {INFINITY, 0.0f, 0.0f, 0xFFFFFFFFu};
    for (uint32_t j = 0; j < K; ++j) {
      jb->hits[r * K + j] = j < nk ? mb[j] : miss;
      if (jb->which) jb->which[r * K + j] = j < nk ? mbw[j] : 0xFFFFFFFFu;
    }
    if (jb->nhits) jb->nhits[r] = nk;
  } else {
    if (jb->which) jb->which[r] = which;
    jb->hits[r] = best;
  }
  if (jb->counts) jb->counts[r] = c;
  return bad;
}

static void* wworker(void* arg) {
  wjob_t* jb = (wjob_t*)arg;
  const uint64_t chunk = 1024;
  for (;;) {
    uint64_t s = __atomic_fetch_add(&jb->next, chunk, __ATOMIC_RELAXED);
    if (s >= jb->n) break;
    uint64_t e = s + chunk < jb->n ? s + chunk : jb->n;
    for (uint64_t r = s; r < e; ++r)
      if (walk_one(jb, r)) __atomic_store_n(&jb->err, 1, __ATOMIC_RELAXED);
  }
  return NULL;
}

static int walker_run(wjob_t* jb, int nthreads);

int walker_trace(const or_bvh* b, const float* rays, uint64_t n, int query, int isect,
                 float thr, uint32_t M, or_hit* hits, or_counts* counts, int nthreads) {
  if (!b || !rays || !hits) return -1;
  if (query != OR_CLOSEST && query != OR_ANY) return -1;
  if (isect < OR_NONE || isect > OR_ALPHA_PROC_UV) return -1;
  if ((isect == OR_ALPHA_PROC || isect == OR_ALPHA_PROC_UV) && M == 0) return -1;
  wjob_t jb;
  memset(&jb, 0, sizeof jb);
  jb.b = b; jb.rays = rays; jb.n = n; jb.query = query; jb.isect = isect; jb.thr = thr;
  jb.M = M; jb.hits = hits; jb.counts = counts;
  return walker_run(&jb, nthreads);
}

int walker_trace_multi(const or_bvh* b, const float* rays, uint64_t n, uint32_t K, int isect,
                       float thr, uint32_t M, or_hit* hits, uint32_t* nhits, or_counts* counts,
                       int nthreads) {
  if (!b || !rays || !hits || K < 1 || K > MAX_MULTI) return -1;
  if (isect < OR_NONE || isect > OR_ALPHA_PROC_UV) return -1;
  if ((isect == OR_ALPHA_PROC || isect == OR_ALPHA_PROC_UV) && M == 0) return -1;
  wjob_t jb;
  memset(&jb, 0, sizeof jb);
  jb.b = b; jb.rays = rays; jb.n = n; jb.query = OR_CLOSEST; jb.isect = isect; jb.thr = thr;
  jb.M = M; jb.hits = hits; jb.counts = counts; jb.K = K; jb.nhits = nhits;
  return walker_run(&jb, nthreads);
}

int walker_trace_list(const or_bvh* list, uint32_t nlist, const float* rays, uint64_t n,
                      int query, int isect, float thr, uint32_t M, or_hit* hits, uint32_t* which,
                      or_counts* counts, int nthreads) {
  if (!list || nlist < 1 || !rays || !hits) return -1;
  if (query != OR_CLOSEST && query != OR_ANY) return -1;
  if (isect < OR_NONE || isect > OR_ALPHA_PROC_UV) return -1;
  if ((isect == OR_ALPHA_PROC || isect == OR_ALPHA_PROC_UV) && M == 0) return -1;
  wjob_t jb;
  memset(&jb, 0, sizeof jb);
  jb.b = list; jb.list = list; jb.nlist = nlist; jb.which = which;
  jb.rays = rays; jb.n = n; jb.query = query; jb.isect = isect; jb.thr = thr;
  jb.M = M; jb.hits = hits; jb.counts = counts;
  return walker_run(&jb, nthreads);
}

int walker_trace_list_multi(const or_bvh* list, uint32_t nlist, const float* rays, uint64_t n,
                            uint32_t K, int isect, float thr, uint32_t M, or_hit* hits,
                            uint32_t* nhits, uint32_t* which, or_counts* counts, int nthreads) {
  if (!list || nlist < 1 || !rays || !hits || K < 1 || K > MAX_MULTI) return -1;
  if (isect < OR_NONE || isect > OR_ALPHA_PROC_UV) return -1;
  if ((isect == OR_ALPHA_PROC || isect == OR_ALPHA_PROC_UV) && M == 0) return -1;
  wjob_t jb;
  memset(&jb, 0, sizeof jb);
  jb.b = list; jb.list = list; jb.nlist = nlist; jb.which = which;
  jb.rays = rays; jb.n = n; jb.query = OR_CLOSEST; jb.isect = isect; jb.thr = thr;
  jb.M = M; jb.hits = hits; jb.counts = counts; jb.K = K; jb.nhits = nhits;
  return walker_run(&jb, nthreads);
}

static int walker_run(wjob_t* jb, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) {
    wworker(jb);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, wworker, jb);
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
    free(th);
  }
  return jb->err ? -1 : 0;
}

/* ====================== two-level instancing (walker C) ===================== */

void oracle_ray_to_object(const float* m, const float* ray, float* out) {
  const float* o = ray;
  const float* d = ray + 4;
  for (int i = 0; i < 3; ++i) {
    const float* r = m + 4 * i;
    out[i] = ((r[0] * o[0] + r[1] * o[1]) + r[2] * o[2]) + r[3];
    out[4 + i] = (r[0] * d[0] + r[1] * d[1]) + r[2] * d[2];
  }
  out[3] = ray[3];
  out[7] = ray[7];
}

typedef struct {
  or_hit best;
  float best_t;
  int have;
  or_counts c;
  int bad;
  /* multi-hit (K > 0): the kept hits, ascending t, with their instance index */
  or_hit mb[MAX_MULTI];
  uint32_t mbw[MAX_MULTI];
  uint32_t nk, K, src;
} istate_t;

typedef struct {
  const or_bvh* top;
  const or_instance* recs;
  const or_bvh* bottoms;
  uint32_t nbottoms;
  const float* rays;
  uint64_t n;
  int query, isect;
  float thr;
  uint32_t M;
  or_hit* hits;
  uint32_t* inst;
  or_counts* counts;
  uint32_t K;        /* multi-hit: hits kept per ray (0 = closest / any) */
  uint32_t* nhits;
  float r_safe;      /* origins with max |o_k| > r_safe skip the top level (reading A27) */
  uint64_t next;
  int err;
} ijob_t;

/* One bottom BVH with the running state (the while-while loop of walk_one,
 * closest / any only).  Returns 1 when an any-hit query accepted a hit. */
static int walk_bottom(const ijob_t* jb, const or_bvh* b, const float* ray, istate_t* S) {
  const float* o = ray;
  const float* d = ray + 4;
  const float tmin = ray[3];
  float inv[3];
  for (int a = 0; a < 3; ++a) {
    float dk = d[a];
    inv[a] = 1.0f / (fabsf(dk) > 0x1p-80f ? dk : copysignf(0x1p-80f, dk));
  }
  uint32_t st_ref[MAX_STACK];
  float st_tn[MAX_STACK];
  int sp = 0;
  float tn;
  S->c.boxes++;
  if (!slab(b->root_lo, b->root_hi, o, inv, tmin, S->best_t, &tn)) return 0;
  uint32_t cur = b->root_ref;
  for (;;) {
    while (!(cur & LEAF_BIT)) {
      if (cur >= b->num_nodes) { S->bad = 1; return 0; }
      const or_node* nd = &b->nodes[cur];
      float tn0, tn1, lo0[3], hi0[3], lo1[3], hi1[3];
      S->c.boxes += 2;
      get_child_box(nd, 0, lo0, hi0);
      get_child_box(nd, 1, lo1, hi1);
      int h0 = slab(lo0, hi0, o, inv, tmin, S->best_t, &tn0);
      int h1 = slab(lo1, hi1, o, inv, tmin, S->best_t, &tn1);
      if (h0 && h1) {
        if (sp >= MAX_STACK) { S->bad = 1; return 0; }
        if (tn1 < tn0) { st_ref[sp] = nd->ref[0]; st_tn[sp] = tn0; cur = nd->ref[1]; }
        else { st_ref[sp] = nd->ref[1]; st_tn[sp] = tn1; cur = nd->ref[0]; }
        sp++;
      } else if (h0) {
        cur = nd->ref[0];
      } else if (h1) {
        cur = nd->ref[1];
      } else {
        goto pop;
      }
    }
    {
      uint32_t first = cur & 0x03FFFFFFu;
      uint32_t cnt = ((cur >> 26) & 31u) + 1u;
      if ((uint64_t)first + cnt > b->num_tris) { S->bad = 1; return 0; }
      for (uint32_t k = first; k < first + cnt; ++k) {
        const or_tri* tr = &b->tris[k];
        float t, u, v;
        S->c.tris++;
        if (!mt_tri(tr, o, d, tmin, S->best_t, &t, &u, &v)) continue;
        if (jb->isect == OR_ALPHA_TEX) S->c.alpha++;
        if (!walk_filter(b, k, jb->isect, u, v, jb->thr, jb->M)) continue;
        if (S->K) {   /* multi-hit: as walk_one, the instance index kept beside each hit */
          if (S->nk < S->K || t < S->best_t) {
            uint32_t pos = S->nk < S->K ? S->nk : S->K - 1;
            while (pos > 0 && S->mb[pos - 1].t > t) {
              S->mb[pos] = S->mb[pos - 1];
              S->mbw[pos] = S->mbw[pos - 1];
              pos--;
            }
            S->mb[pos].t = t; S->mb[pos].u = u; S->mb[pos].v = v; S->mb[pos].prim = tr->prim;
            S->mbw[pos] = S->src;
            if (S->nk < S->K) S->nk++;
            if (S->nk == S->K) S->best_t = S->mb[S->K - 1].t;
          }
          continue;
        }
        if (jb->query == OR_ANY) {
          S->best.t = t; S->best.u = u; S->best.v = v; S->best.prim = tr->prim;
          S->have = 1;
          return 1;
        }
        if (!S->have || t < S->best_t) {
          S->best.t = t; S->best.u = u; S->best.v = v; S->best.prim = tr->prim;
          S->best_t = t;
          S->have = 1;
        }
      }
    }
  pop:
    for (;;) {
      if (sp == 0) return 0;
      sp--;
      if (st_tn[sp] > cull_bound(o, inv, S->best_t)) continue;
      cur = st_ref[sp];
      break;
    }
  }
}

/* Instance record k: map the ray (oracle_ray_to_object), walk its bottom BVH with the
 * running state.  Returns 1 when the query is finished (any-hit accepted). */
static int inst_visit(ijob_t* jb, const float* ray, uint32_t k, istate_t* S, uint32_t* which) {
  const or_instance* in = &jb->recs[k];
  if (in->bvh >= jb->nbottoms) { S->bad = 1; return 1; }
  float oray[8];
  oracle_ray_to_object(in->m, ray, oray);
  const int had = S->have;
  const float bt = S->best_t;
  S->src = in->index;
  const int stop = walk_bottom(jb, &jb->bottoms[in->bvh], oray, S);
  if (S->bad) return 1;
  if ((S->have && !had) || S->best_t < bt) *which = in->index;
  return stop;
}

static void walk_instances_one(ijob_t* jb, uint64_t r) {
  const float* ray = jb->rays + r * 8;
  const float* o = ray;
  const float* d = ray + 4;
  const float tmin = ray[3];
  const or_bvh* top = jb->top;
  float inv[3];
  for (int a = 0; a < 3; ++a) {
    float dk = d[a];
    inv[a] = 1.0f / (fabsf(dk) > 0x1p-80f ? dk : copysignf(0x1p-80f, dk));
  }
  istate_t S;
  memset(&S, 0, sizeof S);
  S.best.t = INFINITY;
  S.best.prim = 0xFFFFFFFFu;
  S.best_t = ray[7];
  S.K = jb->K;
  uint32_t which = 0xFFFFFFFFu;
  uint32_t st_ref[MAX_STACK];
  float st_tn[MAX_STACK];
  int sp = 0;
  float tn;
  S.c.boxes++;
  {
    const int root_hit = slab(top->root_lo, top->root_hi, o, inv, tmin, S.best_t, &tn);
    if (fmaxf(fmaxf(fabsf(o[0]), fabsf(o[1])), fabsf(o[2])) > jb->r_safe) {
      /* beyond the proven range: every instance in leaf order, the top level unused */
      for (uint32_t k = 0; k < top->num_tris; ++k)
        if (inst_visit(jb, ray, k, &S, &which)) goto done;
      goto done;
    }
    if (!root_hit) goto done;
  }
  uint32_t cur = top->root_ref;
  for (;;) {
    while (!(cur & LEAF_BIT)) {
      if (cur >= top->num_nodes) { S.bad = 1; goto done; }
      const or_node* nd = &top->nodes[cur];
      float tn0, tn1, lo0[3], hi0[3], lo1[3], hi1[3];
      S.c.boxes += 2;
      get_child_box(nd, 0, lo0, hi0);
      get_child_box(nd, 1, lo1, hi1);
      int h0 = slab(lo0, hi0, o, inv, tmin, S.best_t, &tn0);
      int h1 = slab(lo1, hi1, o, inv, tmin, S.best_t, &tn1);
      if (h0 && h1) {
        if (sp >= MAX_STACK) { S.bad = 1; goto done; }
        if (tn1 < tn0) { st_ref[sp] = nd->ref[0]; st_tn[sp] = tn0; cur = nd->ref[1]; }
        else { st_ref[sp] = nd->ref[1]; st_tn[sp] = tn1; cur = nd->ref[0]; }
        sp++;
      } else if (h0) {
        cur = nd->ref[0];
      } else if (h1) {
        cur = nd->ref[1];
      } else {
        goto pop;
      }
    }
    {
      /* top-level leaf: its instances in stored order (the BVH's "primitives") */
      uint32_t first = cur & 0x03FFFFFFu;
      uint32_t cnt = ((cur >> 26) & 31u) + 1u;
      if ((uint64_t)first + cnt > top->num_tris) { S.bad = 1; goto done; }
      for (uint32_t k = first; k < first + cnt; ++k)
        if (inst_visit(jb, ray, k, &S, &which)) goto done;
    }
  pop:
    for (;;) {
      if (sp == 0) goto done;
      sp--;
      if (st_tn[sp] > cull_bound(o, inv, S.best_t)) continue;
      cur = st_ref[sp];
      break;
    }
  }
done:
  if (S.K) {
    const or_hit miss = {INFINITY, 0.0f, 0.0f, 0xFFFFFFFFu};
    for (uint32_t j = 0; j < S.K; ++j) {
      jb->hits[r * S.K + j] = j < S.nk ? S.mb[j] : miss;
      if (jb->inst) jb->inst[r * S.K + j] = j < S.nk ? S.mbw[j] : 0xFFFFFFFFu;
    }
    if (jb->nhits) jb->nhits[r] = S.nk;
  } else {
    jb->hits[r] = S.best;
    if (jb->inst) jb->inst[r] = which;
  }
  if (jb->counts) jb->counts[r] = S.c;
  if (S.bad) __atomic_store_n(&jb->err, 1, __ATOMIC_RELAXED);
}

static void* iworker(void* arg) {
  ijob_t* jb = (ijob_t*)arg;
  const uint64_t chunk = 256;
  for (;;) {
    uint64_t s = __atomic_fetch_add(&jb->next, chunk, __ATOMIC_RELAXED);
    if (s >= jb->n) break;
    uint64_t e = s + chunk < jb->n ? s + chunk : jb->n;
    for (uint64_t r = s; r < e; ++r) walk_instances_one(jb, r);
  }
  return NULL;
}

int walker_trace_instances(const or_bvh* top, const or_instance* recs, const or_bvh* bottoms,
                           uint32_t nbottoms, const float* rays, uint64_t n, int query,
                           int isect, float thr, uint32_t M, or_hit* hits, uint32_t* inst,
                           or_counts* counts, float r_safe, int nthreads) {
  return walker_trace_instances_multi(top, recs, bottoms, nbottoms, rays, n, query, 0, isect, thr,
                                      M, hits, NULL, inst, counts, r_safe, nthreads);
}

int walker_trace_instances_multi(const or_bvh* top, const or_instance* recs,
                                 const or_bvh* bottoms, uint32_t nbottoms, const float* rays,
                                 uint64_t n, int query, uint32_t K, int isect, float thr,
                                 uint32_t M, or_hit* hits, uint32_t* nhits, uint32_t* inst,
                                 or_counts* counts, float r_safe, int nthreads) {
  if (!top || !recs || !bottoms || nbottoms < 1 || !rays || !hits) return -1;
  if (query != OR_CLOSEST && query != OR_ANY) return -1;
  if (K > MAX_MULTI) return -1;
  if (isect < OR_NONE || isect > OR_ALPHA_PROC_UV) return -1;
  if ((isect == OR_ALPHA_PROC || isect == OR_ALPHA_PROC_UV) && M == 0) return -1;
  ijob_t jb;
  memset(&jb, 0, sizeof jb);
  jb.top = top; jb.recs = recs; jb.bottoms = bottoms; jb.nbottoms = nbottoms;
  jb.rays = rays; jb.n = n; jb.query = query; jb.isect = isect; jb.thr = thr; jb.M = M;
  jb.hits = hits; jb.inst = inst; jb.counts = counts; jb.K = K; jb.nhits = nhits;
  jb.r_safe = r_safe;
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) {
    iworker(&jb);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, iworker, &jb);
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
    free(th);
  }
  return jb.err ? -1 : 0;
}


/* ====================== 8-wide compressed BVH walker ======================= */
/* DESIGN.md §9h.  Written from the documented layout and traversal order; it
 * shares nothing with the product's wide.cu / bvh8_build.cpp. */
typedef struct {
  const or_bvh* b;
  const or_wnode* nodes;
  uint32_t num_nodes;
  const float* rays;
  uint64_t n;
  int query, isect;
  float thr;
  uint32_t M;
  or_hit* hits;
  or_counts* counts;
  uint64_t next;
  int err;
} wwjob_t;

static float wide_plane(uint8_t q, uint8_t e, float pm) {
  uint32_t bits = (uint32_t)e << 23;
  float scale;
  memcpy(&scale, &bits, 4);
  return fmaf(8388608.0f + (float)q, scale, pm);
}

static int walk_wide_one(const wwjob_t* jb, uint64_t r) {
  const or_bvh* b = jb->b;
  const float* ray = jb->rays + r * 8;
  const float* o = ray;
  const float* d = ray + 4;
  const float tmin = ray[3];
  float inv[3];
  for (int a = 0; a < 3; ++a) {
    float dk = d[a];
    inv[a] = 1.0f / (fabsf(dk) > 0x1p-80f ? dk : copysignf(0x1p-80f, dk));
  }
  const uint32_t oct = (uint32_t)(signbit(inv[0]) != 0) | (uint32_t)(signbit(inv[1]) != 0) << 1 |
                       (uint32_t)(signbit(inv[2]) != 0) << 2;
  or_hit best = {INFINITY, 0.0f, 0.0f, 0xFFFFFFFFu};
  float best_t = ray[7];
  int have = 0, bad = 0;
  or_counts c = {0, 0, 0};
  uint32_t st_base[MAX_STACK], st_imask[MAX_STACK], st_keys[MAX_STACK];
  int sp = 0;
  float tn;
  c.boxes++;
  if (!slab(b->root_lo, b->root_hi, o, inv, tmin, best_t, &tn)) goto done;
  uint32_t node = 0;
  for (;;) {
    if (node >= jb->num_nodes) { bad = 1; goto done; }
    const or_wnode* w = &jb->nodes[node];
    uint32_t valid = 0, hits = 0;
    for (int s = 0; s < 8; ++s)
      if (w->meta[s] != 0xFF) valid |= 1u << s;
    c.boxes += (uint32_t)__builtin_popcount(valid);
    for (int s = 0; s < 8; ++s) {
      if (!(valid >> s & 1u)) continue;
      float lo[3], hi[3];
      for (int a = 0; a < 3; ++a) {
        lo[a] = wide_plane(w->qlo[a][s], w->e[a], w->pm[a]);
        hi[a] = wide_plane(w->qhi[a][s], w->e[a], w->pm[a]);
      }
      if (slab(lo, hi, o, inv, tmin, best_t, &tn)) hits |= 1u << s;
    }
    /* leaf children, keys ascending */
    for (uint32_t k = 0; k < 8; ++k) {
      const uint32_t s = k ^ oct;
      if (!(hits >> s & 1u) || (w->imask >> s & 1u)) continue;
      const uint32_t m = w->meta[s];
      const uint32_t first = w->tri_base + (m & 31u), cnt = (m >> 5) + 1u;
      if ((uint64_t)first + cnt > b->num_tris) { bad = 1; goto done; }
      for (uint32_t t_i = first; t_i < first + cnt; ++t_i) {
        const or_tri* tr = &b->tris[t_i];
        float t, u, v;
        c.tris++;
        if (!mt_tri(tr, o, d, tmin, best_t, &t, &u, &v)) continue;
        if (jb->isect == OR_ALPHA_TEX) c.alpha++;
        if (!walk_filter(b, t_i, jb->isect, u, v, jb->thr, jb->M)) continue;
        if (jb->query == OR_ANY) {
          best.t = t; best.u = u; best.v = v; best.prim = tr->prim;
          goto done;
        }
        if (!have || t < best_t) {
          best.t = t; best.u = u; best.v = v; best.prim = tr->prim;
          best_t = t;
          have = 1;
        }
      }
    }
    /* inner children: descend into the smallest key, keep the others as a group (base =
     * the parent node: a closest-hit query re-tests a pending child against the current
     * best_t when it is popped, one counted box test on its decoded box) */
    uint32_t keys = 0;
    for (uint32_t s = 0; s < 8; ++s)
      if ((hits >> s & 1u) && (w->imask >> s & 1u)) keys |= 1u << (s ^ oct);
    if (keys) {
      const uint32_t k0 = (uint32_t)__builtin_ctz(keys);
      keys &= keys - 1u;
      if (keys) {
        if (sp >= MAX_STACK) { bad = 1; goto done; }
        st_base[sp] = node; st_imask[sp] = w->imask; st_keys[sp] = keys;
        sp++;
      }
      const uint32_t s0 = k0 ^ oct;
      node = w->child_base + (uint32_t)__builtin_popcount(w->imask & ((1u << s0) - 1u));
      continue;
    }
    for (;;) {
      if (sp == 0) goto done;
      const uint32_t parent = st_base[sp - 1], imask = st_imask[sp - 1];
      uint32_t pk = st_keys[sp - 1];
      const uint32_t k0 = (uint32_t)__builtin_ctz(pk);
      pk &= pk - 1u;
      if (pk) st_keys[sp - 1] = pk;
      else sp--;
      const uint32_t s0 = k0 ^ oct;
      if (parent >= jb->num_nodes) { bad = 1; goto done; }
      const or_wnode* pw = &jb->nodes[parent];
      if (jb->query == OR_CLOSEST) {
        float lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
          lo[a] = wide_plane(pw->qlo[a][s0], pw->e[a], pw->pm[a]);
          hi[a] = wide_plane(pw->qhi[a][s0], pw->e[a], pw->pm[a]);
        }
        c.boxes++;
        if (!slab(lo, hi, o, inv, tmin, best_t, &tn)) continue;
      }
      node = pw->child_base + (uint32_t)__builtin_popcount(imask & ((1u << s0) - 1u));
      break;
    }
  }
done:
  jb->hits[r] = best;
  if (jb->counts) jb->counts[r] = c;
  return bad;
}

static void* wwworker(void* arg) {
  wwjob_t* jb = (wwjob_t*)arg;
  const uint64_t chunk = 1024;
  for (;;) {
    uint64_t s = __atomic_fetch_add(&jb->next, chunk, __ATOMIC_RELAXED);
    if (s >= jb->n) break;
    uint64_t e = s + chunk < jb->n ? s + chunk : jb->n;
    for (uint64_t r = s; r < e; ++r)
      if (walk_wide_one(jb, r)) __atomic_store_n(&jb->err, 1, __ATOMIC_RELAXED);
  }
  return NULL;
}

int walker_trace_wide(const or_bvh* b, const or_wnode* nodes, uint32_t num_nodes,
                      const float* rays, uint64_t n, int query, int isect, float thr, uint32_t M,
                      or_hit* hits, or_counts* counts, int nthreads) {
  if (!b || !nodes || num_nodes == 0 || !rays || !hits) return -1;
  if (query != OR_CLOSEST && query != OR_ANY) return -1;
  if (isect < OR_NONE || isect > OR_ALPHA_PROC_UV) return -1;
  if ((isect == OR_ALPHA_PROC || isect == OR_ALPHA_PROC_UV) && M == 0) return -1;
  wwjob_t jb;
  memset(&jb, 0, sizeof jb);
  jb.b = b; jb.nodes = nodes; jb.num_nodes = num_nodes; jb.rays = rays; jb.n = n;
  jb.query = query; jb.isect = isect; jb.thr = thr; jb.M = M; jb.hits = hits; jb.counts = counts;
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) {
    wwworker(&jb);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, wwworker, &jb);
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
    free(th);
  }
  return jb.err ? -2 : 0;
}
