/*
 * oracle.c — oracle S: brute-force reference for the custom-intersector
 * queries of arXiv 1912.12786.  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * The plain definition: for ray r and triangles
 * i = 0..N-1 in caller order
 *   1. geometric test  (hit_i, t_i, u_i, v_i) = MT(r, v0_i, v1_i-v0_i, v2_i-v0_i)
 *      — "the intersect function that tests if a ray intersects the
 *      primitive" (PAPER.md:115-132 [§3.1]); Möller–Trumbore, no culling,
 *      |det| < 1e-12 -> miss, t in [tmin, tmax] inclusive.
 *   2. filter F_I, applied per candidate, inside the loop (PAPER.md:248-252,
 *      "statically replaced with the calls to operator()"):
 *        NONE / DEFAULT / COUNT : true
 *        ALPHA_TEX  : tex2D(textures[geom], lerp(tc[3p..3p+2], u, v)).w >= .01f
 *                                             (PAPER.md:296-316 [§4 listing])
 *        ALPHA_PROC : (floor(u*M) + floor(v*M)) even   (
 *                     reading A4/A5 of DESIGN.md: barycentric checker, M = 8)
 *   3. accepted set A = { i : hit_i && F_I(i) }
 *   4. CLOSEST = argmin_{i in A} t_i, ties -> lowest index
 *   5. ANY     = any element of A; this oracle returns the lowest index
 *                ("the first encountered hit point").
 * Nothing is blocked, fused or reordered: every ray is tested against every
 * triangle in index order.
 *
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math (no FMA contraction).
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- vector helpers (fp32, textbook order) ------------------ */
static void sub3(const float* a, const float* b, float* o) {
  o[0] = a[0] - b[0];
  o[1] = a[1] - b[1];
  o[2] = a[2] - b[2];
}
/* cross(a,b) = (a.y*b.z - a.z*b.y, a.z*b.x - a.x*b.z, a.x*b.y - a.y*b.x) */
static void cross3(const float* a, const float* b, float* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
/* dot(a,b) = (a.x*b.x + a.y*b.y) + a.z*b.z */
static float dot3(const float* a, const float* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

/* Möller–Trumbore, textbook order.
 * ray = (o.xyz, tmin, d.xyz, tmax). Returns hit; t,u,v written always
 * (zeros when det is rejected). */
int oracle_mt(const float* ray, const float* v0, const float* v1, const float* v2,
              float tmax_cur, float* t, float* u, float* v) {
  const float* o = ray;
  const float* d = ray + 4;
  float e1[3], e2[3], p[3], s[3], q[3];
  sub3(v1, v0, e1);
  sub3(v2, v0, e2);
  cross3(d, e2, p);
  float det = dot3(e1, p);
  *t = 0.0f; *u = 0.0f; *v = 0.0f;
  if (!(fabsf(det) >= 1e-12f)) return 0;
  float inv = 1.0f / det;
  sub3(o, v0, s);
  *u = dot3(s, p) * inv;
  cross3(s, e1, q);
  *v = dot3(d, q) * inv;
  *t = dot3(e2, q) * inv;
  float tmin = ray[3];
  return (*u >= 0.0f) && (*u <= 1.0f) && (*v >= 0.0f) && (*u + *v <= 1.0f) &&
         (*t >= tmin) && (*t <= tmax_cur);
}

/* lerp(a,b,c,u,v) = (1-u-v)*a + u*b + v*c,
 * evaluated as w = (1-u)-v; (w*a + u*b) + v*c. */
void oracle_lerp2(const float* a, const float* b, const float* c, float u, float v,
                  float* out) {
  float w = (1.0f - u) - v;
  out[0] = (w * a[0] + u * b[0]) + v * c[0];
  out[1] = (w * a[1] + u * b[1]) + v * c[1];
}

/* tex2D, nearest filter, wrap addressing, texel centres at (i+.5)/W
 * (PAPER.md:311 is silent; reading A6 in DESIGN.md).
 * Returns alpha as a8/255.0f (reading A7). */
static long wrap_index(float x, uint32_t n) {
  long i = (long)floorf(x * (float)n);
  long m = (long)n;
  return ((i % m) + m) % m;
}
float oracle_tex_alpha(uint32_t w, uint32_t h, const uint8_t* rgba, float s, float t) {
  long i = wrap_index(s, w);
  long j = wrap_index(t, h);
  uint8_t a8 = rgba[((size_t)j * w + (size_t)i) * 4 + 3];
  return (float)a8 / 255.0f;
}

static long wrap_long(long i, long m) { return ((i % m) + m) % m; }

float oracle_tex_alpha_bilinear(uint32_t w, uint32_t h, const uint8_t* rgba, float s, float t) {
  float x = s * (float)w - 0.5f;
  float y = t * (float)h - 0.5f;
  float x0 = floorf(x), y0 = floorf(y);
  float fx = x - x0, fy = y - y0;
  long i0 = wrap_long((long)x0, w), i1 = wrap_long((long)x0 + 1, w);
  long j0 = wrap_long((long)y0, h), j1 = wrap_long((long)y0 + 1, h);
  float a00 = (float)rgba[((size_t)j0 * w + (size_t)i0) * 4 + 3] / 255.0f;
  float a10 = (float)rgba[((size_t)j0 * w + (size_t)i1) * 4 + 3] / 255.0f;
  float a01 = (float)rgba[((size_t)j1 * w + (size_t)i0) * 4 + 3] / 255.0f;
  float a11 = (float)rgba[((size_t)j1 * w + (size_t)i1) * 4 + 3] / 255.0f;
  return ((1.0f - fx) * a00 + fx * a10) * (1.0f - fy) + ((1.0f - fx) * a01 + fx * a11) * fy;
}

static double W_of(const or_scene* s, uint32_t k) { return (double)s->tex_w[k]; }
static double H_of(const or_scene* s, uint32_t k) { return (double)s->tex_h[k]; }

/* bilinear alpha in double (flags only) */
static double bilinear_double(uint32_t w, uint32_t h, const uint8_t* rgba, double s, double t) {
  double x = s * w - 0.5, y = t * h - 0.5;
  double x0 = floor(x), y0 = floor(y);
  double fx = x - x0, fy = y - y0;
  long i0 = wrap_long((long)x0, w), i1 = wrap_long((long)x0 + 1, w);
  long j0 = wrap_long((long)y0, h), j1 = wrap_long((long)y0 + 1, h);
  double a00 = rgba[((size_t)j0 * w + (size_t)i0) * 4 + 3] / 255.0;
  double a10 = rgba[((size_t)j0 * w + (size_t)i1) * 4 + 3] / 255.0;
  double a01 = rgba[((size_t)j1 * w + (size_t)i0) * 4 + 3] / 255.0;
  double a11 = rgba[((size_t)j1 * w + (size_t)i1) * 4 + 3] / 255.0;
  return ((1 - fx) * a00 + fx * a10) * (1 - fy) + ((1 - fx) * a01 + fx * a11) * fy;
}

static uint32_t tri_texture(const or_scene* s, uint32_t i) {
  uint32_t g = s->geom_ids ? s->geom_ids[i] : 0u;
  return s->geom_texture ? s->geom_texture[g] : g;
}

/* The filter F_I of one candidate that hit geometrically. */
static int filter(const or_scene* s, uint32_t i, int isect, float u, float v, float thr,
                  uint32_t M) {
  if (isect == OR_ALPHA_TEX) {
    /* textures[hr.geom_id], tex_coords[prim_id*3+k], lerp, tex2D,
       hr.hit &= color.w >= .01f */
    const float* tc = s->texcoords + (size_t)i * 6;
    float coord[2];
    oracle_lerp2(tc, tc + 2, tc + 4, u, v, coord);
    uint32_t k = tri_texture(s, i);
    float a = oracle_tex_alpha(s->tex_w[k], s->tex_h[k], s->tex_rgba[k], coord[0], coord[1]);
    return a >= thr;
  }
  if (isect == OR_ALPHA_PROC) {
    float fm = (float)M;
    int cu = (int)floorf(u * fm);
    int cv = (int)floorf(v * fm);
    return ((cu + cv) % 2) == 0;
  }
  if (isect == OR_ALPHA_BILIN || isect == OR_ALPHA_PROC_UV) {
    const float* tc = s->texcoords + (size_t)i * 6;
    float coord[2];
    oracle_lerp2(tc, tc + 2, tc + 4, u, v, coord);
    if (isect == OR_ALPHA_PROC_UV) {   /* checker on the texcoords (reading A28) */
      float fm = (float)M;
      long cs = (long)floorf(coord[0] * fm), ct = (long)floorf(coord[1] * fm);
      return ((cs + ct) & 1L) == 0;
    }
    uint32_t k = tri_texture(s, i);
    float a = oracle_tex_alpha_bilinear(s->tex_w[k], s->tex_h[k], s->tex_rgba[k], coord[0],
                                        coord[1]);
    return a >= thr;
  }
  return 1; /* NONE, DEFAULT, COUNT */
}

/* Degenerate triangles (|e1 x e2| = 0) never enter the scene.
 * Tested exactly: the fp32 edges' cross product evaluated in double, where
 * every product of two floats is exact. */
static int degenerate(const float* vt) {
  float e1[3], e2[3];
  sub3(vt + 3, vt, e1);
  sub3(vt + 6, vt, e2);
  double cx = (double)e1[1] * e2[2] - (double)e1[2] * e2[1];
  double cy = (double)e1[2] * e2[0] - (double)e1[0] * e2[2];
  double cz = (double)e1[0] * e2[1] - (double)e1[1] * e2[0];
  return cx == 0.0 && cy == 0.0 && cz == 0.0;
}

int oracle_eval_pair(const or_scene* s, const float* ray, uint32_t prim, int isect,
                     float thr, uint32_t M, or_hit* out) {
  const float* vt = s->vertices + (size_t)prim * 9;
  float t, u, v;
  int hit = oracle_mt(ray, vt, vt + 3, vt + 6, ray[7], &t, &u, &v);
  if (degenerate(vt)) hit = 0;
  out->t = t; out->u = u; out->v = v; out->prim = prim;
  return hit && filter(s, prim, isect, u, v, thr, M);
}

/* oracle_eval_pair over n (ray, prim) pairs: acc[i] = accepted, out[i] = (t, u, v, prim). */
int oracle_eval_pairs(const or_scene* s, const float* rays, const uint32_t* prims, uint64_t n,
                      int isect, float thr, uint32_t M, uint8_t* acc, or_hit* out) {
  if (!s || !rays || !prims || !acc || !out) return -1;
  for (uint64_t i = 0; i < n; ++i) {
    if (prims[i] >= s->num_tris) return -1;
    acc[i] = (uint8_t)oracle_eval_pair(s, rays + i * 8, prims[i], isect, thr, M, out + i);
  }
  return 0;
}

/* ---------------- double shadow (ambiguity flags only) ------------------- */
static int mt_double(const float* ray, const float* vt, double* t, double* u, double* v) {
  double o[3] = {ray[0], ray[1], ray[2]}, d[3] = {ray[4], ray[5], ray[6]};
  double a[3] = {vt[0], vt[1], vt[2]};
  double e1[3] = {(double)vt[3] - a[0], (double)vt[4] - a[1], (double)vt[5] - a[2]};
  double e2[3] = {(double)vt[6] - a[0], (double)vt[7] - a[1], (double)vt[8] - a[2]};
  double p[3] = {d[1] * e2[2] - d[2] * e2[1], d[2] * e2[0] - d[0] * e2[2],
                 d[0] * e2[1] - d[1] * e2[0]};
  double det = e1[0] * p[0] + e1[1] * p[1] + e1[2] * p[2];
  if (det == 0.0) return 0;
  double s[3] = {o[0] - a[0], o[1] - a[1], o[2] - a[2]};
  double q[3] = {s[1] * e1[2] - s[2] * e1[1], s[2] * e1[0] - s[0] * e1[2],
                 s[0] * e1[1] - s[1] * e1[0]};
  *u = (s[0] * p[0] + s[1] * p[1] + s[2] * p[2]) / det;
  *v = (d[0] * q[0] + d[1] * q[1] + d[2] * q[2]) / det;
  *t = (e2[0] * q[0] + e2[1] * q[1] + e2[2] * q[2]) / det;
  return 1;
}

static double dist_to_int(double x) { return fabs(x - floor(x + 0.5)); }

/* ---------------- per-ray brute force ------------------------------------ */
typedef struct {
  const or_scene* s;
  const float* rays;
  uint64_t n;
  int query, isect;
  float thr;
  uint32_t M;
  or_hit* hits;
  uint32_t* flags;
  uint32_t* ntie;
  uint32_t K;       /* multi-hit query: hits per ray (0 = closest/any) */
  uint32_t* nhits;  /* multi-hit: accepted hits kept per ray (may be NULL) */
  uint64_t chunk; /* rays per claim */
  uint64_t next;  /* atomic chunk counter */
} job_t;

/* Multi-hit query, plain definition ("the first N hit
 * points"): all accepted candidates of the ray (same test as
 * above, tmax = ray.tmax), sorted ascending by t (equal t: lower index
 * first), the first K kept; remaining slots hold the miss record. */
typedef struct { float t, u, v; uint32_t prim; } cand_t;
static int cmp_cand(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->t < y->t) return -1;
  if (x->t > y->t) return 1;
  return x->prim < y->prim ? -1 : (x->prim > y->prim ? 1 : 0);
}

static void trace_one_multi(const job_t* jb, uint64_t r) {
  const or_scene* s = jb->s;
  const float* ray = jb->rays + r * 8;
  size_t cap = 64, cnt = 0;
  cand_t* c = (cand_t*)malloc(sizeof(cand_t) * cap);
  for (uint32_t i = 0; i < s->num_tris; ++i) {
    const float* vt = s->vertices + (size_t)i * 9;
    float t, u, v;
    if (!oracle_mt(ray, vt, vt + 3, vt + 6, ray[7], &t, &u, &v)) continue;
    if (degenerate(vt)) continue;
    if (!filter(s, i, jb->isect, u, v, jb->thr, jb->M)) continue;
    if (cnt == cap) {
      cap *= 2;
      c = (cand_t*)realloc(c, sizeof(cand_t) * cap);
    }
    c[cnt].t = t; c[cnt].u = u; c[cnt].v = v; c[cnt].prim = i;
    cnt++;
  }
  qsort(c, cnt, sizeof(cand_t), cmp_cand);
  const uint32_t K = jb->K;
  for (uint32_t j = 0; j < K; ++j) {
    or_hit* h = &jb->hits[r * K + j];
    if (j < cnt) { h->t = c[j].t; h->u = c[j].u; h->v = c[j].v; h->prim = c[j].prim; }
    else { h->t = INFINITY; h->u = 0.0f; h->v = 0.0f; h->prim = 0xFFFFFFFFu; }
  }
  if (jb->nhits) jb->nhits[r] = (uint32_t)(cnt < K ? cnt : K);
  /* ties at the cut: how many accepted candidates share the K-th t (for parity) */
  if (jb->ntie) {
    uint32_t ties = 0;
    if (cnt > K && K > 0)
      for (size_t q = 0; q < cnt; ++q) ties += (c[q].t == c[K - 1].t);
    jb->ntie[r] = ties;
  }
  free(c);
}

static void trace_one(const job_t* jb, uint64_t r) {
  const or_scene* s = jb->s;
  const float* ray = jb->rays + r * 8;
  or_hit best = {INFINITY, 0.0f, 0.0f, 0xFFFFFFFFu};
  float second_t = INFINITY;
  int have = 0;
  uint32_t ties = 0;
  for (uint32_t i = 0; i < s->num_tris; ++i) {
    const float* vt = s->vertices + (size_t)i * 9;
    float t, u, v;
    if (!oracle_mt(ray, vt, vt + 3, vt + 6, ray[7], &t, &u, &v)) continue;
    if (degenerate(vt)) continue;
    if (!filter(s, i, jb->isect, u, v, jb->thr, jb->M)) continue;
    /* accepted */
    if (jb->query == OR_ANY) {
      if (!have) { best.t = t; best.u = u; best.v = v; best.prim = i; have = 1; }
      if (!jb->flags && !jb->ntie) break; /* first (lowest-index) element of A */
      continue;
    }
    if (!have || t < best.t) {
      second_t = have ? best.t : second_t;
      best.t = t; best.u = u; best.v = v; best.prim = i;
      have = 1;
      ties = 1;
    } else {
      if (t == best.t) ties++;
      if (t < second_t) second_t = t;
    }
  }
  jb->hits[r] = best;
  if (jb->ntie) jb->ntie[r] = have ? ties : 0;
  if (!jb->flags) return;

  /* ambiguity classes, SURVEY.md §8(c) X1..X4 (double shadow) */
  uint32_t f = 0;
  if (jb->query == OR_CLOSEST && have && second_t < INFINITY &&
      (double)second_t - (double)best.t < 1e-5 * fabs((double)best.t))
    f |= OR_X1_NEAR_TIE;
  double lim = have && jb->query == OR_CLOSEST ? (double)best.t * (1.0 + 1e-5) : INFINITY;
  for (uint32_t i = 0; i < s->num_tris; ++i) {
    const float* vt = s->vertices + (size_t)i * 9;
    double t, u, v;
    if (!mt_double(ray, vt, &t, &u, &v)) continue;
    if (!(t >= (double)ray[3] * (1 - 1e-6) - 1e-9 && t <= (double)ray[7] && t <= lim)) continue;
    double w = 1.0 - u - v;
    double m = u < v ? u : v;
    m = m < w ? m : w;
    if (fabs(m) < 1e-6) f |= OR_X2_EDGE_GRAZE;
    if (m < -1e-6) continue; /* clearly outside: no alpha/checker decision */
    if (jb->isect == OR_ALPHA_TEX) {
      const float* tc = s->texcoords + (size_t)i * 6;
      uint32_t k = tri_texture(s, i);
      double W = s->tex_w[k], H = s->tex_h[k];
      double ss = w * tc[0] + u * tc[2] + v * tc[4];
      double tt = w * tc[1] + u * tc[3] + v * tc[5];
      if (dist_to_int(ss * W) < 1e-5 || dist_to_int(tt * H) < 1e-5) {
        /* straddle check: do the two candidate texels decide differently? */
        float a0 = oracle_tex_alpha(s->tex_w[k], s->tex_h[k], s->tex_rgba[k],
                                    (float)(ss - 2e-5 / W), (float)(tt - 2e-5 / H));
        float a1 = oracle_tex_alpha(s->tex_w[k], s->tex_h[k], s->tex_rgba[k],
                                    (float)(ss + 2e-5 / W), (float)(tt + 2e-5 / H));
        float a2 = oracle_tex_alpha(s->tex_w[k], s->tex_h[k], s->tex_rgba[k],
                                    (float)(ss - 2e-5 / W), (float)(tt + 2e-5 / H));
        float a3 = oracle_tex_alpha(s->tex_w[k], s->tex_h[k], s->tex_rgba[k],
                                    (float)(ss + 2e-5 / W), (float)(tt - 2e-5 / H));
        int d0 = a0 >= jb->thr, d1 = a1 >= jb->thr, d2 = a2 >= jb->thr, d3 = a3 >= jb->thr;
        if (d0 != d1 || d0 != d2 || d0 != d3) f |= OR_X3_TEXEL_EDGE;
      }
    } else if (jb->isect == OR_ALPHA_PROC) {
      double M = (double)jb->M;
      if (dist_to_int(u * M) < 1e-6 * M || dist_to_int(v * M) < 1e-6 * M) f |= OR_X4_CHECKER_EDGE;
    } else if (jb->isect == OR_ALPHA_BILIN || jb->isect == OR_ALPHA_PROC_UV) {
      const float* tc = s->texcoords + (size_t)i * 6;
      double ss = w * tc[0] + u * tc[2] + v * tc[4];
      double tt = w * tc[1] + u * tc[3] + v * tc[5];
      if (jb->isect == OR_ALPHA_PROC_UV) {
        double M = (double)jb->M;
        if (dist_to_int(ss * M) < 1e-5 * (1.0 + fabs(ss * M)) ||
            dist_to_int(tt * M) < 1e-5 * (1.0 + fabs(tt * M)))
          f |= OR_X4_CHECKER_EDGE;
      } else {
        uint32_t k = tri_texture(s, i);
        double a = bilinear_double(s->tex_w[k], s->tex_h[k], s->tex_rgba[k], ss, tt);
        /* X5 band (reading A28): north_star's 1e-6, which also covers
         * the fp32 bilinear formula's own rounding (7 ops on values in [0, 1]:
         * <= 7 * 2^-24 = 4.2e-7), plus the first-order propagation of the fp32
         * texcoords' deviation from the double ones: alpha is piecewise bilinear
         * with |d alpha / d s| <= W and |d alpha / d t| <= H (texel alphas in
         * [0, 1]), so |alpha32 - alpha64| <~ W |s32 - s64| + H |t32 - t64|;
         * doubled for second-order terms.  With no fp32 hit there is no fp32
         * decision to be wrong and the band is the floor. */
        double band = 1e-6;
        float t32, u32, v32;
        if (oracle_mt(ray, vt, vt + 3, vt + 6, ray[7], &t32, &u32, &v32)) {
          float st32[2];
          oracle_lerp2(tc, tc + 2, tc + 4, u32, v32, st32);
          band += 2.0 * (W_of(s, k) * fabs((double)st32[0] - ss) +
                         H_of(s, k) * fabs((double)st32[1] - tt));
        }
        if (fabs(a - (double)jb->thr) < band) f |= OR_X5_ALPHA_NEAR;
      }
    }
  }
  jb->flags[r] = f;
}

static void* worker(void* arg) {
  job_t* jb = (job_t*)arg;
  const uint64_t chunk = jb->chunk;
  for (;;) {
    uint64_t b = __atomic_fetch_add(&jb->next, chunk, __ATOMIC_RELAXED);
    if (b >= jb->n) break;
    uint64_t e = b + chunk < jb->n ? b + chunk : jb->n;
    for (uint64_t r = b; r < e; ++r) {
      if (jb->K) trace_one_multi(jb, r);
      else trace_one(jb, r);
    }
  }
  return NULL;
}

static int run_job(job_t* jb, int nthreads);

int oracle_trace(const or_scene* s, const float* rays, uint64_t n, int query, int isect,
                 float thr, uint32_t M, or_hit* hits, uint32_t* flags, uint32_t* ntie,
                 int nthreads) {
  if (!s || !rays || !hits) return -1;
  if (query != OR_CLOSEST && query != OR_ANY) return -1;
  if (isect < OR_NONE || isect > OR_ALPHA_PROC_UV) return -1;
  if ((isect == OR_ALPHA_PROC || isect == OR_ALPHA_PROC_UV) && M == 0) return -1;
  job_t jb;
  memset(&jb, 0, sizeof jb);
  jb.s = s; jb.rays = rays; jb.n = n; jb.query = query; jb.isect = isect;
  jb.thr = thr; jb.M = M; jb.hits = hits; jb.flags = flags; jb.ntie = ntie; jb.next = 0;
  return run_job(&jb, nthreads);
}

int oracle_trace_multi(const or_scene* s, const float* rays, uint64_t n, uint32_t K, int isect,
                       float thr, uint32_t M, or_hit* hits, uint32_t* nhits, uint32_t* ncut,
                       int nthreads) {
  if (!s || !rays || !hits || K < 1) return -1;
  if (isect < OR_NONE || isect > OR_ALPHA_PROC_UV) return -1;
  if ((isect == OR_ALPHA_PROC || isect == OR_ALPHA_PROC_UV) && M == 0) return -1;
  job_t jb;
  memset(&jb, 0, sizeof jb);
  jb.s = s; jb.rays = rays; jb.n = n; jb.query = OR_CLOSEST; jb.isect = isect;
  jb.thr = thr; jb.M = M; jb.hits = hits; jb.K = K; jb.nhits = nhits; jb.ntie = ncut;
  return run_job(&jb, nthreads);
}

static int run_job(job_t* jbp, int nthreads) {
  job_t jb = *jbp;
  if (nthreads < 1) nthreads = 1;
  /* up to 1024 rays per claim, fewer for small inputs so every thread gets work */
  jb.chunk = jb.n / ((uint64_t)nthreads * 4);
  if (jb.chunk < 1) jb.chunk = 1;
  if (jb.chunk > 1024) jb.chunk = 1024;
  if (nthreads == 1) {
    worker(&jb);
    return 0;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, worker, &jb);
  for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
  free(th);
  return 0;
}
