// intersectors.cuh — the paper's intersector API on the device.
//
// PAPER.md §3.1: the customization point `intersect(ray, prim) -> hit_record`
// is the default behaviour; a custom intersector derives
// from `basic_intersector<Derived>` (CRTP), re-exports the
// base operator() and overrides the hook it wants.  The
// traversal calls the intersector at both call sites — box and primitive —
// (PAPER.md:248-260), and extra box arguments such as the inverse ray
// direction are forwarded untouched (PAPER.md:337-376 variadic pass-through).
//
// Everything here is resolved at compile time: a kernel instantiated with an
// intersector contains exactly that intersector's code and nothing else
// (PAPER.md:83-89), and the default intersector inlines to the same
// instructions as calling `intersect` directly.
//
// Box tests come in two shapes: a single `Aabb` (the root) and an `AabbPair`
// (both children of a 64-B pair node, tested together with Blackwell's packed
// f32x2 add/mul — one instruction computes the same IEEE result for both
// boxes).  A box hook on an AabbPair stands for two box-hook calls.
//
// Arithmetic follows DESIGN.md §3 "Arithmetic contract" (IEEE fp32 RN, no FMA:
// the translation unit is compiled with -fmad=false and IEEE division).
#pragma once
#include <cstdint>
#include <type_traits>

#include "layout.hpp"

// Bounds-checked builds (-DVSR_CHECKED=1; compute-sanitizer is closed on this GPU pool):
// every node, triangle, sidecar, texel, bit-plane word and stack index is checked on the
// device and a violation traps (the launch fails; tests/test_gpu_checked.py).
#ifndef VSR_CHECKED
#define VSR_CHECKED 0
#endif
#if VSR_CHECKED
#define VSR_CHECK(c) \
  do {               \
    if (!(c)) __trap(); \
  } while (0)
#else
#define VSR_CHECK(c) ((void)0)
#endif

#ifndef VSR_LDG256
#define VSR_LDG256 0   // 1: 256-bit node / ray loads — measured 3-4.5 % SLOWER (profiles/r02_tuning.md)
#endif

namespace vsr {

// ---------------------------------------------------------------------------
// packed fp32x2 helpers (sm_100a FADD2 / FMUL2; each lane is an IEEE RN op)
// ---------------------------------------------------------------------------
typedef unsigned long long f2_t;

__device__ __forceinline__ f2_t pk(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(f2_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t sub2(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// a * b + c with ONE rounding per lane (FFMA2): the slab contract's explicit fma
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

struct RayCtx {
  float ox, oy, oz, tmin;
  float dx, dy, dz;
  float ix, iy, iz;          // guarded reciprocal direction (reading A20)
  float nx, ny, nz;          // noi = -(o * inv), clamped to +-FLT_MAX (slab contract r02)
  float pad;                 // 4 max_k |o_k inv_k + noi_k|: the fma-form slab's allowance
};

// Slab contract r02 (DESIGN.md §3 A.2): a box plane's crossing is ONE fused
// multiply-add, t = fma(plane, inv, noi) with noi = -(o * inv) rounded once per
// ray, instead of (plane - o) * inv.  Error: with e_k = o_k inv_k + noi_k the
// EXACT rounding error of noi_k (fma(o, inv, noi) computes it exactly),
// t = (t*(1+d0) + e)(1+d2): <= 2u relative (covered by the tf widening
// 1 + 2 gamma_3, as before) plus the absolute e, covered by `pad` = 4 max_k |e_k|
// added to tf and to the best_t bound.  Axes with a power-of-two inv (axis-
// parallel rays' guarded 2^80, unit directions) have e = 0.  The clamp keeps every
// value finite (no NaN for any finite input); an overflowing origin term makes
// e, hence pad, infinite: the test then never culls (conservative).
__device__ __forceinline__ float clamp_noi(float x) {
  return fminf(fmaxf(x, -3.40282347e38f), 3.40282347e38f);
}

__device__ __forceinline__ void make_ray(RayCtx& r, float4 a, float4 b) {
  r.ox = a.x; r.oy = a.y; r.oz = a.z; r.tmin = a.w;
  r.dx = b.x; r.dy = b.y; r.dz = b.z;
  r.ix = 1.0f / (fabsf(b.x) > 0x1p-80f ? b.x : copysignf(0x1p-80f, b.x));
  r.iy = 1.0f / (fabsf(b.y) > 0x1p-80f ? b.y : copysignf(0x1p-80f, b.y));
  r.iz = 1.0f / (fabsf(b.z) > 0x1p-80f ? b.z : copysignf(0x1p-80f, b.z));
  r.nx = clamp_noi(-(a.x * r.ix));
  r.ny = clamp_noi(-(a.y * r.iy));
  r.nz = clamp_noi(-(a.z * r.iz));
  const float ex = __fmaf_rn(a.x, r.ix, r.nx), ey = __fmaf_rn(a.y, r.iy, r.ny),
              ez = __fmaf_rn(a.z, r.iz, r.nz);
  r.pad = fmaxf(fmaxf(fabsf(ex), fabsf(ey)), fabsf(ez)) * 4.0f;
}

// Three-input min/max (sm_100 FMNMX3).  min/max are exact and, NaN operands
// being ignored, associative: max3(a, b, c) == fmaxf(fmaxf(a, b), c) bit for bit.
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

struct Aabb {
  float lx, ly, lz, hx, hy, hz;
};

// Both children of a pair node, as stored: per axis (lo0, lo1, hi0, hi1).
struct AabbPair {
  float4 x, y, z;
};

struct BoxPairHit {
  bool h0, h1;
  float tn0, tn1;
};

// Triangle as loaded: v0 (+prim id bits in w), e1, e2 (SPEC S:47 v0/e1/e2).
struct TriData {
  float4 a, b, c;
};

// hit_record<Ray, primitive<unsigned>>: hit flag, t, barycentrics
// and the primitive's position k in the leaf-ordered arrays (the sidecar index;
// PAPER.md:306-308 reads tex_coords[prim_id*3 + i], reading A9).
struct hit_record {
  bool hit;
  float t, u, v;
  uint32_t k;
};

__device__ __forceinline__ float4 ldg4(const void* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

// 256-bit read-only load (sm_100 LDG.E.ENL2.256): 32 B per lane in ONE load
// instruction — a 64-B pair node is two loads instead of four, halving the
// L1 data-pipe wavefronts of a divergent warp's node fetch.  `p` 32-B aligned.
__device__ __forceinline__ void ldg8(const void* p, float4& a, float4& b) {
#if VSR_LDG256
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
#else
  a = __ldg(reinterpret_cast<const float4*>(p));
  b = __ldg(reinterpret_cast<const float4*>(p) + 1);
#endif
}
// the same without L1 allocation (streamed data read once: rays)
__device__ __forceinline__ void ldg8_na(const void* p, float4& a, float4& b) {
#if VSR_LDG256
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
#else
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(p));
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "l"(reinterpret_cast<const float4*>(p) + 1));
#endif
}

// ---------------------------------------------------------------------------
// Default primitive tests (the `intersect` customization points).
// ---------------------------------------------------------------------------

// The culling bound a box test compares tn against: best_t plus the slab's
// absolute error allowance (contract r02), so a box holding a hit at t <= best_t
// is never culled.  Loop-invariant in the inner-node loop (best_t only changes
// in the leaf loop), so it is computed once per descent.
__device__ __forceinline__ float cull_t(const RayCtx& r, float best_t) { return best_t + r.pad; }

// Ray/AABB slab test with the caller-supplied inverse direction (the "special
// interface" of PAPER.md:371-376), clipped to [tmin, best_t]; tf widened by
// (1 + 2*gamma_3) (reading A23) plus `pad` (contract r02).  min/max are exact,
// so their order is free.
__device__ __forceinline__ bool intersect(const RayCtx& r, const Aabb& b, float best_t,
                                          float& tn) {
  const float t0x = __fmaf_rn(b.lx, r.ix, r.nx), t1x = __fmaf_rn(b.hx, r.ix, r.nx);
  const float t0y = __fmaf_rn(b.ly, r.iy, r.ny), t1y = __fmaf_rn(b.hy, r.iy, r.ny);
  const float t0z = __fmaf_rn(b.lz, r.iz, r.nz), t1z = __fmaf_rn(b.hz, r.iz, r.nz);
  const float n = fmax3(fminf(t0x, t1x), fminf(t0y, t1y), fmaxf(fminf(t0z, t1z), r.tmin));
  float f = __fmaf_rn(fmin3(fmaxf(t0x, t1x), fmaxf(t0y, t1y), fmaxf(t0z, t1z)), 1.0000003576f,
                      r.pad);
  f = fminf(f, cull_t(r, best_t));
  tn = n;
  return n <= f;
}

// The same test on both children of a pair node at once: every fma is the
// scalar contract's operation, done two at a time (FFMA2).
__device__ __forceinline__ BoxPairHit intersect(const RayCtx& r, const AabbPair& b,
                                                float best_t) {
  float t0x0, t0x1, t1x0, t1x1, t0y0, t0y1, t1y0, t1y1, t0z0, t0z1, t1z0, t1z1;
  // (noi.k, noi.k) and (inv.k, inv.k) are broadcast operands (SASS ".F32" form)
  const f2_t nx2 = pk(r.nx, r.nx), ny2 = pk(r.ny, r.ny), nz2 = pk(r.nz, r.nz);
  const f2_t ix2 = pk(r.ix, r.ix), iy2 = pk(r.iy, r.iy), iz2 = pk(r.iz, r.iz);
  upk(fma2(pk(b.x.x, b.x.y), ix2, nx2), t0x0, t0x1);
  upk(fma2(pk(b.x.z, b.x.w), ix2, nx2), t1x0, t1x1);
  upk(fma2(pk(b.y.x, b.y.y), iy2, ny2), t0y0, t0y1);
  upk(fma2(pk(b.y.z, b.y.w), iy2, ny2), t1y0, t1y1);
  upk(fma2(pk(b.z.x, b.z.y), iz2, nz2), t0z0, t0z1);
  upk(fma2(pk(b.z.z, b.z.w), iz2, nz2), t1z0, t1z1);
  BoxPairHit h;
  h.tn0 = fmax3(fminf(t0x0, t1x0), fminf(t0y0, t1y0), fmaxf(fminf(t0z0, t1z0), r.tmin));
  h.tn1 = fmax3(fminf(t0x1, t1x1), fminf(t0y1, t1y1), fmaxf(fminf(t0z1, t1z1), r.tmin));
  const float f0 = fmin3(fmaxf(t0x0, t1x0), fmaxf(t0y0, t1y0), fmaxf(t0z0, t1z0));
  const float f1 = fmin3(fmaxf(t0x1, t1x1), fmaxf(t0y1, t1y1), fmaxf(t0z1, t1z1));
  float g0, g1;
  upk(fma2(pk(f0, f1), pk(1.0000003576f, 1.0000003576f), pk(r.pad, r.pad)), g0, g1);
  const float bt = cull_t(r, best_t);
  h.h0 = h.tn0 <= fminf(g0, bt);
  h.h1 = h.tn1 <= fminf(g1, bt);
  return h;
}

// ---------------------------------------------------------------------------
// The 8 quantized child boxes of a wide node (wide.hpp, SURVEY.md §8(f)
// NEXT-3), as loaded: h = (pm.x, pm.y, pm.z, e bytes | imask << 24); per axis
// the lower and upper plane codes of slots 0-3 and 4-7 (one byte each):
// q0 = (lo.x 0-3, lo.x 4-7, lo.y 0-3, lo.y 4-7), q1 = (lo.z 0-3, lo.z 4-7,
// hi.x 0-3, hi.x 4-7), q2 = (hi.y 0-3, hi.y 4-7, hi.z 0-3, hi.z 4-7).
// A box hook on an AabbOct stands for one box-hook call per VALID child.
// ---------------------------------------------------------------------------
struct AabbOct {
  float4 h;
  uint4 q0, q1, q2;
};

// 2^23 + byte j of w, as a float (PRMT: the byte becomes the mantissa)
__device__ __forceinline__ float qbyte(uint32_t w, int j) {
  return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u | (uint32_t)j));
}

// t of the 8 slots' planes on one axis: plane = fma(2^23 + q, scale, pm) (the
// decode, one rounding), then the r02 slab crossing fma(plane, inv, noi).
__device__ __forceinline__ void oct_axis(uint32_t w03, uint32_t w47, float scale, float pm,
                                         float inv, float noi, float (&t)[8]) {
  const f2_t s2 = pk(scale, scale), p2 = pk(pm, pm), i2 = pk(inv, inv), n2 = pk(noi, noi);
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const uint32_t w = j < 4 ? w03 : w47;
    upk(fma2(fma2(pk(qbyte(w, j & 3), qbyte(w, (j & 3) + 1)), s2, p2), i2, n2), t[j], t[j + 1]);
  }
}

__device__ __forceinline__ float oct_scale(uint32_t hw, int a) {
  return __uint_as_float(((hw >> (8 * a)) & 0xFFu) << 23);
}

// Slot hit mask of the 8 children (generic: per-axis min/max).  Bits of slots
// that are not valid children are meaningless (the caller masks them).
__device__ __forceinline__ uint32_t intersect(const RayCtx& r, const AabbOct& b, float best_t,
                                              uint32_t /*valid*/) {
  const uint32_t hw = __float_as_uint(b.h.w);
  // axis by axis, folded into the running entry / exit so at most 4 arrays live
  float tn[8], tf[8], a[8], c[8];
  oct_axis(b.q0.x, b.q0.y, oct_scale(hw, 0), b.h.x, r.ix, r.nx, a);
  oct_axis(b.q1.z, b.q1.w, oct_scale(hw, 0), b.h.x, r.ix, r.nx, c);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    tn[j] = fmaxf(fminf(a[j], c[j]), r.tmin);
    tf[j] = fmaxf(a[j], c[j]);
  }
  oct_axis(b.q0.z, b.q0.w, oct_scale(hw, 1), b.h.y, r.iy, r.ny, a);
  oct_axis(b.q2.x, b.q2.y, oct_scale(hw, 1), b.h.y, r.iy, r.ny, c);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    tn[j] = fmaxf(tn[j], fminf(a[j], c[j]));
    tf[j] = fminf(tf[j], fmaxf(a[j], c[j]));
  }
  oct_axis(b.q1.x, b.q1.y, oct_scale(hw, 2), b.h.z, r.iz, r.nz, a);
  oct_axis(b.q2.z, b.q2.w, oct_scale(hw, 2), b.h.z, r.iz, r.nz, c);
  const float bt = cull_t(r, best_t);
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float n0 = fmaxf(tn[j], fminf(a[j], c[j])), n1 = fmaxf(tn[j + 1], fminf(a[j + 1], c[j + 1]));
    float g0, g1;
    upk(fma2(pk(fminf(tf[j], fmaxf(a[j], c[j])), fminf(tf[j + 1], fmaxf(a[j + 1], c[j + 1]))),
             pk(1.0000003576f, 1.0000003576f), pk(r.pad, r.pad)),
        g0, g1);
    m |= (n0 <= fminf(g0, bt) ? 1u : 0u) << j;
    m |= (n1 <= fminf(g1, bt) ? 1u : 0u) << (j + 1);
  }
  return m;
}

// Ray octant (sign bits of inv.x, inv.y, inv.z) known at compile time: an
// extra box-hook argument, forwarded like the paper's inverse direction
// (PAPER.md:371-376).
template <int OCT>
struct octant {};

// Octant-specialised pair slab test.  With lo <= hi (validated on import) and
// inv never 0 or NaN (guarded reciprocal), the exact products lo*inv and hi*inv
// are ordered, the addend noi is shared and rounding is monotone, so
// min(fma(lo,inv,noi), fma(hi,inv,noi)) is exactly the near-plane term and max
// the far one: selecting the planes at compile time gives bit-identical tn/tf to
// the generic test above without its 12 per-axis min/max.
template <int OCT>
__device__ __forceinline__ BoxPairHit intersect(const RayCtx& r, const AabbPair& b, float best_t,
                                                octant<OCT>) {
  constexpr bool sx = OCT & 1, sy = OCT & 2, sz = OCT & 4;
  const f2_t nx2 = pk(r.nx, r.nx), ny2 = pk(r.ny, r.ny), nz2 = pk(r.nz, r.nz);
  const f2_t ix2 = pk(r.ix, r.ix), iy2 = pk(r.iy, r.iy), iz2 = pk(r.iz, r.iz);
  const f2_t lox = pk(b.x.x, b.x.y), hix = pk(b.x.z, b.x.w);
  const f2_t loy = pk(b.y.x, b.y.y), hiy = pk(b.y.z, b.y.w);
  const f2_t loz = pk(b.z.x, b.z.y), hiz = pk(b.z.z, b.z.w);
  float nx0, nx1, fx0, fx1, ny0, ny1, fy0, fy1, nz0, nz1, fz0, fz1;
  upk(fma2(sx ? hix : lox, ix2, nx2), nx0, nx1);
  upk(fma2(sx ? lox : hix, ix2, nx2), fx0, fx1);
  upk(fma2(sy ? hiy : loy, iy2, ny2), ny0, ny1);
  upk(fma2(sy ? loy : hiy, iy2, ny2), fy0, fy1);
  upk(fma2(sz ? hiz : loz, iz2, nz2), nz0, nz1);
  upk(fma2(sz ? loz : hiz, iz2, nz2), fz0, fz1);
  BoxPairHit h;
  h.tn0 = fmax3(nx0, ny0, fmaxf(nz0, r.tmin));
  h.tn1 = fmax3(nx1, ny1, fmaxf(nz1, r.tmin));
  float g0, g1;
  upk(fma2(pk(fmin3(fx0, fy0, fz0), fmin3(fx1, fy1, fz1)),
           pk(1.0000003576f, 1.0000003576f), pk(r.pad, r.pad)),
      g0, g1);
  const float bt = cull_t(r, best_t);
  h.h0 = h.tn0 <= fminf(g0, bt);
  h.h1 = h.tn1 <= fminf(g1, bt);
  return h;
}

// Octant-specialised slot hit mask: the near / far code words of each axis are
// chosen at compile time (the same monotonicity argument as the pair test:
// plane(q) is nondecreasing in q and fma(plane, inv, noi) is monotone in the
// plane, so for inv > 0 the lower code gives the entry crossing).
template <int OCT>
__device__ __forceinline__ uint32_t intersect(const RayCtx& r, const AabbOct& b, float best_t,
                                              uint32_t /*valid*/, octant<OCT>) {
  constexpr bool sx = OCT & 1, sy = OCT & 2, sz = OCT & 4;
  const uint32_t hw = __float_as_uint(b.h.w);
  // axis by axis, folded into the running entry / exit so at most 4 arrays live
  float tn[8], tf[8], a[8], c[8];
  oct_axis(sx ? b.q1.z : b.q0.x, sx ? b.q1.w : b.q0.y, oct_scale(hw, 0), b.h.x, r.ix, r.nx, tn);
  oct_axis(sx ? b.q0.x : b.q1.z, sx ? b.q0.y : b.q1.w, oct_scale(hw, 0), b.h.x, r.ix, r.nx, tf);
  oct_axis(sy ? b.q2.x : b.q0.z, sy ? b.q2.y : b.q0.w, oct_scale(hw, 1), b.h.y, r.iy, r.ny, a);
  oct_axis(sy ? b.q0.z : b.q2.x, sy ? b.q0.w : b.q2.y, oct_scale(hw, 1), b.h.y, r.iy, r.ny, c);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    tn[j] = fmax3(tn[j], a[j], r.tmin);
    tf[j] = fminf(tf[j], c[j]);
  }
  oct_axis(sz ? b.q2.z : b.q1.x, sz ? b.q2.w : b.q1.y, oct_scale(hw, 2), b.h.z, r.iz, r.nz, a);
  oct_axis(sz ? b.q1.x : b.q2.z, sz ? b.q1.y : b.q2.w, oct_scale(hw, 2), b.h.z, r.iz, r.nz, c);
  const float bt = cull_t(r, best_t);
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float n0 = fmaxf(tn[j], a[j]), n1 = fmaxf(tn[j + 1], a[j + 1]);
    float g0, g1;
    upk(fma2(pk(fminf(tf[j], c[j]), fminf(tf[j + 1], c[j + 1])),
             pk(1.0000003576f, 1.0000003576f), pk(r.pad, r.pad)),
        g0, g1);
    m |= (n0 <= fminf(g0, bt) ? 1u : 0u) << j;
    m |= (n1 <= fminf(g1, bt) ? 1u : 0u) << (j + 1);
  }
  return m;
}

__device__ __forceinline__ int ray_octant(const RayCtx& r) {
  return (int)(__float_as_uint(r.ix) >> 31) | (int)((__float_as_uint(r.iy) >> 31) << 1) |
         (int)((__float_as_uint(r.iz) >> 31) << 2);
}

// Ray/triangle: Möller–Trumbore in textbook order (DESIGN.md
// A.1), no culling, |det| < 1e-12 -> miss, t in [tmin, tmax_cur] inclusive.
__device__ __forceinline__ hit_record intersect(const RayCtx& r, const TriData& tri, uint32_t k,
                                                float tmax_cur) {
  hit_record hr;
  hr.k = k;
  const float e1x = tri.b.x, e1y = tri.b.y, e1z = tri.b.z;
  const float e2x = tri.c.x, e2y = tri.c.y, e2z = tri.c.z;
#ifdef VSR_SCALAR_MT
  // p = cross(d, e2)
  const float px = r.dy * e2z - r.dz * e2y;
  const float py = r.dz * e2x - r.dx * e2z;
  const float pz = r.dx * e2y - r.dy * e2x;
  const float det = (e1x * px + e1y * py) + e1z * pz;
  const float inv = 1.0f / det;
  const float sx = r.ox - tri.a.x, sy = r.oy - tri.a.y, sz = r.oz - tri.a.z;
  const float u = ((sx * px + sy * py) + sz * pz) * inv;
  // q = cross(s, e1)
  const float qx = sy * e1z - sz * e1y;
  const float qy = sz * e1x - sx * e1z;
  const float qz = sx * e1y - sy * e1x;
  const float v = ((r.dx * qx + r.dy * qy) + r.dz * qz) * inv;
  const float t = ((e2x * qx + e2y * qy) + e2z * qz) * inv;
#else
  // The same operations, the independent (x, y) pairs issued as FMUL2/FADD2
  // (each lane one IEEE RN op, so every value is bit-identical to the scalar
  // textbook order of DESIGN.md A.1; VSR_SCALAR_MT builds the scalar form).
  // p = cross(d, e2)
  const float px = r.dy * e2z - r.dz * e2y;
  const float py = r.dz * e2x - r.dx * e2z;
  const float pz = r.dx * e2y - r.dy * e2x;
  const f2_t pxy = pk(px, py);
  float ax, ay;
  upk(mul2(pk(e1x, e1y), pxy), ax, ay);                 // (e1x*px, e1y*py)
  const float det = (ax + ay) + e1z * pz;
  const float inv = 1.0f / det;
  float sx, sy;
  upk(sub2(pk(r.ox, r.oy), pk(tri.a.x, tri.a.y)), sx, sy);
  const float sz = r.oz - tri.a.z;
  float bx, by;
  upk(mul2(pk(sx, sy), pxy), bx, by);                   // (sx*px, sy*py)
  const float U = (bx + by) + sz * pz;
  // q = cross(s, e1)
  const float qx = sy * e1z - sz * e1y;
  const float qy = sz * e1x - sx * e1z;
  const float qz = sx * e1y - sy * e1x;
  const f2_t qxy = pk(qx, qy);
  float cx, cy, gx, gy;
  upk(mul2(pk(r.dx, r.dy), qxy), cx, cy);               // (dx*qx, dy*qy)
  upk(mul2(pk(e2x, e2y), qxy), gx, gy);                 // (e2x*qx, e2y*qy)
  const float V = (cx + cy) + r.dz * qz;
  const float T = (gx + gy) + e2z * qz;
  float u, v;
  upk(mul2(pk(U, V), pk(inv, inv)), u, v);
  const float t = T * inv;
#endif
  hr.t = t;
  hr.u = u;
  hr.v = v;
  hr.hit = (fabsf(det) >= 1e-12f) && (u >= 0.0f) && (u <= 1.0f) && (v >= 0.0f) &&
           (u + v <= 1.0f) && (t >= r.tmin) && (t <= tmax_cur);
  return hr;
}

// ---------------------------------------------------------------------------
// basic_intersector<Derived>: both hooks forward.
// ---------------------------------------------------------------------------
template <class Derived>
struct basic_intersector {
  static constexpr bool kCounts = false;
  template <class... Args>
  __device__ __forceinline__ bool operator()(const RayCtx& r, const Aabb& b, Args&&... args) {
    return intersect(r, b, static_cast<Args&&>(args)...);
  }
  template <class... Args>
  __device__ __forceinline__ BoxPairHit operator()(const RayCtx& r, const AabbPair& b,
                                                   Args&&... args) {
    return intersect(r, b, static_cast<Args&&>(args)...);
  }
  template <class... Args>
  __device__ __forceinline__ uint32_t operator()(const RayCtx& r, const AabbOct& b, float best_t,
                                                 uint32_t valid, Args&&... args) {
    return intersect(r, b, best_t, valid, static_cast<Args&&>(args)...);
  }
  __device__ __forceinline__ hit_record operator()(const RayCtx& r, const TriData& t, uint32_t k,
                                                   float tmax_cur) {
    return intersect(r, t, k, tmax_cur);
  }
  __device__ __forceinline__ void reset() {}
  __device__ __forceinline__ uint32_t lookups() const { return 0u; }
};

// Tag for the default overload without an intersector:
// the traversal calls `intersect` itself.
struct no_intersector {
  static constexpr bool kCounts = false;
  __device__ __forceinline__ void reset() {}
  __device__ __forceinline__ uint32_t lookups() const { return 0u; }
};

// DEFAULT: a user intersector that overrides nothing.
struct default_intersector : basic_intersector<default_intersector> {
  using basic_intersector<default_intersector>::operator();
};

// nearest + wrap addressing on the integer texel index (reading A6)
__device__ __forceinline__ uint32_t wrap_texel(float x, uint32_t n) {
  const int i = (int)floorf(x * (float)n);
  if ((n & (n - 1u)) == 0u) return (uint32_t)i & (n - 1u);
  const int m = (int)n;
  return (uint32_t)(((i % m) + m) % m);
}

// The §4 alpha-mask filter body: lerp the three texcoords with (u, v), tex2D,
// test alpha against the threshold.
__device__ __forceinline__ bool alpha_keep(const IsectData& d, const float4 s0, const float4 s1,
                                           float u, float v) {
  const float w = (1.0f - u) - v;
  const float s = (w * s0.x + u * s0.z) + v * s1.x;
  const float t = (w * s0.y + u * s0.w) + v * s1.y;
  const uint32_t dims = __float_as_uint(s1.w);
  const uint32_t tw = (dims & 0xFFFFu) + 1u, th = (dims >> 16) + 1u;
  const uint32_t i = wrap_texel(s, tw);
  const uint32_t j = wrap_texel(t, th);
  VSR_CHECK((uint64_t)__float_as_uint(s1.z) + (uint64_t)j * tw + i < d.num_texels);
  const uint32_t a8 = __ldg(d.texels + (uint64_t)__float_as_uint(s1.z) + (uint64_t)j * tw + i);
  return a8 >= d.a_min;
}

__device__ __forceinline__ bool alpha_keep(const IsectData& d, uint32_t k, float u, float v) {
  return alpha_keep(d, ldg4(d.sides + k), ldg4(reinterpret_cast<const float4*>(d.sides + k) + 1),
                    u, v);
}

// The same decision read from the 1-bit plane (a8 >= a_min) of the call's
// threshold (SURVEY.md §8(f) NEXT-4 "1-bit alpha plane"): texel (i, j) of a
// texture whose A8 texels start at offset O is bit (i & 31) of word
// O/32 + ((j/32)·(W/32) + i/32)·32 + (j & 31) — 32×32-texel tiles of 32 words,
// one 128-B line each, so rays landing near each other on a billboard share
// lines in both directions. Same (i, j) as alpha_keep, same comparison made
// once per texel on the host's behalf: identical results. Only used when every
// texture's W and H are multiples of 32 (O is then a multiple of 1024).
__device__ __forceinline__ bool alpha_keep_bits(const IsectData& d, uint32_t k, float u, float v) {
  const float4 s0 = ldg4(d.sides + k);
  const float4 s1 = ldg4(reinterpret_cast<const float4*>(d.sides + k) + 1);
  const float w = (1.0f - u) - v;
  const float s = (w * s0.x + u * s0.z) + v * s1.x;
  const float t = (w * s0.y + u * s0.w) + v * s1.y;
  const uint32_t dims = __float_as_uint(s1.w);
  const uint32_t tw = (dims & 0xFFFFu) + 1u, th = (dims >> 16) + 1u;
  const uint32_t i = wrap_texel(s, tw);
  const uint32_t j = wrap_texel(t, th);
  const uint32_t word = (__float_as_uint(s1.z) >> 5) +
                        ((((j >> 5) * (tw >> 5) + (i >> 5)) << 5) | (j & 31u));
  VSR_CHECK(word < d.num_texels / 32);
  return (__ldg(d.bits + word) >> (i & 31u)) & 1u;
}

// NEXT-4 variant (reading A28): bilinear tex2D of the A8 plane, texel centres at
// (i+.5)/W, wrap; the filtered alpha is compared with the threshold itself.
// |texcoord| <= 1024 and W <= 65536 keep every index within int32
__device__ __forceinline__ uint32_t wrap_i(int i, uint32_t n) {
  if ((n & (n - 1u)) == 0u) return (uint32_t)i & (n - 1u);
  const int m = (int)n;
  return (uint32_t)(((i % m) + m) % m);
}

__device__ __forceinline__ bool alpha_bilinear_keep(const IsectData& d, uint32_t k, float u,
                                                    float v) {
  const float4 s0 = ldg4(d.sides + k);
  const float4 s1 = ldg4(reinterpret_cast<const float4*>(d.sides + k) + 1);
  const float w = (1.0f - u) - v;
  const float s = (w * s0.x + u * s0.z) + v * s1.x;
  const float t = (w * s0.y + u * s0.w) + v * s1.y;
  const uint32_t dims = __float_as_uint(s1.w);
  const uint32_t tw = (dims & 0xFFFFu) + 1u, th = (dims >> 16) + 1u;
  const float x = s * (float)tw - 0.5f, y = t * (float)th - 0.5f;
  const float x0 = floorf(x), y0 = floorf(y);
  const float fx = x - x0, fy = y - y0;
  const uint32_t i0 = wrap_i((int)x0, tw), i1 = wrap_i((int)x0 + 1, tw);
  const uint64_t r0 = (uint64_t)wrap_i((int)y0, th) * tw, r1 = (uint64_t)wrap_i((int)y0 + 1, th) * tw;
  const uint8_t* p = d.texels + __float_as_uint(s1.z);
  VSR_CHECK((uint64_t)__float_as_uint(s1.z) + r0 + i0 < d.num_texels &&
            (uint64_t)__float_as_uint(s1.z) + r0 + i1 < d.num_texels &&
            (uint64_t)__float_as_uint(s1.z) + r1 + i0 < d.num_texels &&
            (uint64_t)__float_as_uint(s1.z) + r1 + i1 < d.num_texels);
  const float a00 = (float)__ldg(p + r0 + i0) / 255.0f;
  const float a10 = (float)__ldg(p + r0 + i1) / 255.0f;
  const float a01 = (float)__ldg(p + r1 + i0) / 255.0f;
  const float a11 = (float)__ldg(p + r1 + i1) / 255.0f;
  const float a = ((1.0f - fx) * a00 + fx * a10) * (1.0f - fy) + ((1.0f - fx) * a01 + fx * a11) * fy;
  return a >= d.thr;
}

// NEXT-4 variant (reading A28): the procedural checker on the interpolated
// texcoords (s, t) instead of the barycentrics.
__device__ __forceinline__ bool checker_uv_keep(const IsectData& d, uint32_t k, float u, float v) {
  const float4 s0 = ldg4(d.sides + k);
  const float4 s1 = ldg4(reinterpret_cast<const float4*>(d.sides + k) + 1);
  const float w = (1.0f - u) - v;
  const float s = (w * s0.x + u * s0.z) + v * s1.x;
  const float t = (w * s0.y + u * s0.w) + v * s1.y;
  const long long cs = (long long)floorf(s * d.fm), ct = (long long)floorf(t * d.fm);
  return ((cs + ct) & 1ll) == 0;   // s*M may exceed int32 (|s| <= 1024, M <= 2^24)
}

// §4 procedural mask, read as a barycentric checkerboard (readings A4/A5).
__device__ __forceinline__ bool checker_keep(float fm, float u, float v) {
  const int cu = (int)floorf(u * fm);
  const int cv = (int)floorf(v * fm);
  return ((cu + cv) & 1) == 0;
}

// ALPHA_TEXTURE: the §4 listing.  Only the triangle hook is
// overridden; the box hooks are inherited (SPEC S:226 design decision).
struct alpha_texture_intersector : basic_intersector<alpha_texture_intersector> {
  using basic_intersector<alpha_texture_intersector>::operator();
  IsectData d;
  uint32_t n_lookups = 0;
  __device__ __forceinline__ hit_record operator()(const RayCtx& r, const TriData& t, uint32_t k,
                                                   float tmax_cur) {
    hit_record hr = intersect(r, t, k, tmax_cur);
    if (hr.hit) {   // look up only on a geometric hit (reading A3); fetching the
      ++n_lookups;  // sidecar before the test was measured slower (+8 registers)
      hr.hit &= alpha_keep(d, hr.k, hr.u, hr.v);
    }
    return hr;
  }
  __device__ __forceinline__ void reset() { n_lookups = 0; }
  __device__ __forceinline__ uint32_t lookups() const { return n_lookups; }
};

// ALPHA_TEXTURE through the 1-bit plane (alpha_keep_bits): chosen by the host
// for VSR_ISECT_ALPHA_TEXTURE when the scene's plane for the call's threshold
// exists; otherwise alpha_texture_intersector reads the A8 plane.
#ifndef VSR_SIDE_PF
#define VSR_SIDE_PF 0   // 1: prefetch the triangle's alpha sidecar into L1 before the MT test
#endif
struct alpha_bits_intersector : alpha_texture_intersector {
  using alpha_texture_intersector::operator();
  __device__ __forceinline__ hit_record operator()(const RayCtx& r, const TriData& t, uint32_t k,
                                                   float tmax_cur) {
#if VSR_SIDE_PF
    asm volatile("prefetch.global.L1 [%0];" ::"l"(d.sides + k));
#endif
    hit_record hr = intersect(r, t, k, tmax_cur);
    if (hr.hit) {
      ++n_lookups;
      hr.hit &= alpha_keep_bits(d, hr.k, hr.u, hr.v);
    }
    return hr;
  }
};

// ALPHA_PROCEDURAL.
struct alpha_procedural_intersector : basic_intersector<alpha_procedural_intersector> {
  using basic_intersector<alpha_procedural_intersector>::operator();
  float fm;
  __device__ __forceinline__ hit_record operator()(const RayCtx& r, const TriData& t, uint32_t k,
                                                   float tmax_cur) {
    hit_record hr = intersect(r, t, k, tmax_cur);
    if (hr.hit) hr.hit &= checker_keep(fm, hr.u, hr.v);
    return hr;
  }
};

// ALPHA_TEXTURE_BILINEAR / ALPHA_PROCEDURAL_UV: the NEXT-4 sampling variants
// (reading A28), reported apart from the headline.
struct alpha_bilinear_intersector : basic_intersector<alpha_bilinear_intersector> {
  using basic_intersector<alpha_bilinear_intersector>::operator();
  IsectData d;
  __device__ __forceinline__ hit_record operator()(const RayCtx& r, const TriData& t, uint32_t k,
                                                   float tmax_cur) {
    hit_record hr = intersect(r, t, k, tmax_cur);
    if (hr.hit) hr.hit &= alpha_bilinear_keep(d, hr.k, hr.u, hr.v);
    return hr;
  }
};

struct alpha_procedural_uv_intersector : basic_intersector<alpha_procedural_uv_intersector> {
  using basic_intersector<alpha_procedural_uv_intersector>::operator();
  IsectData d;
  __device__ __forceinline__ hit_record operator()(const RayCtx& r, const TriData& t, uint32_t k,
                                                   float tmax_cur) {
    hit_record hr = intersect(r, t, k, tmax_cur);
    if (hr.hit) hr.hit &= checker_uv_keep(d, hr.k, hr.u, hr.v);
    return hr;
  }
};

// bvh_costs: intercept and count both hooks, then forward.
// Stacked on any other intersector (Inner), the counts are those of Inner's
// traversal; COUNT uses the default one, as in the listing.
template <class Inner>
struct cost_intersector : Inner {
  static constexpr bool kCounts = true;
  uint32_t num_boxes = 0;
  uint32_t num_tris = 0;
  template <class... Args>
  __device__ __forceinline__ bool operator()(const RayCtx& r, const Aabb& b, Args&&... args) {
    ++num_boxes;
    return Inner::operator()(r, b, static_cast<Args&&>(args)...);
  }
  template <class... Args>
  __device__ __forceinline__ BoxPairHit operator()(const RayCtx& r, const AabbPair& b,
                                                   Args&&... args) {
    num_boxes += 2;   // two box tests: one per child
    return Inner::operator()(r, b, static_cast<Args&&>(args)...);
  }
  template <class... Args>
  __device__ __forceinline__ uint32_t operator()(const RayCtx& r, const AabbOct& b, float best_t,
                                                 uint32_t valid, Args&&... args) {
    num_boxes += (uint32_t)__popc(valid);   // one box test per valid child of the wide node
    return Inner::operator()(r, b, best_t, valid, static_cast<Args&&>(args)...);
  }
  __device__ __forceinline__ hit_record operator()(const RayCtx& r, const TriData& t, uint32_t k,
                                                   float tmax_cur) {
    ++num_tris;
    return Inner::operator()(r, t, k, tmax_cur);
  }
  __device__ __forceinline__ void reset() {
    num_boxes = 0;
    num_tris = 0;
    Inner::reset();
  }
};

// ---------------------------------------------------------------------------
// Measurement controls (never a default path): the run-time alternatives the
// paper contrasts with (Embree intersection filter / OptiX
// any-hit program).  Same traversal; the filter is chosen while tracing.
// ---------------------------------------------------------------------------
enum : int { kFilterDefault = 1, kFilterAlphaTex = 2, kFilterAlphaProc = 3 };

struct runtime_switch_intersector : basic_intersector<runtime_switch_intersector> {
  using basic_intersector<runtime_switch_intersector>::operator();
  IsectData d;
  int kind;
  __device__ __forceinline__ hit_record operator()(const RayCtx& r, const TriData& t, uint32_t k,
                                                   float tmax_cur) {
    hit_record hr = intersect(r, t, k, tmax_cur);
    if (hr.hit) {
      switch (kind) {
        case kFilterAlphaTex: hr.hit &= alpha_keep(d, hr.k, hr.u, hr.v); break;
        case kFilterAlphaProc: hr.hit &= checker_keep(d.fm, hr.u, hr.v); break;
        default: break;
      }
    }
    return hr;
  }
};

typedef bool (*filter_fn_t)(const IsectData*, uint32_t, float, float);

struct runtime_fnptr_intersector : basic_intersector<runtime_fnptr_intersector> {
  using basic_intersector<runtime_fnptr_intersector>::operator();
  IsectData d;
  filter_fn_t fn;   // nullptr == no filter registered
  __device__ __forceinline__ hit_record operator()(const RayCtx& r, const TriData& t, uint32_t k,
                                                   float tmax_cur) {
    hit_record hr = intersect(r, t, k, tmax_cur);
    if (hr.hit && fn != nullptr) hr.hit &= fn(&d, hr.k, hr.u, hr.v);
    return hr;
  }
};

}  // namespace vsr
