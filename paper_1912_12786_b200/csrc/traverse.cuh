// traverse.cuh — the traversal core every trace kernel shares (
// PAPER.md §3.2): hooks, per-lane state, ray fetch / generation, the inner-node
// and leaf loops, the hit write, the launch-slot -> ray-block mapping of the
// longest-first order, and the PDL launch helper.  Included by trace.cu (plain,
// multi-hit, pinhole, persistent kernels and the order pass), compound.cu
// (lists and instances) and prims.cu (primitive lists).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <string>
#include <utility>

#include "intersectors.cuh"
#include "trace.hpp"

namespace vsr {

#ifndef VSR_BLOCK
#define VSR_BLOCK 128
#endif
constexpr int kBlock = VSR_BLOCK;   // rays per thread block (= per order-pass unit)
constexpr uint32_t kMissPrim = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xFFFFFFFFu;
enum : int { kClosest = 0, kAny = 1, kMulti = 2 };

template <class I>
__device__ __forceinline__ bool box_hook(I& isect, const RayCtx& r, const Aabb& b, float best_t,
                                         float& tn) {
  if constexpr (std::is_same<I, no_intersector>::value) return intersect(r, b, best_t, tn);
  else return isect(r, b, best_t, tn);
}

template <class I, class... Args>
__device__ __forceinline__ BoxPairHit box_pair_hook(I& isect, const RayCtx& r, const AabbPair& b,
                                                    float best_t, Args... args) {
  if constexpr (std::is_same<I, no_intersector>::value) return intersect(r, b, best_t, args...);
  else return isect(r, b, best_t, args...);
}

template <class I>
__device__ __forceinline__ hit_record tri_hook(I& isect, const RayCtx& r, const TriData& t,
                                               uint32_t k, float tmax_cur) {
  if constexpr (std::is_same<I, no_intersector>::value) return intersect(r, t, k, tmax_cur);
  else return isect(r, t, k, tmax_cur);
}

// Per-lane traversal state of one ray.
struct Trav {
  RayCtx r;
  float best_t;   // tmax of the moment; the kept hit's t once prim != kMissPrim
  float u, v;
  uint32_t prim;  // kMissPrim until a hit is kept (the "have" flag)
  uint32_t cur;
  int sp;
};

// Pop the next entry not farther than the current best (reading A14), with the
// same culling bound as the box test (best_t + pad, contract r02).
__device__ __forceinline__ bool pop(Trav& T, const float2* stack) {
  const float bt = cull_t(T.r, T.best_t);
  while (T.sp > 0) {
    --T.sp;
    const float2 e = stack[T.sp];
    if (e.y <= bt) {
      T.cur = __float_as_uint(e.x);
      return true;
    }
  }
  return false;
}

// Any-hit stack: ref only.  Until the first accepted hit ends an any-hit query
// its tmax never shrinks, and every entry was pushed with tnear <= that tmax,
// so the cull above can never fire: dropping tnear changes no result (reading
// A14) and halves the stack's local-memory traffic.
__device__ __forceinline__ bool pop(Trav& T, const uint32_t* stack) {
  if (T.sp == 0) return false;
  T.cur = stack[--T.sp];
  return true;
}

__device__ __forceinline__ void push(Trav& T, float2* stack, uint32_t ref, float tn) {
  VSR_CHECK(T.sp < kMaxStack);
  stack[T.sp++] = make_float2(__uint_as_float(ref), tn);
}
__device__ __forceinline__ void push(Trav& T, uint32_t* stack, uint32_t ref, float) {
  VSR_CHECK(T.sp < kMaxStack);
  stack[T.sp++] = ref;
}

// Stack entry of a query: any-hit keeps refs only (see pop above).
#ifndef VSR_ANY_REFSTACK
#define VSR_ANY_REFSTACK 1
#endif
template <int Q>
using StackEntry =
    typename std::conditional<Q == kAny && VSR_ANY_REFSTACK, uint32_t, float2>::type;

// ---- fused primary-ray generation (vsr.h vsr_pinhole) ----
// Ray `id` of the (8x8 tile, sample, y, x) order, computed with exactly the
// fp64 operations of the input recipe (workloads.pinhole_rays)
// and rounded to fp32, so it is bit-identical to the host-generated ray.
__device__ __forceinline__ uint32_t pcg_hash32(uint64_t x) {
  x &= 0xFFFFFFFFull;
  const uint64_t state = (x * 747796405ull + 2891336453ull) & 0xFFFFFFFFull;
  const uint64_t shift = (state >> 28) + 4ull;
  const uint64_t word = (((state >> shift) ^ state) * 277803737ull) & 0xFFFFFFFFull;
  return (uint32_t)((word >> 22) ^ word);
}

__device__ __forceinline__ void gen_ray(const Pinhole& c, uint64_t id, float4& a, float4& b) {
  const uint64_t per_tile = 64ull * c.spp;
  const uint64_t tile = id / per_tile, rem = id % per_tile;
  const uint32_t smp = (uint32_t)(rem >> 6), q = (uint32_t)(rem & 63u);
  const uint64_t tx = c.width >> 3;
  const uint64_t px = (tile % tx) * 8ull + (q & 7u), py = (tile / tx) * 8ull + (q >> 3);
  double jx = 0.5, jy = 0.5;
  if (c.spp > 1) {
    const uint64_t key = (py * c.width + px) * c.spp + smp;
    const uint64_t seed = (uint64_t)c.seed * 7919ull;
    const double r1 = (double)pcg_hash32(key * 2ull + seed) / 4294967296.0;
    const double r2 = (double)pcg_hash32(key * 2ull + (1ull + seed)) / 4294967296.0;
    jx = ((double)(smp % c.side) + r1) / (double)c.side;
    jy = ((double)(smp / c.side) + r2) / (double)c.side;
  }
  const double sx = 2.0 * ((double)px + jx) / (double)c.width - 1.0;
  const double sy = 1.0 - 2.0 * ((double)py + jy) / (double)c.height;
  const double A = sx * c.tan_half * c.aspect, B = sy * c.tan_half;
  a = make_float4(__double2float_rn(c.eye[0]), __double2float_rn(c.eye[1]),
                  __double2float_rn(c.eye[2]), c.tmin);
  b = make_float4(__double2float_rn((c.w[0] + A * c.u[0]) + B * c.v[0]),
                  __double2float_rn((c.w[1] + A * c.u[1]) + B * c.v[1]),
                  __double2float_rn((c.w[2] + A * c.u[2]) + B * c.v[2]), c.tmax);
}

#ifndef VSR_RAY_NA
#define VSR_RAY_NA 1   // measured +1 % (profiles/r01_tuning.md); 0 = plain __ldg
#endif
template <bool GEN>
__device__ __forceinline__ void fetch_ray(const TraceParams& p, uint64_t id, float4& a, float4& b) {
  if constexpr (GEN) {
    gen_ray(p.cam, id, a, b);
  } else {
#if VSR_RAY_NA
    // rays are read once: no L1 allocation, so they do not evict node lines
    ldg8_na(p.rays + 2 * id, a, b);
#else
    a = __ldg(p.rays + 2 * id);
    b = __ldg(p.rays + 2 * id + 1);
#endif
  }
}

// Load (or generate) ray `id`, test the root box once (counted, reading A11).
// Returns true if the ray needs traversal.
template <bool GEN = false, class I>
__device__ __forceinline__ bool start_ray(const TraceParams& p, Trav& T, I& isect, uint64_t id) {
  float4 a, b;
  fetch_ray<GEN>(p, id, a, b);
  make_ray(T.r, a, b);
  T.best_t = b.w;
  T.u = 0.0f;
  T.v = 0.0f;
  T.prim = kMissPrim;
  T.sp = 0;
  T.cur = p.scene.root_ref;
  isect.reset();
  const Aabb root{p.scene.root_lo[0], p.scene.root_lo[1], p.scene.root_lo[2],
                  p.scene.root_hi[0], p.scene.root_hi[1], p.scene.root_hi[2]};
  float tn;
  return box_hook(isect, T.r, root, T.best_t, tn);
}

// ---- inner-node loop: "while node is inner" ----
// OCT >= 0: the warp's rays all share octant OCT (specialised slab test);
// OCT < 0: generic min/max slab test.  Returns false when the ray is done
// (nothing left to visit), true when T.cur is a leaf.
__device__ __forceinline__ void prefetch_ref(const DevScene& S, uint32_t ref) {
  const void* ptr = (ref & kLeafBit) ? static_cast<const void*>(S.tris + (ref & kLeafFirstMask))
                                     : static_cast<const void*>(S.nodes + ref);
#if VSR_PREFETCH == 1
  asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr));
#elif VSR_PREFETCH == 2
  asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
#else
  (void)ptr;
#endif
}

template <int OCT, class I, class SE>
__device__ __forceinline__ bool descend(const DevScene& S, Trav& T, I& isect, SE* stack) {
  while (!(T.cur & kLeafBit)) {
    VSR_CHECK(T.cur < S.num_nodes);
    const float4* np = reinterpret_cast<const float4*>(S.nodes + T.cur);
    float4 nx, ny, nz, nr;
    ldg8(np, nx, ny);
    ldg8(np + 2, nz, nr);
#if VSR_PREFETCH
    // both children towards L1 while the box tests run (scheduling only)
    prefetch_ref(S, __float_as_uint(nr.x));
    prefetch_ref(S, __float_as_uint(nr.y));
#endif
    BoxPairHit h;
    if constexpr (OCT >= 0) h = box_pair_hook(isect, T.r, AabbPair{nx, ny, nz}, T.best_t, octant<OCT>{});
    else h = box_pair_hook(isect, T.r, AabbPair{nx, ny, nz}, T.best_t);
    const uint32_t r0 = __float_as_uint(nr.x), r1 = __float_as_uint(nr.y);
    if (h.h0 && h.h1) {
      const bool swap = h.tn1 < h.tn0;   // nearer child first, ties -> child 0 (reading A13)
      push(T, stack, swap ? r0 : r1, swap ? h.tn0 : h.tn1);
      T.cur = swap ? r1 : r0;
    } else if (h.h0) {
      T.cur = r0;
    } else if (h.h1) {
      T.cur = r1;
    } else if (!pop(T, stack)) {
      return false;
    }
  }
  return true;
}

// ---- any-hit inner loop without divergent branches (VSR_ANY_SENTINEL) ----
// The any-hit stack holds refs only, and its traversal pushes a sentinel ref
// (leaf bit set) below its entries: the inner loop then never needs an "is the
// stack empty" exit — "neither child hit" pops unconditionally, and popping the
// sentinel leaves the loop as a leaf would.  Push, pop and the next-node choice
// become predicated selects; the node sequence is exactly descend's (same test,
// same order), so results and counts are unchanged.
#ifndef VSR_ANY_SENTINEL
#define VSR_ANY_SENTINEL 0   // 1: measured C2 any +-0 %, C5 any -3.4 % (profiles/r02_tuning.md)
#endif
constexpr uint32_t kSentinel = 0xFFFFFFFFu;

template <int OCT, class I>
__device__ __forceinline__ void descend_any(const DevScene& S, Trav& T, I& isect, uint32_t* stack) {
  while (!(T.cur & kLeafBit)) {
    VSR_CHECK(T.cur < S.num_nodes);
    const float4* np = reinterpret_cast<const float4*>(S.nodes + T.cur);
    const float4 nx = __ldg(np), ny = __ldg(np + 1), nz = __ldg(np + 2);
    const uint2 nr = __ldg(reinterpret_cast<const uint2*>(np + 3));
    // the top entry, read unconditionally (the floor keeps T.sp >= 1): its load
    // overlaps the node's, and the pop needs no branch
    const uint32_t top = stack[T.sp - 1];
    BoxPairHit h;
    if constexpr (OCT >= 0) h = box_pair_hook(isect, T.r, AabbPair{nx, ny, nz}, T.best_t, octant<OCT>{});
    else h = box_pair_hook(isect, T.r, AabbPair{nx, ny, nz}, T.best_t);
    const bool swap = h.tn1 < h.tn0;   // nearer child first, ties -> child 0 (reading A13)
    const uint32_t nearr = (h.h0 && !(h.h1 && swap)) ? nr.x : nr.y;
    if (h.h0 && h.h1) {
      VSR_CHECK(T.sp < kMaxStack);
      stack[T.sp++] = swap ? nr.x : nr.y;
    }
    const bool any = h.h0 || h.h1;
    T.cur = any ? nearr : top;
    T.sp -= any ? 0 : 1;
  }
}

template <class I>
__device__ __forceinline__ void descend_any_oct(const DevScene& S, Trav& T, I& isect,
                                                uint32_t* stack, int oct) {
  switch (oct) {
    case 0: descend_any<0>(S, T, isect, stack); break;
    case 1: descend_any<1>(S, T, isect, stack); break;
    case 2: descend_any<2>(S, T, isect, stack); break;
    case 3: descend_any<3>(S, T, isect, stack); break;
    case 4: descend_any<4>(S, T, isect, stack); break;
    case 5: descend_any<5>(S, T, isect, stack); break;
    case 6: descend_any<6>(S, T, isect, stack); break;
    case 7: descend_any<7>(S, T, isect, stack); break;
    default: descend_any<-1>(S, T, isect, stack); break;
  }
}

// Multi-hit accumulator ("the first N hit points"; SPEC
// S:285-293): the maxk smallest-t accepted hits, ascending t, equal t in
// discovery order; once full, tmax shrinks to the worst kept t.
struct NoMulti {};
template <int K, bool SRC = false>
struct MultiBuf {
  static constexpr bool kSrc = SRC;
  float t[K], u[K], v[K];
  uint32_t prim[K];
  uint32_t src[SRC ? K : 1];   // list / instance index of each kept hit (compound queries)
  uint32_t cur_src;            // the element being traversed
  int n;
  int maxk;
};

// Stable insertion by t into the sorted buffer (equal t keep discovery order); a
// full buffer drops its worst, then tmax shrinks to the new worst.  For K <= 8
// every array index is a compile-time constant (the insertion is a carry that
// walks the K slots: at the first slot holding a larger t it swaps in, every
// later occupied slot shifts, the first empty slot absorbs the carry), so the
// buffer lives in registers instead of local memory.
#ifndef VSR_MULTI_REG
#define VSR_MULTI_REG 0   // 1: register-resident K <= 8 insertion — measured 6 % SLOWER (profiles/r02_tuning.md)
#endif
template <int K, bool SRC>
__device__ __forceinline__ void multi_insert(MultiBuf<K, SRC>& mb, Trav& T, float t, float u,
                                             float v, uint32_t prim) {
  if constexpr (K <= 8 && VSR_MULTI_REG) {
    float ct = t, cu = u, cv = v;
    uint32_t cp = prim, cs = mb.cur_src;
    bool carry = true, shifting = false;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (j < mb.maxk) {
        const bool occ = j < mb.n;
        if (carry && (!occ || shifting || mb.t[j] > ct)) {
          const float t0 = mb.t[j], u0 = mb.u[j], v0 = mb.v[j];
          const uint32_t p0 = mb.prim[j];
          mb.t[j] = ct; mb.u[j] = cu; mb.v[j] = cv; mb.prim[j] = cp;
          ct = t0; cu = u0; cv = v0; cp = p0;
          if constexpr (SRC) {
            const uint32_t s0 = mb.src[j];
            mb.src[j] = cs;
            cs = s0;
          }
          if (occ) shifting = true;
          else carry = false;
        }
      }
    }
    if (mb.n < mb.maxk) ++mb.n;
    if (mb.n == mb.maxk) {
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (j == mb.maxk - 1) T.best_t = mb.t[j];
    }
  } else {
    int pos = mb.n < mb.maxk ? mb.n : mb.maxk - 1;   // a full buffer drops its worst
    while (pos > 0 && mb.t[pos - 1] > t) {          // stable insertion by t
      mb.t[pos] = mb.t[pos - 1];
      mb.u[pos] = mb.u[pos - 1];
      mb.v[pos] = mb.v[pos - 1];
      mb.prim[pos] = mb.prim[pos - 1];
      if constexpr (SRC) mb.src[pos] = mb.src[pos - 1];
      --pos;
    }
    mb.t[pos] = t;
    mb.u[pos] = u;
    mb.v[pos] = v;
    mb.prim[pos] = prim;
    if constexpr (SRC) mb.src[pos] = mb.cur_src;
    if (mb.n < mb.maxk) ++mb.n;
    if (mb.n == mb.maxk) T.best_t = mb.t[mb.maxk - 1];
  }
}

// ---- leaf loop: "while node contains untested primitives" ----
// Returns true when the query is finished (any-hit accepted a primitive).
template <int Q, class I, class M>
__device__ __forceinline__ bool leaf(const DevScene& S, Trav& T, I& isect, M& mb) {
  const uint32_t first = T.cur & kLeafFirstMask;
  const uint32_t end = first + ((T.cur >> kLeafCountShift) & 31u) + 1u;
  VSR_CHECK(end <= S.num_tris);
  for (uint32_t k = first; k < end; ++k) {
    const float4* tp = reinterpret_cast<const float4*>(S.tris + k);
    const TriData td{__ldg(tp), __ldg(tp + 1), __ldg(tp + 2)};
    const hit_record hr = tri_hook(isect, T.r, td, k, T.best_t);
    if constexpr (Q == kMulti) {
      if (hr.hit && (mb.n < mb.maxk || hr.t < T.best_t))
        multi_insert(mb, T, hr.t, hr.u, hr.v, __float_as_uint(td.a.w));
    } else if (Q == kAny) {
      if (hr.hit) {   // any-hit: the first accepted hit ends the query
        T.best_t = hr.t;
        T.u = hr.u;
        T.v = hr.v;
        T.prim = __float_as_uint(td.a.w);
        return true;
      }
    } else if (hr.hit && (T.prim == kMissPrim || hr.t < T.best_t)) {
      // closest-hit: accepted hits shrink tmax; vetoed ones do not
      T.best_t = hr.t;
      T.u = hr.u;
      T.v = hr.v;
      T.prim = __float_as_uint(td.a.w);
    }
  }
  return false;
}

// One outer iteration of "while ray not terminated": descend
// to the next leaf, run its primitives, pop.  Returns true when the ray is done.
template <int Q, int OCT, class I, class SE>
__device__ __forceinline__ bool advance(const DevScene& S, Trav& T, I& isect, SE* stack) {
  NoMulti none;
  if (!descend<OCT>(S, T, isect, stack)) return true;
  if (leaf<Q>(S, T, isect, none)) return true;
  return !pop(T, stack);
}

// Whole traversal of one ray.  `oct` is warp-uniform: 0..7 if every lane of
// the warp has that octant (primary rays: all but the centre row/column
// tiles), 8 otherwise; the switch is taken once per leaf, uniformly.
template <class I, class SE>
__device__ __forceinline__ bool descend_oct(const DevScene& S, Trav& T, I& isect, SE* stack,
                                            int oct) {
  switch (oct) {
    case 0: return descend<0>(S, T, isect, stack);
    case 1: return descend<1>(S, T, isect, stack);
    case 2: return descend<2>(S, T, isect, stack);
    case 3: return descend<3>(S, T, isect, stack);
    case 4: return descend<4>(S, T, isect, stack);
    case 5: return descend<5>(S, T, isect, stack);
    case 6: return descend<6>(S, T, isect, stack);
    case 7: return descend<7>(S, T, isect, stack);
    default: return descend<-1>(S, T, isect, stack);
  }
}

// ---- speculative while-while (Aila & Laine, HPG 2009, "postponed leaves") ----
// The paper's while-while lets a lane that reaches a leaf sit
// idle until every lane of its warp has left the inner-node loop.  Here a lane
// that reaches its first leaf POSTPONES it (keeps the ref in `lf`) and keeps
// descending from its next stack entry; the warp leaves the inner loop once no
// converged lane is still without a postponed leaf, then every lane runs its
// postponed leaf — and the leaf it stands on, if any — in one pass.  Each
// lane's own sequence is still a complete traversal with conservative culls
// (only the ORDER of leaves and inner nodes changes; a closest-hit lane may
// visit nodes with a best_t that a postponed leaf will shrink), so the closest
// t and hit / miss are those of the plain loop; the prim on an exact t tie
// and the hit an any-hit query returns may differ (both are valid answers).
// Counting intersectors keep the plain loop: their counts define walker C's
// visit order (reading A29 / SURVEY §8(c).6).
#ifndef VSR_SPEC
#define VSR_SPEC 0
#endif
constexpr uint32_t kNoRef = 0xFFFFFFFFu;   // never a valid ref (leaf range past kMaxTris)

template <int OCT, class I, class SE>
__device__ __forceinline__ void descend_spec(const DevScene& S, Trav& T, I& isect, SE* stack,
                                             uint32_t& lf) {
  while (!(T.cur & kLeafBit)) {
    VSR_CHECK(T.cur < S.num_nodes);
    const float4* np = reinterpret_cast<const float4*>(S.nodes + T.cur);
    float4 nx, ny, nz, nr;
    ldg8(np, nx, ny);
    ldg8(np + 2, nz, nr);
    BoxPairHit h;
    if constexpr (OCT >= 0) h = box_pair_hook(isect, T.r, AabbPair{nx, ny, nz}, T.best_t, octant<OCT>{});
    else h = box_pair_hook(isect, T.r, AabbPair{nx, ny, nz}, T.best_t);
    const uint32_t r0 = __float_as_uint(nr.x), r1 = __float_as_uint(nr.y);
    if (h.h0 && h.h1) {
      const bool swap = h.tn1 < h.tn0;   // nearer child first, ties -> child 0 (reading A13)
      push(T, stack, swap ? r0 : r1, swap ? h.tn0 : h.tn1);
      T.cur = swap ? r1 : r0;
    } else if (h.h0) {
      T.cur = r0;
    } else if (h.h1) {
      T.cur = r1;
    } else if (!pop(T, stack)) {
      T.cur = kNoRef;
    }
    if ((T.cur & kLeafBit) && T.cur != kNoRef && lf == kNoRef) {   // first leaf: postpone it
      lf = T.cur;
      if (!pop(T, stack)) T.cur = kNoRef;
    }
    if (!__any_sync(__activemask(), lf == kNoRef)) break;   // every lane holds a leaf
  }
}

template <class I, class SE>
__device__ __forceinline__ void descend_spec_oct(const DevScene& S, Trav& T, I& isect, SE* stack,
                                                 int oct, uint32_t& lf) {
  switch (oct) {
    case 0: descend_spec<0>(S, T, isect, stack, lf); break;
    case 1: descend_spec<1>(S, T, isect, stack, lf); break;
    case 2: descend_spec<2>(S, T, isect, stack, lf); break;
    case 3: descend_spec<3>(S, T, isect, stack, lf); break;
    case 4: descend_spec<4>(S, T, isect, stack, lf); break;
    case 5: descend_spec<5>(S, T, isect, stack, lf); break;
    case 6: descend_spec<6>(S, T, isect, stack, lf); break;
    case 7: descend_spec<7>(S, T, isect, stack, lf); break;
    default: descend_spec<-1>(S, T, isect, stack, lf); break;
  }
}

template <int Q, class I, class SE>
__device__ __forceinline__ void traverse_spec(const DevScene& S, Trav& T, I& isect, SE* stack,
                                              int oct) {
  NoMulti none;
  uint32_t lf = kNoRef;
  if (T.cur & kLeafBit) {   // the root is a leaf
    lf = T.cur;
    T.cur = kNoRef;
  }
  for (;;) {
    if (T.cur != kNoRef) descend_spec_oct(S, T, isect, stack, oct, lf);
    while (lf != kNoRef) {   // the postponed leaf, then the one this lane stands on
      const uint32_t at = T.cur;
      T.cur = lf;
      if (leaf<Q>(S, T, isect, none)) return;   // any-hit accepted a primitive
      T.cur = at;
      lf = kNoRef;
      if ((at & kLeafBit) && at != kNoRef) {
        lf = at;
        if (!pop(T, stack)) T.cur = kNoRef;
      }
    }
    if (T.cur == kNoRef) return;
  }
}

// Octant dispatch outside the while-while (OUTER): one switch per ray instead of
// one per leaf, at the price of one leaf-loop copy per octant.  The direct
// trace kernel uses it for its default-occupancy instantiation (measured C2 any
// +1.6 %, closest +1.5 %, C4 any -0.5 %); the 12-CTA variant for scenes larger
// than L2 keeps the per-leaf switch (C5 any -2.1 % with it; profiles/r02_tuning.md).
#ifndef VSR_OCT_OUTER
#define VSR_OCT_OUTER 1   // 0: every kernel keeps the per-leaf switch
#endif
template <int Q, int OCT, class I, class SE, class M>
__device__ __forceinline__ void traverse_fixed(const DevScene& S, Trav& T, I& isect, SE* stack,
                                               M& mb) {
  for (;;) {
    const bool at_leaf = descend<OCT>(S, T, isect, stack);
    if (!at_leaf || leaf<Q>(S, T, isect, mb) || !pop(T, stack)) return;
  }
}

template <int Q, bool OUTER = false, class I, class SE, class M = NoMulti>
__device__ __forceinline__ void traverse(const DevScene& S, Trav& T, I& isect, SE* stack,
                                         int oct, M& mb) {
  if constexpr (VSR_SPEC && Q != kMulti && !I::kCounts && std::is_same<M, NoMulti>::value) {
    traverse_spec<Q>(S, T, isect, stack, oct);
  } else if constexpr (std::is_same<SE, uint32_t>::value && VSR_ANY_SENTINEL) {
    stack[T.sp++] = kSentinel;   // the stack's floor (see descend_any)
    for (;;) {
      descend_any_oct(S, T, isect, stack, oct);
      if (T.cur == kSentinel) return;                 // popped the floor: done
      if (leaf<Q>(S, T, isect, mb)) return;           // any-hit accepted a primitive
      T.cur = stack[--T.sp];                          // next entry (possibly the floor)
    }
  } else if constexpr (OUTER && VSR_OCT_OUTER) {
    switch (oct) {   // once per ray: the whole while-while is specialised per octant
      case 0: traverse_fixed<Q, 0>(S, T, isect, stack, mb); break;
      case 1: traverse_fixed<Q, 1>(S, T, isect, stack, mb); break;
      case 2: traverse_fixed<Q, 2>(S, T, isect, stack, mb); break;
      case 3: traverse_fixed<Q, 3>(S, T, isect, stack, mb); break;
      case 4: traverse_fixed<Q, 4>(S, T, isect, stack, mb); break;
      case 5: traverse_fixed<Q, 5>(S, T, isect, stack, mb); break;
      case 6: traverse_fixed<Q, 6>(S, T, isect, stack, mb); break;
      case 7: traverse_fixed<Q, 7>(S, T, isect, stack, mb); break;
      default: traverse_fixed<Q, -1>(S, T, isect, stack, mb); break;
    }
  } else {
    for (;;) {
      const bool at_leaf = descend_oct(S, T, isect, stack, oct);
      if (!at_leaf || leaf<Q>(S, T, isect, mb) || !pop(T, stack)) return;
    }
  }
}

// Warp-uniform octant of the converged lanes' rays, 8 when they disagree.
__device__ __forceinline__ int warp_octant(const RayCtx& r) {
  const unsigned live = __activemask();
  const int oct = ray_octant(r);
  return __match_any_sync(live, oct) == live ? oct : 8;
}

template <class I>
__device__ __forceinline__ void finish(const TraceParams& p, const Trav& T, const I& isect,
                                       uint64_t id) {
  uint64_t o = id;
  if (p.out_world) {   // vsr_trace_tiles: local tile j is frame tile j*world + rank
    const uint32_t local = (uint32_t)id, tile = local / p.out_tile;
    o = ((uint64_t)tile * p.out_world + p.out_rank) * p.out_tile + (local - tile * p.out_tile);
  }
  // hits may live in a peer GPU's frame buffer (CUDA IPC over NVLink): plain stores,
  // complete when this kernel is
  const float t = T.prim != kMissPrim ? T.best_t : __int_as_float(0x7f800000);
  p.hits[o] = make_float4(t, T.u, T.v, __uint_as_float(T.prim));
  if constexpr (I::kCounts) {
    p.counts[o] = make_uint4(isect.num_boxes, isect.num_tris, isect.lookups(), 0u);
  }
}

template <class I>
__device__ __forceinline__ I make_isect(const TraceParams& p) {
  I isect{};
  if constexpr (std::is_base_of<alpha_texture_intersector, I>::value ||
                std::is_same<I, alpha_bilinear_intersector>::value ||
                std::is_same<I, alpha_procedural_uv_intersector>::value) {
    isect.d = p.data;
  } else if constexpr (std::is_base_of<alpha_procedural_intersector, I>::value) {
    isect.fm = p.data.fm;
  } else if constexpr (std::is_same<I, runtime_switch_intersector>::value) {
    isect.d = p.data;
    isect.kind = p.runtime_kind;
  } else if constexpr (std::is_same<I, runtime_fnptr_intersector>::value) {
    isect.d = p.data;
    isect.fn = reinterpret_cast<filter_fn_t>(p.filter_fn);
  }
  return isect;
}

#ifndef VSR_MINB
#define VSR_MINB 0
#endif
// multi-hit: 10 CTAs/SM (45 registers, no spills) measured +1-3 % over ptxas's own 40 + spills;
// the instance kernel keeps its 64 (bounding it to 10 spills 272 B: -8 %)
#ifndef VSR_MULTI_MINB
#define VSR_MULTI_MINB 10
#endif
#ifndef VSR_INST_MINB
#define VSR_INST_MINB VSR_MINB
#endif
#ifndef VSR_CHUNK
#define VSR_CHUNK 32
#endif
constexpr unsigned kChunk = VSR_CHUNK;   // rays a warp claims per atomicAdd

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// Longest-first block order (scheduling only; results do not depend on it).
// The last rays to start bound a launch's tail by their own latency, so the
// blocks whose rays cross the most of the scene are launched first.  Cost
// proxy per 128-ray block: the longest segment of 4 sample rays inside the
// padded root box, in 128 buckets of the root diagonal; a counting sort
// (histogram + scatter, most expensive bucket first) gives the permutation.
// ---------------------------------------------------------------------------
#ifndef VSR_ORDER_BUCKETS
#define VSR_ORDER_BUCKETS 128
#endif
constexpr int kOrderBuckets = VSR_ORDER_BUCKETS;   // multiple of 32, <= 1024
static_assert(kOrderBuckets % 32 == 0 && kOrderBuckets <= 1024, "bucket count");

// First statement of every trace kernel.  After an order pass the kernel is a
// programmatic dependent launch (PDL): its CTAs may be resident before the
// scatter kernel ends, so it waits for it here (a no-op for a plain launch),
// then reads the permutation through L2 (.cg: no L1 line from an earlier
// launch of the same scratch can be hit) and re-zeroes the histogram for the
// scratch's next use (the stream orders that after this launch).
__device__ __forceinline__ uint64_t launch_block(const TraceParams& p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.hist_reset && blockIdx.x == 0)
    for (int i = threadIdx.x; i < kOrderBuckets; i += blockDim.x) p.hist_reset[i] = 0u;
  return p.perm ? (uint64_t)__ldcg(p.perm + blockIdx.x) : (uint64_t)blockIdx.x;
}

// Point a mask intersector at list element s's texture data (the alpha
// listing's "member variables", differ per BVH).
template <class I>
__device__ __forceinline__ void bind_scene_data(I& isect, const IsectData& d) {
  if constexpr (std::is_base_of<alpha_texture_intersector, I>::value ||
                std::is_same<I, alpha_bilinear_intersector>::value ||
                std::is_same<I, alpha_procedural_uv_intersector>::value) {
    isect.d.sides = d.sides;   // threshold / checker frequency stay the call's
    isect.d.descs = d.descs;
    isect.d.texels = d.texels;
    isect.d.bits = d.bits;     // the element's 1-bit plane (alpha_bits_intersector)
    isect.d.num_texels = d.num_texels;
  } else {
    (void)d;
  }
}

// <<<grid, block, 0, st>>>, as a programmatic dependent launch when `pdl`
// (the kernel starts with griddepcontrol.wait, see launch_block).
// VSR_CARVEOUT=<percent> (tuning knob): the preferred shared-memory carveout of every kernel
// this library launches (0 = the most L1), set once per kernel.
void apply_carveout(const void* kernel);

template <typename... Args, typename... Act>
cudaError_t launch_k(void (*k)(Args...), uint64_t grid, unsigned block, bool pdl, cudaStream_t st,
                     Act&&... args) {
  apply_carveout(reinterpret_cast<const void*>(k));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(block);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Act>(args)...);
}

// Kernels launched by this library (all translation units), for vsr_launch_count.
std::atomic<uint64_t>& launch_counter();

}  // namespace vsr
