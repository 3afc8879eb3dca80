// trace.cu — the hot path: per-ray BVH traversal + ray/triangle intersection
// with a compile-time intersector (§3.2).
//
// Traversal: the while-while scheme of Aila & Laine cited by the paper
// (PAPER.md:228-247): an inner-node loop that calls the intersector's box
// hook on both children of a 64-B pair node, then a leaf loop that calls its
// triangle hook on each primitive.  Every decision is a function of the ray
// alone (no warp-voted speculation), so results and the counting
// intersector's numbers do not depend on which lanes share a warp — they are
// deterministic and match the CPU walker bit for bit.
//
// Scheduling (B200), measured in profiles/r01_tuning.md: one thread per ray,
// 128-ray blocks launched longest-first (a small order pass estimates each
// block's cost from its rays' segment inside the root box), so the blocks
// whose single-ray latency would set the tail start first.  A persistent
// dynamic-fetch kernel (warps claim rays from a global counter and refill
// idle lanes) is kept as VSR_SCHED=persistent; it loses on coherent primary
// rays.
//
// Build: -gencode arch=compute_100a,code=sm_100a -fmad=false (IEEE fp32
// contract).
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

// Pop the next entry not farther than the current best (reading A14).
__device__ __forceinline__ bool pop(Trav& T, const float2* stack) {
  while (T.sp > 0) {
    --T.sp;
    const float2 e = stack[T.sp];
    if (e.y <= T.best_t) {
      T.cur = __float_as_uint(e.x);
      return true;
    }
  }
  return false;
}

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

template <bool GEN>
__device__ __forceinline__ void fetch_ray(const TraceParams& p, uint64_t id, float4& a, float4& b) {
  if constexpr (GEN) {
    gen_ray(p.cam, id, a, b);
  } else {
    a = __ldg(p.rays + 2 * id);
    b = __ldg(p.rays + 2 * id + 1);
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

template <int OCT, class I>
__device__ __forceinline__ bool descend(const DevScene& S, Trav& T, I& isect, float2* stack) {
  while (!(T.cur & kLeafBit)) {
    const float4* np = reinterpret_cast<const float4*>(S.nodes + T.cur);
    const float4 nx = __ldg(np), ny = __ldg(np + 1), nz = __ldg(np + 2), nr = __ldg(np + 3);
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
      stack[T.sp] = make_float2(__uint_as_float(swap ? r0 : r1), swap ? h.tn0 : h.tn1);
      ++T.sp;
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

// ---- leaf loop: "while node contains untested primitives" ----
// Returns true when the query is finished (any-hit accepted a primitive).
template <int Q, class I, class M>
__device__ __forceinline__ bool leaf(const DevScene& S, Trav& T, I& isect, M& mb) {
  const uint32_t first = T.cur & kLeafFirstMask;
  const uint32_t end = first + ((T.cur >> kLeafCountShift) & 31u) + 1u;
  for (uint32_t k = first; k < end; ++k) {
    const float4* tp = reinterpret_cast<const float4*>(S.tris + k);
    const TriData td{__ldg(tp), __ldg(tp + 1), __ldg(tp + 2)};
    const hit_record hr = tri_hook(isect, T.r, td, k, T.best_t);
    if constexpr (Q == kMulti) {
      if (hr.hit && (mb.n < mb.maxk || hr.t < T.best_t)) {
        int pos = mb.n < mb.maxk ? mb.n : mb.maxk - 1;   // a full buffer drops its worst
        while (pos > 0 && mb.t[pos - 1] > hr.t) {       // stable insertion by t
          mb.t[pos] = mb.t[pos - 1];
          mb.u[pos] = mb.u[pos - 1];
          mb.v[pos] = mb.v[pos - 1];
          mb.prim[pos] = mb.prim[pos - 1];
          if constexpr (M::kSrc) mb.src[pos] = mb.src[pos - 1];
          --pos;
        }
        mb.t[pos] = hr.t;
        mb.u[pos] = hr.u;
        mb.v[pos] = hr.v;
        mb.prim[pos] = __float_as_uint(td.a.w);
        if constexpr (M::kSrc) mb.src[pos] = mb.cur_src;
        if (mb.n < mb.maxk) ++mb.n;
        if (mb.n == mb.maxk) T.best_t = mb.t[mb.maxk - 1];
      }
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
template <int Q, int OCT, class I>
__device__ __forceinline__ bool advance(const DevScene& S, Trav& T, I& isect, float2* stack) {
  NoMulti none;
  if (!descend<OCT>(S, T, isect, stack)) return true;
  if (leaf<Q>(S, T, isect, none)) return true;
  return !pop(T, stack);
}

// Whole traversal of one ray.  `oct` is warp-uniform: 0..7 if every lane of
// the warp has that octant (primary rays: all but the centre row/column
// tiles), 8 otherwise; the switch is taken once per leaf, uniformly.
template <class I>
__device__ __forceinline__ bool descend_oct(const DevScene& S, Trav& T, I& isect, float2* stack,
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

template <int Q, class I, class M = NoMulti>
__device__ __forceinline__ void traverse(const DevScene& S, Trav& T, I& isect, float2* stack,
                                         int oct, M& mb) {
  for (;;) {
    const bool at_leaf = descend_oct(S, T, isect, stack, oct);
    if (!at_leaf || leaf<Q>(S, T, isect, mb) || !pop(T, stack)) return;
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

template <bool GEN>
__global__ void __launch_bounds__(256) order_cost_kernel(const TraceParams p, uint32_t nblocks,
                                                         uint32_t* hist, uint32_t* slot) {
  asm volatile("griddepcontrol.launch_dependents;");   // let the scatter kernel's CTAs launch
  const uint32_t t = blockIdx.x * 256 + threadIdx.x;   // 4 sample rays per 128-ray block
  const uint32_t b = t >> 2;
  float len = 0.0f;
  if (b < nblocks) {
    const uint64_t id = (uint64_t)b * kBlock + (t & 3u) * (uint32_t)((kBlock - 1) / 3);
    if (id < p.n) {
      float4 a, d;
      fetch_ray<GEN>(p, id, a, d);
      RayCtx r;
      make_ray(r, a, d);
      const float t0x = (p.scene.root_lo[0] - r.ox) * r.ix, t1x = (p.scene.root_hi[0] - r.ox) * r.ix;
      const float t0y = (p.scene.root_lo[1] - r.oy) * r.iy, t1y = (p.scene.root_hi[1] - r.oy) * r.iy;
      const float t0z = (p.scene.root_lo[2] - r.oz) * r.iz, t1z = (p.scene.root_hi[2] - r.oz) * r.iz;
      const float tn = fmaxf(fmaxf(fminf(t0x, t1x), fminf(t0y, t1y)), fmaxf(fminf(t0z, t1z), a.w));
      const float tf = fminf(fminf(fmaxf(t0x, t1x), fmaxf(t0y, t1y)), fminf(fmaxf(t0z, t1z), d.w));
      if (tf > tn) len = (tf - tn) * sqrtf(d.x * d.x + d.y * d.y + d.z * d.z);
    }
  }
  len = fmaxf(len, __shfl_xor_sync(0xFFFFFFFFu, len, 1));
  len = fmaxf(len, __shfl_xor_sync(0xFFFFFFFFu, len, 2));
  // CTA-local histogram first: a handful of buckets take almost all blocks,
  // so per-block global atomics would serialise on a few addresses.
  __shared__ uint32_t lh[kOrderBuckets], lbase[kOrderBuckets];
  for (int i = threadIdx.x; i < kOrderBuckets; i += 256) lh[i] = 0;
  __syncthreads();
  const bool leader = (t & 3u) == 0u && b < nblocks;
  int q = 0;
  uint32_t lpos = 0;
  if (leader) {
    const float dx = p.scene.root_hi[0] - p.scene.root_lo[0];
    const float dy = p.scene.root_hi[1] - p.scene.root_lo[1];
    const float dz = p.scene.root_hi[2] - p.scene.root_lo[2];
    const float diag = sqrtf(dx * dx + dy * dy + dz * dz);
    q = diag > 0.0f ? (int)(len / diag * kOrderBuckets) : 0;
    q = q < 0 ? 0 : (q >= kOrderBuckets ? kOrderBuckets - 1 : q);
    lpos = atomicAdd(lh + q, 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kOrderBuckets; i += 256)
    if (lh[i]) lbase[i] = atomicAdd(hist + i, lh[i]);
  __syncthreads();
  if (leader) slot[b] = ((uint32_t)q << 24) | (lbase[q] + lpos);
}

__global__ void __launch_bounds__(256) order_scatter_kernel(uint32_t nblocks, const uint32_t* hist,
                                                            const uint32_t* slot, uint32_t* perm) {
  __shared__ uint32_t start[kOrderBuckets];
  asm volatile("griddepcontrol.launch_dependents;");   // the trace kernel may launch now ...
  asm volatile("griddepcontrol.wait;" ::: "memory");    // ... and this one waits for the cost pass
  if (threadIdx.x < 32) {   // exclusive scan over buckets, most expensive first
    constexpr int R = kOrderBuckets / 32;   // consecutive buckets per lane
    const int lane = (int)threadIdx.x;
    uint32_t cnt[R], sum = 0;
    for (int k = 0; k < R; ++k) {
      cnt[k] = __ldcg(hist + (kOrderBuckets - 1 - (lane * R + k)));
      sum += cnt[k];
    }
    uint32_t incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += v;
    }
    uint32_t run = incl - sum;
    for (int k = 0; k < R; ++k) {
      start[kOrderBuckets - 1 - (lane * R + k)] = run;
      run += cnt[k];
    }
  }
  __syncthreads();
  const uint32_t b = blockIdx.x * 256 + threadIdx.x;
  if (b >= nblocks) return;
  const uint32_t s = __ldcg(slot + b);
  perm[start[s >> 24] + (s & 0xFFFFFFu)] = b;
}

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

// Direct schedule (default): one thread per ray; launch slot i traces the 128
// rays of block perm[i] (block i when no order was computed), and the
// hardware block scheduler balances the blocks across the 148 SMs.
template <int Q, class I, bool GEN = false>
__global__ void __launch_bounds__(kBlock, VSR_MINB) trace_kernel(const TraceParams p) {
#ifdef VSR_TIMELINE
  const uint64_t t0 = global_ns();
#endif
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
  if (id < p.n) {
    I isect = make_isect<I>(p);
    Trav T;
    float2 stack[kMaxStack];   // (ref bits, tnear); depth <= 64 guaranteed by build/import
    const bool go = start_ray<GEN>(p, T, isect, id);
    // warp-uniform octant: specialised slab test when all live lanes agree
    const unsigned live = __activemask();
    const int oct = ray_octant(T.r);
    const int woct = __match_any_sync(live, oct) == live ? oct : 8;
    NoMulti none;
    if (go) traverse<Q>(p.scene, T, isect, stack, woct, none);
    // the ray index is recomputed (perm re-read through L2) rather than kept live
    // across the traversal: one register less in the hot loop
    const uint64_t blk2 = p.perm ? (uint64_t)__ldcg(p.perm + blockIdx.x) : (uint64_t)blockIdx.x;
    finish(p, T, isect, blk2 * kBlock + threadIdx.x);
  }
#ifdef VSR_TIMELINE
  // diagnostic build only: per-warp (SM id, start ns, end ns) into counts[warp]
  __syncwarp();
  if ((threadIdx.x & 31u) == 0 && !I::kCounts) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    const uint64_t t1 = global_ns();
    p.counts[id / 32] = make_uint4(smid, (unsigned)t0, (unsigned)t1, (unsigned)(t0 >> 32));
  }
#endif
}

// Multi-hit query: same traversal, the leaf accepts into a K-entry sorted
// buffer (runtime max_hits <= K).  Output ray-major: hits[id*max_hits + j].
template <class I, int K>
__global__ void __launch_bounds__(kBlock, VSR_MINB) trace_multi_kernel(const TraceParams p) {
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
  if (id >= p.n) return;
  I isect = make_isect<I>(p);
  Trav T;
  float2 stack[kMaxStack];
  MultiBuf<K> mb;
  mb.n = 0;
  mb.maxk = p.max_hits;
  const bool go = start_ray(p, T, isect, id);
  const unsigned live = __activemask();
  const int oct = ray_octant(T.r);
  const int woct = __match_any_sync(live, oct) == live ? oct : 8;
  if (go) traverse<kMulti>(p.scene, T, isect, stack, woct, mb);
  float4* out = p.hits + id * (uint64_t)p.max_hits;
  for (int j = 0; j < mb.maxk; ++j) {
    out[j] = j < mb.n ? make_float4(mb.t[j], mb.u[j], mb.v[j], __uint_as_float(mb.prim[j]))
                      : make_float4(__int_as_float(0x7f800000), 0.0f, 0.0f,
                                    __uint_as_float(kMissPrim));
  }
  if (p.num_hits) p.num_hits[id] = (uint32_t)mb.n;
  if constexpr (I::kCounts) {
    p.counts[id] = make_uint4(isect.num_boxes, isect.num_tris, isect.lookups(), 0u);
  }
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
  } else {
    (void)d;
  }
}

// Query over a LIST of BVHs (BVHs act as compound
// primitives; the intersector is passed on into each BVH's traversal).  The
// list is walked linearly in order; every element's root box is tested (and
// counted) with the current best_t, so a closer hit in an earlier BVH prunes
// later ones.  `which` records the list index of the kept hit.
template <int Q, class I>
__global__ void __launch_bounds__(kBlock, VSR_MINB) trace_list_kernel(const TraceParams p) {
  const DevScene* list = p.list;
  const IsectData* ldata = p.list_data;
  const uint32_t count = p.list_count;
  uint32_t* which = p.which;
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
  if (id >= p.n) return;
  I isect = make_isect<I>(p);
  Trav T;
  float2 stack[kMaxStack];
  start_ray(p, T, isect, id);   // loads the ray; p.scene is element 0 (root test redone below)
  isect.reset();
  const unsigned live = __activemask();
  const int oct = ray_octant(T.r);
  const int woct = __match_any_sync(live, oct) == live ? oct : 8;
  uint32_t hit_in = 0xFFFFFFFFu;
  NoMulti none;
  for (uint32_t s = 0; s < count; ++s) {
    const DevScene S = list[s];
    bind_scene_data(isect, ldata[s]);
    const Aabb root{S.root_lo[0], S.root_lo[1], S.root_lo[2], S.root_hi[0], S.root_hi[1], S.root_hi[2]};
    float tn;
    if (!box_hook(isect, T.r, root, T.best_t, tn)) continue;
    const float t_before = T.best_t;
    const uint32_t prim_before = T.prim;
    T.cur = S.root_ref;
    T.sp = 0;
    traverse<Q>(S, T, isect, stack, woct, none);
    if (T.best_t != t_before || T.prim != prim_before) hit_in = s;
    if (Q == kAny && T.prim != kMissPrim) break;   // any-hit: the first accepted hit ends it
  }
  finish(p, T, isect, id);
  if (which) which[id] = hit_in;
}

// ---------------------------------------------------------------------------
// Two-level instancing ("the BVH will store BVHs as
// primitives").  p.scene is the top level (pair nodes over instance world
// boxes; a leaf's range indexes p.instances); p.list / p.list_data are the
// instanced scenes.  A top-level leaf runs, per instance, the whole bottom
// traversal with the ray mapped to object space (reading A27) and the shared
// best_t; the bottom's stack entries sit above the top level's.
// ---------------------------------------------------------------------------
constexpr int kInstStack = 2 * kMaxStack;

__device__ __forceinline__ void to_object(const float4 r0, const float4 r1, const float4 r2,
                                          const RayCtx& w, float4& a, float4& b) {
  a.x = ((r0.x * w.ox + r0.y * w.oy) + r0.z * w.oz) + r0.w;
  a.y = ((r1.x * w.ox + r1.y * w.oy) + r1.z * w.oz) + r1.w;
  a.z = ((r2.x * w.ox + r2.y * w.oy) + r2.z * w.oz) + r2.w;
  a.w = w.tmin;
  b.x = (r0.x * w.dx + r0.y * w.dy) + r0.z * w.dz;
  b.y = (r1.x * w.dx + r1.y * w.dy) + r1.z * w.dz;
  b.z = (r2.x * w.dx + r2.y * w.dy) + r2.z * w.dz;
}

// Instance k of the current top-level leaf.  Returns true when the query is
// finished (any-hit accepted a primitive).
template <int Q, class I>
__device__ __forceinline__ bool instance_leaf(const TraceParams& p, Trav& T, I& isect,
                                              float2* stack, uint32_t k, uint32_t& hit_in) {
  const float4* ip = reinterpret_cast<const float4*>(p.instances + k);
  const float4 r0 = __ldg(ip), r1 = __ldg(ip + 1), r2 = __ldg(ip + 2), ex = __ldg(ip + 3);
  const uint32_t b = __float_as_uint(ex.x);
  const DevScene& S = p.list[b];
  bind_scene_data(isect, p.list_data[b]);
  Trav B = T;   // running best (t, u, v, prim, have, best_t) carried in and out
  float4 oa, ob;
  to_object(r0, r1, r2, T.r, oa, ob);
  make_ray(B.r, oa, ob);
  B.sp = 0;
  B.cur = S.root_ref;
  const Aabb root{S.root_lo[0], S.root_lo[1], S.root_lo[2], S.root_hi[0], S.root_hi[1], S.root_hi[2]};
  float tn;
  if (!box_hook(isect, B.r, root, B.best_t, tn)) return false;
  NoMulti none;
  traverse<Q>(S, B, isect, stack, warp_octant(B.r), none);
  const bool better = Q == kAny ? B.prim != kMissPrim
                                : (B.prim != kMissPrim && (T.prim == kMissPrim || B.best_t < T.best_t));
  if (better) {
    T.best_t = B.best_t;
    T.u = B.u;
    T.v = B.v;
    T.prim = B.prim;
    hit_in = __float_as_uint(ex.y);
  }
  return Q == kAny && better;
}

template <int Q, class I>
__global__ void __launch_bounds__(kBlock, VSR_MINB) trace_instances_kernel(const TraceParams p) {
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
  if (id >= p.n) return;
  I isect = make_isect<I>(p);
  Trav T;
  float2 stack[kInstStack];   // top level below, the current instance's entries above
  uint32_t hit_in = 0xFFFFFFFFu;
  if (start_ray(p, T, isect, id)) {   // world ray; counted test of the top-level root box
    const int woct = warp_octant(T.r);
    for (;;) {
      if (!descend_oct(p.scene, T, isect, stack, woct)) break;
      const uint32_t first = T.cur & kLeafFirstMask;
      const uint32_t end = first + ((T.cur >> kLeafCountShift) & 31u) + 1u;
      bool done = false;
      for (uint32_t k = first; k < end && !done; ++k)
        done = instance_leaf<Q>(p, T, isect, stack + T.sp, k, hit_in);
      if (done || !pop(T, stack)) break;
    }
  }
  finish(p, T, isect, id);
  if (p.which) p.which[id] = hit_in;
}

// Multi-hit query over a LIST of BVHs / over instances (the
// visibility queries closest_hit, any_hit AND multi_hit iterate over lists
// whose elements may be BVHs): one K-entry buffer across all elements, each
// kept hit tagged with its element (list index, or the caller's instance
// index); output as trace_multi_kernel plus `which` per kept hit.
template <class I, int K>
__device__ __forceinline__ void write_multi(const TraceParams& p, uint64_t id,
                                            const MultiBuf<K, true>& mb, const I& isect) {
  float4* out = p.hits + id * (uint64_t)p.max_hits;
  uint32_t* wout = p.which ? p.which + id * (uint64_t)p.max_hits : nullptr;
  for (int j = 0; j < mb.maxk; ++j) {
    const bool kept = j < mb.n;
    out[j] = kept ? make_float4(mb.t[j], mb.u[j], mb.v[j], __uint_as_float(mb.prim[j]))
                  : make_float4(__int_as_float(0x7f800000), 0.0f, 0.0f, __uint_as_float(kMissPrim));
    if (wout) wout[j] = kept ? mb.src[j] : kMissPrim;
  }
  if (p.num_hits) p.num_hits[id] = (uint32_t)mb.n;
  if constexpr (I::kCounts) {
    p.counts[id] = make_uint4(isect.num_boxes, isect.num_tris, isect.lookups(), 0u);
  }
}

template <class I, int K>
__global__ void __launch_bounds__(kBlock, VSR_MINB) trace_list_multi_kernel(const TraceParams p) {
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
  if (id >= p.n) return;
  I isect = make_isect<I>(p);
  Trav T;
  float2 stack[kMaxStack];
  MultiBuf<K, true> mb;
  mb.n = 0;
  mb.maxk = p.max_hits;
  start_ray(p, T, isect, id);   // loads the ray (the list's roots are tested below)
  isect.reset();
  const int woct = warp_octant(T.r);
  for (uint32_t s = 0; s < p.list_count; ++s) {
    const DevScene S = p.list[s];
    bind_scene_data(isect, p.list_data[s]);
    const Aabb root{S.root_lo[0], S.root_lo[1], S.root_lo[2], S.root_hi[0], S.root_hi[1], S.root_hi[2]};
    float tn;
    if (!box_hook(isect, T.r, root, T.best_t, tn)) continue;
    T.cur = S.root_ref;
    T.sp = 0;
    mb.cur_src = s;
    traverse<kMulti>(S, T, isect, stack, woct, mb);
  }
  write_multi<I, K>(p, id, mb, isect);
}

template <class I, int K>
__global__ void __launch_bounds__(kBlock, VSR_MINB) trace_instances_multi_kernel(const TraceParams p) {
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
  if (id >= p.n) return;
  I isect = make_isect<I>(p);
  Trav T;
  float2 stack[kInstStack];
  MultiBuf<K, true> mb;
  mb.n = 0;
  mb.maxk = p.max_hits;
  if (start_ray(p, T, isect, id)) {   // world ray; counted test of the top-level root box
    const int woct = warp_octant(T.r);
    for (;;) {
      if (!descend_oct(p.scene, T, isect, stack, woct)) break;
      const uint32_t first = T.cur & kLeafFirstMask;
      const uint32_t end = first + ((T.cur >> kLeafCountShift) & 31u) + 1u;
      for (uint32_t k = first; k < end; ++k) {
        const float4* ip = reinterpret_cast<const float4*>(p.instances + k);
        const float4 r0 = __ldg(ip), r1 = __ldg(ip + 1), r2 = __ldg(ip + 2), ex = __ldg(ip + 3);
        const uint32_t b = __float_as_uint(ex.x);
        const DevScene& S = p.list[b];
        bind_scene_data(isect, p.list_data[b]);
        Trav B = T;
        float4 oa, ob;
        to_object(r0, r1, r2, T.r, oa, ob);
        make_ray(B.r, oa, ob);
        B.sp = 0;
        B.cur = S.root_ref;
        const Aabb root{S.root_lo[0], S.root_lo[1], S.root_lo[2], S.root_hi[0], S.root_hi[1],
                        S.root_hi[2]};
        float tn;
        if (!box_hook(isect, B.r, root, B.best_t, tn)) continue;
        mb.cur_src = __float_as_uint(ex.y);
        traverse<kMulti>(S, B, isect, stack + T.sp, warp_octant(B.r), mb);
        T.best_t = B.best_t;   // a full buffer's worst kept t prunes the rest
      }
      if (!pop(T, stack)) break;
    }
  }
  write_multi<I, K>(p, id, mb, isect);
}

// ---------------------------------------------------------------------------
// Query on a plain LIST of primitives, no BVH ("the user
// might decide that a BVH is not required and just pass iterators to a linear
// list of primitives to the query routines"; the custom intersector then
// replaces the primitive test inside the loop).  p.scene.tris / p.data.sides
// are the scene's triangles in CALLER order (prim field 0xFFFFFFFF for the
// excluded degenerate ones); blocks stage 128 triangles at a time in shared
// memory and every thread tests its ray against them in order, so closest
// keeps the lowest index among equal t and any-hit the first accepted index —
// the brute-force definition itself.
// ---------------------------------------------------------------------------
template <int Q, class I>
__global__ void __launch_bounds__(kBlock) trace_prims_kernel(const TraceParams p) {
  __shared__ float4 tile[3 * kBlock];
  const uint64_t id = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
  const bool live = id < p.n;
  I isect = make_isect<I>(p);
  isect.reset();
  Trav T;
  bool done = !live;
  if (live) {
    const float4 a = __ldg(p.rays + 2 * id), b = __ldg(p.rays + 2 * id + 1);
    make_ray(T.r, a, b);
    T.best_t = b.w;
    T.u = T.v = 0.0f;
    T.prim = kMissPrim;
  }
  const uint32_t total = p.scene.num_tris;
  for (uint32_t base = 0; base < total; base += kBlock) {
    const uint32_t k = base + threadIdx.x;
    if (k < total) {
      const float4* tp = reinterpret_cast<const float4*>(p.scene.tris + k);
      tile[3 * threadIdx.x] = __ldg(tp);
      tile[3 * threadIdx.x + 1] = __ldg(tp + 1);
      tile[3 * threadIdx.x + 2] = __ldg(tp + 2);
    }
    __syncthreads();
    if (!done) {
      const uint32_t cnt = min((uint32_t)kBlock, total - base);
      for (uint32_t j = 0; j < cnt; ++j) {
        const TriData td{tile[3 * j], tile[3 * j + 1], tile[3 * j + 2]};
        const uint32_t prim = __float_as_uint(td.a.w);
        if (prim == kMissPrim) continue;   // degenerate: not in the scene
        const hit_record hr = tri_hook(isect, T.r, td, base + j, T.best_t);
        if constexpr (Q == kAny) {
          if (hr.hit) {
            T.best_t = hr.t;
            T.u = hr.u;
            T.v = hr.v;
            T.prim = prim;
            done = true;
            break;
          }
        } else if (hr.hit && (T.prim == kMissPrim || hr.t < T.best_t)) {
          T.best_t = hr.t;
          T.u = hr.u;
          T.v = hr.v;
          T.prim = prim;
        }
      }
    }
    __syncthreads();
  }
  if (live) finish(p, T, isect, id);
}

// Persistent schedule (VSR_SCHED=persistent): grid sized to residency; warps
// claim kChunk rays per atomicAdd and refill idle lanes after each leaf once
// `refill` lanes are idle.  Measured slower than the direct schedule on the
// coherent primary rays of C2 (profiles/r01_tuning.md); kept for incoherent
// workloads and as a measured alternative.
template <int Q, class I>
__global__ void __launch_bounds__(kBlock, VSR_MINB) trace_kernel_persistent(const TraceParams p) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned below = (1u << lane) - 1u;
  unsigned long long* ctr = p.counter;
  I isect = make_isect<I>(p);
  Trav T;
  float2 stack[kMaxStack];   // (ref bits, tnear); depth <= 64 guaranteed by build/import
  bool active = false;
  // warp-uniform work queue: [next, next + left) of the warp's claimed chunk
  unsigned long long next = 0;
  unsigned left = 0;
  uint64_t my_id = 0;
  bool drained = false;      // the global counter ran past n
  for (;;) {
    // converged refill point: ballot/popc compaction of the idle lanes
    const unsigned idle = __ballot_sync(kFull, !active);
    if (idle != 0u && (idle == kFull || __popc(idle) >= p.refill) && !(drained && left == 0)) {
      if (left == 0) {   // claim a new chunk: one atomicAdd per kChunk rays
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ctr, (unsigned long long)kChunk);
        base = __shfl_sync(kFull, base, 0);
        next = base;
        left = base >= p.n ? 0u : (unsigned)min((unsigned long long)kChunk, p.n - base);
        drained = base + kChunk >= p.n;
      }
      const unsigned take = min((unsigned)__popc(idle), left);
      if (!active) {
        const unsigned rank = __popc(idle & below);
        if (rank < take) {
          my_id = next + rank;
          active = start_ray(p, T, isect, my_id);
          if (!active) finish(p, T, isect, my_id);   // missed the root box: a miss record
        }
      }
      next += take;
      left -= take;
    } else if (idle == kFull && drained && left == 0) {
      break;
    }
    if (active && advance<Q, -1>(p.scene, T, isect, stack)) {
      finish(p, T, isect, my_id);
      active = false;
    }
  }
  // The launch's last warp resets the counter slot for a later launch.
  if (lane == 0) {
    __threadfence();
    const unsigned long long warps = (unsigned long long)gridDim.x * (kBlock / 32);
    if (atomicAdd(ctr + 1, 1ull) == warps - 1ull) {
      atomicExch(ctr, 0ull);
      atomicExch(ctr + 1, 0ull);
    }
  }
}

// Device filter functions for the function-pointer control (OptiX-style).
__device__ bool fn_alpha_tex(const IsectData* d, uint32_t k, float u, float v) {
  return alpha_keep(*d, k, u, v);
}
__device__ bool fn_alpha_proc(const IsectData* d, uint32_t, float u, float v) {
  return checker_keep(d->fm, u, v);
}
__device__ filter_fn_t g_fn_alpha_tex = fn_alpha_tex;
__device__ filter_fn_t g_fn_alpha_proc = fn_alpha_proc;

namespace {
std::atomic<uint64_t> g_launches{0};

int sm_count() {
  static std::atomic<int> cache[64];   // zero-initialised (static storage)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = n > 0 ? n : 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// <<<grid, block, 0, st>>>, as a programmatic dependent launch when `pdl`
// (the kernel starts with griddepcontrol.wait, see launch_block).
template <typename... Args, typename... Act>
cudaError_t launch_k(void (*k)(Args...), uint64_t grid, unsigned block, bool pdl, cudaStream_t st,
                     Act&&... args) {
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

template <int Q, class I>
cudaError_t launch(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (p.sched == kSchedPersistent) {
    static std::atomic<int> per_sm_cache{0};   // resident blocks per SM for this instantiation
    int per_sm = per_sm_cache.load(std::memory_order_relaxed);
    if (per_sm == 0) {
      int nb = 0;
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &nb, trace_kernel_persistent<Q, I>, kBlock, 0);
      if (e != cudaSuccess) return e;
      per_sm = nb > 0 ? nb : 1;
      per_sm_cache.store(per_sm, std::memory_order_relaxed);
    }
    const uint64_t full = (uint64_t)per_sm * sm_count();
    const unsigned blocks = (unsigned)(need < full ? need : full);
    trace_kernel_persistent<Q, I><<<blocks, kBlock, 0, st>>>(p);
  } else {
    if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
    cudaError_t e;
    if (p.gen) {   // fused ray generation: not built for the run-time controls
      if constexpr (std::is_same<I, runtime_switch_intersector>::value ||
                    std::is_same<I, runtime_fnptr_intersector>::value)
        return cudaErrorInvalidValue;
      else
        e = launch_k(trace_kernel<Q, I, true>, need, kBlock, p.perm && p.pdl, st, p);
    } else {
      e = launch_k(trace_kernel<Q, I>, need, kBlock, p.perm && p.pdl, st, p);
    }
    if (e != cudaSuccess) return e;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <class I>
cudaError_t launch_multi(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const bool pdl = p.perm && p.pdl;
  cudaError_t e = p.max_hits <= 4 ? launch_k(trace_multi_kernel<I, 4>, need, kBlock, pdl, st, p)
                                  : launch_k(trace_multi_kernel<I, 16>, need, kBlock, pdl, st, p);
  if (e != cudaSuccess) return e;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t dispatch_multi(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch_multi<no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch_multi<default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE: return launch_multi<alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch_multi<alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch_multi<alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch_multi<alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch_multi<cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch_multi<cost_intersector<alpha_texture_intersector>>(p, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int Q, class I>
cudaError_t launch_list(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  cudaError_t e = launch_k(trace_list_kernel<Q, I>, need, kBlock, p.perm && p.pdl, st, p);
  if (e != cudaSuccess) return e;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <class I>
cudaError_t launch_compound_multi(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const bool pdl = p.perm && p.pdl;
  cudaError_t e;
  if (p.instances)
    e = p.max_hits <= 4 ? launch_k(trace_instances_multi_kernel<I, 4>, need, kBlock, pdl, st, p)
                        : launch_k(trace_instances_multi_kernel<I, 16>, need, kBlock, pdl, st, p);
  else
    e = p.max_hits <= 4 ? launch_k(trace_list_multi_kernel<I, 4>, need, kBlock, pdl, st, p)
                        : launch_k(trace_list_multi_kernel<I, 16>, need, kBlock, pdl, st, p);
  if (e != cudaSuccess) return e;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t dispatch_compound_multi(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch_compound_multi<no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch_compound_multi<default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE: return launch_compound_multi<alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch_compound_multi<alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch_compound_multi<alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch_compound_multi<alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch_compound_multi<cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch_compound_multi<cost_intersector<alpha_texture_intersector>>(p, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int Q, class I>
cudaError_t launch_inst(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  cudaError_t e = launch_k(trace_instances_kernel<Q, I>, need, kBlock, p.perm && p.pdl, st, p);
  if (e != cudaSuccess) return e;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int Q>
cudaError_t dispatch_inst(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch_inst<Q, no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch_inst<Q, default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE: return launch_inst<Q, alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch_inst<Q, alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch_inst<Q, alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch_inst<Q, alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch_inst<Q, cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch_inst<Q, cost_intersector<alpha_texture_intersector>>(p, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int Q>
cudaError_t dispatch_list(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch_list<Q, no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch_list<Q, default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE: return launch_list<Q, alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch_list<Q, alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch_list<Q, alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch_list<Q, alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch_list<Q, cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch_list<Q, cost_intersector<alpha_texture_intersector>>(p, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int Q>
cudaError_t dispatch_isect(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch<Q, no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch<Q, default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE: return launch<Q, alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch<Q, alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch<Q, alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch<Q, alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch<Q, cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch<Q, cost_intersector<alpha_texture_intersector>>(p, st);
    case VSR_ISECT_RUNTIME_SWITCH_DEFAULT:
    case VSR_ISECT_RUNTIME_SWITCH_ALPHA_TEXTURE:
    case VSR_ISECT_RUNTIME_SWITCH_ALPHA_PROCEDURAL:
      return launch<Q, runtime_switch_intersector>(p, st);
    case VSR_ISECT_RUNTIME_FNPTR_DEFAULT:
    case VSR_ISECT_RUNTIME_FNPTR_ALPHA_TEXTURE:
    case VSR_ISECT_RUNTIME_FNPTR_ALPHA_PROCEDURAL:
      return launch<Q, runtime_fnptr_intersector>(p, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

cudaError_t filter_fn_pointer(int kind, void** out) {
  filter_fn_t f = nullptr;
  cudaError_t e = cudaSuccess;
  if (kind == kFilterAlphaTex) e = cudaMemcpyFromSymbol(&f, g_fn_alpha_tex, sizeof f);
  else if (kind == kFilterAlphaProc) e = cudaMemcpyFromSymbol(&f, g_fn_alpha_proc, sizeof f);
  *out = reinterpret_cast<void*>(f);
  return e;
}

// Profiling hook (thread-local): events recorded right before and after the
// trace kernel itself, i.e. excluding the block-order pass.
thread_local void* g_kernel_events[2] = {nullptr, nullptr};

void set_kernel_events(void* start, void* stop) {
  g_kernel_events[0] = start;
  g_kernel_events[1] = stop;
}

size_t order_scratch_bytes(uint64_t n) {
  const uint64_t nblocks = (n + kBlock - 1) / kBlock;
  return sizeof(uint32_t) * (kOrderBuckets + 2 * (size_t)nblocks);
}

cudaError_t launch_trace(int query, int isect, const TraceParams& p_in, cudaStream_t st) {
  if (p_in.n == 0) return cudaSuccess;
  TraceParams p = p_in;
  p.perm = nullptr;
  p.hist_reset = nullptr;
  const uint64_t nblocks = (p.n + kBlock - 1) / kBlock;
  void* scratch = nullptr;
  bool owned = false;
  if (p.order && p.sched == kSchedDirect && nblocks >= 2ull * sm_count() && nblocks < (1u << 24)) {
    // the owner's per-stream scratch (api.cpp ScratchSet); a stream-ordered
    // allocation only past 16 streams per owner
    const size_t bytes = order_scratch_bytes(p.n);
    cudaError_t e = cudaSuccess;
    if (p.order_scratch && p.order_scratch_bytes >= bytes) {
      scratch = p.order_scratch;   // caller-provided, stream-ordered (per-stream scene scratch)
    } else {
      if ((e = cudaMallocAsync(&scratch, bytes, st)) != cudaSuccess) return e;
      owned = true;
    }
    uint32_t* hist = static_cast<uint32_t*>(scratch);
    uint32_t* slot = hist + kOrderBuckets;
    uint32_t* perm = slot + nblocks;
    const bool zeroed = !owned;   // caller scratch: zero at entry, kept so by the trace kernel
    if (!zeroed &&
        (e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kOrderBuckets, st)) != cudaSuccess)
      return e;
    if (p.gen)
      order_cost_kernel<true><<<(unsigned)((4 * nblocks + 255) / 256), 256, 0, st>>>(
          p, (uint32_t)nblocks, hist, slot);
    else
      order_cost_kernel<false><<<(unsigned)((4 * nblocks + 255) / 256), 256, 0, st>>>(
          p, (uint32_t)nblocks, hist, slot);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = launch_k(order_scatter_kernel, (nblocks + 255) / 256, 256, p.pdl != 0, st,
                      (uint32_t)nblocks, (const uint32_t*)hist, (const uint32_t*)slot, perm)) !=
        cudaSuccess) {
      if (zeroed) cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kOrderBuckets, st);
      return e;
    }
    g_launches.fetch_add(2, std::memory_order_relaxed);
    if (!owned) p.hist_reset = hist;   // the trace kernel re-zeroes it for the next launch
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    p.perm = perm;
  }
  if (g_kernel_events[0]) cudaEventRecord(static_cast<cudaEvent_t>(g_kernel_events[0]), st);
  cudaError_t e = (p.list && query == kMulti) ? dispatch_compound_multi(isect, p, st)
                  : p.instances ? (query == kAny ? dispatch_inst<kAny>(isect, p, st)
                                                : dispatch_inst<kClosest>(isect, p, st))
                  : p.list ? (query == kAny ? dispatch_list<kAny>(isect, p, st)
                                          : dispatch_list<kClosest>(isect, p, st))
                  : query == kMulti ? dispatch_multi(isect, p, st)
                  : query == kAny ? dispatch_isect<kAny>(isect, p, st)
                                  : dispatch_isect<kClosest>(isect, p, st);
  if (g_kernel_events[1]) cudaEventRecord(static_cast<cudaEvent_t>(g_kernel_events[1]), st);
  if (e != cudaSuccess && p.hist_reset)   // the trace kernel did not run: restore the invariant
    cudaMemsetAsync(p.hist_reset, 0, sizeof(uint32_t) * kOrderBuckets, st);
  if (owned) {
    cudaError_t f = cudaFreeAsync(scratch, st);
    if (e == cudaSuccess) e = f;
  }
  return e;
}

namespace {
template <int Q, class I>
cudaError_t launch_prims_as(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  trace_prims_kernel<Q, I><<<(unsigned)need, kBlock, 0, st>>>(p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int Q>
cudaError_t dispatch_prims(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch_prims_as<Q, no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch_prims_as<Q, default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE: return launch_prims_as<Q, alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch_prims_as<Q, alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch_prims_as<Q, alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch_prims_as<Q, alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch_prims_as<Q, cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch_prims_as<Q, cost_intersector<alpha_texture_intersector>>(p, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

cudaError_t launch_prims(int query, int isect, const TraceParams& p, cudaStream_t st) {
  if (p.n == 0) return cudaSuccess;
  return query == kAny ? dispatch_prims<kAny>(isect, p, st) : dispatch_prims<kClosest>(isect, p, st);
}

uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

}  // namespace vsr
