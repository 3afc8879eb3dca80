// compound.cu — queries over compound primitives: lists of
// BVHs / multiple roots, two-level instancing, and the multi-hit query over
// both.  The intersector is passed on into every element's traversal.
#include "traverse.cuh"

namespace vsr {

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
  StackEntry<Q> stack[kMaxStack];   // any-hit: refs only (traverse.cuh pop)
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
// The bottom traversal reads the instanced scene's DevScene through a private copy: through
// a reference into p.list the compiler reloads S.nodes from global memory at every node
// (a store to the local stack may alias a generic pointer), a dependent L1 round trip per
// visit.  Measured instanced forest any +2.0 %, closest +2.7 % (profiles/r02_tuning.md).
#ifndef VSR_INST_SCOPY
#define VSR_INST_SCOPY 1
#endif
#ifndef VSR_INST_OUTER
#define VSR_INST_OUTER 0   // 1: octant dispatch once per instance visit (measured -14 / -29 %)
#endif

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
template <int Q, class I, class SE>
__device__ __forceinline__ bool instance_leaf(const TraceParams& p, Trav& T, I& isect,
                                              SE* stack, uint32_t k, uint32_t& hit_in) {
  VSR_CHECK(k < p.num_instances);
  const float4* ip = reinterpret_cast<const float4*>(p.instances + k);
  const float4 r0 = __ldg(ip), r1 = __ldg(ip + 1), r2 = __ldg(ip + 2), ex = __ldg(ip + 3);
  const uint32_t b = __float_as_uint(ex.x);
  VSR_CHECK(b < p.list_count);
#if VSR_INST_SCOPY
  const DevScene S = p.list[b];   // a private copy: the bottom loop keeps its pointers in registers
#else
  const DevScene& S = p.list[b];
#endif
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
  traverse<Q, VSR_INST_OUTER != 0>(S, B, isect, stack, warp_octant(B.r), none);
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

// A ray whose origin lies beyond the instances' proven range (|o|_inf > r_safe).
__device__ __forceinline__ bool far_origin(const TraceParams& p, const RayCtx& r) {
  return fmax3(fabsf(r.ox), fabsf(r.oy), fabsf(r.oz)) > p.inst_r_safe;
}

template <int Q, class I>
__global__ void __launch_bounds__(kBlock, VSR_INST_MINB) trace_instances_kernel(const TraceParams p) {
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
  if (id >= p.n) return;
  I isect = make_isect<I>(p);
  Trav T;
  StackEntry<Q> stack[kInstStack];   // top level below, the current instance's entries above
  uint32_t hit_in = 0xFFFFFFFFu;
  const bool go = start_ray(p, T, isect, id);   // world ray; counted test of the top-level root box
  if (far_origin(p, T.r)) {
    // beyond r_safe the world boxes are not proven conservative for the fp32 ray map:
    // every instance in leaf order, whatever the top level says (reading A27)
    for (uint32_t k = 0; k < p.num_instances; ++k)
      if (instance_leaf<Q>(p, T, isect, stack, k, hit_in)) break;
  } else if (go) {
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
#pragma unroll
  for (int j = 0; j < K; ++j) {   // static indices: the buffer stays in registers
    if (j >= mb.maxk) break;
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

// Instance k of the multi-hit query: the bottom traversal into the shared K-buffer.
template <class I, int K>
__device__ __forceinline__ void instance_leaf_multi(const TraceParams& p, Trav& T, I& isect,
                                                    float2* stack, uint32_t k,
                                                    MultiBuf<K, true>& mb) {
  VSR_CHECK(k < p.num_instances);
  const float4* ip = reinterpret_cast<const float4*>(p.instances + k);
  const float4 r0 = __ldg(ip), r1 = __ldg(ip + 1), r2 = __ldg(ip + 2), ex = __ldg(ip + 3);
  const uint32_t b = __float_as_uint(ex.x);
  VSR_CHECK(b < p.list_count);
#if VSR_INST_SCOPY
  const DevScene S = p.list[b];   // a private copy: the bottom loop keeps its pointers in registers
#else
  const DevScene& S = p.list[b];
#endif
  bind_scene_data(isect, p.list_data[b]);
  Trav B = T;
  float4 oa, ob;
  to_object(r0, r1, r2, T.r, oa, ob);
  make_ray(B.r, oa, ob);
  B.sp = 0;
  B.cur = S.root_ref;
  const Aabb root{S.root_lo[0], S.root_lo[1], S.root_lo[2], S.root_hi[0], S.root_hi[1], S.root_hi[2]};
  float tn;
  if (!box_hook(isect, B.r, root, B.best_t, tn)) return;
  mb.cur_src = __float_as_uint(ex.y);
  traverse<kMulti>(S, B, isect, stack, warp_octant(B.r), mb);
  T.best_t = B.best_t;   // a full buffer's worst kept t prunes the rest
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
  const bool go = start_ray(p, T, isect, id);   // world ray; counted test of the top-level root box
  if (far_origin(p, T.r)) {   // beyond r_safe: every instance (reading A27)
    for (uint32_t k = 0; k < p.num_instances; ++k) instance_leaf_multi(p, T, isect, stack, k, mb);
  } else if (go) {
    const int woct = warp_octant(T.r);
    for (;;) {
      if (!descend_oct(p.scene, T, isect, stack, woct)) break;
      const uint32_t first = T.cur & kLeafFirstMask;
      const uint32_t end = first + ((T.cur >> kLeafCountShift) & 31u) + 1u;
      for (uint32_t k = first; k < end; ++k) instance_leaf_multi(p, T, isect, stack + T.sp, k, mb);
      if (!pop(T, stack)) break;
    }
  }
  write_multi<I, K>(p, id, mb, isect);
}

namespace {
template <int Q, class I>
cudaError_t launch_list(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  cudaError_t e = launch_k(trace_list_kernel<Q, I>, need, kBlock, p.perm && p.pdl, st, p);
  if (e != cudaSuccess) return e;
  launch_counter().fetch_add(1, std::memory_order_relaxed);
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
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t dispatch_compound_multi(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch_compound_multi<no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch_compound_multi<default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE:
      return p.data.bits ? launch_compound_multi<alpha_bits_intersector>(p, st)
                         : launch_compound_multi<alpha_texture_intersector>(p, st);
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
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int Q>
cudaError_t dispatch_inst(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch_inst<Q, no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch_inst<Q, default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE:
      return p.data.bits ? launch_inst<Q, alpha_bits_intersector>(p, st)
                         : launch_inst<Q, alpha_texture_intersector>(p, st);
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
    case VSR_ISECT_ALPHA_TEXTURE:
      return p.data.bits ? launch_list<Q, alpha_bits_intersector>(p, st)
                         : launch_list<Q, alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch_list<Q, alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch_list<Q, alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch_list<Q, alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch_list<Q, cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch_list<Q, cost_intersector<alpha_texture_intersector>>(p, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

cudaError_t launch_compound(int query, int isect, const TraceParams& p, cudaStream_t st) {
  if (query == kMulti) return dispatch_compound_multi(isect, p, st);
  if (p.instances)
    return query == kAny ? dispatch_inst<kAny>(isect, p, st) : dispatch_inst<kClosest>(isect, p, st);
  return query == kAny ? dispatch_list<kAny>(isect, p, st) : dispatch_list<kClosest>(isect, p, st);
}

}  // namespace vsr
