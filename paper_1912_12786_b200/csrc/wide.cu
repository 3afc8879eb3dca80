// wide.cu — traversal of the 8-wide compressed BVH (wide.hpp; SURVEY.md §8(f)
// NEXT-3) with the same compile-time intersectors as the binary kernels.
//
// The while-while scheme of PAPER.md:228-247, one level wider: visiting a
// node calls the box hook once on its 8 quantized children (AabbOct; a
// counting intersector counts one box test per valid child), then the
// triangle hook on every triangle of each hit LEAF child (in child order),
// then descends into the first hit INNER child and keeps the others as a
// pending group.  Child order is a function of the ray alone: slot s is
// visited at key s ^ octant(ray), ascending (the builder placed near children
// in the slot of the octant they suit).  A group on the stack is (child_base,
// slot mask of inner children, pending keys); a pending child is visited even
// if best_t has since shrunk below its entry (its own children are tested
// against the new best_t) — the stack holds no t.  Deterministic per ray, so
// the counts and hits match walker C's walk_wide bit for bit.
#include "traverse.cuh"
#include "wide.hpp"

namespace vsr {

#ifndef VSR_WIDE_MINB
#define VSR_WIDE_MINB 0
#endif

template <class I, class... Args>
__device__ __forceinline__ uint32_t box_oct_hook(I& isect, const RayCtx& r, const AabbOct& b,
                                                 float best_t, uint32_t valid, Args... args) {
  if constexpr (std::is_same<I, no_intersector>::value) return intersect(r, b, best_t, valid, args...);
  else return isect(r, b, best_t, valid, args...);
}

// bit s of m moves to bit s ^ oct (three conditional swaps: XOR permutes the 3 index bits)
template <int OCT>
__device__ __forceinline__ uint32_t keyperm(uint32_t m, int oct) {
  const int o = OCT >= 0 ? OCT : oct;
  if (o & 1) m = ((m & 0x55u) << 1) | ((m >> 1) & 0x55u);
  if (o & 2) m = ((m & 0x33u) << 2) | ((m >> 2) & 0x33u);
  if (o & 4) m = ((m & 0x0Fu) << 4) | ((m >> 4) & 0x0Fu);
  return m;
}

// slots whose meta byte has bit 7 clear (leaf children)
__device__ __forceinline__ uint32_t leaf_slots(uint32_t m03, uint32_t m47) {
  const uint32_t a = ~m03 & 0x80808080u, b = ~m47 & 0x80808080u;
  const uint32_t lo = (a >> 7 | a >> 14 | a >> 21 | a >> 28) & 0xFu;
  const uint32_t hi = (b >> 7 | b >> 14 | b >> 21 | b >> 28) & 0xFu;
  return lo | hi << 4;
}

// Whole traversal of one ray over the wide tree (root = node 0; the root box
// was tested by start_ray).  OCT >= 0: warp-uniform octant (specialised slab).
template <int Q, int OCT, class I>
__device__ __forceinline__ void traverse_wide(const TraceParams& p, Trav& T, I& isect, uint2* stack,
                                              int oct) {
  const WideNode* W = p.wide;
  NoMulti none;
  uint32_t node = 0;
  int sp = 0;
  for (;;) {
    VSR_CHECK(node < p.num_wide);
    const float4* np = reinterpret_cast<const float4*>(W + node);
    AabbOct b;
    b.h = __ldg(np);
    const uint4 w1 = __ldg(reinterpret_cast<const uint4*>(np + 1));
    b.q0 = __ldg(reinterpret_cast<const uint4*>(np + 2));
    b.q1 = __ldg(reinterpret_cast<const uint4*>(np + 3));
    b.q2 = __ldg(reinterpret_cast<const uint4*>(np + 4));
    const uint32_t imask = __float_as_uint(b.h.w) >> 24;
    const uint32_t valid = imask | leaf_slots(w1.z, w1.w);
    uint32_t hits;
    if constexpr (OCT >= 0) hits = box_oct_hook(isect, T.r, b, T.best_t, valid, octant<OCT>{});
    else hits = box_oct_hook(isect, T.r, b, T.best_t, valid);
    hits &= valid;
    // leaf children first, in key order
    uint32_t lk = keyperm<OCT>(hits & ~imask, oct);
    while (lk) {
      const int s = (__ffs(lk) - 1) ^ (OCT >= 0 ? OCT : oct);
      lk &= lk - 1;
      const uint32_t m = ((s < 4 ? w1.z : w1.w) >> (8 * (s & 3))) & 0xFFu;
      T.cur = kLeafBit | (m >> 5) << kLeafCountShift | (w1.y + (m & 31u));
      if (leaf<Q>(p.scene, T, isect, none)) return;   // any-hit accepted a primitive
    }
    uint32_t ik = keyperm<OCT>(hits & imask, oct);
    if (ik) {   // descend into the first inner child, keep the rest as a group
      const int s = (__ffs(ik) - 1) ^ (OCT >= 0 ? OCT : oct);
      ik &= ik - 1;
      VSR_CHECK(sp < kMaxStack);
      if constexpr (Q == kClosest) {   // closest: the group remembers its PARENT (re-test on pop)
        if (ik) stack[sp++] = make_uint2(node, ik);
      } else {
        if (ik) stack[sp++] = make_uint2(w1.x, imask | ik << 8);
      }
      node = w1.x + __popc(imask & ((1u << s) - 1u));
      continue;
    }
    if constexpr (Q == kClosest) {
      // closest-hit: a pending child is re-tested against the CURRENT best_t before its node
      // is fetched (one box hook on its decoded box, counted); culled ones are skipped
      for (;;) {
        if (sp == 0) return;
        const uint2 e = stack[sp - 1];
        uint32_t keys = e.y;
        const int s = (__ffs(keys) - 1) ^ (OCT >= 0 ? OCT : oct);
        keys &= keys - 1;
        if (keys) stack[sp - 1].y = keys;
        else --sp;
        VSR_CHECK(e.x < p.num_wide);
        const float4* pp = reinterpret_cast<const float4*>(W + e.x);
        const float4 ph = __ldg(pp);
        const uint4 pw1 = __ldg(reinterpret_cast<const uint4*>(pp + 1));
        const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(pp + 2));
        const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(pp + 3));
        const uint4 q2 = __ldg(reinterpret_cast<const uint4*>(pp + 4));
        const uint32_t hw = __float_as_uint(ph.w), pim = hw >> 24;
        const uint32_t lo_w[3] = {s < 4 ? q0.x : q0.y, s < 4 ? q0.z : q0.w, s < 4 ? q1.x : q1.y};
        const uint32_t hi_w[3] = {s < 4 ? q1.z : q1.w, s < 4 ? q2.x : q2.y, s < 4 ? q2.z : q2.w};
        const float pm[3] = {ph.x, ph.y, ph.z};
        float lo[3], hi[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const float sc = oct_scale(hw, a);
          lo[a] = __fmaf_rn(qbyte(lo_w[a], s & 3), sc, pm[a]);
          hi[a] = __fmaf_rn(qbyte(hi_w[a], s & 3), sc, pm[a]);
        }
        float tn;
        if (!box_hook(isect, T.r, Aabb{lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]}, T.best_t, tn))
          continue;
        node = pw1.x + __popc(pim & ((1u << s) - 1u));
        break;
      }
    } else {
      if (sp == 0) return;
      const uint2 e = stack[sp - 1];
      uint32_t keys = e.y >> 8;
      const uint32_t im = e.y & 0xFFu;
      const int s = (__ffs(keys) - 1) ^ (OCT >= 0 ? OCT : oct);
      keys &= keys - 1;
      if (keys) stack[sp - 1].y = im | keys << 8;
      else --sp;
      node = e.x + __popc(im & ((1u << s) - 1u));
    }
  }
}

template <int Q, class I>
__device__ __forceinline__ void traverse_wide_oct(const TraceParams& p, Trav& T, I& isect,
                                                  uint2* stack, int woct, int oct) {
  switch (woct) {
    case 0: traverse_wide<Q, 0>(p, T, isect, stack, oct); break;
    case 1: traverse_wide<Q, 1>(p, T, isect, stack, oct); break;
    case 2: traverse_wide<Q, 2>(p, T, isect, stack, oct); break;
    case 3: traverse_wide<Q, 3>(p, T, isect, stack, oct); break;
    case 4: traverse_wide<Q, 4>(p, T, isect, stack, oct); break;
    case 5: traverse_wide<Q, 5>(p, T, isect, stack, oct); break;
    case 6: traverse_wide<Q, 6>(p, T, isect, stack, oct); break;
    case 7: traverse_wide<Q, 7>(p, T, isect, stack, oct); break;
    default: traverse_wide<Q, -1>(p, T, isect, stack, oct); break;
  }
}

template <int Q, class I>
__global__ void __launch_bounds__(kBlock, VSR_WIDE_MINB) trace_wide_kernel(const TraceParams p) {
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
  if (id >= p.n) return;
  I isect = make_isect<I>(p);
  Trav T;
  uint2 stack[kMaxStack];   // (child_base, inner slot mask | pending keys << 8)
  const bool go = start_ray(p, T, isect, id);
  const unsigned live = __activemask();
  const int oct = ray_octant(T.r);
  const int woct = __match_any_sync(live, oct) == live ? oct : 8;
  if (go) traverse_wide_oct<Q>(p, T, isect, stack, woct, oct);
  finish(p, T, isect, id);
}

namespace {

template <int Q, class I>
cudaError_t launch_w(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  cudaError_t e = launch_k(trace_wide_kernel<Q, I>, need, kBlock, p.perm && p.pdl, st, p);
  if (e != cudaSuccess) return e;
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int Q>
cudaError_t dispatch_w(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch_w<Q, no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch_w<Q, default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE:
      return p.data.bits ? launch_w<Q, alpha_bits_intersector>(p, st)
                         : launch_w<Q, alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch_w<Q, alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch_w<Q, alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch_w<Q, alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch_w<Q, cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch_w<Q, cost_intersector<alpha_texture_intersector>>(p, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_wide(int query, int isect, const TraceParams& p, cudaStream_t st) {
  return query == kAny ? dispatch_w<kAny>(isect, p, st) : dispatch_w<kClosest>(isect, p, st);
}

}  // namespace vsr
