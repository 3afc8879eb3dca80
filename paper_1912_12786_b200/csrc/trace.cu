// trace.cu — the hot path: per-ray BVH traversal + ray/triangle intersection
// with a compile-time intersector (§3.2).
//
// One thread per ray.  The traversal is the while-while scheme of Aila &
// Laine cited by the paper: an inner-node loop that calls
// the intersector's box hook on both children of a 64-B pair node, then a
// leaf loop that calls its triangle hook on each primitive.  Every decision
// is a function of the ray alone (no warp-voted speculation), so the
// counting intersector's numbers are deterministic and match the CPU walker
// bit for bit.
//
// Build: -gencode arch=compute_100a,code=sm_100a -fmad=false (IEEE fp32
// contract; see DESIGN.md A.1-A.3).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <string>

#include "intersectors.cuh"
#include "trace.hpp"

namespace vsr {

constexpr int kBlock = 128;
constexpr uint32_t kMissPrim = 0xFFFFFFFFu;
enum : int { kClosest = 0, kAny = 1 };

template <class I>
__device__ __forceinline__ bool box_hook(I& isect, const RayCtx& r, const Aabb& b, float best_t,
                                         float& tn) {
  if constexpr (std::is_same<I, no_intersector>::value) return intersect(r, b, best_t, tn);
  else return isect(r, b, best_t, tn);
}

template <class I>
__device__ __forceinline__ hit_record tri_hook(I& isect, const RayCtx& r, const TriData& t,
                                               uint32_t k, float tmax_cur) {
  if constexpr (std::is_same<I, no_intersector>::value) return intersect(r, t, k, tmax_cur);
  else return isect(r, t, k, tmax_cur);
}

struct Result {
  float t, u, v;
  uint32_t prim;
};

// intersect(ray, BVH, isect) — PAPER.md:228-247, both call sites hooked
// (PAPER.md:248-252).
template <int Q, class I>
__device__ __forceinline__ Result traverse(const DevScene& S, const RayCtx& r, float tmax,
                                           I& isect) {
  Result res{__int_as_float(0x7f800000), 0.0f, 0.0f, kMissPrim};
  float best_t = tmax;
  bool have = false;
  float tn;
  const Aabb root{S.root_lo[0], S.root_lo[1], S.root_lo[2],
                  S.root_hi[0], S.root_hi[1], S.root_hi[2]};
  // The root box is tested (and counted) once before the loop (reading A11).
  if (!box_hook(isect, r, root, best_t, tn)) return res;

  float2 stack[kMaxStack];   // (ref bits, tnear); depth <= 64 guaranteed by the build
  int sp = 0;
  uint32_t cur = S.root_ref;
  for (;;) {
    // ---- inner-node loop: "while node is inner" ----
    while (!(cur & kLeafBit)) {
      const float4* np = reinterpret_cast<const float4*>(S.nodes + cur);
      const float4 n0 = __ldg(np), n1 = __ldg(np + 1), n2 = __ldg(np + 2), n3 = __ldg(np + 3);
      const Aabb b0{n0.x, n0.y, n0.z, n0.w, n1.x, n1.y};
      const Aabb b1{n1.z, n1.w, n2.x, n2.y, n2.z, n2.w};
      float tn0, tn1;
      const bool h0 = box_hook(isect, r, b0, best_t, tn0);
      const bool h1 = box_hook(isect, r, b1, best_t, tn1);
      const uint32_t r0 = __float_as_uint(n3.x), r1 = __float_as_uint(n3.y);
      if (h0 && h1) {
        const bool swap = tn1 < tn0;   // nearer child first, ties -> child 0 (reading A13)
        stack[sp] = make_float2(__uint_as_float(swap ? r0 : r1), swap ? tn0 : tn1);
        ++sp;
        cur = swap ? r1 : r0;
      } else if (h0) {
        cur = r0;
      } else if (h1) {
        cur = r1;
      } else {
        goto pop;
      }
    }
    // ---- leaf loop: "while node contains untested primitives" ----
    {
      const uint32_t first = cur & kLeafFirstMask;
      const uint32_t end = first + ((cur >> kLeafCountShift) & 31u) + 1u;
      for (uint32_t k = first; k < end; ++k) {
        const float4* tp = reinterpret_cast<const float4*>(S.tris + k);
        const TriData td{__ldg(tp), __ldg(tp + 1), __ldg(tp + 2)};
        const hit_record hr = tri_hook(isect, r, td, k, best_t);
        if (Q == kAny) {
          if (hr.hit) {   // any-hit: the first accepted hit ends the query
            res = Result{hr.t, hr.u, hr.v, __float_as_uint(td.a.w)};
            return res;
          }
        } else if (hr.hit && (!have || hr.t < best_t)) {
          // closest-hit: accepted hits shrink tmax; vetoed ones do not
          best_t = hr.t;
          have = true;
          res = Result{hr.t, hr.u, hr.v, __float_as_uint(td.a.w)};
        }
      }
    }
  pop:
    for (;;) {   // entries farther than the current best are dropped unhooked (A14)
      if (sp == 0) return res;
      --sp;
      const float2 e = stack[sp];
      if (e.y <= best_t) {
        cur = __float_as_uint(e.x);
        break;
      }
    }
  }
}

template <class I>
__device__ __forceinline__ I make_isect(const TraceParams& p) {
  I isect{};
  if constexpr (std::is_base_of<alpha_texture_intersector, I>::value) {
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

template <int Q, class I>
__global__ void __launch_bounds__(kBlock) trace_kernel(const TraceParams p) {
  const uint64_t i = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
  if (i >= p.n) return;
  const float4 a = __ldg(p.rays + 2 * i);
  const float4 b = __ldg(p.rays + 2 * i + 1);
  RayCtx r;
  r.ox = a.x; r.oy = a.y; r.oz = a.z; r.tmin = a.w;
  r.dx = b.x; r.dy = b.y; r.dz = b.z;
  // guarded reciprocal (reading A20): no 0*inf NaN in the slab test
  r.ix = 1.0f / (fabsf(b.x) > 0x1p-80f ? b.x : copysignf(0x1p-80f, b.x));
  r.iy = 1.0f / (fabsf(b.y) > 0x1p-80f ? b.y : copysignf(0x1p-80f, b.y));
  r.iz = 1.0f / (fabsf(b.z) > 0x1p-80f ? b.z : copysignf(0x1p-80f, b.z));
  I isect = make_isect<I>(p);
  const Result res = traverse<Q>(p.scene, r, b.w, isect);
  p.hits[i] = make_float4(res.t, res.u, res.v, __uint_as_float(res.prim));
  if constexpr (I::kCounts) {
    p.counts[i] = make_uint4(isect.num_boxes, isect.num_tris, isect.lookups(), 0u);
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

template <int Q, class I>
cudaError_t launch(const TraceParams& p, cudaStream_t st) {
  const uint64_t blocks = (p.n + kBlock - 1) / kBlock;
  trace_kernel<Q, I><<<(unsigned)blocks, kBlock, 0, st>>>(p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int Q>
cudaError_t dispatch_isect(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch<Q, no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch<Q, default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE: return launch<Q, alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch<Q, alpha_procedural_intersector>(p, st);
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

cudaError_t launch_trace(int query, int isect, const TraceParams& p, cudaStream_t st) {
  if (p.n == 0) return cudaSuccess;
  return query == kAny ? dispatch_isect<kAny>(isect, p, st) : dispatch_isect<kClosest>(isect, p, st);
}

uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

}  // namespace vsr
