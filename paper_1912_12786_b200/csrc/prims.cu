// prims.cu — the query on a plain list of primitives, without a BVH
// (PAPER.md:270-274).
#include "traverse.cuh"

namespace vsr {

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

namespace {
template <int Q, class I>
cudaError_t launch_prims_as(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  trace_prims_kernel<Q, I><<<(unsigned)need, kBlock, 0, st>>>(p);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
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

}  // namespace vsr
