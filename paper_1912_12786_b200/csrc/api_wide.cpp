// api_wide.cpp — C ABI of the 8-wide compressed BVH (include/vsr.h
// vsr_bvh8_build / vsr_bvh8_export / vsr_trace_bvh8).
#include "api_internal.hpp"

namespace {

template <class T>
vsr_status upload_vec(T** dst, const std::vector<T>& v, const char* what) {
  *dst = nullptr;
  if (v.empty()) return VSR_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), v.size() * sizeof(T));
  if (e != cudaSuccess) {
    *dst = nullptr;
    return e == cudaErrorMemoryAllocation ? fail(VSR_ERR_OOM, what) : cuda_fail(e, what);
  }
  e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e == cudaSuccess ? VSR_OK : cuda_fail(e, what);
}

}  // namespace

extern "C" {

vsr_status vsr_bvh8_build(vsr_scene* s) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  if (!s->built && !s->host_built) return fail(VSR_ERR_NOT_BUILT, "scene has no BVH");
  auto t0 = std::chrono::steady_clock::now();
  // the binary BVH on the host (host-only scenes keep it; device scenes copy it back)
  HostBvh hb;
  const HostBvh* src = &s->host_bvh;
  if (!s->host_built) {
    const DevScene& d = s->dev;
    hb.root_ref = d.root_ref;
    for (int a = 0; a < 3; ++a) {
      hb.root_lo[a] = d.root_lo[a];
      hb.root_hi[a] = d.root_hi[a];
    }
    try {
      hb.nodes.resize(d.num_nodes);
      hb.tris.resize(d.num_tris);
      hb.sides.resize(d.num_tris);
    } catch (const std::bad_alloc&) {
      return fail(VSR_ERR_OOM, "wide build host copies");
    }
    DeviceGuard g(s->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaError_t e;
    if ((d.num_nodes && (e = cudaMemcpy(hb.nodes.data(), s->d_nodes, d.num_nodes * sizeof(PairNode),
                                        cudaMemcpyDeviceToHost)) != cudaSuccess) ||
        (e = cudaMemcpy(hb.tris.data(), s->d_tris, d.num_tris * sizeof(Tri),
                        cudaMemcpyDeviceToHost)) != cudaSuccess ||
        (e = cudaMemcpy(hb.sides.data(), s->d_sides, d.num_tris * sizeof(Side),
                        cudaMemcpyDeviceToHost)) != cudaSuccess)
      return cuda_fail(e, "wide build copies");
    src = &hb;
  }
  HostWide hw;
  std::string err;
  vsr_status st;
  try {
    st = build_wide(*src, hw, err);
  } catch (const std::bad_alloc&) {
    return fail(VSR_ERR_OOM, "wide build");
  }
  if (st != VSR_OK) return fail(st, err);
  if (s->device >= 0) {
    DeviceGuard g(s->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    s->free_wide();
    if ((st = upload_vec(&s->d_wnodes, hw.nodes, "wide nodes")) != VSR_OK ||
        (st = upload_vec(&s->d_wtris, hw.tris, "wide triangles")) != VSR_OK ||
        (st = upload_vec(&s->d_wsides, hw.sides, "wide sidecars")) != VSR_OK) {
      s->free_wide();
      return st;
    }
    s->num_wnodes = (uint32_t)hw.nodes.size();
    s->wide_depth = hw.max_depth;
    s->host_wide = HostWide{};
    for (int a = 0; a < 3; ++a) {
      s->host_wide.root_lo[a] = hw.root_lo[a];
      s->host_wide.root_hi[a] = hw.root_hi[a];
    }
  } else {
    s->num_wnodes = (uint32_t)hw.nodes.size();
    s->wide_depth = hw.max_depth;
    s->host_wide = std::move(hw);
  }
  s->wide_built = true;
  s->wide_build_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return VSR_OK;
}

vsr_status vsr_bvh8_export(const vsr_scene* s, vsr_bvh8_view* v) {
  g_err.clear();
  if (!s || !v) return fail(VSR_ERR_INVALID_ARG, "NULL scene or view");
  if (!s->wide_built) return fail(VSR_ERR_NOT_BUILT, "scene has no wide BVH: call vsr_bvh8_build");
  v->num_nodes = s->num_wnodes;
  v->num_tris = s->dev.num_tris;
  v->max_depth = s->wide_depth;
  v->pad = 0;
  v->build_ms = s->wide_build_ms;
  for (int a = 0; a < 3; ++a) {
    v->root_lo[a] = s->dev.root_lo[a];
    v->root_hi[a] = s->dev.root_hi[a];
  }
  const size_t nb = (size_t)s->num_wnodes * sizeof(WideNode), tb = (size_t)v->num_tris * sizeof(Tri),
               sb = (size_t)v->num_tris * sizeof(Side);
  if (s->device < 0) {
    if (v->nodes) std::memcpy(v->nodes, s->host_wide.nodes.data(), nb);
    if (v->tris) std::memcpy(v->tris, s->host_wide.tris.data(), tb);
    if (v->sides) std::memcpy(v->sides, s->host_wide.sides.data(), sb);
    return VSR_OK;
  }
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaError_t e;
  if ((v->nodes && (e = cudaMemcpy(v->nodes, s->d_wnodes, nb, cudaMemcpyDefault)) != cudaSuccess) ||
      (v->tris && (e = cudaMemcpy(v->tris, s->d_wtris, tb, cudaMemcpyDefault)) != cudaSuccess) ||
      (v->sides && (e = cudaMemcpy(v->sides, s->d_wsides, sb, cudaMemcpyDefault)) != cudaSuccess))
    return cuda_fail(e, "wide export copy");
  return VSR_OK;
}

vsr_status vsr_trace_bvh8(vsr_scene* s, const vsr_ray* d_rays, uint64_t n, vsr_query query,
                          vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                          vsr_counts* d_counts, void* stream) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  if ((int)isect >= 100 && valid_isect(isect))
    return fail(VSR_ERR_UNSUPPORTED, "run-time controls are not provided for the wide BVH");
  TraceParams p;
  vsr_status st = make_params(s, query, isect, params, p, true, stream);
  if (st != VSR_OK) return st;
  if (s->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only scene (device -1) cannot be traced");
  if (!s->built) return fail(VSR_ERR_NOT_BUILT, "scene has no BVH: call vsr_bvh_build first");
  if (!s->wide_built) return fail(VSR_ERR_NOT_BUILT, "scene has no wide BVH: call vsr_bvh8_build");
  if (n == 0) return VSR_OK;
  if (!d_rays || !d_hits) return fail(VSR_ERR_INVALID_ARG, "NULL rays or hits buffer");
  if (!aligned16(d_rays) || !aligned16(d_hits))
    return fail(VSR_ERR_INVALID_ARG, "rays/hits buffers must be 16-byte aligned");
  if (needs_counts(isect)) {
    if (!d_counts) return fail(VSR_ERR_INVALID_ARG, "COUNT intersector needs a counts buffer");
    if (!aligned16(d_counts)) return fail(VSR_ERR_INVALID_ARG, "counts buffer not 16-B aligned");
  }
  p.rays = reinterpret_cast<const float4*>(d_rays);
  p.hits = reinterpret_cast<float4*>(d_hits);
  p.counts = reinterpret_cast<uint4*>(d_counts);
  p.n = n;
  p.sched = kSchedDirect;
  p.wide = s->d_wnodes;
  p.num_wide = s->num_wnodes;
  p.scene.tris = s->d_wtris;     // the wide leaf order
  p.data.sides = s->d_wsides;
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaError_t e = launch_with_scratch(s->scratch, query, isect, p, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "wide trace launch");
  return VSR_OK;
}

}  // extern "C"
