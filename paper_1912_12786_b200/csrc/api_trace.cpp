// api_trace.cpp — the per-scene trace entry points of the C ABI (include/vsr.h,
// SURVEY.md §8(b)): vsr_trace, vsr_trace_multi, vsr_trace_pinhole,
// vsr_trace_primitives, vsr_trace_tiles (+ the raw device-memory / IPC helpers
// the multi-GPU tile path uses) and vsr_trace_host. Each maps (query,
// intersector) to ONE kernel instantiation per call.
#include "api_internal.hpp"

extern "C" {

vsr_status vsr_trace_tiles(vsr_scene* s, const vsr_ray* d_rays, uint64_t n, uint32_t tile_rays,
                           uint32_t rank, uint32_t world, vsr_query query, vsr_isect isect,
                           const vsr_isect_params* params, vsr_hit* d_hits, vsr_counts* d_counts,
                           void* stream) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  TraceParams p;
  vsr_status st = make_params(s, query, isect, params, p, true, stream);
  if (st != VSR_OK) return st;
  if (s->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only scene (device -1) cannot be traced");
  if (!s->built) return fail(VSR_ERR_NOT_BUILT, "scene has no BVH: call vsr_bvh_build first");
  if (tile_rays == 0 || world == 0 || rank >= world)
    return fail(VSR_ERR_INVALID_ARG, "need tile_rays > 0 and rank < world");
  if (n % tile_rays) return fail(VSR_ERR_INVALID_ARG, "n must be a whole number of tiles");
  if (n >= (1ull << 32) || (n / tile_rays) * (uint64_t)world * tile_rays >= (1ull << 40))
    return fail(VSR_ERR_INVALID_ARG, "shard too large");
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
  p.out_tile = tile_rays;
  p.out_rank = rank;
  p.out_world = world;
  p.sched = kSchedDirect;
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaError_t e = launch_with_scratch(s->scratch, query, isect, p, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tile trace launch");
  return VSR_OK;
}

vsr_status vsr_device_alloc(uint64_t bytes, int device, void** d_ptr) {
  g_err.clear();
  if (!d_ptr || bytes == 0 || device < 0) return fail(VSR_ERR_INVALID_ARG, "bad allocation request");
  DeviceGuard g(device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaError_t e = cudaMalloc(d_ptr, bytes);
  if (e != cudaSuccess) {
    *d_ptr = nullptr;
    return e == cudaErrorMemoryAllocation ? fail(VSR_ERR_OOM, "cudaMalloc") : cuda_fail(e, "cudaMalloc");
  }
  return VSR_OK;
}

vsr_status vsr_device_free(void* d_ptr, int device) {
  g_err.clear();
  if (!d_ptr) return VSR_OK;
  DeviceGuard g(device);
  cudaError_t e = cudaFree(d_ptr);
  return e == cudaSuccess ? VSR_OK : cuda_fail(e, "cudaFree");
}

vsr_status vsr_ipc_handle(const void* d_ptr, void* handle64) {
  g_err.clear();
  if (!d_ptr || !handle64) return fail(VSR_ERR_INVALID_ARG, "NULL pointer or handle");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  std::memcpy(handle64, &h, sizeof h);
  return VSR_OK;
}

vsr_status vsr_ipc_open(const void* handle64, int device, void** d_ptr) {
  g_err.clear();
  if (!handle64 || !d_ptr || device < 0) return fail(VSR_ERR_INVALID_ARG, "bad IPC open request");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  DeviceGuard g(device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    *d_ptr = nullptr;
    return cuda_fail(e, "cudaIpcOpenMemHandle");
  }
  return VSR_OK;
}

vsr_status vsr_ipc_close(void* d_ptr, int device) {
  g_err.clear();
  if (!d_ptr) return VSR_OK;
  DeviceGuard g(device);
  cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  return e == cudaSuccess ? VSR_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

}  // extern "C"

namespace {
// The scene's triangles and sidecars in caller order (prim id order), for the
// primitive-list query; ids the build excluded (degenerate) keep prim = ~0.
vsr_status ensure_caller_order(vsr_scene* s) {
  std::lock_guard<std::mutex> lk(s->caller_mu);
  if (s->d_tris_caller) return VSR_OK;
  const uint32_t m = s->dev.num_tris;
  std::vector<Tri> tris(m);
  std::vector<Side> sides(m);
  cudaError_t e;
  if ((e = cudaMemcpy(tris.data(), s->d_tris, sizeof(Tri) * m, cudaMemcpyDeviceToHost)) !=
          cudaSuccess ||
      (e = cudaMemcpy(sides.data(), s->d_sides, sizeof(Side) * m, cudaMemcpyDeviceToHost)) !=
          cudaSuccess)
    return cuda_fail(e, "caller-order copy");
  uint32_t P = s->num_tris_input;
  for (const Tri& t : tris) P = std::max(P, t.prim + 1u);
  Tri none{};
  none.prim = 0xFFFFFFFFu;
  std::vector<Tri> ct(P, none);
  std::vector<Side> cs(P, Side{});
  for (uint32_t k = 0; k < m; ++k) {
    ct[tris[k].prim] = tris[k];
    cs[tris[k].prim] = sides[k];
  }
  vsr_status st;
  if ((st = dev_upload(&s->d_tris_caller, ct.data(), P, "caller-order triangles")) != VSR_OK ||
      (st = dev_upload(&s->d_sides_caller, cs.data(), P, "caller-order sidecars")) != VSR_OK)
    return st;
  s->num_caller = P;
  return VSR_OK;
}
}  // namespace

extern "C" {

vsr_status vsr_trace_primitives(vsr_scene* s, const vsr_ray* d_rays, uint64_t n, vsr_query query,
                                vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                                vsr_counts* d_counts, void* stream) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  if ((int)isect >= 100 && valid_isect(isect))
    return fail(VSR_ERR_UNSUPPORTED, "run-time controls are not provided for primitive lists");
  TraceParams p;
  vsr_status st = make_params(s, query, isect, params, p, false);
  if (st != VSR_OK) return st;
  if (s->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only scene (device -1) cannot be traced");
  if (!s->built) return fail(VSR_ERR_NOT_BUILT, "scene has no triangles on the device: build first");
  if (n == 0) return VSR_OK;
  if (!d_rays || !d_hits) return fail(VSR_ERR_INVALID_ARG, "NULL rays or hits buffer");
  if (!aligned16(d_rays) || !aligned16(d_hits))
    return fail(VSR_ERR_INVALID_ARG, "rays/hits buffers must be 16-byte aligned");
  if (needs_counts(isect)) {
    if (!d_counts) return fail(VSR_ERR_INVALID_ARG, "COUNT intersector needs a counts buffer");
    if (!aligned16(d_counts)) return fail(VSR_ERR_INVALID_ARG, "counts buffer not 16-B aligned");
  }
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  if ((st = ensure_caller_order(s)) != VSR_OK) return st;
  p.scene.tris = s->d_tris_caller;
  p.scene.num_tris = s->num_caller;
  p.data.sides = s->d_sides_caller;
  p.rays = reinterpret_cast<const float4*>(d_rays);
  p.hits = reinterpret_cast<float4*>(d_hits);
  p.counts = reinterpret_cast<uint4*>(d_counts);
  p.n = n;
  cudaError_t e = launch_prims(query, isect, p, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "primitive-list trace launch");
  return VSR_OK;
}

vsr_status vsr_trace_pinhole(vsr_scene* s, const vsr_pinhole* cam, vsr_query query,
                             vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                             vsr_counts* d_counts, void* stream) {
  g_err.clear();
  if (!s || !cam) return fail(VSR_ERR_INVALID_ARG, "NULL scene or camera");
  if ((int)isect >= 100 && valid_isect(isect))
    return fail(VSR_ERR_UNSUPPORTED, "run-time controls are not provided with in-kernel ray generation");
  TraceParams p;
  vsr_status st = make_params(s, query, isect, params, p, true, stream);
  if (st != VSR_OK) return st;
  if (s->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only scene (device -1) cannot be traced");
  if (!s->built) return fail(VSR_ERR_NOT_BUILT, "scene has no BVH: call vsr_bvh_build first");
  if (cam->width == 0 || cam->height == 0 || cam->width % 8 || cam->height % 8)
    return fail(VSR_ERR_INVALID_ARG, "width and height must be positive multiples of 8");
  uint32_t side = 1;
  while (side * side < cam->spp && side < 65536) ++side;
  if (cam->spp == 0 || side * side != cam->spp)
    return fail(VSR_ERR_INVALID_ARG, "spp must be a perfect square >= 1");
  const double* vals[] = {cam->eye, cam->w, cam->u, cam->v};
  for (const double* vv : vals)
    for (int k = 0; k < 3; ++k)
      if (!std::isfinite(vv[k])) return fail(VSR_ERR_INVALID_ARG, "non-finite camera");
  if (!std::isfinite(cam->tan_half_vfov) || !std::isfinite(cam->aspect) || std::isnan(cam->tmin) ||
      std::isnan(cam->tmax))
    return fail(VSR_ERR_INVALID_ARG, "non-finite camera");
  const uint64_t n = (uint64_t)cam->width * cam->height * cam->spp;
  if (!d_hits) return fail(VSR_ERR_INVALID_ARG, "NULL hits buffer");
  if (!aligned16(d_hits)) return fail(VSR_ERR_INVALID_ARG, "hits buffer must be 16-byte aligned");
  if (needs_counts(isect)) {
    if (!d_counts) return fail(VSR_ERR_INVALID_ARG, "COUNT intersector needs a counts buffer");
    if (!aligned16(d_counts)) return fail(VSR_ERR_INVALID_ARG, "counts buffer not 16-B aligned");
  }
  p.gen = 1;
  for (int k = 0; k < 3; ++k) {
    p.cam.eye[k] = cam->eye[k];
    p.cam.w[k] = cam->w[k];
    p.cam.u[k] = cam->u[k];
    p.cam.v[k] = cam->v[k];
  }
  p.cam.tan_half = cam->tan_half_vfov;
  p.cam.aspect = cam->aspect;
  p.cam.width = cam->width;
  p.cam.height = cam->height;
  p.cam.spp = cam->spp;
  p.cam.seed = cam->jitter_seed;
  p.cam.side = side;
  p.cam.tmin = cam->tmin;
  p.cam.tmax = cam->tmax;
  p.sched = kSchedDirect;   // the persistent schedule reads a ray buffer
  p.rays = nullptr;
  p.hits = reinterpret_cast<float4*>(d_hits);
  p.counts = reinterpret_cast<uint4*>(d_counts);
  p.n = n;
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaError_t e = launch_with_scratch(s->scratch, query, isect, p, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pinhole trace launch");
  return VSR_OK;
}

vsr_status vsr_trace(vsr_scene* s, const vsr_ray* d_rays, uint64_t n, vsr_query query,
                     vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                     vsr_counts* d_counts, void* stream) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  TraceParams p;
  vsr_status st = make_params(s, query, isect, params, p, true, stream);
  if (st != VSR_OK) return st;
  if (s->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only scene (device -1) cannot be traced");
  if (!s->built) return fail(VSR_ERR_NOT_BUILT, "scene has no BVH: call vsr_bvh_build first");
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
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  p.counter = next_counter(s);
  cudaError_t e = launch_with_scratch(s->scratch, query, isect, p, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "trace kernel launch");
  return VSR_OK;
}

vsr_status vsr_trace_multi(vsr_scene* s, const vsr_ray* d_rays, uint64_t n, uint32_t max_hits,
                           vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                           uint32_t* d_num_hits, vsr_counts* d_counts, void* stream) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  if (max_hits < 1 || max_hits > 16) return fail(VSR_ERR_INVALID_ARG, "max_hits must be in [1, 16]");
  if ((int)isect >= 100 && valid_isect(isect))
    return fail(VSR_ERR_UNSUPPORTED, "run-time controls are not provided for the multi-hit query");
  TraceParams p;
  vsr_status st = make_params(s, VSR_QUERY_CLOSEST, isect, params, p, true, stream);
  if (st != VSR_OK) return st;
  if (s->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only scene (device -1) cannot be traced");
  if (!s->built) return fail(VSR_ERR_NOT_BUILT, "scene has no BVH: call vsr_bvh_build first");
  if (n == 0) return VSR_OK;
  if (!d_rays || !d_hits) return fail(VSR_ERR_INVALID_ARG, "NULL rays or hits buffer");
  if (!aligned16(d_rays) || !aligned16(d_hits))
    return fail(VSR_ERR_INVALID_ARG, "rays/hits buffers must be 16-byte aligned");
  if (d_num_hits && (reinterpret_cast<uintptr_t>(d_num_hits) & 3u))
    return fail(VSR_ERR_INVALID_ARG, "num_hits buffer must be 4-byte aligned");
  if (needs_counts(isect)) {
    if (!d_counts) return fail(VSR_ERR_INVALID_ARG, "COUNT intersector needs a counts buffer");
    if (!aligned16(d_counts)) return fail(VSR_ERR_INVALID_ARG, "counts buffer not 16-B aligned");
  }
  p.rays = reinterpret_cast<const float4*>(d_rays);
  p.hits = reinterpret_cast<float4*>(d_hits);
  p.counts = reinterpret_cast<uint4*>(d_counts);
  p.n = n;
  p.max_hits = (int)max_hits;
  p.num_hits = d_num_hits;
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  p.counter = next_counter(s);
  cudaError_t e = launch_with_scratch(s->scratch, 2 /* multi */, isect, p, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "multi-hit trace launch");
  return VSR_OK;
}

}  // extern "C"

extern "C" {

vsr_status vsr_trace_host(vsr_scene* s, const vsr_ray* h_rays, uint64_t n, vsr_query query,
                          vsr_isect isect, const vsr_isect_params* params, vsr_hit* h_hits,
                          vsr_counts* h_counts, void* stream) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  TraceParams p;
  vsr_status st = make_params(s, query, isect, params, p, true, stream);
  if (st != VSR_OK) return st;
  if (s->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only scene (device -1) cannot be traced");
  if (!s->built) return fail(VSR_ERR_NOT_BUILT, "scene has no BVH: call vsr_bvh_build first");
  if (n == 0) return VSR_OK;
  if (!h_rays || !h_hits) return fail(VSR_ERR_INVALID_ARG, "NULL rays or hits buffer");
  const bool cnt = needs_counts(isect);
  if (cnt && !h_counts) return fail(VSR_ERR_INVALID_ARG, "COUNT intersector needs counts");
  std::lock_guard<std::mutex> lk(s->stage_mu);
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  // Chunked pipeline on three streams: every chunk's H2D copy goes on s_in,
  // its trace on s_run, its D2H copy on s_out, chained by per-chunk events, so
  // the host-to-device copy engine never waits behind a device-to-host copy or
  // a kernel (both directions of the link and the SMs work at once). Chunk
  // buffers form a ring of kSlots; a slot's next H2D waits for its last D2H.
  // Chunk size: n/8 within [256 Ki, 1 Mi] rays (measured, profiles/r01_tuning.md).
  const char* ec = std::getenv("VSR_HOST_CHUNK");   // tuning knob: rays per chunk
  const uint64_t want = ec ? std::max<uint64_t>(4096, std::strtoull(ec, nullptr, 10))
                           : std::min<uint64_t>(1u << 20, std::max<uint64_t>(1u << 18, n / 8));
  const uint64_t chunk = std::min<uint64_t>(n, want);
  cudaError_t e;
  if (s->stage_cap < chunk || (cnt && !s->stage_counts)) {
    s->free_stage();
    bool ok = true;
    for (int k = 0; k < vsr_scene::kSlots && ok; ++k) {
      ok = (e = cudaMalloc(&s->d_in[k], chunk * 32)) == cudaSuccess &&
           (e = cudaMalloc(&s->d_out[k], chunk * 16)) == cudaSuccess &&
           (!cnt || (e = cudaMalloc(&s->d_cnt[k], chunk * 16)) == cudaSuccess) &&
           (e = cudaEventCreateWithFlags(&s->ev_in[k], cudaEventDisableTiming)) == cudaSuccess &&
           (e = cudaEventCreateWithFlags(&s->ev_run[k], cudaEventDisableTiming)) == cudaSuccess &&
           (e = cudaEventCreateWithFlags(&s->ev_out[k], cudaEventDisableTiming)) == cudaSuccess;
    }
    ok = ok && (e = cudaStreamCreateWithFlags(&s->s_in, cudaStreamNonBlocking)) == cudaSuccess &&
         (e = cudaStreamCreateWithFlags(&s->s_run, cudaStreamNonBlocking)) == cudaSuccess &&
         (e = cudaStreamCreateWithFlags(&s->s_out, cudaStreamNonBlocking)) == cudaSuccess &&
         (e = cudaEventCreateWithFlags(&s->ev_start, cudaEventDisableTiming)) == cudaSuccess;
    if (!ok) {
      s->free_stage();
      return e == cudaErrorMemoryAllocation ? fail(VSR_ERR_OOM, "staging allocation")
                                            : cuda_fail(e, "staging allocation");
    }
    s->stage_cap = chunk;
    s->stage_counts = cnt;
  }
  cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
  if ((e = cudaEventRecord(s->ev_start, user)) != cudaSuccess) return cuda_fail(e, "event");
  for (cudaStream_t ss : {s->s_in, s->s_run, s->s_out})
    if ((e = cudaStreamWaitEvent(ss, s->ev_start, 0)) != cudaSuccess)
      return cuda_fail(e, "stream wait");
  const char* src = reinterpret_cast<const char*>(h_rays);
  char* dst = reinterpret_cast<char*>(h_hits);
  char* cdst = reinterpret_cast<char*>(h_counts);
  uint64_t c = 0;
  for (uint64_t b = 0; b < n; b += chunk, ++c) {
    const int k = (int)(c % vsr_scene::kSlots);
    const uint64_t m = std::min(chunk, n - b);
    if (c >= (uint64_t)vsr_scene::kSlots &&   // the slot's previous hits are out
        (e = cudaStreamWaitEvent(s->s_in, s->ev_out[k], 0)) != cudaSuccess)
      return cuda_fail(e, "stream wait");
    if ((e = cudaMemcpyAsync(s->d_in[k], src + b * 32, m * 32, cudaMemcpyHostToDevice,
                             s->s_in)) != cudaSuccess)
      return cuda_fail(e, "H2D rays");
    if ((e = cudaEventRecord(s->ev_in[k], s->s_in)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s->s_run, s->ev_in[k], 0)) != cudaSuccess)
      return cuda_fail(e, "event");
    p.rays = s->d_in[k];
    p.hits = s->d_out[k];
    p.counts = s->d_cnt[k];
    p.n = m;
    p.counter = next_counter(s);
    if ((e = launch_with_scratch(s->scratch, query, isect, p, s->s_run)) != cudaSuccess)
      return cuda_fail(e, "trace launch");
    if ((e = cudaEventRecord(s->ev_run[k], s->s_run)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s->s_out, s->ev_run[k], 0)) != cudaSuccess)
      return cuda_fail(e, "event");
    if ((e = cudaMemcpyAsync(dst + b * 16, s->d_out[k], m * 16, cudaMemcpyDeviceToHost,
                             s->s_out)) != cudaSuccess)
      return cuda_fail(e, "D2H hits");
    if (cnt && (e = cudaMemcpyAsync(cdst + b * 16, s->d_cnt[k], m * 16, cudaMemcpyDeviceToHost,
                                    s->s_out)) != cudaSuccess)
      return cuda_fail(e, "D2H counts");
    if ((e = cudaEventRecord(s->ev_out[k], s->s_out)) != cudaSuccess)
      return cuda_fail(e, "event");
  }
  // s_out's last copy follows every trace and every H2D (event chains)
  if ((e = cudaEventRecord(s->ev_start, s->s_out)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(user, s->ev_start, 0)) != cudaSuccess)
    return cuda_fail(e, "stream wait");
  if ((e = cudaStreamSynchronize(user)) != cudaSuccess) return cuda_fail(e, "trace (host)");
  return VSR_OK;
}

}  // extern "C"
