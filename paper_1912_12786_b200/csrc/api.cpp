// api.cpp — the C ABI declared in include/vsr.h.
//
// Host-side responsibilities: argument validation, scene ingest (SPEC
// S:433-436), BVH build + upload (untimed setup), export/import of the
// flattened structure for multi-GPU replication, and the host dispatch that
// maps (query, intersector) to ONE kernel instantiation per call (PAPER.md:
// 74-78: the choice is made once, outside the innermost loop).
//
// The trace entry points live in api_trace.cpp, lists and instancing in
// api_compound.cpp; the state they share is in api_internal.hpp.
#include "api_internal.hpp"

namespace vsr_api {

thread_local std::string g_err;

vsr_status fail(vsr_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

vsr_status cuda_fail(cudaError_t e, const char* what) {
  return fail(VSR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Copy `bytes` from src (host or device memory) into host memory.
cudaError_t to_host(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, src);
  if (e != cudaSuccess || at.type == cudaMemoryTypeUnregistered || at.type == cudaMemoryTypeHost) {
    cudaGetLastError();   // clear a sticky "no device" / invalid value from the query
    std::memcpy(dst, src, bytes);
    return cudaSuccess;
  }
  return cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
}

// Upload flattened arrays (host or device sources) and fill scene->dev.
vsr_status upload(vsr_scene* s, uint32_t root_ref, const float* root_lo, const float* root_hi,
                  const void* nodes, uint32_t num_nodes, const void* tris, const void* sides,
                  uint32_t num_tris, const void* texdescs, uint32_t num_textures,
                  const void* texels, uint64_t num_texels) {
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  s->free_device();
  vsr_status st;
  if ((st = dev_upload(&s->d_nodes, nodes, num_nodes, "nodes")) != VSR_OK) return st;
  if ((st = dev_upload(&s->d_tris, tris, num_tris, "triangles")) != VSR_OK) return st;
  if ((st = dev_upload(&s->d_sides, sides, num_tris, "sidecars")) != VSR_OK) return st;
  if ((st = dev_upload(&s->d_texdescs, texdescs, num_textures, "texdescs")) != VSR_OK) return st;
  if ((st = dev_upload(&s->d_texels, texels, num_texels, "texels")) != VSR_OK) return st;
  {
    const size_t cbytes = sizeof(unsigned long long) * 2 * kCounterSlots;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&s->d_counters), cbytes);
    if (e != cudaSuccess) return cuda_fail(e, "counters");
    if ((e = cudaMemset(s->d_counters, 0, cbytes)) != cudaSuccess) return cuda_fail(e, "counters");
    // cudaMemset may return before the zeroes land; the build is synchronous, so
    // wait here rather than rely on legacy-stream ordering against later streams
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cuda_fail(e, "counters");
  }
  s->num_texels = num_texels;
  DevScene& d = s->dev;
  d.counters = s->d_counters;
  d.nodes = s->d_nodes;
  d.tris = s->d_tris;
  d.sides = s->d_sides;
  d.texdescs = s->d_texdescs;
  d.texels = s->d_texels;
  d.root_ref = root_ref;
  for (int a = 0; a < 3; ++a) {
    d.root_lo[a] = root_lo[a];
    d.root_hi[a] = root_hi[a];
  }
  d.num_nodes = num_nodes;
  d.num_tris = num_tris;
  d.num_textures = num_textures;
  {   // density grid: the order pass's cost proxy (scheduling only; results never depend on it)
    density_grid_dims(d.root_lo, d.root_hi, d.gdim, d.gscale);
    const size_t cells = density_grid_words(d.gdim);
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&s->d_grid), cells * sizeof(uint32_t));
    if (e != cudaSuccess) return cuda_fail(e, "density grid");
    if ((e = cudaMemset(s->d_grid, 0, cells * sizeof(uint32_t))) != cudaSuccess ||
        (e = build_density_grid(s->d_tris, num_tris, d.root_lo, d.gdim, d.gscale, s->d_grid,
                                nullptr)) != cudaSuccess ||
        (e = cudaDeviceSynchronize()) != cudaSuccess)
      return cuda_fail(e, "density grid");
    d.grid = s->d_grid;
  }
  s->stats.num_nodes = num_nodes;
  s->stats.num_tris = num_tris;
  s->stats.num_textures = num_textures;
  s->stats.num_texels = num_texels;
  s->stats.device_bytes = (uint64_t)num_nodes * 64 + (uint64_t)num_tris * 80 +
                          (uint64_t)num_textures * 16 + num_texels;
  s->built = true;
  s->stats.built = 1;
  return VSR_OK;
}

// smallest a8 in [0,255] with (float)a8 / 255.0f >= thr, evaluated with the
// exact fp32 expression of the listing (reading A7); 256 = none.
uint32_t alpha_min_a8(float thr) {
  for (uint32_t a = 0; a < 256; ++a)
    if ((float)a / 255.0f >= thr) return a;
  return 256;
}

bool valid_isect(int k) {
  switch (k) {
    case VSR_ISECT_NONE:
    case VSR_ISECT_DEFAULT:
    case VSR_ISECT_ALPHA_TEXTURE:
    case VSR_ISECT_ALPHA_PROCEDURAL:
    case VSR_ISECT_COUNT:
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR:
    case VSR_ISECT_ALPHA_PROCEDURAL_UV:
    case VSR_ISECT_RUNTIME_SWITCH_DEFAULT:
    case VSR_ISECT_RUNTIME_SWITCH_ALPHA_TEXTURE:
    case VSR_ISECT_RUNTIME_SWITCH_ALPHA_PROCEDURAL:
    case VSR_ISECT_RUNTIME_FNPTR_DEFAULT:
    case VSR_ISECT_RUNTIME_FNPTR_ALPHA_TEXTURE:
    case VSR_ISECT_RUNTIME_FNPTR_ALPHA_PROCEDURAL: return true;
    default: return false;
  }
}

// The scene's 1-bit alpha plane for a_min (alpha_keep_bits), built on first
// use; nullptr when the textures are not 32-aligned, the cache is full or the
// build fails (the A8 path then runs: same results). VSR_ALPHA_BITS=0 disables.
const uint32_t* alpha_plane(vsr_scene* s, uint32_t a_min, void* stream) {
  const char* eb = std::getenv("VSR_ALPHA_BITS");
  if ((eb && std::strcmp(eb, "0") == 0) || !s->built || s->dev.num_textures == 0) return nullptr;
  std::lock_guard<std::mutex> lk(s->bits_mu);
  const uint32_t nt = s->dev.num_textures;
  for (int i = 0; i < s->num_planes; ++i)
    if (s->plane_amin[i] == a_min) return s->d_planes[i];
  // no synchronous build while the call's stream is being captured into a graph
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(reinterpret_cast<cudaStream_t>(stream), &cs) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (cs != cudaStreamCaptureStatusNone) return nullptr;
  if (s->bits_ok < 0) {   // once per device state: are all textures 32-aligned?
    std::vector<TexDesc> descs(nt);
    if (cudaMemcpy(descs.data(), s->d_texdescs, nt * sizeof(TexDesc), cudaMemcpyDeviceToHost) !=
        cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    bool ok = s->num_texels % 32 == 0;
    uint64_t max_words = 0;
    for (const TexDesc& d : descs) {
      ok = ok && d.w % 32 == 0 && d.h % 32 == 0 && d.offset % 1024 == 0;
      max_words = std::max<uint64_t>(max_words, (uint64_t)d.w * d.h / 32);
    }
    s->bits_ok = ok ? 1 : 0;
    s->bits_max_words = max_words;
  }
  if (s->bits_ok != 1) return nullptr;
  const uint64_t max_words = s->bits_max_words;
  if (s->num_planes == vsr_scene::kMaxPlanes) return nullptr;
  DeviceGuard g(s->device);
  uint32_t* d = nullptr;
  cudaStream_t st = nullptr;
  bool ok = cudaMalloc(&d, s->num_texels / 8) == cudaSuccess &&
            cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
            build_alpha_bits(s->d_texdescs, nt, s->d_texels, a_min, d, max_words, st) ==
                cudaSuccess &&
            cudaStreamSynchronize(st) == cudaSuccess;
  if (st) cudaStreamDestroy(st);
  if (!ok) {
    cudaGetLastError();
    cudaFree(d);
    return nullptr;
  }
  s->plane_amin[s->num_planes] = a_min;
  s->d_planes[s->num_planes++] = d;
  return d;
}

vsr_status make_params(vsr_scene* s, vsr_query query, vsr_isect isect,
                       const vsr_isect_params* params, TraceParams& p, bool alpha_bits,
                       void* stream) {
  if (query != VSR_QUERY_CLOSEST && query != VSR_QUERY_ANY)
    return fail(VSR_ERR_INVALID_ARG, "invalid query");
  if (!valid_isect(isect)) return fail(VSR_ERR_INVALID_ARG, "invalid intersector kind");
  vsr_isect_params ip{0.01f, 8u};
  if (params) ip = *params;
  if (std::isnan(ip.alpha_threshold)) return fail(VSR_ERR_INVALID_ARG, "alpha_threshold is NaN");
  if (ip.checker_freq < 1u || ip.checker_freq > (1u << 24))
    return fail(VSR_ERR_INVALID_ARG, "checker_freq must be in [1, 2^24]");
  std::memset(&p, 0, sizeof p);
  p.scene = s->dev;
  p.data.sides = s->d_sides;
  p.data.descs = s->d_texdescs;
  p.data.texels = s->d_texels;
  p.data.num_texels = s->num_texels;
  p.data.a_min = alpha_min_a8(ip.alpha_threshold);
  p.data.fm = (float)ip.checker_freq;
  p.data.thr = ip.alpha_threshold;
  if (alpha_bits && isect == VSR_ISECT_ALPHA_TEXTURE)
    p.data.bits = alpha_plane(s, p.data.a_min, stream);
  int kind = 0;
  if (isect >= 200) kind = isect - 200;
  else if (isect >= 100) kind = isect - 100;
  p.runtime_kind = kind;
  if (isect >= 200 && kind != 1) {
    if (!s->fn_cached[kind]) {
      DeviceGuard g(s->device);
      cudaError_t e = filter_fn_pointer(kind, &s->fn_cache[kind]);
      if (e != cudaSuccess) return cuda_fail(e, "filter function pointer");
      s->fn_cached[kind] = true;
    }
    p.filter_fn = s->fn_cache[kind];
  }
  // Scheduling knobs (read per call; defaults are the measured best):
  // VSR_SCHED=persistent selects the persistent kernel, VSR_REFILL its refill threshold.
  const char* ev = std::getenv("VSR_REFILL");
  const int refill = ev ? std::atoi(ev) : 32;
  p.refill = refill < 1 ? 1 : (refill > 32 ? 32 : refill);
  const char* es = std::getenv("VSR_SCHED");
  p.sched = (es && std::strcmp(es, "persistent") == 0) ? kSchedPersistent
            : (es && std::strcmp(es, "warp") == 0)      ? kSchedWarp
            : (es && std::strcmp(es, "region") == 0)    ? kSchedRegion
                                                         : kSchedDirect;
  const char* eo = std::getenv("VSR_ORDER");   // "0" disables longest-first block order
  p.order = (eo && std::strcmp(eo, "0") == 0) ? 0 : 1;
  // order pass cost proxy: "grid" (density-grid line integral, 16 samples), "len" (segment
  // length in the root box), "mix" (mean of a 4-sample grid bucket and the length bucket);
  // unset = auto: grid for instanced queries (measured +4-5 %), mix otherwise (C2 +1.2 %,
  // C4 +0.8 %, C5 -0.2 % against len; pure grid: C4 -8 to -25 %; profiles/r02_tuning.md)
  const char* eg = std::getenv("VSR_ORDER_PROXY");
  p.order_proxy = !eg ? 2
                  : (std::strcmp(eg, "grid") == 0 ? 1 : std::strcmp(eg, "mix") == 0 ? 3 : 0);
  const char* ep = std::getenv("VSR_PDL");   // "0": plain launches after the order pass
  p.pdl = (ep && std::strcmp(ep, "0") == 0) ? 0 : 1;
  // 12-CTA occupancy variant for scenes that do not fit in L2 (VSR_OCC=0/1 forces it)
  const char* eo2 = std::getenv("VSR_OCC");
  if (eo2) {
    p.occ = std::strcmp(eo2, "0") != 0;
  } else {
    int l2 = 0;
    if (s->device >= 0 &&
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, s->device) != cudaSuccess) {
      cudaGetLastError();
      l2 = 0;
    }
    p.occ = l2 > 0 && s->stats.device_bytes > (uint64_t)l2;
  }
  return VSR_OK;
}

// Launch with the owner's scratch for stream `st` (created or grown on first
// use; the launch waits for the scratch's previous use, then records its own).
// Caller holds no lock; n must be the launch's ray count.
cudaError_t launch_with_scratch(ScratchSet& set, int query, int isect, TraceParams& p,
                                cudaStream_t st) {
  // Under stream capture (CUDA graphs) the owner's event-guarded scratch is not
  // used: launch_trace takes a stream-ordered allocation instead, which the
  // graph records as its own memory nodes, so every replay has private scratch.
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) cudaGetLastError();
  if (cs != cudaStreamCaptureStatusNone) {
    p.order_scratch = nullptr;
    p.order_scratch_bytes = 0;
    return launch_trace(query, isect, p, st);
  }
  std::lock_guard<std::mutex> lk(set.mu);
  const size_t bytes = order_scratch_bytes(p.n);
  ScratchSet::OrderScratch* o = nullptr;
  for (auto& e : set.v)
    if (e.st == st) o = &e;
  cudaError_t e = cudaSuccess;
  if (!o && set.v.size() < 16) {
    ScratchSet::OrderScratch n{st, nullptr, 0, nullptr};
    if ((e = cudaEventCreateWithFlags(&n.ev, cudaEventDisableTiming)) != cudaSuccess) return e;
    set.v.push_back(n);
    o = &set.v.back();
  }
  p.order_scratch = nullptr;
  p.order_scratch_bytes = 0;
  if (o) {
    if (o->cap < bytes) {
      cudaEventSynchronize(o->ev);
      cudaFree(o->ptr);
      o->ptr = nullptr;
      o->cap = 0;
      if ((e = cudaMalloc(&o->ptr, bytes)) != cudaSuccess) return e;
      // the order histogram must be zero at each launch's entry (launch_trace
      // keeps it so: the trace kernel re-zeroes it).  Zeroed on the launch
      // stream itself: a legacy-stream memset is not ordered before kernels on
      // a non-blocking stream, and the event wait below is a no-op on first use.
      if ((e = cudaMemsetAsync(o->ptr, 0, bytes, st)) != cudaSuccess) {
        cudaFree(o->ptr);
        o->ptr = nullptr;
        return e;
      }
      o->cap = bytes;
    }
    if ((e = cudaStreamWaitEvent(st, o->ev, 0)) != cudaSuccess) return e;
    p.order_scratch = o->ptr;
    p.order_scratch_bytes = o->cap;
  }
  e = launch_trace(query, isect, p, st);
  // recorded even when the launch failed part-way: kernels touching the
  // scratch may already be queued, and the next user must wait for them
  if (o) {
    const cudaError_t r = cudaEventRecord(o->ev, st);
    if (e == cudaSuccess) e = r;
  }
  return e;
}

// A fresh work-counter slot per launch (self-reset by the launch's last warp).
unsigned long long* next_counter(vsr_scene* s) {
  const uint32_t slot = s->launch_seq.fetch_add(1, std::memory_order_relaxed) % kCounterSlots;
  return s->d_counters + 2 * (size_t)slot;
}

}  // namespace vsr_api

extern "C" {

uint32_t vsr_abi_version(void) { return VSR_ABI_VERSION; }

const char* vsr_last_error(void) { return g_err.c_str(); }

uint64_t vsr_launch_count(void) { return launch_count(); }

vsr_status vsr_set_kernel_events(void* start, void* stop) {
  g_err.clear();
  if ((start == nullptr) != (stop == nullptr))
    return fail(VSR_ERR_INVALID_ARG, "set both events or neither");
  set_kernel_events(start, stop);
  return VSR_OK;
}

vsr_status vsr_scene_create(const vsr_scene_desc* desc, vsr_scene** out) {
  g_err.clear();
  if (!desc || !out) return fail(VSR_ERR_INVALID_ARG, "NULL desc or out");
  *out = nullptr;
  const uint32_t n = desc->num_tris;
  if (n > 0 && !desc->vertices) return fail(VSR_ERR_INVALID_ARG, "vertices is NULL");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0 &&
      (desc->device < -1 || desc->device >= ndev))
    return fail(VSR_ERR_INVALID_ARG, "device ordinal out of range");
  for (size_t i = 0; i < (size_t)n * 9; ++i)
    if (!std::isfinite(desc->vertices[i]))
      return fail(VSR_ERR_NONFINITE, "non-finite vertex coordinate at triangle " +
                                         std::to_string(i / 9));
  if (desc->texcoords) {
    for (size_t i = 0; i < (size_t)n * 6; ++i) {
      float v = desc->texcoords[i];
      if (!std::isfinite(v))
        return fail(VSR_ERR_NONFINITE, "non-finite texcoord at triangle " + std::to_string(i / 6));
      if (std::fabs(v) > 1024.0f)
        return fail(VSR_ERR_INVALID_ARG, "|texcoord| > 1024 at triangle " + std::to_string(i / 6));
    }
  }
  const uint32_t ntex = desc->num_textures;
  if (ntex > 0 && !desc->textures) return fail(VSR_ERR_INVALID_ARG, "textures is NULL");
  for (uint32_t k = 0; k < ntex; ++k) {
    const vsr_texture_desc& t = desc->textures[k];
    if (t.width < 1 || t.height < 1 || t.width > 65536 || t.height > 65536 || !t.rgba8)
      return fail(VSR_ERR_INVALID_ARG, "texture " + std::to_string(k) + " has a bad size/pointer");
  }
  const uint32_t eff_tex = ntex ? ntex : 1u;
  if (desc->geom_texture) {
    for (uint32_t g = 0; g < desc->num_geoms; ++g)
      if (desc->geom_texture[g] >= eff_tex)
        return fail(VSR_ERR_INVALID_ARG, "geom_texture[" + std::to_string(g) + "] out of range");
  }
  vsr_scene* s = new (std::nothrow) vsr_scene();
  if (!s) return fail(VSR_ERR_OOM, "scene allocation");
  try {
    s->device = desc->device;
    s->num_tris_input = n;
    s->vertices.assign(desc->vertices, desc->vertices + (size_t)n * 9);
    s->has_texcoords = desc->texcoords != nullptr;
    if (desc->texcoords) s->texcoords.assign(desc->texcoords, desc->texcoords + (size_t)n * 6);
    s->tri_tex.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
      uint32_t g = desc->geom_ids ? desc->geom_ids[i] : 0u;
      uint32_t t;
      if (desc->geom_texture) {
        if (g >= desc->num_geoms) {
          delete s;
          return fail(VSR_ERR_INVALID_ARG, "geom_id of triangle " + std::to_string(i) +
                                               " >= num_geoms");
        }
        t = desc->geom_texture[g];
      } else {
        t = ntex ? g : 0u;
      }
      if (t >= eff_tex) {
        delete s;
        return fail(VSR_ERR_INVALID_ARG, "texture index of triangle " + std::to_string(i) +
                                             " out of range");
      }
      s->tri_tex[i] = t;
    }
    if (ntex == 0) {
      s->textures.push_back(HostTexture{1, 1, {255u}});   // implicit opaque white
    } else {
      // Only the alpha channel is kept: the mask listing reads color.w alone
      // (PAPER.md:311-313), so the device pool is an A8 plane.
      s->textures.resize(ntex);
      for (uint32_t k = 0; k < ntex; ++k) {
        const vsr_texture_desc& t = desc->textures[k];
        HostTexture& h = s->textures[k];
        h.w = t.width;
        h.h = t.height;
        size_t cnt = (size_t)t.width * t.height;
        h.texels.resize(cnt);
        const uint8_t* p = t.rgba8;
        for (size_t q = 0; q < cnt; ++q) h.texels[q] = p[4 * q + 3];
      }
    }
  } catch (const std::bad_alloc&) {
    delete s;
    return fail(VSR_ERR_OOM, "host copy of the scene");
  }
  s->stats.num_tris_input = n;
  *out = s;
  return VSR_OK;
}

vsr_status vsr_bvh_build(vsr_scene* s, const vsr_build_params* params) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  if (s->vertices.empty() && s->num_tris_input == 0 && s->built)
    return fail(VSR_ERR_INVALID_ARG, "imported scenes cannot be rebuilt");
  vsr_build_params prm{2u, 16u, 1.0f, 1.0f};   // max_leaf 2: measured best (A22)
  if (params) prm = *params;
  if (prm.max_leaf_size < 1 || prm.max_leaf_size > kMaxLeafSize)
    return fail(VSR_ERR_INVALID_ARG, "max_leaf_size must be in [1, 32]");
  if (prm.sah_bins < 2 || prm.sah_bins > 256)
    return fail(VSR_ERR_INVALID_ARG, "sah_bins must be in [2, 256]");
  if (!(prm.traversal_cost >= 0.0f) || !(prm.intersection_cost > 0.0f))
    return fail(VSR_ERR_INVALID_ARG, "costs must be finite, intersection_cost > 0");
  if (s->num_tris_input == 0) return fail(VSR_ERR_EMPTY_SCENE, "empty scene: zero triangles");
  auto t0 = std::chrono::steady_clock::now();
  // texture pool (A8 plane) and per-texture descriptors
  std::vector<TexDesc> descs(s->textures.size());
  uint64_t total = 0;
  for (size_t k = 0; k < s->textures.size(); ++k) {
    descs[k].offset = total;
    descs[k].w = s->textures[k].w;
    descs[k].h = s->textures[k].h;
    total += (uint64_t)descs[k].w * descs[k].h;
  }
  if (total > 0xFFFFFFFFull)
    return fail(VSR_ERR_UNSUPPORTED, "more than 2^32 texels in total (32-bit sidecar offsets)");
  std::vector<uint8_t> pool(total);
  for (size_t k = 0; k < s->textures.size(); ++k)
    std::memcpy(pool.data() + descs[k].offset, s->textures[k].texels.data(),
                s->textures[k].texels.size());
  HostBvh hb;
  std::string err;
  BuildInput in{s->vertices.data(), s->num_tris_input,
                s->has_texcoords ? s->texcoords.data() : nullptr, s->tri_tex.data(),
                descs.data()};
  vsr_status st;
  try {
    st = build_bvh(in, prm, hb, err);
  } catch (const std::bad_alloc&) {
    return fail(VSR_ERR_OOM, "host BVH build");
  }
  if (st != VSR_OK) return fail(st, err);
  if (s->device < 0) {
    // host-only scene: keep the flattened arrays for export (no device copy)
    s->free_device();
    s->stats.num_nodes = (uint32_t)hb.nodes.size();
    s->stats.num_tris = (uint32_t)hb.tris.size();
    s->stats.num_textures = (uint32_t)descs.size();
    s->stats.num_texels = total;
    s->stats.device_bytes = 0;
    s->stats.built = 1;
    s->dev.root_ref = hb.root_ref;
    for (int a = 0; a < 3; ++a) {
      s->dev.root_lo[a] = hb.root_lo[a];
      s->dev.root_hi[a] = hb.root_hi[a];
    }
    s->dev.num_nodes = s->stats.num_nodes;
    s->dev.num_tris = s->stats.num_tris;
    s->dev.num_textures = s->stats.num_textures;
    s->num_texels = total;
    s->host_bvh = std::move(hb);
    s->host_descs = std::move(descs);
    s->host_pool = std::move(pool);
    s->host_built = true;
  } else {
    st = upload(s, hb.root_ref, hb.root_lo, hb.root_hi, hb.nodes.data(),
                (uint32_t)hb.nodes.size(), hb.tris.data(), hb.sides.data(),
                (uint32_t)hb.tris.size(), descs.data(), (uint32_t)descs.size(), pool.data(), total);
    if (st != VSR_OK) return st;
  }
  s->stats.num_degenerate = hb.num_degenerate;
  s->stats.num_leaves = hb.num_leaves;
  s->stats.max_depth = hb.max_depth;
  s->stats.build_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return VSR_OK;
}

}  // extern "C"

namespace {
vsr_status build_on_gpu(vsr_scene* s, uint32_t max_leaf_size, int ploc_radius) {
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  if (s->vertices.empty() && s->num_tris_input == 0 && s->built)
    return fail(VSR_ERR_INVALID_ARG, "imported scenes cannot be rebuilt");
  if (max_leaf_size < 1 || max_leaf_size > kMaxLeafSize)
    return fail(VSR_ERR_INVALID_ARG, "max_leaf_size must be in [1, 32]");
  if (s->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only scene: use vsr_bvh_build");
  if (s->num_tris_input == 0) return fail(VSR_ERR_EMPTY_SCENE, "empty scene: zero triangles");
  auto t0 = std::chrono::steady_clock::now();
  std::vector<TexDesc> descs(s->textures.size());
  uint64_t total = 0;
  for (size_t k = 0; k < s->textures.size(); ++k) {
    descs[k].offset = total;
    descs[k].w = s->textures[k].w;
    descs[k].h = s->textures[k].h;
    total += (uint64_t)descs[k].w * descs[k].h;
  }
  if (total > 0xFFFFFFFFull)
    return fail(VSR_ERR_UNSUPPORTED, "more than 2^32 texels in total (32-bit sidecar offsets)");
  std::vector<uint8_t> pool(total);
  for (size_t k = 0; k < s->textures.size(); ++k)
    std::memcpy(pool.data() + descs[k].offset, s->textures[k].texels.data(),
                s->textures[k].texels.size());
  DeviceGuard g(s->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  const uint32_t n = s->num_tris_input;
  float* d_v = nullptr;
  float* d_tc = nullptr;
  uint32_t* d_tt = nullptr;
  TexDesc* d_desc = nullptr;
  auto cleanup = [&] {
    cudaFree(d_v);
    cudaFree(d_tc);
    cudaFree(d_tt);
    cudaFree(d_desc);
  };
  vsr_status st;
  if ((st = dev_upload(&d_v, s->vertices.data(), 9 * (size_t)n, "vertices")) != VSR_OK ||
      (s->has_texcoords &&
       (st = dev_upload(&d_tc, s->texcoords.data(), 6 * (size_t)n, "texcoords")) != VSR_OK) ||
      (st = dev_upload(&d_tt, s->tri_tex.data(), n, "texture indices")) != VSR_OK ||
      (st = dev_upload(&d_desc, descs.data(), descs.size(), "texdescs")) != VSR_OK) {
    cleanup();
    return st;
  }
  GpuBvh gb;
  std::string err;
  st = build_bvh_gpu(d_v, d_tc, d_tt, d_desc, n, max_leaf_size, gb, err, ploc_radius);
  cleanup();
  if (st != VSR_OK) return fail(st, err);
  st = upload(s, gb.root_ref, gb.root_lo, gb.root_hi, gb.nodes, gb.num_nodes, gb.tris, gb.sides,
              gb.num_tris, descs.data(), (uint32_t)descs.size(), pool.data(), total);
  cudaFree(gb.nodes);
  cudaFree(gb.tris);
  cudaFree(gb.sides);
  if (st != VSR_OK) return st;
  s->stats.num_degenerate = gb.num_degenerate;
  s->stats.num_leaves = gb.num_leaves;
  s->stats.max_depth = gb.max_depth;
  s->stats.build_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return VSR_OK;
}
}  // namespace

extern "C" {

vsr_status vsr_bvh_build_gpu(vsr_scene* s, uint32_t max_leaf_size) {
  g_err.clear();
  return build_on_gpu(s, max_leaf_size, 0);
}

vsr_status vsr_bvh_build_ploc(vsr_scene* s, uint32_t max_leaf_size, uint32_t radius) {
  g_err.clear();
  if (radius < 1 || radius > 256) return fail(VSR_ERR_INVALID_ARG, "radius must be in [1, 256]");
  return build_on_gpu(s, max_leaf_size, (int)radius);
}

}  // extern "C"

extern "C" {

vsr_status vsr_destroy(vsr_scene* s) {
  g_err.clear();
  if (!s) return VSR_OK;
  if (s->device >= 0) {
    DeviceGuard g(s->device);
    s->free_stage();
    s->scratch.release();
    s->free_device();
  }
  delete s;
  return VSR_OK;
}

vsr_status vsr_bvh_export(const vsr_scene* s, vsr_bvh_view* view) {
  g_err.clear();
  if (!s || !view) return fail(VSR_ERR_INVALID_ARG, "NULL scene or view");
  if (!s->built && !s->host_built) return fail(VSR_ERR_NOT_BUILT, "scene has no BVH");
  const DevScene& d = s->dev;
  view->root_ref = d.root_ref;
  for (int a = 0; a < 3; ++a) {
    view->root_lo[a] = d.root_lo[a];
    view->root_hi[a] = d.root_hi[a];
  }
  view->num_nodes = d.num_nodes;
  view->num_tris = d.num_tris;
  view->num_textures = d.num_textures;
  view->num_texels = s->num_texels;
  struct Item { void* dst; const void* src; size_t bytes; };
  if (s->host_built) {
    // host-only scene: plain host copies (destinations must be host memory)
    const HostBvh& h = s->host_bvh;
    const Item items[] = {{view->nodes, h.nodes.data(), (size_t)d.num_nodes * 64},
                          {view->tris, h.tris.data(), (size_t)d.num_tris * 48},
                          {view->sides, h.sides.data(), (size_t)d.num_tris * 32},
                          {view->texdescs, s->host_descs.data(), (size_t)d.num_textures * 16},
                          {view->texels, s->host_pool.data(), (size_t)s->num_texels}};
    for (const Item& it : items)
      if (it.dst && it.bytes) std::memcpy(it.dst, it.src, it.bytes);
    return VSR_OK;
  }
  DeviceGuard g(s->device);
  const Item items[] = {{view->nodes, s->d_nodes, (size_t)d.num_nodes * 64},
                        {view->tris, s->d_tris, (size_t)d.num_tris * 48},
                        {view->sides, s->d_sides, (size_t)d.num_tris * 32},
                        {view->texdescs, s->d_texdescs, (size_t)d.num_textures * 16},
                        {view->texels, s->d_texels, (size_t)s->num_texels}};
  for (const Item& it : items) {
    if (!it.dst || it.bytes == 0) continue;
    cudaError_t e = cudaMemcpy(it.dst, it.src, it.bytes, cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_fail(e, "export copy");
  }
  return VSR_OK;
}

vsr_status vsr_scene_import(const vsr_bvh_view* v, int device, vsr_scene** out) {
  g_err.clear();
  if (!v || !out) return fail(VSR_ERR_INVALID_ARG, "NULL view or out");
  *out = nullptr;
  if (v->num_tris == 0) return fail(VSR_ERR_EMPTY_SCENE, "imported BVH has no triangles");
  if (v->num_tris > kMaxTris) return fail(VSR_ERR_UNSUPPORTED, "more than 2^26 triangles");
  if (v->num_texels > 0xFFFFFFFFull) return fail(VSR_ERR_UNSUPPORTED, "more than 2^32 texels");
  if (!v->tris || !v->sides || (v->num_nodes && !v->nodes) || !v->texdescs || !v->texels ||
      v->num_textures == 0)
    return fail(VSR_ERR_INVALID_ARG, "NULL array in view (or zero textures)");
  int ndev = 0;
  if (device < -1) return fail(VSR_ERR_INVALID_ARG, "device ordinal out of range");
  if (device >= 0 && cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0 && device >= ndev)
    return fail(VSR_ERR_INVALID_ARG, "device ordinal out of range");
  // Host copies for validation (the source may be device memory).
  std::vector<PairNode> nodes(v->num_nodes);
  std::vector<Side> sides(v->num_tris);
  std::vector<TexDesc> descs(v->num_textures);
  {
    cudaError_t e;
    if (v->num_nodes && (e = to_host(nodes.data(), v->nodes, nodes.size() * 64)) != cudaSuccess)
      return cuda_fail(e, "import nodes");
    if ((e = to_host(sides.data(), v->sides, sides.size() * 32)) != cudaSuccess)
      return cuda_fail(e, "import sidecars");
    if ((e = to_host(descs.data(), v->texdescs, descs.size() * 16)) != cudaSuccess)
      return cuda_fail(e, "import texdescs");
  }
  for (uint32_t k = 0; k < v->num_textures; ++k) {
    const TexDesc& t = descs[k];
    if (t.w < 1 || t.h < 1 || t.w > 65536 || t.h > 65536 ||
        t.offset + (uint64_t)t.w * t.h > v->num_texels)
      return fail(VSR_ERR_INVALID_ARG, "texture descriptor " + std::to_string(k) + " out of range");
  }
  // Every sidecar must name one of the descriptors exactly (offset and dims): the
  // 1-bit-plane eligibility is decided on the descriptors, and alpha_keep_bits
  // indexes the plane with the sidecar's own (offset, dims).
  std::vector<uint64_t> keys(v->num_textures);
  for (uint32_t k = 0; k < v->num_textures; ++k)
    keys[k] = descs[k].offset << 32 | (uint64_t)((descs[k].w - 1u) | (descs[k].h - 1u) << 16);
  std::sort(keys.begin(), keys.end());
  for (uint32_t k = 0; k < v->num_tris; ++k) {
    if ((uint64_t)sides[k].texel_offset + (uint64_t)((sides[k].dims & 0xFFFFu) + 1u) *
                                              ((sides[k].dims >> 16) + 1u) > v->num_texels)
      return fail(VSR_ERR_INVALID_ARG, "sidecar " + std::to_string(k) + " texture out of range");
    const uint64_t key = (uint64_t)sides[k].texel_offset << 32 | sides[k].dims;
    if (!std::binary_search(keys.begin(), keys.end(), key))
      return fail(VSR_ERR_INVALID_ARG,
                  "sidecar " + std::to_string(k) + " does not match any texture descriptor");
  }
  // Structure: reachable refs in range, every triangle in exactly one leaf, depth <= 64.
  std::vector<uint8_t> seen_tri(v->num_tris, 0), seen_node(v->num_nodes, 0);
  struct Item { uint32_t ref; uint32_t depth; };
  std::vector<Item> st{{v->root_ref, 0}};
  uint32_t max_depth = 0, leaves = 0;
  while (!st.empty()) {
    Item it = st.back();
    st.pop_back();
    if (it.depth > (uint32_t)kMaxStack)
      return fail(VSR_ERR_BVH_TOO_DEEP, "imported BVH deeper than 64 levels");
    max_depth = std::max(max_depth, it.depth);
    if (it.ref & kLeafBit) {
      uint32_t first = it.ref & kLeafFirstMask;
      uint32_t cnt = ((it.ref >> kLeafCountShift) & 31u) + 1u;
      if ((uint64_t)first + cnt > v->num_tris)
        return fail(VSR_ERR_INVALID_ARG, "leaf range out of bounds");
      for (uint32_t k = first; k < first + cnt; ++k) {
        if (seen_tri[k]) return fail(VSR_ERR_INVALID_ARG, "triangle referenced by two leaves");
        seen_tri[k] = 1;
      }
      ++leaves;
      continue;
    }
    if (it.ref >= v->num_nodes) return fail(VSR_ERR_INVALID_ARG, "node ref out of range");
    if (seen_node[it.ref]) return fail(VSR_ERR_INVALID_ARG, "node reachable twice (not a tree)");
    {
      const PairNode& nd = nodes[it.ref];
      const float* ax[3] = {nd.x, nd.y, nd.z};
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 2; ++c)
          if (!std::isfinite(ax[a][c]) || !std::isfinite(ax[a][2 + c]) || !(ax[a][c] <= ax[a][2 + c]))
            return fail(VSR_ERR_INVALID_ARG, "node " + std::to_string(it.ref) +
                                                 " has a non-finite or inverted child box");
    }
    seen_node[it.ref] = 1;
    st.push_back({nodes[it.ref].ref[1], it.depth + 1});
    st.push_back({nodes[it.ref].ref[0], it.depth + 1});
  }
  for (uint32_t k = 0; k < v->num_tris; ++k)
    if (!seen_tri[k]) return fail(VSR_ERR_INVALID_ARG, "triangle not referenced by any leaf");
  vsr_scene* s = new (std::nothrow) vsr_scene();
  if (!s) return fail(VSR_ERR_OOM, "scene allocation");
  s->device = device;
  if (device < 0) {
    // host-only import (e.g. a CPU rank relaying a broadcast): keep host copies
    try {
      HostBvh& h = s->host_bvh;
      h.nodes = std::move(nodes);
      h.tris.resize(v->num_tris);
      h.sides = std::move(sides);
      s->host_descs = std::move(descs);
      s->host_pool.resize(v->num_texels);
      cudaError_t e;
      if ((e = to_host(h.tris.data(), v->tris, (size_t)v->num_tris * 48)) != cudaSuccess ||
          (e = to_host(s->host_pool.data(), v->texels, (size_t)v->num_texels)) != cudaSuccess) {
        delete s;
        return cuda_fail(e, "import copy");
      }
    } catch (const std::bad_alloc&) {
      delete s;
      return fail(VSR_ERR_OOM, "host import");
    }
    DevScene& d = s->dev;
    d.root_ref = v->root_ref;
    for (int a = 0; a < 3; ++a) {
      d.root_lo[a] = v->root_lo[a];
      d.root_hi[a] = v->root_hi[a];
    }
    d.num_nodes = v->num_nodes;
    d.num_tris = v->num_tris;
    d.num_textures = v->num_textures;
    s->num_texels = v->num_texels;
    s->host_built = true;
    s->stats.built = 1;
    s->stats.num_nodes = v->num_nodes;
    s->stats.num_tris = v->num_tris;
    s->stats.num_textures = v->num_textures;
    s->stats.num_texels = v->num_texels;
    s->stats.num_tris_input = v->num_tris;
    s->stats.num_leaves = leaves;
    s->stats.max_depth = max_depth;
    *out = s;
    return VSR_OK;
  }
  vsr_status rc = upload(s, v->root_ref, v->root_lo, v->root_hi, v->nodes, v->num_nodes, v->tris,
                         v->sides, v->num_tris, v->texdescs, v->num_textures, v->texels,
                         v->num_texels);
  if (rc != VSR_OK) {
    vsr_destroy(s);
    return rc;
  }
  s->stats.num_tris_input = v->num_tris;
  s->stats.num_leaves = leaves;
  s->stats.max_depth = max_depth;
  *out = s;
  return VSR_OK;
}

vsr_status vsr_scene_stats(const vsr_scene* s, vsr_stats* out) {
  g_err.clear();
  if (!s || !out) return fail(VSR_ERR_INVALID_ARG, "NULL scene or out");
  *out = s->stats;
  return VSR_OK;
}

}  // extern "C"
