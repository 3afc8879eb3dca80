// api.cpp — the C ABI declared in include/vsr.h.
//
// Host-side responsibilities: argument validation, scene ingest (SPEC
// S:433-436), BVH build + upload (untimed setup), export/import of the
// flattened structure for multi-GPU replication, and the host dispatch that
// maps (query, intersector) to ONE kernel instantiation per call (PAPER.md:
// 74-78: the choice is made once, outside the innermost loop).
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/vsr.h"
#include "builder.hpp"
#include "layout.hpp"
#include "trace.hpp"

using namespace vsr;

namespace {
thread_local std::string g_err;

vsr_status fail(vsr_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

vsr_status cuda_fail(cudaError_t e, const char* what) {
  return fail(VSR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

struct HostTexture {
  uint32_t w, h;
  std::vector<uint8_t> texels;    // alpha channel (A8)
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

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

}  // namespace

// Per-stream scratch of the longest-first order pass, owned by whatever is
// traced (scene, group, instances): reused in stream order behind an event, so
// launches on other streams never share it and steady-state launches allocate
// nothing.
struct ScratchSet {
  struct OrderScratch {
    cudaStream_t st;
    void* ptr;
    size_t cap;
    cudaEvent_t ev;   // last use; the next use waits on it (stream-ordered reuse)
  };
  std::mutex mu;
  std::vector<OrderScratch> v;

  void release() {
    for (OrderScratch& o : v) {
      cudaEventSynchronize(o.ev);
      cudaFree(o.ptr);
      cudaEventDestroy(o.ev);
    }
    v.clear();
  }
};

struct vsr_scene {
  int device = 0;
  // ---- host copies (vsr_scene_create) ----
  uint32_t num_tris_input = 0;
  std::vector<float> vertices, texcoords;
  std::vector<uint32_t> tri_tex;
  std::vector<HostTexture> textures;
  bool has_texcoords = false;
  // ---- device state (vsr_bvh_build / vsr_scene_import) ----
  bool built = false;
  // host-only scenes (device == -1) keep the flattened arrays here instead
  bool host_built = false;
  HostBvh host_bvh;
  std::vector<TexDesc> host_descs;
  std::vector<uint8_t> host_pool;
  DevScene dev{};
  PairNode* d_nodes = nullptr;
  Tri* d_tris = nullptr;
  Side* d_sides = nullptr;
  // caller-order copies for vsr_trace_primitives (built on first use)
  std::mutex caller_mu;
  Tri* d_tris_caller = nullptr;
  Side* d_sides_caller = nullptr;
  uint32_t num_caller = 0;
  TexDesc* d_texdescs = nullptr;
  uint8_t* d_texels = nullptr;
  unsigned long long* d_counters = nullptr;   // persistent-kernel work counters
  std::atomic<uint32_t> launch_seq{0};
  uint64_t num_texels = 0;
  vsr_stats stats{};
  // ---- vsr_trace_host staging ----
  std::mutex stage_mu;
  static constexpr int kSlots = 3;
  uint64_t stage_cap = 0;   // rays per slot
  float4* d_in[kSlots] = {};
  float4* d_out[kSlots] = {};
  uint4* d_cnt[kSlots] = {};
  cudaStream_t streams[kSlots] = {};
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_done[kSlots] = {};
  void* fn_cache[4] = {};
  bool fn_cached[4] = {};
  ScratchSet scratch;   // per-stream scratch of the longest-first order pass

  void free_device() {
    cudaFree(d_nodes);
    cudaFree(d_tris);
    cudaFree(d_sides);
    cudaFree(d_tris_caller);
    cudaFree(d_sides_caller);
    d_tris_caller = nullptr;
    d_sides_caller = nullptr;
    num_caller = 0;
    cudaFree(d_texdescs);
    cudaFree(d_texels);
    cudaFree(d_counters);
    d_nodes = nullptr;
    d_tris = nullptr;
    d_sides = nullptr;
    d_texdescs = nullptr;
    d_texels = nullptr;
    d_counters = nullptr;
    built = false;
  }
  void free_stage() {
    for (int s = 0; s < kSlots; ++s) {
      cudaFree(d_in[s]);
      cudaFree(d_out[s]);
      cudaFree(d_cnt[s]);
      d_in[s] = nullptr;
      d_out[s] = nullptr;
      d_cnt[s] = nullptr;
      if (streams[s]) cudaStreamDestroy(streams[s]);
      if (ev_done[s]) cudaEventDestroy(ev_done[s]);
      streams[s] = nullptr;
      ev_done[s] = nullptr;
    }
    if (ev_start) cudaEventDestroy(ev_start);
    ev_start = nullptr;
    stage_cap = 0;
  }
};

namespace {

template <class T>
vsr_status dev_upload(T** dst, const void* src, size_t count, const char* what) {
  size_t bytes = count * sizeof(T);
  if (bytes == 0) bytes = sizeof(T);   // keep a valid pointer for empty arrays
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), bytes);
  if (e != cudaSuccess) {
    *dst = nullptr;
    return e == cudaErrorMemoryAllocation ? fail(VSR_ERR_OOM, std::string("cudaMalloc ") + what)
                                          : cuda_fail(e, what);
  }
  if (count) {
    e = cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_fail(e, what);
  }
  return VSR_OK;
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

bool needs_counts(int k) { return k == VSR_ISECT_COUNT || k == VSR_ISECT_COUNT_ALPHA_TEXTURE; }

vsr_status make_params(vsr_scene* s, vsr_query query, vsr_isect isect,
                       const vsr_isect_params* params, TraceParams& p) {
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
  p.data.a_min = alpha_min_a8(ip.alpha_threshold);
  p.data.fm = (float)ip.checker_freq;
  p.data.thr = ip.alpha_threshold;
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
  p.sched = (es && std::strcmp(es, "persistent") == 0) ? kSchedPersistent : kSchedDirect;
  const char* eo = std::getenv("VSR_ORDER");   // "0" disables longest-first block order
  p.order = (eo && std::strcmp(eo, "0") == 0) ? 0 : 1;
  const char* ep = std::getenv("VSR_PDL");   // "0": plain launches after the order pass
  p.pdl = (ep && std::strcmp(ep, "0") == 0) ? 0 : 1;
  return VSR_OK;
}

// Launch with the owner's scratch for stream `st` (created or grown on first
// use; the launch waits for the scratch's previous use, then records its own).
// Caller holds no lock; n must be the launch's ray count.
cudaError_t launch_with_scratch(ScratchSet& set, int query, int isect, TraceParams& p,
                                cudaStream_t st) {
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
      // keeps it so: the trace kernel re-zeroes it)
      if ((e = cudaMemset(o->ptr, 0, bytes)) != cudaSuccess) return e;
      o->cap = bytes;
    }
    if ((e = cudaStreamWaitEvent(st, o->ev, 0)) != cudaSuccess) return e;
    p.order_scratch = o->ptr;
    p.order_scratch_bytes = o->cap;
  }
  e = launch_trace(query, isect, p, st);
  if (e == cudaSuccess && o) e = cudaEventRecord(o->ev, st);
  return e;
}

// A fresh work-counter slot per launch (self-reset by the launch's last warp).
unsigned long long* next_counter(vsr_scene* s) {
  const uint32_t slot = s->launch_seq.fetch_add(1, std::memory_order_relaxed) % kCounterSlots;
  return s->d_counters + 2 * (size_t)slot;
}

}  // namespace

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

vsr_status vsr_trace_tiles(vsr_scene* s, const vsr_ray* d_rays, uint64_t n, uint32_t tile_rays,
                           uint32_t rank, uint32_t world, vsr_query query, vsr_isect isect,
                           const vsr_isect_params* params, vsr_hit* d_hits, vsr_counts* d_counts,
                           void* stream) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  TraceParams p;
  vsr_status st = make_params(s, query, isect, params, p);
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
  vsr_status st = make_params(s, query, isect, params, p);
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
  vsr_status st = make_params(s, query, isect, params, p);
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
  vsr_status st = make_params(s, query, isect, params, p);
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
  vsr_status st = make_params(s, VSR_QUERY_CLOSEST, isect, params, p);
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

struct vsr_group {
  int device = 0;
  ScratchSet scratch;
  std::vector<vsr_scene*> scenes;
  DevScene* d_list = nullptr;
  IsectData* d_data = nullptr;
  float lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};   // union of the roots (order-pass proxy)
};

extern "C" {

vsr_status vsr_group_create(vsr_scene* const* scenes, uint32_t count, vsr_group** out) {
  g_err.clear();
  if (!scenes || !out) return fail(VSR_ERR_INVALID_ARG, "NULL scenes or out");
  *out = nullptr;
  if (count < 1 || count > 1024) return fail(VSR_ERR_INVALID_ARG, "count must be in [1, 1024]");
  for (uint32_t k = 0; k < count; ++k) {
    if (!scenes[k]) return fail(VSR_ERR_INVALID_ARG, "NULL scene in list");
    if (scenes[k]->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only scene in list");
    if (!scenes[k]->built) return fail(VSR_ERR_NOT_BUILT, "scene " + std::to_string(k) + " not built");
    if (scenes[k]->device != scenes[0]->device)
      return fail(VSR_ERR_INVALID_ARG, "all scenes of a group must be on one device");
  }
  vsr_group* g = new (std::nothrow) vsr_group();
  if (!g) return fail(VSR_ERR_OOM, "group allocation");
  g->device = scenes[0]->device;
  g->scenes.assign(scenes, scenes + count);
  std::vector<DevScene> list(count);
  std::vector<IsectData> data(count);
  for (int a = 0; a < 3; ++a) {
    g->lo[a] = INFINITY;
    g->hi[a] = -INFINITY;
  }
  for (uint32_t k = 0; k < count; ++k) {
    list[k] = scenes[k]->dev;
    data[k] = IsectData{scenes[k]->d_sides, scenes[k]->d_texdescs, scenes[k]->d_texels, 0u, 0.0f, 0.0f};
    for (int a = 0; a < 3; ++a) {
      g->lo[a] = std::min(g->lo[a], scenes[k]->dev.root_lo[a]);
      g->hi[a] = std::max(g->hi[a], scenes[k]->dev.root_hi[a]);
    }
  }
  DeviceGuard dg(g->device);
  cudaError_t e;
  if ((e = cudaMalloc(&g->d_list, sizeof(DevScene) * count)) != cudaSuccess ||
      (e = cudaMalloc(&g->d_data, sizeof(IsectData) * count)) != cudaSuccess ||
      (e = cudaMemcpy(g->d_list, list.data(), sizeof(DevScene) * count, cudaMemcpyHostToDevice)) !=
          cudaSuccess ||
      (e = cudaMemcpy(g->d_data, data.data(), sizeof(IsectData) * count, cudaMemcpyHostToDevice)) !=
          cudaSuccess) {
    cudaFree(g->d_list);
    cudaFree(g->d_data);
    delete g;
    return cuda_fail(e, "group upload");
  }
  *out = g;
  return VSR_OK;
}

vsr_status vsr_group_destroy(vsr_group* g) {
  g_err.clear();
  if (!g) return VSR_OK;
  {
    DeviceGuard dg(g->device);
    g->scratch.release();
    cudaFree(g->d_list);
    cudaFree(g->d_data);
  }
  delete g;
  return VSR_OK;
}

}  // extern "C"

namespace {
// query: 0 closest, 1 any, 2 multi-hit (max_hits per ray, d_which max_hits per ray)
vsr_status group_trace(vsr_group* g, const vsr_ray* d_rays, uint64_t n, int query,
                       uint32_t max_hits, vsr_isect isect, const vsr_isect_params* params,
                       vsr_hit* d_hits, uint32_t* d_num_hits, uint32_t* d_which,
                       vsr_counts* d_counts, void* stream) {
  g_err.clear();
  if (!g) return fail(VSR_ERR_INVALID_ARG, "NULL group");
  if ((int)isect >= 100 && valid_isect(isect))
    return fail(VSR_ERR_UNSUPPORTED, "run-time controls are not provided for list queries");
  if (query == 2 && (max_hits < 1 || max_hits > 16))
    return fail(VSR_ERR_INVALID_ARG, "max_hits must be in [1, 16]");
  TraceParams p;
  vsr_status st = make_params(g->scenes[0], query == 2 ? VSR_QUERY_CLOSEST : (vsr_query)query,
                              isect, params, p);
  if (st != VSR_OK) return st;
  if (n == 0) return VSR_OK;
  if (d_num_hits && (reinterpret_cast<uintptr_t>(d_num_hits) & 3u))
    return fail(VSR_ERR_INVALID_ARG, "num_hits buffer must be 4-byte aligned");
  p.max_hits = (int)max_hits;
  p.num_hits = d_num_hits;
  if (!d_rays || !d_hits) return fail(VSR_ERR_INVALID_ARG, "NULL rays or hits buffer");
  if (!aligned16(d_rays) || !aligned16(d_hits))
    return fail(VSR_ERR_INVALID_ARG, "rays/hits buffers must be 16-byte aligned");
  if (d_which && (reinterpret_cast<uintptr_t>(d_which) & 3u))
    return fail(VSR_ERR_INVALID_ARG, "which buffer must be 4-byte aligned");
  if (needs_counts(isect)) {
    if (!d_counts) return fail(VSR_ERR_INVALID_ARG, "COUNT intersector needs a counts buffer");
    if (!aligned16(d_counts)) return fail(VSR_ERR_INVALID_ARG, "counts buffer not 16-B aligned");
  }
  for (int a = 0; a < 3; ++a) {   // the order pass's cost proxy uses the union of the roots
    p.scene.root_lo[a] = g->lo[a];
    p.scene.root_hi[a] = g->hi[a];
  }
  p.rays = reinterpret_cast<const float4*>(d_rays);
  p.hits = reinterpret_cast<float4*>(d_hits);
  p.counts = reinterpret_cast<uint4*>(d_counts);
  p.n = n;
  p.list = g->d_list;
  p.list_data = g->d_data;
  p.list_count = (uint32_t)g->scenes.size();
  p.which = d_which;
  DeviceGuard dg(g->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  cudaError_t e = launch_with_scratch(g->scratch, query, isect, p,
                                      reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "list trace launch");
  return VSR_OK;
}
}  // namespace

extern "C" {

vsr_status vsr_trace_group(vsr_group* g, const vsr_ray* d_rays, uint64_t n, vsr_query query,
                           vsr_isect isect, const vsr_isect_params* params, vsr_hit* d_hits,
                           uint32_t* d_which, vsr_counts* d_counts, void* stream) {
  if ((int)query != VSR_QUERY_CLOSEST && (int)query != VSR_QUERY_ANY) {
    g_err.clear();
    return fail(VSR_ERR_INVALID_ARG, "invalid query");
  }
  return group_trace(g, d_rays, n, (int)query, 0, isect, params, d_hits, nullptr, d_which,
                     d_counts, stream);
}

vsr_status vsr_trace_group_multi(vsr_group* g, const vsr_ray* d_rays, uint64_t n,
                                 uint32_t max_hits, vsr_isect isect,
                                 const vsr_isect_params* params, vsr_hit* d_hits,
                                 uint32_t* d_num_hits, uint32_t* d_which, vsr_counts* d_counts,
                                 void* stream) {
  return group_trace(g, d_rays, n, 2, max_hits, isect, params, d_hits, d_num_hits, d_which,
                     d_counts, stream);
}

}  // extern "C"

// Two-level instancing: the top level lives here; the instanced scenes are
// referenced, not owned.
struct vsr_instances {
  int device = 0;
  ScratchSet scratch;
  std::vector<vsr_scene*> scenes;
  HostBvh top;                       // host copy of the top-level nodes (export)
  std::vector<Instance> records;     // leaf order (export)
  DevScene dev{};                    // top level: nodes, root ref / box
  PairNode* d_nodes = nullptr;
  Instance* d_records = nullptr;
  DevScene* d_list = nullptr;
  IsectData* d_data = nullptr;
};

namespace {

// World box of an instance: the 8 corners of the scene's (padded) root box
// mapped by the fp64 inverse of [A | b], then padded by 2^-10 (diagonal +
// max |coordinate|) and rounded outward (reading A27).  False if A is singular.
bool instance_world_box(const float* m, const float* lo, const float* hi, float* out) {
  const double a[3][3] = {{m[0], m[1], m[2]}, {m[4], m[5], m[6]}, {m[8], m[9], m[10]}};
  const double bv[3] = {m[3], m[7], m[11]};
  const double det = a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
                     a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
                     a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
  if (!(std::fabs(det) > 1e-30) || !std::isfinite(det)) return false;
  double inv[3][3];
  inv[0][0] = (a[1][1] * a[2][2] - a[1][2] * a[2][1]) / det;
  inv[0][1] = (a[0][2] * a[2][1] - a[0][1] * a[2][2]) / det;
  inv[0][2] = (a[0][1] * a[1][2] - a[0][2] * a[1][1]) / det;
  inv[1][0] = (a[1][2] * a[2][0] - a[1][0] * a[2][2]) / det;
  inv[1][1] = (a[0][0] * a[2][2] - a[0][2] * a[2][0]) / det;
  inv[1][2] = (a[0][2] * a[1][0] - a[0][0] * a[1][2]) / det;
  inv[2][0] = (a[1][0] * a[2][1] - a[1][1] * a[2][0]) / det;
  inv[2][1] = (a[0][1] * a[2][0] - a[0][0] * a[2][1]) / det;
  inv[2][2] = (a[0][0] * a[1][1] - a[0][1] * a[1][0]) / det;
  double wlo[3] = {INFINITY, INFINITY, INFINITY}, whi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int c = 0; c < 8; ++c) {
    const double p[3] = {(c & 1) ? hi[0] : lo[0], (c & 2) ? hi[1] : lo[1], (c & 4) ? hi[2] : lo[2]};
    for (int i = 0; i < 3; ++i) {
      const double w = inv[i][0] * (p[0] - bv[0]) + inv[i][1] * (p[1] - bv[1]) +
                       inv[i][2] * (p[2] - bv[2]);
      wlo[i] = std::min(wlo[i], w);
      whi[i] = std::max(whi[i], w);
    }
  }
  double diag = 0.0, mag = 0.0;
  for (int i = 0; i < 3; ++i) {
    diag += (whi[i] - wlo[i]) * (whi[i] - wlo[i]);
    mag = std::max(mag, std::max(std::fabs(wlo[i]), std::fabs(whi[i])));
  }
  const double pad = std::ldexp(std::sqrt(diag) + mag, -10);
  for (int i = 0; i < 3; ++i) {
    const double l = wlo[i] - pad, h = whi[i] + pad;
    float lf = (float)l, hf = (float)h;
    if ((double)lf > l) lf = std::nextafter(lf, -INFINITY);
    if ((double)hf < h) hf = std::nextafter(hf, INFINITY);
    if (!std::isfinite(lf) || !std::isfinite(hf)) return false;
    out[i] = lf;
    out[3 + i] = hf;
  }
  return true;
}

void free_instances(vsr_instances* I) {
  if (I->device < 0) return;
  DeviceGuard dg(I->device);
  I->scratch.release();
  cudaFree(I->d_nodes);
  cudaFree(I->d_records);
  cudaFree(I->d_list);
  cudaFree(I->d_data);
}

}  // namespace

extern "C" {

vsr_status vsr_instances_create(vsr_scene* const* scenes, uint32_t num_scenes,
                                const vsr_instance* instances, uint32_t num_instances,
                                const vsr_build_params* params, vsr_instances** out) {
  g_err.clear();
  if (!scenes || !instances || !out) return fail(VSR_ERR_INVALID_ARG, "NULL scenes, instances or out");
  *out = nullptr;
  if (num_scenes < 1 || num_scenes > 1024)
    return fail(VSR_ERR_INVALID_ARG, "num_scenes must be in [1, 1024]");
  if (num_instances < 1 || num_instances > kMaxTris)
    return fail(VSR_ERR_INVALID_ARG, "num_instances must be in [1, 2^26]");
  for (uint32_t k = 0; k < num_scenes; ++k) {
    if (!scenes[k]) return fail(VSR_ERR_INVALID_ARG, "NULL scene in list");
    const bool host = scenes[k]->device < 0;   // host-only: build + export, no trace
    if (!(host ? scenes[k]->host_built : scenes[k]->built))
      return fail(VSR_ERR_NOT_BUILT, "scene " + std::to_string(k) + " not built");
    if (scenes[k]->device != scenes[0]->device)
      return fail(VSR_ERR_INVALID_ARG, "all scenes must be on one device");
  }
  vsr_build_params prm{1u, 16u, 1.0f, 1.0f};
  if (params) prm = *params;
  if (prm.max_leaf_size < 1 || prm.max_leaf_size > kMaxLeafSize || prm.sah_bins < 2 ||
      prm.sah_bins > 256 || !(prm.traversal_cost >= 0.0f) || !(prm.intersection_cost > 0.0f))
    return fail(VSR_ERR_INVALID_ARG, "invalid build params");
  std::vector<float> boxes(6 * (size_t)num_instances);
  for (uint32_t i = 0; i < num_instances; ++i) {
    const vsr_instance& in = instances[i];
    if (in.bvh >= num_scenes)
      return fail(VSR_ERR_INVALID_ARG, "instance " + std::to_string(i) + ": bvh index out of range");
    for (float x : in.object_from_world)
      if (!std::isfinite(x))
        return fail(VSR_ERR_INVALID_ARG, "instance " + std::to_string(i) + ": non-finite matrix");
    const DevScene& d = scenes[in.bvh]->dev;
    if (!instance_world_box(in.object_from_world, d.root_lo, d.root_hi, boxes.data() + 6 * (size_t)i))
      return fail(VSR_ERR_INVALID_ARG, "instance " + std::to_string(i) + ": singular matrix");
  }
  vsr_instances* I = new (std::nothrow) vsr_instances();
  if (!I) return fail(VSR_ERR_OOM, "instances allocation");
  I->device = scenes[0]->device;
  I->scenes.assign(scenes, scenes + num_scenes);
  std::vector<uint32_t> order;
  std::string err;
  vsr_status st = build_top(boxes.data(), num_instances, prm, I->top, order, err);
  if (st != VSR_OK) {
    delete I;
    return fail(st, err);
  }
  I->records.resize(num_instances);
  for (uint32_t k = 0; k < num_instances; ++k) {
    const vsr_instance& in = instances[order[k]];
    Instance& r = I->records[k];
    std::memcpy(r.m, in.object_from_world, sizeof r.m);
    r.bvh = in.bvh;
    r.index = order[k];
    r.pad[0] = r.pad[1] = 0;
  }
  const size_t nn = I->top.nodes.size();
  I->dev = DevScene{};
  I->dev.root_ref = I->top.root_ref;
  for (int a = 0; a < 3; ++a) {
    I->dev.root_lo[a] = I->top.root_lo[a];
    I->dev.root_hi[a] = I->top.root_hi[a];
  }
  I->dev.num_nodes = (uint32_t)nn;
  I->dev.num_tris = num_instances;
  if (I->device < 0) {   // host-only: nothing to upload
    *out = I;
    return VSR_OK;
  }
  std::vector<DevScene> list(num_scenes);
  std::vector<IsectData> data(num_scenes);
  for (uint32_t k = 0; k < num_scenes; ++k) {
    list[k] = scenes[k]->dev;
    data[k] = IsectData{scenes[k]->d_sides, scenes[k]->d_texdescs, scenes[k]->d_texels, 0u, 0.0f, 0.0f};
  }
  DeviceGuard dg(I->device);
  cudaError_t e;
  if ((nn && (e = cudaMalloc(&I->d_nodes, nn * sizeof(PairNode))) != cudaSuccess) ||
      (e = cudaMalloc(&I->d_records, num_instances * sizeof(Instance))) != cudaSuccess ||
      (e = cudaMalloc(&I->d_list, sizeof(DevScene) * num_scenes)) != cudaSuccess ||
      (e = cudaMalloc(&I->d_data, sizeof(IsectData) * num_scenes)) != cudaSuccess ||
      (nn && (e = cudaMemcpy(I->d_nodes, I->top.nodes.data(), nn * sizeof(PairNode),
                             cudaMemcpyHostToDevice)) != cudaSuccess) ||
      (e = cudaMemcpy(I->d_records, I->records.data(), num_instances * sizeof(Instance),
                      cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(I->d_list, list.data(), sizeof(DevScene) * num_scenes,
                      cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(I->d_data, data.data(), sizeof(IsectData) * num_scenes,
                      cudaMemcpyHostToDevice)) != cudaSuccess) {
    free_instances(I);
    delete I;
    return cuda_fail(e, "instances upload");
  }
  I->dev.nodes = I->d_nodes;
  *out = I;
  return VSR_OK;
}

vsr_status vsr_instances_destroy(vsr_instances* I) {
  g_err.clear();
  if (!I) return VSR_OK;
  free_instances(I);
  delete I;
  return VSR_OK;
}

vsr_status vsr_instances_export(const vsr_instances* I, vsr_instances_view* v) {
  g_err.clear();
  if (!I || !v) return fail(VSR_ERR_INVALID_ARG, "NULL instances or view");
  v->root_ref = I->top.root_ref;
  for (int a = 0; a < 3; ++a) {
    v->root_lo[a] = I->top.root_lo[a];
    v->root_hi[a] = I->top.root_hi[a];
  }
  v->num_nodes = (uint32_t)I->top.nodes.size();
  v->num_instances = (uint32_t)I->records.size();
  v->max_depth = I->top.max_depth;
  if (v->nodes && !I->top.nodes.empty())
    std::memcpy(v->nodes, I->top.nodes.data(), I->top.nodes.size() * sizeof(PairNode));
  if (v->records) std::memcpy(v->records, I->records.data(), I->records.size() * sizeof(Instance));
  return VSR_OK;
}

}  // extern "C"

namespace {
vsr_status instances_trace(vsr_instances* I, const vsr_ray* d_rays, uint64_t n, int query,
                           uint32_t max_hits, vsr_isect isect, const vsr_isect_params* params,
                           vsr_hit* d_hits, uint32_t* d_num_hits, uint32_t* d_inst,
                           vsr_counts* d_counts, void* stream) {
  g_err.clear();
  if (!I) return fail(VSR_ERR_INVALID_ARG, "NULL instances");
  if ((int)isect >= 100 && valid_isect(isect))
    return fail(VSR_ERR_UNSUPPORTED, "run-time controls are not provided for instanced queries");
  if (query == 2 && (max_hits < 1 || max_hits > 16))
    return fail(VSR_ERR_INVALID_ARG, "max_hits must be in [1, 16]");
  TraceParams p;
  vsr_status st = make_params(I->scenes[0], query == 2 ? VSR_QUERY_CLOSEST : (vsr_query)query,
                              isect, params, p);
  if (st != VSR_OK) return st;
  if (d_num_hits && (reinterpret_cast<uintptr_t>(d_num_hits) & 3u))
    return fail(VSR_ERR_INVALID_ARG, "num_hits buffer must be 4-byte aligned");
  p.max_hits = (int)max_hits;
  p.num_hits = d_num_hits;
  if (I->device < 0) return fail(VSR_ERR_UNSUPPORTED, "host-only instances cannot be traced");
  if (n == 0) return VSR_OK;
  if (!d_rays || !d_hits) return fail(VSR_ERR_INVALID_ARG, "NULL rays or hits buffer");
  if (!aligned16(d_rays) || !aligned16(d_hits))
    return fail(VSR_ERR_INVALID_ARG, "rays/hits buffers must be 16-byte aligned");
  if (d_inst && (reinterpret_cast<uintptr_t>(d_inst) & 3u))
    return fail(VSR_ERR_INVALID_ARG, "instance buffer must be 4-byte aligned");
  if (needs_counts(isect)) {
    if (!d_counts) return fail(VSR_ERR_INVALID_ARG, "COUNT intersector needs a counts buffer");
    if (!aligned16(d_counts)) return fail(VSR_ERR_INVALID_ARG, "counts buffer not 16-B aligned");
  }
  p.scene = I->dev;   // top level (the order pass's cost proxy uses its root box)
  p.rays = reinterpret_cast<const float4*>(d_rays);
  p.hits = reinterpret_cast<float4*>(d_hits);
  p.counts = reinterpret_cast<uint4*>(d_counts);
  p.n = n;
  p.list = I->d_list;
  p.list_data = I->d_data;
  p.list_count = (uint32_t)I->scenes.size();
  p.instances = I->d_records;
  p.which = d_inst;
  DeviceGuard dg(I->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  cudaError_t e = launch_with_scratch(I->scratch, query, isect, p,
                                      reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "instanced trace launch");
  return VSR_OK;
}
}  // namespace

extern "C" {

vsr_status vsr_trace_instances(vsr_instances* I, const vsr_ray* d_rays, uint64_t n,
                               vsr_query query, vsr_isect isect, const vsr_isect_params* params,
                               vsr_hit* d_hits, uint32_t* d_inst, vsr_counts* d_counts,
                               void* stream) {
  if ((int)query != VSR_QUERY_CLOSEST && (int)query != VSR_QUERY_ANY) {
    g_err.clear();
    return fail(VSR_ERR_INVALID_ARG, "invalid query");
  }
  return instances_trace(I, d_rays, n, (int)query, 0, isect, params, d_hits, nullptr, d_inst,
                         d_counts, stream);
}

vsr_status vsr_trace_instances_multi(vsr_instances* I, const vsr_ray* d_rays, uint64_t n,
                                     uint32_t max_hits, vsr_isect isect,
                                     const vsr_isect_params* params, vsr_hit* d_hits,
                                     uint32_t* d_num_hits, uint32_t* d_inst,
                                     vsr_counts* d_counts, void* stream) {
  return instances_trace(I, d_rays, n, 2, max_hits, isect, params, d_hits, d_num_hits, d_inst,
                         d_counts, stream);
}

vsr_status vsr_trace_host(vsr_scene* s, const vsr_ray* h_rays, uint64_t n, vsr_query query,
                          vsr_isect isect, const vsr_isect_params* params, vsr_hit* h_hits,
                          vsr_counts* h_counts, void* stream) {
  g_err.clear();
  if (!s) return fail(VSR_ERR_INVALID_ARG, "NULL scene");
  TraceParams p;
  vsr_status st = make_params(s, query, isect, params, p);
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
  // Chunked pipeline over kSlots streams: chunk c's H2D copy, kernel and D2H
  // copy run on stream c % kSlots, so copies of one chunk overlap the kernel
  // of another (copy engines and SMs work concurrently).
  const char* ec = std::getenv("VSR_HOST_CHUNKS");   // tuning knob: chunks per call
  // 4 chunks measured best on C2 (2/4/8/16/32: 1.64/1.44/1.51/1.61/1.81 ms per frame)
  const uint64_t nchunks = ec ? std::max(1, std::atoi(ec)) : 4;
  const uint64_t chunk = std::min<uint64_t>(n, std::max<uint64_t>(65536, (n + nchunks - 1) / nchunks));
  cudaError_t e;
  if (s->stage_cap < chunk || (cnt && !s->d_cnt[0])) {
    s->free_stage();
    for (int k = 0; k < vsr_scene::kSlots; ++k) {
      if ((e = cudaMalloc(&s->d_in[k], chunk * 32)) != cudaSuccess ||
          (e = cudaMalloc(&s->d_out[k], chunk * 16)) != cudaSuccess ||
          (e = cudaMalloc(&s->d_cnt[k], chunk * 16)) != cudaSuccess ||
          (e = cudaStreamCreateWithFlags(&s->streams[k], cudaStreamNonBlocking)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&s->ev_done[k], cudaEventDisableTiming)) != cudaSuccess) {
        s->free_stage();
        return cuda_fail(e, "staging allocation");
      }
    }
    if ((e = cudaEventCreateWithFlags(&s->ev_start, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "event");
    s->stage_cap = chunk;
  }
  cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
  if ((e = cudaEventRecord(s->ev_start, user)) != cudaSuccess) return cuda_fail(e, "event");
  for (int k = 0; k < vsr_scene::kSlots; ++k)
    if ((e = cudaStreamWaitEvent(s->streams[k], s->ev_start, 0)) != cudaSuccess)
      return cuda_fail(e, "stream wait");
  const char* src = reinterpret_cast<const char*>(h_rays);
  char* dst = reinterpret_cast<char*>(h_hits);
  char* cdst = reinterpret_cast<char*>(h_counts);
  uint64_t c = 0;
  for (uint64_t b = 0; b < n; b += chunk, ++c) {
    const int k = (int)(c % vsr_scene::kSlots);
    const uint64_t m = std::min(chunk, n - b);
    cudaStream_t ss = s->streams[k];
    if ((e = cudaMemcpyAsync(s->d_in[k], src + b * 32, m * 32, cudaMemcpyHostToDevice, ss)) !=
        cudaSuccess)
      return cuda_fail(e, "H2D rays");
    p.rays = s->d_in[k];
    p.hits = s->d_out[k];
    p.counts = s->d_cnt[k];
    p.n = m;
    p.counter = next_counter(s);
    if ((e = launch_with_scratch(s->scratch, query, isect, p, ss)) != cudaSuccess)
      return cuda_fail(e, "trace launch");
    if ((e = cudaMemcpyAsync(dst + b * 16, s->d_out[k], m * 16, cudaMemcpyDeviceToHost, ss)) !=
        cudaSuccess)
      return cuda_fail(e, "D2H hits");
    if (cnt && (e = cudaMemcpyAsync(cdst + b * 16, s->d_cnt[k], m * 16, cudaMemcpyDeviceToHost,
                                    ss)) != cudaSuccess)
      return cuda_fail(e, "D2H counts");
  }
  for (int k = 0; k < vsr_scene::kSlots; ++k) {
    if ((e = cudaEventRecord(s->ev_done[k], s->streams[k])) != cudaSuccess)
      return cuda_fail(e, "event");
    if ((e = cudaStreamWaitEvent(user, s->ev_done[k], 0)) != cudaSuccess)
      return cuda_fail(e, "stream wait");
  }
  if ((e = cudaStreamSynchronize(user)) != cudaSuccess) return cuda_fail(e, "trace (host)");
  return VSR_OK;
}

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
  for (uint32_t k = 0; k < v->num_tris; ++k)
    if ((uint64_t)sides[k].texel_offset + (uint64_t)((sides[k].dims & 0xFFFFu) + 1u) *
                                              ((sides[k].dims >> 16) + 1u) > v->num_texels)
      return fail(VSR_ERR_INVALID_ARG, "sidecar " + std::to_string(k) + " texture out of range");
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
