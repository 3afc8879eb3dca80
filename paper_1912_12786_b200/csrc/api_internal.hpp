// api_internal.hpp — host-side state shared by the C-ABI translation units
// (api.cpp: helpers, scene lifecycle, builds, export/import; api_trace.cpp:
// the per-scene trace entry points; api_compound.cpp: lists and instancing).
// Not part of the ABI: include/vsr.h is.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
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

namespace vsr_api {

extern thread_local std::string g_err;

vsr_status fail(vsr_status s, const std::string& msg);
vsr_status cuda_fail(cudaError_t e, const char* what);

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

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Copy `bytes` from src (host or device memory) into host memory.
cudaError_t to_host(void* dst, const void* src, size_t bytes);

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

}  // namespace vsr_api

struct vsr_scene {
  int device = 0;
  // ---- host copies (vsr_scene_create) ----
  uint32_t num_tris_input = 0;
  std::vector<float> vertices, texcoords;
  std::vector<uint32_t> tri_tex;
  std::vector<vsr_api::HostTexture> textures;
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
  uint32_t* d_grid = nullptr;                  // density grid (order-pass cost proxy)
  std::atomic<uint32_t> launch_seq{0};
  uint64_t num_texels = 0;
  vsr_stats stats{};
  // ---- vsr_trace_host staging ----
  std::mutex stage_mu;
  // ring of kSlots chunk buffers; copy-in, trace and copy-out each on their
  // own stream, chained per chunk by events (vsr_trace_host)
  static constexpr int kSlots = 8;
  uint64_t stage_cap = 0;   // rays per slot
  bool stage_counts = false;
  float4* d_in[kSlots] = {};
  float4* d_out[kSlots] = {};
  uint4* d_cnt[kSlots] = {};
  cudaStream_t s_in = nullptr, s_run = nullptr, s_out = nullptr;
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_in[kSlots] = {}, ev_run[kSlots] = {}, ev_out[kSlots] = {};
  void* fn_cache[4] = {};
  bool fn_cached[4] = {};
  vsr_api::ScratchSet scratch;   // per-stream scratch of the longest-first order pass
  // 1-bit alpha planes, one per threshold seen (cache; built on first use, kept until
  // the device state is freed; at most kMaxPlanes, then the A8 path is used)
  static constexpr int kMaxPlanes = 8;
  std::mutex bits_mu;
  int bits_ok = -1;   // -1 unknown, 0 textures not 32-aligned, 1 eligible
  uint64_t bits_max_words = 0;   // largest texture's W*H/32
  uint32_t plane_amin[kMaxPlanes] = {};
  uint32_t* d_planes[kMaxPlanes] = {};
  int num_planes = 0;
  // ---- 8-wide compressed BVH (vsr_bvh8_build; NEXT-3) ----
  bool wide_built = false;
  HostWide host_wide;   // host-only scenes keep it here; device scenes upload it
  WideNode* d_wnodes = nullptr;
  Tri* d_wtris = nullptr;
  Side* d_wsides = nullptr;
  uint32_t num_wnodes = 0, wide_depth = 0;
  double wide_build_ms = 0.0;

  void free_wide() {
    cudaFree(d_wnodes);
    cudaFree(d_wtris);
    cudaFree(d_wsides);
    d_wnodes = nullptr;
    d_wtris = nullptr;
    d_wsides = nullptr;
    num_wnodes = wide_depth = 0;
    host_wide = HostWide{};
    wide_built = false;
  }

  void free_device() {
    free_wide();
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
    cudaFree(d_grid);
    d_grid = nullptr;
    d_nodes = nullptr;
    d_tris = nullptr;
    d_sides = nullptr;
    d_texdescs = nullptr;
    d_texels = nullptr;
    d_counters = nullptr;
    for (int i = 0; i < num_planes; ++i) cudaFree(d_planes[i]);
    num_planes = 0;
    bits_ok = -1;
    built = false;
  }
  void free_stage() {
    if (s_out) cudaStreamSynchronize(s_out);
    for (int s = 0; s < kSlots; ++s) {
      cudaFree(d_in[s]);
      cudaFree(d_out[s]);
      cudaFree(d_cnt[s]);
      d_in[s] = nullptr;
      d_out[s] = nullptr;
      d_cnt[s] = nullptr;
      for (cudaEvent_t* ev : {&ev_in[s], &ev_run[s], &ev_out[s]}) {
        if (*ev) cudaEventDestroy(*ev);
        *ev = nullptr;
      }
    }
    for (cudaStream_t* st : {&s_in, &s_run, &s_out}) {
      if (*st) cudaStreamDestroy(*st);
      *st = nullptr;
    }
    if (ev_start) cudaEventDestroy(ev_start);
    ev_start = nullptr;
    stage_counts = false;
    stage_cap = 0;
  }
};

namespace vsr_api {

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
                  const void* texels, uint64_t num_texels);

// smallest a8 in [0,255] with (float)a8 / 255.0f >= thr (reading A7); 256 = none.
uint32_t alpha_min_a8(float thr);
bool valid_isect(int k);
inline bool needs_counts(int k) {
  return k == VSR_ISECT_COUNT || k == VSR_ISECT_COUNT_ALPHA_TEXTURE;
}
// alpha_bits: look up (or build) the scene's 1-bit alpha plane for ALPHA_TEXTURE
// (plain per-scene traces; compounds keep the A8 path)
// (stream: the call's stream — no plane is built while it is being captured)
vsr_status make_params(vsr_scene* s, vsr_query query, vsr_isect isect,
                       const vsr_isect_params* params, TraceParams& p, bool alpha_bits = true,
                       void* stream = nullptr);

// Launch with the owner's scratch for stream `st` (see the definition).
cudaError_t launch_with_scratch(ScratchSet& set, int query, int isect, TraceParams& p,
                                cudaStream_t st);

// The scene's 1-bit alpha plane for threshold a_min (built on first use, cached), or
// nullptr (textures not 32-aligned, cache full, disabled, or `stream` capturing).
const uint32_t* alpha_plane(vsr_scene* s, uint32_t a_min, void* stream);

// A fresh work-counter slot per launch (self-reset by the launch's last warp).
unsigned long long* next_counter(vsr_scene* s);

}  // namespace vsr_api

using namespace vsr_api;
