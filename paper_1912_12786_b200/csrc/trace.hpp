// trace.hpp — host-visible launch interface of the trace kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/vsr.h"
#include "layout.hpp"

namespace vsr {

struct WideNode;

enum : int { kSchedDirect = 0, kSchedPersistent = 1, kSchedWarp = 2, kSchedRegion = 3 };

// Kernel parameters (passed by value: they live in the constant parameter bank).
struct TraceParams {
  DevScene scene;
  IsectData data;
  const float4* rays;
  float4* hits;
  uint4* counts;
  uint64_t n;
  unsigned long long* counter;   // {next ray, warps done}: this launch's slot
  int refill;                    // refill a warp once this many lanes are idle
  int sched;                     // kSchedDirect (default) or kSchedPersistent
  int order;                     // 1: launch blocks longest-first (direct schedule)
  const uint32_t* perm;          // longest-first block permutation (set by launch_trace)
  uint32_t* hist_reset;          // order histogram the trace kernel re-zeroes (set by launch_trace)
  int pdl;                       // launch the order pass + trace kernel as PDL dependents
  int occ;                       // the 12-CTA/SM trace-kernel variant (scenes larger than L2)
  void* order_scratch;           // optional stream-ordered scratch for the order pass
  size_t order_scratch_bytes;
  int max_hits;                  // multi-hit query: hits kept per ray (1..16)
  uint32_t* num_hits;            // multi-hit query: optional per-ray hit count
  const DevScene* list;          // list query (device array) or nullptr
  const IsectData* list_data;    // per-element mask data (device array)
  uint32_t list_count;
  uint32_t* which;               // list / instance query: optional per-ray element of the hit
  const Instance* instances;     // instance query: records in top-level leaf order (p.scene = top)
  uint32_t num_instances;        // instance query: number of records
  float inst_r_safe;             // instance query: origins beyond take the linear path (A27)
  uint32_t out_tile, out_rank, out_world;   // vsr_trace_tiles output mapping (world 0: identity)
  int gen;                       // 1: rays generated in-kernel from `cam` (rays unused)
  Pinhole cam;
  int runtime_kind;
  void* filter_fn;
  int order_proxy;               // order pass cost proxy: 0 segment length, 1 density grid, 3 blend
                                 // of the two, 2 auto (grid for instances, blend otherwise)
  const WideNode* wide;          // 8-wide compressed BVH (vsr_trace_bvh8) or nullptr
  uint32_t num_wide;             // its node count (bounds-checked builds)
  uint32_t* region_ctr;          // region schedule: per-region claim counters (set by launch_trace)
  uint32_t regions;              // region schedule: number of regions (= SMs)
};

cudaError_t launch_trace(int query, int isect, const TraceParams& p, cudaStream_t st);
// 1-bit alpha plane of threshold a_min into d_bits (texel_count / 32 words; every
// texture's W, H multiples of 32); max_words = the largest texture's W*H/32.
cudaError_t build_alpha_bits(const TexDesc* d_descs, uint32_t num_textures, const uint8_t* texels,
                             uint32_t a_min, uint32_t* d_bits, uint64_t max_words,
                             cudaStream_t st);
size_t order_scratch_bytes(uint64_t n);
// Density grid of a scene (order-pass cost proxy): dims chosen for ~4096 cells over the root
// box; counts the triangles whose box overlaps each cell into d_grid (zeroed by the caller).
void density_grid_dims(const float* lo, const float* hi, uint32_t* dims, float* scale);
size_t density_grid_words(const uint32_t* dims);   // grid allocation (with its replicas)
cudaError_t build_density_grid(const Tri* d_tris, uint32_t n, const float* lo, const uint32_t* dims,
                               const float* scale, uint32_t* d_grid, cudaStream_t st);
void set_kernel_events(void* start, void* stop);
cudaError_t filter_fn_pointer(int kind, void** out);
uint64_t launch_count();
// Query on the scene's triangles as a plain list (no BVH); p.scene.tris / p.data.sides in
// caller order (vsr_trace_primitives).
cudaError_t launch_prims(int query, int isect, const TraceParams& p, cudaStream_t st);
// Lists of BVHs and instances (p.list set; compound.cu), closest / any / multi.
cudaError_t launch_compound(int query, int isect, const TraceParams& p, cudaStream_t st);
// The 8-wide compressed BVH (p.wide set; wide.cu), closest / any.
cudaError_t launch_wide(int query, int isect, const TraceParams& p, cudaStream_t st);

}  // namespace vsr
