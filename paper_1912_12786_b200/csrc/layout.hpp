// layout.hpp — device/export data layout shared by the host builder, the C ABI
// and the trace kernels (product side only; the oracle re-declares it from
// DESIGN.md and never includes this file).
//
// All arrays are 16-B aligned AoS records sized for 128-bit loads:
//   PairNode 64 B  = 4 x LDG.128   (both children's boxes + refs: one node
//                                   visit tests two boxes)
//   Tri      48 B  = 3 x LDG.128   (v0 + precomputed edges)
//   Side     32 B  = 2 x LDG.128   (alpha sidecar)
//   TexDesc  16 B
#pragma once
#include <cstdint>

namespace vsr {

constexpr uint32_t kLeafBit = 0x80000000u;
constexpr uint32_t kLeafFirstMask = 0x03FFFFFFu;  // 26 bits
constexpr uint32_t kLeafCountShift = 26;
constexpr uint32_t kMaxLeafSize = 32;
constexpr uint32_t kMaxTris = 1u << 26;
constexpr int kMaxStack = 64;

// Per axis k: (lo0.k, lo1.k, hi0.k, hi1.k) — the two children's slab planes
// side by side, so one packed f32x2 op works on both children.
struct alignas(16) PairNode {
  float x[4];
  float y[4];
  float z[4];
  uint32_t ref[2];
  uint32_t pad[2];
};
static_assert(sizeof(PairNode) == 64, "PairNode must be 64 B");

struct alignas(16) Tri {
  float v0[3];
  uint32_t prim;
  float e1[3];
  uint32_t pad1;
  float e2[3];
  uint32_t pad2;
};
static_assert(sizeof(Tri) == 48, "Tri must be 48 B");

// Alpha sidecar: the three texcoords and the triangle's texture resolved to
// its place in the alpha plane (byte offset) and its size, so a lookup is one
// 32-B sidecar read and one byte read, with no descriptor indirection.
struct alignas(16) Side {
  float uv[6];
  uint32_t texel_offset;   // first texel of the texture in the A8 pool
  uint32_t dims;           // (W - 1) | (H - 1) << 16
};
static_assert(sizeof(Side) == 32, "Side must be 32 B");

inline uint32_t pack_dims(uint32_t w, uint32_t h) { return (w - 1u) | ((h - 1u) << 16); }

struct alignas(16) TexDesc {
  uint64_t offset;
  uint32_t w, h;
};
static_assert(sizeof(TexDesc) == 16, "TexDesc must be 16 B");

inline uint32_t make_leaf(uint32_t first, uint32_t count) {
  return kLeafBit | ((count - 1u) << kLeafCountShift) | first;
}

// Device view of a built scene, passed by value in the kernel parameter space.
struct DevScene {
  const PairNode* nodes;
  const Tri* tris;
  const Side* sides;
  const TexDesc* texdescs;
  const uint8_t* texels;   // A8 alpha plane (the listing reads color.w only)
  uint32_t root_ref;
  float root_lo[3], root_hi[3];
  uint32_t num_nodes, num_tris, num_textures;
  unsigned long long* counters;   // kCounterSlots x 2, zero-initialised
  // density grid over the root box (scheduling hint for the order pass only): per cell
  // the number of triangles whose box overlaps it; gscale = cells per unit length
  const uint32_t* grid;
  uint32_t gdim[3];
  float gscale[3];
};

// Work-distribution counters for the persistent trace kernel: slot s holds
// {next ray, warps finished}; the last warp of a launch resets its slot.
constexpr uint32_t kCounterSlots = 256;

// Scene data the mask intersectors read (their "member variables",
// PAPER.md:286-288 "stores a pointer to the texture and texture coordinate
// lists").
struct IsectData {
  const Side* sides;
  const TexDesc* descs;
  const uint8_t* texels;
  uint32_t a_min;   // smallest a8 with (float)a8/255.0f >= threshold (exact, host-derived)
  float fm;         // checker frequency M as float
  float thr;        // the alpha threshold itself (bilinear variant compares filtered alpha)
  const uint32_t* bits;   // 1-bit plane of (a8 >= a_min) for this a_min, or null (see
                          // alpha_keep_bits; built per threshold by the host, a cache)
  uint64_t num_texels;    // size of the A8 plane (bounds-checked builds, VSR_CHECKED)
};

// Pinhole camera for rays generated inside the trace kernel (vsr.h vsr_pinhole;
// `side` = sqrt(spp), precomputed on the host).
struct Pinhole {
  double eye[3], w[3], u[3], v[3];
  double tan_half, aspect;
  uint32_t width, height, spp, seed, side;
  float tmin, tmax;
};

// One instance of a two-level hierarchy (vsr.h vsr_instance), in top-level
// leaf order: the [A | b] map rays take into object space, rows padded to
// float4 so the record is 4 x LDG.128.
struct alignas(16) Instance {
  float m[12];       // row-major 3x4 object_from_world
  uint32_t bvh;      // element of the scene list
  uint32_t index;    // the caller's instance index
  uint32_t pad[2];
};
static_assert(sizeof(Instance) == 64, "Instance must be 64 B");

}  // namespace vsr
