// builder.hpp — host BVH builder interface (product side).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/vsr.h"
#include "layout.hpp"
#include "wide.hpp"

namespace vsr {

struct BuildInput {
  const float* vertices;    // 9 per triangle
  uint32_t num_tris;
  const float* texcoords;   // 6 per triangle or nullptr
  const uint32_t* tri_tex;  // resolved texture index per triangle
  const TexDesc* tex_table; // per texture: offset in the A8 pool, width, height
};

struct HostBvh {
  uint32_t root_ref = 0;
  float root_lo[3] = {0, 0, 0}, root_hi[3] = {0, 0, 0};
  std::vector<PairNode> nodes;
  std::vector<Tri> tris;
  std::vector<Side> sides;
  uint32_t max_depth = 0, num_leaves = 0, num_degenerate = 0;
};

vsr_status build_bvh(const BuildInput& in, const vsr_build_params& prm, HostBvh& out,
                     std::string& err);

// 8-wide compressed BVH collapsed from a built binary BVH (bvh8_build.cpp, NEXT-3):
// nodes breadth-first (root = 0), triangles / sidecars in the wide leaf order.
struct HostWide {
  float root_lo[3] = {0, 0, 0}, root_hi[3] = {0, 0, 0};
  std::vector<WideNode> nodes;
  std::vector<Tri> tris;
  std::vector<Side> sides;
  uint32_t max_depth = 0;
};
vsr_status build_wide(const HostBvh& b, HostWide& out, std::string& err);

// GPU linear BVH (lbvh.cu) on the current device from device inputs (9 floats
// per triangle, optional 6 texcoords, resolved texture index, texture table).
// Outputs are device arrays in the export layout, owned by the caller (cudaFree).
struct GpuBvh {
  PairNode* nodes = nullptr;
  Tri* tris = nullptr;
  Side* sides = nullptr;
  uint32_t num_nodes = 0, num_tris = 0, root_ref = 0;
  uint32_t max_depth = 0, num_leaves = 0, num_degenerate = 0;
  float root_lo[3] = {0, 0, 0}, root_hi[3] = {0, 0, 0};
};
vsr_status build_bvh_gpu(const float* d_vertices, const float* d_texcoords,
                         const uint32_t* d_tri_tex, const TexDesc* d_tex, uint32_t n,
                         uint32_t max_leaf, GpuBvh& out, std::string& err,
                         int ploc_radius = 0);   // 0: LBVH (Karras); > 0: PLOC, +-radius

// Top level of a two-level (instanced) hierarchy: the same binned SAH over
// instance world boxes (6 floats per instance: lo xyz, hi xyz); `order`
// receives the instance indices in leaf order (a leaf's `first` indexes it).
vsr_status build_top(const float* boxes, uint32_t n, const vsr_build_params& prm, HostBvh& out,
                     std::vector<uint32_t>& order, std::string& err);

}  // namespace vsr
