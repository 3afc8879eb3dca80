// wide.hpp — the 8-wide compressed BVH layout (SURVEY.md §8(f) NEXT-3 "wide /
// compressed BVH (8-wide quantized nodes)"), shared by the host collapse
// (bvh8_build.cpp), the C ABI (api_wide.cpp) and the trace kernel (wide.cu).
// Product side only: the oracle's walker re-declares it from DESIGN.md §9h.
//
// One WideNode = 80 B = 5 x LDG.128 holds up to 8 children, each child box
// quantized to 8 bits per plane on a per-node, per-axis grid (Ylitie, Karras
// & Laine, HPG 2017, "compressed wide BVH"):
//   plane(q) = fma(2^23 + q, scale_k, pm_k)        (one rounding; q in 0..255)
// scale_k = 2^(e_k - 127) (a float whose exponent field is e_k).  The builder
// picks pm, e and the codes so that every decoded child box CONTAINS the
// binary tree's (padded) child box — evaluating this exact fp32 expression —
// so the decoded boxes are as conservative as the binary ones and the slab
// test (contract r02) is unchanged.  2^23 + q is the float whose mantissa is q
// (the PRMT byte -> float trick), so decoding is PRMT + FFMA per plane.
#pragma once
#include <cstdint>

#include "layout.hpp"

namespace vsr {

struct alignas(16) WideNode {
  float pm[3];           // decode origin per axis (includes the -2^23 * scale offset)
  uint8_t e[3];          // scale exponent field per axis
  uint8_t imask;         // bit s: slot s holds an inner child
  uint32_t child_base;   // first inner child; inner children contiguous in slot order
  uint32_t tri_base;     // first triangle of the leaf children (slot order)
  uint8_t meta[8];       // slot s: 0xFF empty; 0x80 inner; leaf (count-1) << 5 | offset
  uint8_t qlo[3][8];     // per axis, per slot: lower plane code
  uint8_t qhi[3][8];     // per axis, per slot: upper plane code
};
static_assert(sizeof(WideNode) == 80, "WideNode must be 80 B");

constexpr uint8_t kWideEmpty = 0xFF;
constexpr uint8_t kWideInner = 0x80;
constexpr uint32_t kWideMaxLeaf = 4;   // triangles per leaf child (2-bit count)

}  // namespace vsr
