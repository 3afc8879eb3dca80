// bvh8_build.cpp — collapse a built binary BVH into the 8-wide compressed
// layout of wide.hpp.  Host code, untimed setup.
//
//  1. Collapse (greedy, Ylitie et al. 2017 §3 "wide BVH construction" uses an
//     SAH-optimal DP; this is the common greedy variant): a wide node starts
//     with the binary node's two children and repeatedly replaces its inner
//     child of largest surface area by that child's two children, while fewer
//     than 8 children exist.  Binary leaves (<= 4 triangles) stay leaves.
//  2. Slot order: child c goes to slot s so that rays of octant s (the sign
//     bits of their direction, bit k set = negative along axis k) meet it
//     early: greedy assignment on cost(c, s) = (centroid_c - centroid_parent)
//     . dir(s), smallest first.  The kernel visits slots in order of s ^ octant.
//  3. Quantization per axis (wide.hpp): scale = 2^e, the smallest power of two
//     for which 255 codes span the node; pm = lo - 2^23 scale rounded down
//     until plane(0) <= lo; each child's codes are the tightest q with
//     plane(q_lo) <= child lo and plane(q_hi) >= child hi, evaluated with the
//     kernel's exact fp32 expression (std::fma, one rounding).  A child that
//     does not fit raises e and the axis is redone.
//  4. Layout: breadth-first, inner children of a node contiguous in slot order
//     (child index = child_base + rank of the slot among inner slots); the
//     triangles (and alpha sidecars) of a node's leaf children contiguous in
//     slot order from tri_base — a new triangle order, prim ids unchanged.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "builder.hpp"
#include "wide.hpp"

namespace vsr {

namespace {

struct Cand {
  uint32_t ref;       // binary ref (leaf bit + range, or node index)
  float lo[3], hi[3];
};

double area(const Cand& c) {
  const double dx = (double)c.hi[0] - c.lo[0], dy = (double)c.hi[1] - c.lo[1],
               dz = (double)c.hi[2] - c.lo[2];
  return dx * dy + dy * dz + dz * dx;
}

Cand child_of(const std::vector<PairNode>& nodes, uint32_t node, int c) {
  const PairNode& n = nodes[node];
  Cand k;
  k.ref = n.ref[c];
  k.lo[0] = n.x[c]; k.lo[1] = n.y[c]; k.lo[2] = n.z[c];
  k.hi[0] = n.x[2 + c]; k.hi[1] = n.y[2 + c]; k.hi[2] = n.z[2 + c];
  return k;
}

float scale_of(int efield) {
  uint32_t bits = (uint32_t)efield << 23;
  float s;
  std::memcpy(&s, &bits, 4);
  return s;
}

// plane(q) = fma(2^23 + q, scale, pm): the kernel's decode, bit for bit
float plane(uint32_t q, float scale, float pm) {
  return std::fma(8388608.0f + (float)q, scale, pm);
}

// Quantize axis a of the children into node w; false if some child does not fit.
bool quantize_axis(WideNode& w, int a, const std::vector<Cand>& ch, const int* slot_of, float lo,
                   float hi, int efield) {
  const float s = scale_of(efield);
  float pm = (float)((double)lo - 8388608.0 * (double)s);
  while (plane(0, s, pm) > lo) pm = std::nextafter(pm, -INFINITY);
  if (plane(255, s, pm) < hi) return false;
  w.pm[a] = pm;
  w.e[a] = (uint8_t)efield;
  for (int sl = 0; sl < 8; ++sl) {   // empty slots: an inverted box (lo code > hi code)
    w.qlo[a][sl] = 255;
    w.qhi[a][sl] = 0;
  }
  for (size_t c = 0; c < ch.size(); ++c) {
    const float clo = ch[c].lo[a], chi = ch[c].hi[a];
    // largest q with plane(q) <= clo; smallest q with plane(q) >= chi (plane is monotone
    // in q): start from the real-valued estimate, then step to the exact fp32 answer
    const double base = (double)plane(0, s, pm);
    int ql = (int)std::floor(((double)clo - base) / s);
    ql = std::min(std::max(ql, 0), 255);
    while (ql > 0 && plane((uint32_t)ql, s, pm) > clo) --ql;
    while (ql < 255 && plane((uint32_t)ql + 1, s, pm) <= clo) ++ql;
    int qh = (int)std::ceil(((double)chi - base) / s);
    qh = std::min(std::max(qh, ql), 255);
    while (qh < 255 && plane((uint32_t)qh, s, pm) < chi) ++qh;
    while (qh > ql && plane((uint32_t)qh - 1, s, pm) >= chi) --qh;
    if (plane((uint32_t)qh, s, pm) < chi || plane((uint32_t)ql, s, pm) > clo) return false;
    w.qlo[a][slot_of[c]] = (uint8_t)ql;
    w.qhi[a][slot_of[c]] = (uint8_t)qh;
  }
  return true;
}

}  // namespace

vsr_status build_wide(const HostBvh& b, HostWide& out, std::string& err) {
  out = HostWide{};
  for (int a = 0; a < 3; ++a) {
    out.root_lo[a] = b.root_lo[a];
    out.root_hi[a] = b.root_hi[a];
  }
  // leaf sizes must fit the 2-bit count
  for (const PairNode& n : b.nodes)
    for (int c = 0; c < 2; ++c)
      if ((n.ref[c] & kLeafBit) && ((n.ref[c] >> kLeafCountShift) & 31u) + 1u > kWideMaxLeaf) {
        err = "8-wide BVH needs leaves of at most 4 triangles (build with max_leaf_size <= 4)";
        return VSR_ERR_UNSUPPORTED;
      }
  if ((b.root_ref & kLeafBit) && ((b.root_ref >> kLeafCountShift) & 31u) + 1u > kWideMaxLeaf) {
    err = "8-wide BVH needs leaves of at most 4 triangles (build with max_leaf_size <= 4)";
    return VSR_ERR_UNSUPPORTED;
  }
  struct Job { uint32_t wide; std::vector<Cand> ch; uint32_t depth; };
  std::vector<Job> queue;
  {
    Job root{0, {}, 1};
    if (b.root_ref & kLeafBit) {
      Cand k;
      k.ref = b.root_ref;
      std::memcpy(k.lo, b.root_lo, sizeof k.lo);
      std::memcpy(k.hi, b.root_hi, sizeof k.hi);
      root.ch.push_back(k);
    } else {
      root.ch = {child_of(b.nodes, b.root_ref, 0), child_of(b.nodes, b.root_ref, 1)};
    }
    queue.push_back(root);
  }
  out.nodes.resize(1);
  for (size_t qi = 0; qi < queue.size(); ++qi) {
    Job job = std::move(queue[qi]);
    std::vector<Cand>& ch = job.ch;
    // 1. collapse: open the largest inner child while fewer than 8 children
    for (;;) {
      if (ch.size() >= 8) break;
      int best = -1;
      double ba = -1.0;
      for (size_t c = 0; c < ch.size(); ++c)
        if (!(ch[c].ref & kLeafBit) && area(ch[c]) > ba) {
          ba = area(ch[c]);
          best = (int)c;
        }
      if (best < 0) break;
      const uint32_t node = ch[best].ref;
      ch[best] = child_of(b.nodes, node, 0);
      ch.insert(ch.begin() + best + 1, child_of(b.nodes, node, 1));
    }
    // node box
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (const Cand& c : ch)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], c.lo[a]);
        hi[a] = std::max(hi[a], c.hi[a]);
      }
    // 2. slots by octant
    int slot_of[8];
    {
      double pc[3];
      for (int a = 0; a < 3; ++a) pc[a] = 0.5 * ((double)lo[a] + hi[a]);
      struct P { double cost; int c, s; };
      std::vector<P> pairs;
      for (size_t c = 0; c < ch.size(); ++c)
        for (int s = 0; s < 8; ++s) {
          double cost = 0.0;
          for (int a = 0; a < 3; ++a) {
            const double cc = 0.5 * ((double)ch[c].lo[a] + ch[c].hi[a]) - pc[a];
            cost += ((s >> a) & 1) ? -cc : cc;
          }
          pairs.push_back({cost, (int)c, s});
        }
      std::stable_sort(pairs.begin(), pairs.end(), [](const P& x, const P& y) {
        return x.cost < y.cost;
      });
      bool cused[8] = {}, sused[8] = {};
      for (const P& p : pairs)
        if (!cused[p.c] && !sused[p.s]) {
          cused[p.c] = sused[p.s] = true;
          slot_of[p.c] = p.s;
        }
    }
    WideNode w;
    std::memset(&w, 0, sizeof w);
    // 3. quantize
    for (int a = 0; a < 3; ++a) {
      const double ext = (double)hi[a] - lo[a];
      int ef = ext > 0.0 ? 127 + (int)std::ceil(std::log2(ext / 255.0)) : 1;
      ef = std::max(ef, 1);
      while (!quantize_axis(w, a, ch, slot_of, lo[a], hi[a], ef)) {
        if (++ef > 254) {
          err = "8-wide BVH: node extent beyond the quantization range";
          return VSR_ERR_UNSUPPORTED;
        }
      }
    }
    // 4. children: inner slots in slot order get consecutive node indices; leaf
    //    triangles consecutive from tri_base in slot order
    int cat[8];   // child index at slot, -1 empty
    for (int s = 0; s < 8; ++s) cat[s] = -1;
    for (size_t c = 0; c < ch.size(); ++c) cat[slot_of[c]] = (int)c;
    w.child_base = (uint32_t)out.nodes.size();
    w.tri_base = (uint32_t)out.tris.size();
    uint32_t off = 0;
    for (int s = 0; s < 8; ++s) {
      if (cat[s] < 0) {
        w.meta[s] = kWideEmpty;
        continue;
      }
      const Cand& c = ch[cat[s]];
      if (c.ref & kLeafBit) {
        const uint32_t first = c.ref & kLeafFirstMask, cnt = ((c.ref >> kLeafCountShift) & 31u) + 1u;
        w.meta[s] = (uint8_t)(((cnt - 1u) << 5) | off);
        for (uint32_t k = 0; k < cnt; ++k) {
          out.tris.push_back(b.tris[first + k]);
          out.sides.push_back(b.sides[first + k]);
        }
        off += cnt;
      } else {
        w.meta[s] = kWideInner;
        w.imask |= (uint8_t)(1u << s);
        Job nj{(uint32_t)out.nodes.size(), {}, job.depth + 1};
        nj.ch = {child_of(b.nodes, c.ref, 0), child_of(b.nodes, c.ref, 1)};
        out.nodes.emplace_back();
        queue.push_back(std::move(nj));
      }
    }
    out.nodes[job.wide] = w;
    out.max_depth = std::max(out.max_depth, job.depth);
  }
  if (out.max_depth > (uint32_t)kMaxStack) {
    err = "8-wide BVH deeper than 64 levels";
    return VSR_ERR_BVH_TOO_DEEP;
  }
  return VSR_OK;
}

}  // namespace vsr
