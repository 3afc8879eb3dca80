// bvh_build.cpp — host binned-SAH BVH builder (untimed setup).
//
// The paper assumes a BVH exists ("usually, the ray is tested against a
// bounding volume hierarchy (BVH) built over some primitives", PAPER.md:185-
// 186) and does not describe construction; SPEC S:265-273 fixes binned SAH
// with a median fallback.  Readings (A22/A23):
//   * always split while n > max_leaf (so every leaf holds <= max_leaf);
//   * coincident centroids -> median split in array order;
//   * exported child boxes are padded outward by 2^-20 * max(1,|x|) so the
//     slab test never culls a triangle Möller–Trumbore would hit.
// Large subtrees are built on worker threads; the final node order is a
// deterministic depth-first pre-order regardless of thread timing.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <future>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "builder.hpp"

namespace vsr {
namespace {

struct Box {
  float lo[3] = {INFINITY, INFINITY, INFINITY};
  float hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  void grow(const Box& b) {
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], b.lo[a]);
      hi[a] = std::max(hi[a], b.hi[a]);
    }
  }
  double area() const {
    if (!(lo[0] <= hi[0])) return 0.0;
    double dx = (double)hi[0] - lo[0], dy = (double)hi[1] - lo[1], dz = (double)hi[2] - lo[2];
    return 2.0 * (dx * dy + dy * dz + dz * dx);
  }
};

struct TmpNode {
  Box box[2];
  int32_t child[2];   // >= 0: TmpNode index; < 0: leaf -> ~(leaf index)
};
struct TmpLeaf {
  uint32_t first, count;
};

struct Ctx {
  const std::vector<Box>* pbox;
  const std::vector<float>* cen;   // 3 per prim
  std::vector<uint32_t>* idx;
  uint32_t max_leaf, bins;
  double ct, ci;
  // node/leaf pools, grown under a mutex (rare: one append per node)
  std::mutex mu;
  std::vector<TmpNode> nodes;
  std::vector<TmpLeaf> leaves;
  std::atomic<int> max_depth{0};
  std::atomic<bool> too_deep{false};
};

Box range_box(const Ctx& c, uint32_t b, uint32_t e) {
  Box r;
  const auto& pb = *c.pbox;
  const auto& idx = *c.idx;
  for (uint32_t k = b; k < e; ++k) r.grow(pb[idx[k]]);
  return r;
}

int32_t add_leaf(Ctx& c, uint32_t b, uint32_t e) {
  std::lock_guard<std::mutex> g(c.mu);
  c.leaves.push_back({b, e - b});
  return ~(int32_t)(c.leaves.size() - 1);
}

// Choose the split position of idx[b,e); returns mid.
uint32_t split(Ctx& c, uint32_t b, uint32_t e, const Box& parent) {
  auto& idx = *c.idx;
  const auto& cen = *c.cen;
  const auto& pb = *c.pbox;
  uint32_t n = e - b;
  float cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (uint32_t k = b; k < e; ++k)
    for (int a = 0; a < 3; ++a) {
      float v = cen[3 * (size_t)idx[k] + a];
      cmin[a] = std::min(cmin[a], v);
      cmax[a] = std::max(cmax[a], v);
    }
  const uint32_t B = c.bins;
  double best_cost = INFINITY;
  int best_axis = -1;
  uint32_t best_split = 0;
  std::vector<Box> bb(B);
  std::vector<uint32_t> bn(B);
  std::vector<double> left_cost(B);
  double pa = parent.area();
  if (!(pa > 0.0)) pa = 1.0;
  for (int a = 0; a < 3; ++a) {
    double ext = (double)cmax[a] - cmin[a];
    if (!(ext > 0.0)) continue;
    std::fill(bb.begin(), bb.end(), Box());
    std::fill(bn.begin(), bn.end(), 0u);
    double scale = (double)B / ext;
    for (uint32_t k = b; k < e; ++k) {
      uint32_t p = idx[k];
      int bi = (int)(((double)cen[3 * (size_t)p + a] - cmin[a]) * scale);
      bi = std::min(std::max(bi, 0), (int)B - 1);
      bb[bi].grow(pb[p]);
      bn[bi]++;
    }
    Box acc;
    uint32_t cnt = 0;
    for (uint32_t i = 0; i + 1 < B; ++i) {   // left = bins [0, i]
      acc.grow(bb[i]);
      cnt += bn[i];
      left_cost[i] = cnt ? acc.area() * cnt : 0.0;
      if (!cnt) left_cost[i] = -1.0;
    }
    acc = Box();
    cnt = 0;
    for (uint32_t i = B - 1; i >= 1; --i) {  // right = bins [i, B-1]
      acc.grow(bb[i]);
      cnt += bn[i];
      if (cnt == 0 || cnt == n || left_cost[i - 1] < 0.0) continue;
      double cost = c.ct + c.ci * (left_cost[i - 1] + acc.area() * cnt) / pa;
      if (cost < best_cost) {
        best_cost = cost;
        best_axis = a;
        best_split = i;
      }
    }
  }
  if (best_axis < 0) return b + n / 2;   // coincident centroids: median in array order
  const int a = best_axis;
  const double scale = (double)B / ((double)cmax[a] - cmin[a]);
  const float lo_a = cmin[a];
  auto it = std::partition(idx.begin() + b, idx.begin() + e, [&](uint32_t p) {
    int bi = (int)(((double)cen[3 * (size_t)p + a] - lo_a) * scale);
    bi = std::min(std::max(bi, 0), (int)B - 1);
    return (uint32_t)bi < best_split;
  });
  uint32_t mid = (uint32_t)(it - idx.begin());
  if (mid == b || mid == e) return b + n / 2;   // cannot happen; keep the invariant anyway
  return mid;
}

int32_t build_rec(Ctx& c, uint32_t b, uint32_t e, const Box& box, int depth) {
  int md = c.max_depth.load(std::memory_order_relaxed);
  while (depth > md && !c.max_depth.compare_exchange_weak(md, depth)) {
  }
  if (depth > kMaxStack) {
    c.too_deep = true;
    return add_leaf(c, b, std::min(e, b + 1));
  }
  uint32_t n = e - b;
  if (n <= c.max_leaf) return add_leaf(c, b, e);
  uint32_t mid = split(c, b, e, box);
  Box lb = range_box(c, b, mid), rb = range_box(c, mid, e);
  int32_t me;
  {
    std::lock_guard<std::mutex> g(c.mu);
    c.nodes.push_back(TmpNode{});
    me = (int32_t)(c.nodes.size() - 1);
  }
  int32_t l, r;
  if (n > 65536) {
    auto fut = std::async(std::launch::async, [&] { return build_rec(c, b, mid, lb, depth + 1); });
    r = build_rec(c, mid, e, rb, depth + 1);
    l = fut.get();
  } else {
    l = build_rec(c, b, mid, lb, depth + 1);
    r = build_rec(c, mid, e, rb, depth + 1);
  }
  std::lock_guard<std::mutex> g(c.mu);
  c.nodes[me].box[0] = lb;
  c.nodes[me].box[1] = rb;
  c.nodes[me].child[0] = l;
  c.nodes[me].child[1] = r;
  return me;
}

void pad_out(const Box& in, float* lo, float* hi) {
  for (int a = 0; a < 3; ++a) {
    double l = in.lo[a], h = in.hi[a];
    double dl = std::ldexp(std::max(1.0, std::fabs(l)), -20);
    double dh = std::ldexp(std::max(1.0, std::fabs(h)), -20);
    double ld = l - dl, hd = h + dh;
    float lf = (float)ld, hf = (float)hd;
    if ((double)lf > ld) lf = std::nextafter(lf, -INFINITY);
    if ((double)hf < hd) hf = std::nextafter(hf, INFINITY);
    lo[a] = lf;
    hi[a] = hf;
  }
}

bool degenerate(const float* vt) {
  float e1[3] = {vt[3] - vt[0], vt[4] - vt[1], vt[5] - vt[2]};
  float e2[3] = {vt[6] - vt[0], vt[7] - vt[1], vt[8] - vt[2]};
  double x = (double)e1[1] * e2[2] - (double)e1[2] * e2[1];
  double y = (double)e1[2] * e2[0] - (double)e1[0] * e2[2];
  double z = (double)e1[0] * e2[1] - (double)e1[1] * e2[0];
  return x == 0.0 && y == 0.0 && z == 0.0;
}

template <class F>
void parallel_for(size_t n, F f) {
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 200000 || nt == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  size_t chunk = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    size_t b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    th.emplace_back([=] { f(b, e); });
  }
  for (auto& x : th) x.join();
}

// The tree over prims idx[0, m) with boxes pbox / centroids cen: binned SAH,
// flattened depth-first pre-order with padded child boxes.  Fills out.nodes,
// root_ref, root box, max_depth, num_leaves; idx ends in leaf order (a leaf's
// `first` indexes idx).
vsr_status build_tree(const std::vector<Box>& pbox, const std::vector<float>& cen,
                      std::vector<uint32_t>& idx, const vsr_build_params& prm, HostBvh& out,
                      std::string& err) {
  const uint32_t m = (uint32_t)idx.size();
  Ctx c;
  c.pbox = &pbox;
  c.cen = &cen;
  c.idx = &idx;
  c.max_leaf = prm.max_leaf_size;
  c.bins = prm.sah_bins;
  c.ct = prm.traversal_cost;
  c.ci = prm.intersection_cost;
  c.nodes.reserve(2 * (size_t)m / std::max(1u, prm.max_leaf_size) + 16);
  c.leaves.reserve(2 * (size_t)m / std::max(1u, prm.max_leaf_size) + 16);
  Box root = range_box(c, 0, m);
  int32_t root_tmp = build_rec(c, 0, m, root, 0);
  if (c.too_deep) {
    err = "BVH deeper than 64 levels (traversal stack bound)";
    return VSR_ERR_BVH_TOO_DEEP;
  }
  out.max_depth = (uint32_t)c.max_depth.load();
  out.num_leaves = (uint32_t)c.leaves.size();

  // Flatten: depth-first pre-order, child 0 first.
  out.nodes.clear();
  out.nodes.reserve(c.nodes.size());
  auto leaf_ref = [&](int32_t t) {
    const TmpLeaf& L = c.leaves[~t];
    return make_leaf(L.first, L.count);
  };
  if (root_tmp < 0) {
    out.root_ref = leaf_ref(root_tmp);
  } else {
    // explicit stack of (tmp node, slot to patch)
    struct Item { int32_t tmp; int64_t patch_node; int patch_child; };
    std::vector<Item> st;
    st.push_back({root_tmp, -1, 0});
    while (!st.empty()) {
      Item it = st.back();
      st.pop_back();
      uint32_t me = (uint32_t)out.nodes.size();
      out.nodes.push_back(PairNode{});
      if (it.patch_node >= 0) out.nodes[it.patch_node].ref[it.patch_child] = me;
      const TmpNode& tn = c.nodes[it.tmp];
      PairNode& pn = out.nodes[me];
      float lo[2][3], hi[2][3];
      pad_out(tn.box[0], lo[0], hi[0]);
      pad_out(tn.box[1], lo[1], hi[1]);
      float* axis[3] = {pn.x, pn.y, pn.z};
      for (int a = 0; a < 3; ++a) {
        axis[a][0] = lo[0][a];
        axis[a][1] = lo[1][a];
        axis[a][2] = hi[0][a];
        axis[a][3] = hi[1][a];
      }
      pn.pad[0] = pn.pad[1] = 0;
      for (int k = 1; k >= 0; --k) {       // push child 1 first so child 0 is emitted next
        int32_t ch = tn.child[k];
        if (ch < 0) pn.ref[k] = leaf_ref(ch);
        else st.push_back({ch, (int64_t)me, k});
      }
    }
    out.root_ref = 0;
  }
  pad_out(root, out.root_lo, out.root_hi);
  return VSR_OK;
}

}  // namespace

vsr_status build_bvh(const BuildInput& in, const vsr_build_params& prm, HostBvh& out,
                     std::string& err) {
  const uint32_t N = in.num_tris;
  std::vector<uint8_t> degen(N);
  parallel_for(N, [&](size_t b, size_t e) {
    for (size_t i = b; i < e; ++i) degen[i] = degenerate(in.vertices + 9 * i);
  });
  std::vector<uint32_t> idx;
  idx.reserve(N);
  for (uint32_t i = 0; i < N; ++i)
    if (!degen[i]) idx.push_back(i);
  out.num_degenerate = N - (uint32_t)idx.size();
  const uint32_t m = (uint32_t)idx.size();
  if (m == 0) {
    err = "empty scene: no non-degenerate triangles";
    return VSR_ERR_EMPTY_SCENE;
  }
  if (m > kMaxTris) {
    err = "more than 2^26 triangles are not supported by the 26-bit leaf encoding";
    return VSR_ERR_UNSUPPORTED;
  }
  std::vector<Box> pbox(N);
  std::vector<float> cen(3 * (size_t)N);
  parallel_for(N, [&](size_t b, size_t e) {
    for (size_t i = b; i < e; ++i) {
      const float* vt = in.vertices + 9 * i;
      Box bx;
      for (int a = 0; a < 3; ++a) {
        bx.lo[a] = std::min(std::min(vt[a], vt[3 + a]), vt[6 + a]);
        bx.hi[a] = std::max(std::max(vt[a], vt[3 + a]), vt[6 + a]);
        cen[3 * i + a] = 0.5f * bx.lo[a] + 0.5f * bx.hi[a];
      }
      pbox[i] = bx;
    }
  });
  vsr_status st = build_tree(pbox, cen, idx, prm, out, err);
  if (st != VSR_OK) return st;

  out.tris.resize(m);
  out.sides.resize(m);
  parallel_for(m, [&](size_t b, size_t e) {
    for (size_t k = b; k < e; ++k) {
      uint32_t p = idx[k];
      const float* vt = in.vertices + 9 * (size_t)p;
      Tri& t = out.tris[k];
      for (int a = 0; a < 3; ++a) {
        t.v0[a] = vt[a];
        t.e1[a] = vt[3 + a] - vt[a];
        t.e2[a] = vt[6 + a] - vt[a];
      }
      t.prim = p;
      t.pad1 = t.pad2 = 0;
      Side& s = out.sides[k];
      if (in.texcoords) std::memcpy(s.uv, in.texcoords + 6 * (size_t)p, sizeof s.uv);
      else std::memset(s.uv, 0, sizeof s.uv);
      const TexDesc& td = in.tex_table[in.tri_tex[p]];
      s.texel_offset = (uint32_t)td.offset;
      s.dims = pack_dims(td.w, td.h);
    }
  });
  return VSR_OK;
}

vsr_status build_top(const float* boxes, uint32_t n, const vsr_build_params& prm, HostBvh& out,
                     std::vector<uint32_t>& order, std::string& err) {
  if (n == 0) {
    err = "no instances";
    return VSR_ERR_EMPTY_SCENE;
  }
  if (n > kMaxTris) {
    err = "more than 2^26 instances are not supported by the 26-bit leaf encoding";
    return VSR_ERR_UNSUPPORTED;
  }
  std::vector<Box> pbox(n);
  std::vector<float> cen(3 * (size_t)n);
  for (uint32_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      pbox[i].lo[a] = boxes[6 * (size_t)i + a];
      pbox[i].hi[a] = boxes[6 * (size_t)i + 3 + a];
      cen[3 * (size_t)i + a] = 0.5f * pbox[i].lo[a] + 0.5f * pbox[i].hi[a];
    }
  }
  order.resize(n);
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  out.num_degenerate = 0;
  return build_tree(pbox, cen, order, prm, out, err);
}

}  // namespace vsr
