// lbvh.cu — GPU BVH builder ("GPU builder (LBVH / PLOC)").
//
// The paper assumes a BVH exists and does not describe its
// construction; the host binned-SAH builder (bvh_build.cpp) stays the default.
// This is the linear BVH of Karras (HPG 2012): 63-bit Morton codes of the
// triangle centroids, a device radix sort, one thread per internal node finds
// its key range and split from the longest common prefixes, boxes are unioned
// bottom-up (the second child to arrive at a parent computes it), subtrees of
// <= max_leaf triangles collapse into leaves, and the surviving nodes are
// compacted and written in the same export layout as the host builder:
// 64-B pair nodes with the same 2^-20 outward padding, triangles and sidecars
// gathered into leaf order.  Setup only (untimed); any valid BVH prunes exactly,
// so traversal results do not depend on which builder made the tree.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "builder.hpp"

namespace vsr {
namespace {

constexpr int kT = 256;
constexpr uint64_t kInvalidKey = ~0ull;

__device__ __forceinline__ int f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

struct Box6 {
  float lo[3], hi[3];
};

// Per triangle: degenerate test (as the host builder: e1 x e2 == 0 in fp64 on the
// fp32 edges), bounds, centroid (0.5 lo + 0.5 hi), centroid bounds, valid count.
__global__ void prep_kernel(const float* __restrict__ v, uint32_t n, Box6* __restrict__ box,
                            float* __restrict__ cen, uint8_t* __restrict__ valid,
                            int* __restrict__ cbounds, uint32_t* __restrict__ nvalid) {
  const uint32_t i = blockIdx.x * kT + threadIdx.x;
  float c[3] = {0, 0, 0};
  bool ok = false;
  if (i < n) {
    const float* t = v + 9 * (size_t)i;
    const float e1[3] = {t[3] - t[0], t[4] - t[1], t[5] - t[2]};
    const float e2[3] = {t[6] - t[0], t[7] - t[1], t[8] - t[2]};
    const double x = (double)e1[1] * e2[2] - (double)e1[2] * e2[1];
    const double y = (double)e1[2] * e2[0] - (double)e1[0] * e2[2];
    const double z = (double)e1[0] * e2[1] - (double)e1[1] * e2[0];
    ok = !(x == 0.0 && y == 0.0 && z == 0.0);
    Box6 b;
    for (int a = 0; a < 3; ++a) {
      b.lo[a] = fminf(fminf(t[a], t[3 + a]), t[6 + a]);
      b.hi[a] = fmaxf(fmaxf(t[a], t[3 + a]), t[6 + a]);
      c[a] = 0.5f * b.lo[a] + 0.5f * b.hi[a];
      cen[3 * (size_t)i + a] = c[a];
    }
    box[i] = b;
    valid[i] = ok;
  }
  // centroid bounds of the valid triangles: warp reduce, one atomic per warp
  for (int a = 0; a < 3; ++a) {
    int lo = ok ? f2ord(c[a]) : 0x7FFFFFFF, hi = ok ? f2ord(c[a]) : (int)0x80000000;
    for (int o = 16; o; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(cbounds + a, lo);
      atomicMax(cbounds + 3 + a, hi);
    }
  }
  const unsigned bal = __ballot_sync(0xFFFFFFFFu, ok);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(nvalid, (uint32_t)__popc(bal));
}

__device__ __forceinline__ uint64_t spread21(uint64_t x) {
  x &= 0x1FFFFFull;
  x = (x | x << 32) & 0x1F00000000FFFFull;
  x = (x | x << 16) & 0x1F0000FF0000FFull;
  x = (x | x << 8) & 0x100F00F00F00F00Full;
  x = (x | x << 4) & 0x10C30C30C30C30C3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

__global__ void morton_kernel(const float* __restrict__ cen, const uint8_t* __restrict__ valid,
                              const int* __restrict__ cbounds, uint32_t n,
                              uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint32_t i = blockIdx.x * kT + threadIdx.x;
  if (i >= n) return;
  vals[i] = i;
  if (!valid[i]) {
    keys[i] = kInvalidKey;   // sorts after every valid code (63-bit codes)
    return;
  }
  uint64_t q[3];
  for (int a = 0; a < 3; ++a) {
    const float lo = ord2f(cbounds[a]), hi = ord2f(cbounds[3 + a]);
    const float ext = hi - lo;
    float u = ext > 0.0f ? (cen[3 * (size_t)i + a] - lo) / ext : 0.0f;
    u = fminf(fmaxf(u, 0.0f), 1.0f);
    q[a] = (uint64_t)fminf(u * 2097152.0f, 2097151.0f);
  }
  keys[i] = spread21(q[0]) << 2 | spread21(q[1]) << 1 | spread21(q[2]);
}

// Longest common prefix of sorted keys i and j (index tie-break for equal keys).
__device__ __forceinline__ int delta(const uint64_t* k, int m, int i, int j) {
  if (j < 0 || j >= m) return -1;
  const uint64_t a = k[i], b = k[j];
  return a == b ? 64 + __clz((unsigned)(i ^ j)) : __clzll((long long)(a ^ b));
}

// Karras 2012, Fig. 4: internal node i's range [first, last] and split gamma.
// Children: internal node index in [0, m-1) or leaf j encoded as ~j.
__global__ void karras_kernel(const uint64_t* __restrict__ k, int m, int2* __restrict__ range,
                              int2* __restrict__ child, int* __restrict__ parent_node,
                              int* __restrict__ parent_leaf) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= m - 1) return;
  const int d = delta(k, m, i, i + 1) - delta(k, m, i, i - 1) >= 0 ? 1 : -1;
  const int dmin = delta(k, m, i, i - d);
  int lmax = 2;
  while (delta(k, m, i, i + lmax * d) > dmin) lmax *= 2;
  int l = 0;
  for (int t = lmax / 2; t >= 1; t /= 2)
    if (delta(k, m, i, i + (l + t) * d) > dmin) l += t;
  const int j = i + l * d;
  const int dnode = delta(k, m, i, j);
  int s = 0;
  for (int div = 2;; div *= 2) {
    const int t = (l + div - 1) / div;
    if (delta(k, m, i, i + (s + t) * d) > dnode) s += t;
    if (t <= 1) break;
  }
  const int gamma = i + s * d + min(d, 0);
  const int first = min(i, j), last = max(i, j);
  range[i] = make_int2(first, last);
  const int left = first == gamma ? ~gamma : gamma;
  const int right = last == gamma + 1 ? ~(gamma + 1) : gamma + 1;
  child[i] = make_int2(left, right);
  if (left < 0) parent_leaf[~left] = i; else parent_node[left] = i;
  if (right < 0) parent_leaf[~right] = i; else parent_node[right] = i;
}

__device__ __forceinline__ Box6 unite(const Box6& a, const Box6& b) {
  Box6 r;
  for (int q = 0; q < 3; ++q) {
    r.lo[q] = fminf(a.lo[q], b.lo[q]);
    r.hi[q] = fmaxf(a.hi[q], b.hi[q]);
  }
  return r;
}

__device__ __forceinline__ Box6 load_box(const Box6* p) {
  Box6 b;
  const volatile float* f = reinterpret_cast<const volatile float*>(p);
  for (int q = 0; q < 3; ++q) {
    b.lo[q] = f[q];
    b.hi[q] = f[3 + q];
  }
  return b;
}

// Bottom-up boxes: each leaf climbs; the second arrival at a node unites its children.
__global__ void boxes_kernel(const Box6* __restrict__ prim_box, const uint32_t* __restrict__ order,
                             int m, const int2* __restrict__ child, const int* __restrict__ parent_node,
                             const int* __restrict__ parent_leaf, Box6* node_box,
                             int* __restrict__ arrivals) {
  const int j = blockIdx.x * kT + threadIdx.x;
  if (j >= m) return;
  int p = parent_leaf[j];
  while (p >= 0) {
    __threadfence();
    if (atomicAdd(arrivals + p, 1) == 0) return;   // the sibling subtree is not done yet
    __threadfence();
    const int2 c = child[p];
    const Box6 a = c.x < 0 ? prim_box[order[~c.x]] : load_box(node_box + c.x);
    const Box6 b = c.y < 0 ? prim_box[order[~c.y]] : load_box(node_box + c.y);
    node_box[p] = unite(a, b);
    p = p == 0 ? -1 : parent_node[p];
  }
}

__global__ void live_kernel(const int2* __restrict__ range, int m, uint32_t max_leaf,
                            uint32_t* __restrict__ live) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= m - 1) return;
  live[i] = (uint32_t)(range[i].y - range[i].x + 1) > max_leaf ? 1u : 0u;
}

// Outward padding 2^-20 * max(1, |x|) in fp64, rounded outward to fp32 (the host builder's pad_out).
__device__ __forceinline__ void pad_box(const Box6& b, float* lo, float* hi) {
  for (int q = 0; q < 3; ++q) {
    const double l = b.lo[q], h = b.hi[q];
    const double ld = l - ldexp(fmax(1.0, fabs(l)), -20), hd = h + ldexp(fmax(1.0, fabs(h)), -20);
    float lf = __double2float_rd(ld), hf = __double2float_ru(hd);
    lo[q] = lf;
    hi[q] = hf;
  }
}

__device__ __forceinline__ uint32_t leaf_ref(int first, int count) {
  return kLeafBit | ((uint32_t)(count - 1) << kLeafCountShift) | (uint32_t)first;
}

// Write the surviving nodes (compacted index = exclusive scan of `live`) as pair
// nodes; children at or below max_leaf become leaves over their key range.
__global__ void write_kernel(const int2* __restrict__ range, const int2* __restrict__ child,
                             const uint32_t* __restrict__ live, const uint32_t* __restrict__ newidx,
                             const Box6* __restrict__ node_box, const Box6* __restrict__ prim_box,
                             const uint32_t* __restrict__ order, int m, PairNode* __restrict__ out,
                             const int* __restrict__ parent_node, uint32_t* __restrict__ max_depth,
                             uint32_t* __restrict__ num_leaves) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= m - 1 || !live[i]) return;
  PairNode nd;
  const int2 c = child[i];
  const int cs[2] = {c.x, c.y};
  uint32_t leaves = 0;
  for (int s = 0; s < 2; ++s) {
    const int ch = cs[s];
    Box6 b;
    if (ch < 0) {
      b = prim_box[order[~ch]];
      nd.ref[s] = leaf_ref(~ch, 1);
      ++leaves;
    } else {
      b = node_box[ch];
      if (live[ch]) {
        nd.ref[s] = newidx[ch];
      } else {
        nd.ref[s] = leaf_ref(range[ch].x, range[ch].y - range[ch].x + 1);
        ++leaves;
      }
    }
    float lo[3], hi[3];
    pad_box(b, lo, hi);
    nd.x[s] = lo[0];
    nd.x[2 + s] = hi[0];
    nd.y[s] = lo[1];
    nd.y[2 + s] = hi[1];
    nd.z[s] = lo[2];
    nd.z[2 + s] = hi[2];
  }
  nd.pad[0] = nd.pad[1] = 0;
  out[newidx[i]] = nd;
  // depth of this node's children (root = 0): ancestors are live, so climb
  uint32_t depth = 1;
  for (int p = i; p != 0; p = parent_node[p]) ++depth;
  atomicMax(max_depth, depth);
  if (leaves) atomicAdd(num_leaves, leaves);
}

__global__ void gather_kernel(const float* __restrict__ v, const float* __restrict__ tc,
                              const uint32_t* __restrict__ tri_tex, const TexDesc* __restrict__ tex,
                              const uint32_t* __restrict__ order, int m, Tri* __restrict__ tris,
                              Side* __restrict__ sides) {
  const int k = blockIdx.x * kT + threadIdx.x;
  if (k >= m) return;
  const uint32_t p = order[k];
  const float* t = v + 9 * (size_t)p;
  Tri tr;
  for (int a = 0; a < 3; ++a) {
    tr.v0[a] = t[a];
    tr.e1[a] = t[3 + a] - t[a];
    tr.e2[a] = t[6 + a] - t[a];
  }
  tr.prim = p;
  tr.pad1 = tr.pad2 = 0;
  tris[k] = tr;
  Side sd;
  for (int q = 0; q < 6; ++q) sd.uv[q] = tc ? tc[6 * (size_t)p + q] : 0.0f;
  const TexDesc d = tex[tri_tex[p]];
  sd.texel_offset = (uint32_t)d.offset;
  sd.dims = (d.w - 1u) | ((d.h - 1u) << 16);
  sides[k] = sd;
}

__global__ void root_box_kernel(const Box6* __restrict__ prim_box, const uint32_t* __restrict__ order,
                                int m, const Box6* __restrict__ node_box, float* __restrict__ out) {
  // single thread: the root box is node 0's (m >= 2) or the lone leaf's union
  Box6 b;
  if (m >= 2) {
    b = node_box[0];
  } else {
    b = prim_box[order[0]];
  }
  pad_box(b, out, out + 3);
}

// ---------------------------------------------------------------------------
// PLOC (Meister & Bittner, TVCG 2018): parallel locally-ordered clustering on
// the Morton-sorted leaves.  Each round every cluster finds its nearest
// neighbour (smallest union surface area, ties -> lower index) within +-r
// positions, mutual pairs merge into a new node, and the cluster array is
// compacted; binned-SAH-like trees at LBVH-like cost.  The finished tree is
// re-expressed in the Karras arrays above (root = node 0, every node a
// contiguous range of a depth-first leaf order) so the same collapse / write
// kernels produce the export layout.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float half_area(const Box6& b) {
  const float dx = b.hi[0] - b.lo[0], dy = b.hi[1] - b.lo[1], dz = b.hi[2] - b.lo[2];
  return dx * dy + dy * dz + dz * dx;
}

__global__ void ploc_init_kernel(const Box6* __restrict__ prim_box, const uint32_t* __restrict__ order,
                                 int m, int* __restrict__ cl_node, Box6* __restrict__ cl_box) {
  const int k = blockIdx.x * kT + threadIdx.x;
  if (k >= m) return;
  cl_node[k] = ~k;
  cl_box[k] = prim_box[order[k]];
}

__global__ void ploc_nn_kernel(const Box6* __restrict__ cl_box, int c, int r, int* __restrict__ nn) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= c) return;
  // Ties are broken by a key symmetric in (i, j) — nearer position, then pairs that start
  // at an even position, then the lower pair — so runs of equal boxes pair up (2k, 2k+1)
  // instead of chaining onto the lowest index.
  const Box6 bi = cl_box[i];
  float best = INFINITY;
  int bj = -1;
  uint64_t bkey = ~0ull;
  const int lo = max(0, i - r), hi = min(c - 1, i + r);
  for (int j = lo; j <= hi; ++j) {
    if (j == i) continue;
    const float a = half_area(unite(bi, cl_box[j]));
    const int lo_ij = min(i, j);
    const uint64_t key = ((uint64_t)abs(i - j) << 33) | ((uint64_t)(lo_ij & 1) << 32) |
                         (uint64_t)(uint32_t)lo_ij;
    if (a < best || (a == best && key < bkey)) {
      best = a;
      bj = j;
      bkey = key;
    }
  }
  nn[i] = bj;
}

__global__ void ploc_flags_kernel(const int* __restrict__ nn, int c, uint32_t* __restrict__ fnew,
                                  uint32_t* __restrict__ fkeep) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= c) return;
  const int j = nn[i];
  const bool mutual = j >= 0 && nn[j] == i;
  fnew[i] = mutual && i < j;
  fkeep[i] = !(mutual && i > j);
}

__global__ void ploc_force_kernel(int* nn) {   // no mutual pair this round: merge clusters 0 and 1
  nn[0] = 1;
  nn[1] = 0;
}

__global__ void ploc_apply_kernel(const int* __restrict__ nn, int c, const uint32_t* __restrict__ fnew,
                                  const uint32_t* __restrict__ snew, const uint32_t* __restrict__ fkeep,
                                  const uint32_t* __restrict__ skeep, const int* __restrict__ cl_node,
                                  const Box6* __restrict__ cl_box, int node_base,
                                  int* __restrict__ out_node, Box6* __restrict__ out_box,
                                  int2* __restrict__ nchild, Box6* __restrict__ nbox) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= c || !fkeep[i]) return;
  const uint32_t pos = skeep[i];
  if (fnew[i]) {
    const int j = nn[i];
    const int id = node_base + (int)snew[i];
    const Box6 b = unite(cl_box[i], cl_box[j]);
    nchild[id] = make_int2(cl_node[i], cl_node[j]);
    nbox[id] = b;
    out_node[pos] = id;
    out_box[pos] = b;
  } else {
    out_node[pos] = cl_node[i];
    out_box[pos] = cl_box[i];
  }
}

__global__ void ploc_parents_kernel(const int2* __restrict__ nchild, int nint, int* __restrict__ parent_int,
                                    int* __restrict__ parent_leaf) {
  const int n = blockIdx.x * kT + threadIdx.x;
  if (n >= nint) return;
  const int2 c = nchild[n];
  if (c.x >= 0) parent_int[c.x] = n; else parent_leaf[~c.x] = n;
  if (c.y >= 0) parent_int[c.y] = n; else parent_leaf[~c.y] = n;
}

// leaves per subtree, bottom-up (the second child to arrive sums)
__global__ void ploc_sizes_kernel(int m, const int2* __restrict__ nchild, const int* __restrict__ parent_int,
                                  const int* __restrict__ parent_leaf, int* size, int* __restrict__ arrivals) {
  const int k = blockIdx.x * kT + threadIdx.x;
  if (k >= m) return;
  int p = parent_leaf[k];
  const volatile int* vs = size;
  while (p >= 0) {
    __threadfence();
    if (atomicAdd(arrivals + p, 1) == 0) return;
    __threadfence();
    const int2 c = nchild[p];
    size[p] = (c.x < 0 ? 1 : vs[c.x]) + (c.y < 0 ? 1 : vs[c.y]);
    p = parent_int[p];
  }
}

// first leaf position of subtree x (node id, or ~leaf) in the depth-first leaf order
__device__ __forceinline__ int dfs_start(int x, const int* parent_int, const int* parent_leaf,
                                         const int2* nchild, const int* size) {
  int s = 0;
  int cur = x;
  int p = x >= 0 ? parent_int[x] : parent_leaf[~x];
  while (p >= 0) {
    const int2 c = nchild[p];
    if (c.y == cur) s += c.x < 0 ? 1 : size[c.x];
    cur = p;
    p = parent_int[p];
  }
  return s;
}

__global__ void ploc_layout_kernel(int m, const uint32_t* __restrict__ order, const int* __restrict__ parent_int,
                                   const int* __restrict__ parent_leaf, const int2* __restrict__ nchild,
                                   const int* __restrict__ size, int* __restrict__ pos,
                                   uint32_t* __restrict__ order2, int* __restrict__ start) {
  const int k = blockIdx.x * kT + threadIdx.x;
  if (k < m) {
    const int q = dfs_start(~k, parent_int, parent_leaf, nchild, size);
    pos[k] = q;
    order2[q] = order[k];
  }
  if (k < m - 1) start[k] = dfs_start(k, parent_int, parent_leaf, nchild, size);
}

// node n (creation order, root = m - 2) -> Karras arrays with root 0
__global__ void ploc_export_kernel(int m, const int2* __restrict__ nchild, const Box6* __restrict__ nbox,
                                   const int* __restrict__ size, const int* __restrict__ start,
                                   const int* __restrict__ parent_int, const int* __restrict__ pos,
                                   int2* __restrict__ range, int2* __restrict__ child,
                                   int* __restrict__ parent_node, Box6* __restrict__ node_box) {
  const int n = blockIdx.x * kT + threadIdx.x;
  if (n >= m - 1) return;
  const int root = m - 2, nid = root - n;
  range[nid] = make_int2(start[n], start[n] + size[n] - 1);
  const int2 c = nchild[n];
  child[nid] = make_int2(c.x >= 0 ? root - c.x : ~pos[~c.x], c.y >= 0 ? root - c.y : ~pos[~c.y]);
  parent_node[nid] = parent_int[n] >= 0 ? root - parent_int[n] : -1;
  node_box[nid] = nbox[n];
}

template <class T>
cudaError_t alloc(T** p, size_t count) {
  return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1));
}

}  // namespace

vsr_status build_bvh_gpu(const float* d_vertices, const float* d_texcoords,
                         const uint32_t* d_tri_tex, const TexDesc* d_tex, uint32_t n,
                         uint32_t max_leaf, GpuBvh& out, std::string& err, int ploc_radius) {
  cudaStream_t st = nullptr;
  Box6* box = nullptr;
  float* cen = nullptr;
  uint8_t* valid = nullptr;
  int* cb = nullptr;
  uint32_t* counters = nullptr;   // [0] valid, [1] max depth, [2] leaves
  uint64_t *keys = nullptr, *keys2 = nullptr;
  uint32_t *vals = nullptr, *vals2 = nullptr, *live = nullptr, *newidx = nullptr;
  int2 *range = nullptr, *child = nullptr;
  int *parent_node = nullptr, *parent_leaf = nullptr, *arrivals = nullptr;
  Box6* node_box = nullptr;
  float* root = nullptr;
  void* tmp = nullptr;
  // PLOC scratch
  int *cl_node[2] = {nullptr, nullptr}, *nn = nullptr, *pint = nullptr, *psize = nullptr;
  int *ppos = nullptr, *pstart = nullptr, *parr = nullptr;
  Box6 *cl_box[2] = {nullptr, nullptr}, *nbox = nullptr;
  int2* nchild = nullptr;
  uint32_t *fnew = nullptr, *fkeep = nullptr, *snew = nullptr, *skeep = nullptr, *order2 = nullptr;
  out = GpuBvh{};
  cudaError_t e = cudaSuccess;
  auto fin = [&](vsr_status s, const std::string& msg) {
    cudaFree(box); cudaFree(cen); cudaFree(valid); cudaFree(cb); cudaFree(counters);
    cudaFree(keys); cudaFree(keys2); cudaFree(vals); cudaFree(vals2); cudaFree(live);
    cudaFree(newidx); cudaFree(range); cudaFree(child); cudaFree(parent_node);
    cudaFree(parent_leaf); cudaFree(arrivals); cudaFree(node_box); cudaFree(root); cudaFree(tmp);
    cudaFree(cl_node[0]); cudaFree(cl_node[1]); cudaFree(nn); cudaFree(pint); cudaFree(psize);
    cudaFree(ppos); cudaFree(pstart); cudaFree(parr); cudaFree(cl_box[0]); cudaFree(cl_box[1]);
    cudaFree(nbox); cudaFree(nchild); cudaFree(fnew); cudaFree(fkeep); cudaFree(snew);
    cudaFree(skeep); cudaFree(order2);
    if (s != VSR_OK) {
      cudaFree(out.nodes); cudaFree(out.tris); cudaFree(out.sides);
      out = GpuBvh{};
      err = msg + (e != cudaSuccess ? std::string(": ") + cudaGetErrorString(e) : std::string());
    }
    return s;
  };
#define VSR_TRY(x)                                  \
  if ((e = (x)) != cudaSuccess) return fin(e == cudaErrorMemoryAllocation ? VSR_ERR_OOM : VSR_ERR_CUDA, #x)
  const unsigned g = (n + kT - 1) / kT;
  VSR_TRY(alloc(&box, n));
  VSR_TRY(alloc(&cen, 3 * (size_t)n));
  VSR_TRY(alloc(&valid, n));
  VSR_TRY(alloc(&cb, 6));
  VSR_TRY(alloc(&counters, 3));
  const int init[6] = {0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF, (int)0x80000000, (int)0x80000000,
                       (int)0x80000000};
  VSR_TRY(cudaMemcpy(cb, init, sizeof init, cudaMemcpyHostToDevice));
  VSR_TRY(cudaMemsetAsync(counters, 0, 3 * sizeof(uint32_t), st));   // ordered before prep_kernel
  prep_kernel<<<g, kT, 0, st>>>(d_vertices, n, box, cen, valid, cb, counters);
  VSR_TRY(cudaGetLastError());
  uint32_t m32 = 0;
  VSR_TRY(cudaMemcpy(&m32, counters, sizeof m32, cudaMemcpyDeviceToHost));
  out.num_degenerate = n - m32;
  const int m = (int)m32;
  if (m == 0) return fin(VSR_ERR_EMPTY_SCENE, "empty scene: no non-degenerate triangles");
  if (m32 > kMaxTris)
    return fin(VSR_ERR_UNSUPPORTED, "more than 2^26 triangles are not supported by the 26-bit leaf encoding");
  VSR_TRY(alloc(&keys, n));
  VSR_TRY(alloc(&keys2, n));
  VSR_TRY(alloc(&vals, n));
  VSR_TRY(alloc(&vals2, n));
  morton_kernel<<<g, kT, 0, st>>>(cen, valid, cb, n, keys, vals);
  VSR_TRY(cudaGetLastError());
  size_t tmp_bytes = 0, scan_bytes = 0;
  VSR_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, 64, st));
  VSR_TRY(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, live, newidx, m > 1 ? m - 1 : 1, st));
  VSR_TRY(cudaMalloc(&tmp, tmp_bytes > scan_bytes ? tmp_bytes : scan_bytes));
  // stable LSD radix sort: equal codes keep ascending triangle index
  VSR_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, 64, st));
  const uint32_t* order = vals2;   // sorted triangle indices; the first m are the valid ones
  const unsigned gi = m > 1 ? (unsigned)((m - 1 + kT - 1) / kT) : 1u;
  const unsigned gl = (unsigned)((m + kT - 1) / kT);
  if (m >= 2) {
    VSR_TRY(alloc(&range, m - 1));
    VSR_TRY(alloc(&child, m - 1));
    VSR_TRY(alloc(&parent_node, m - 1));
    VSR_TRY(alloc(&parent_leaf, m));
    VSR_TRY(alloc(&arrivals, m - 1));
    VSR_TRY(alloc(&node_box, m - 1));
    VSR_TRY(alloc(&live, m - 1));
    VSR_TRY(alloc(&newidx, m - 1));
    VSR_TRY(cudaMemsetAsync(arrivals, 0, sizeof(int) * (m - 1), st));
    VSR_TRY(cudaMemsetAsync(parent_node, 0xFF, sizeof(int) * (m - 1), st));
    if (ploc_radius <= 0) {   // LBVH: Karras splits on the Morton codes
      karras_kernel<<<gi, kT, 0, st>>>(keys2, m, range, child, parent_node, parent_leaf);
      VSR_TRY(cudaGetLastError());
      boxes_kernel<<<gl, kT, 0, st>>>(box, order, m, child, parent_node, parent_leaf, node_box,
                                      arrivals);
      VSR_TRY(cudaGetLastError());
    } else {                  // PLOC clustering, then the same arrays
      VSR_TRY(alloc(&cl_node[0], m));
      VSR_TRY(alloc(&cl_node[1], m));
      VSR_TRY(alloc(&cl_box[0], m));
      VSR_TRY(alloc(&cl_box[1], m));
      VSR_TRY(alloc(&nn, m));
      VSR_TRY(alloc(&fnew, m));
      VSR_TRY(alloc(&fkeep, m));
      VSR_TRY(alloc(&snew, m));
      VSR_TRY(alloc(&skeep, m));
      VSR_TRY(alloc(&nchild, m - 1));
      VSR_TRY(alloc(&nbox, m - 1));
      size_t sb = 0;
      VSR_TRY(cub::DeviceScan::ExclusiveSum(nullptr, sb, fnew, snew, m, st));
      if (sb > scan_bytes && sb > tmp_bytes) {
        cudaFree(tmp);
        tmp = nullptr;
        VSR_TRY(cudaMalloc(&tmp, sb));
        tmp_bytes = sb;
      }
      const size_t tb = tmp_bytes > scan_bytes ? tmp_bytes : scan_bytes;
      ploc_init_kernel<<<gl, kT, 0, st>>>(box, order, m, cl_node[0], cl_box[0]);
      VSR_TRY(cudaGetLastError());
      int c = m, node_base = 0, cur = 0;
      while (c > 1) {
        const unsigned gc = (unsigned)((c + kT - 1) / kT);
        ploc_nn_kernel<<<gc, kT, 0, st>>>(cl_box[cur], c, ploc_radius, nn);
        ploc_flags_kernel<<<gc, kT, 0, st>>>(nn, c, fnew, fkeep);
        VSR_TRY(cudaGetLastError());
        size_t b1 = tb, b2 = tb;
        VSR_TRY(cub::DeviceScan::ExclusiveSum(tmp, b1, fnew, snew, c, st));
        uint32_t tail[2];
        VSR_TRY(cudaMemcpy(&tail[0], snew + (c - 1), 4, cudaMemcpyDeviceToHost));
        VSR_TRY(cudaMemcpy(&tail[1], fnew + (c - 1), 4, cudaMemcpyDeviceToHost));
        int made = (int)(tail[0] + tail[1]);
        if (made == 0) {   // cannot happen with a strict order on (area, index); stay safe
          ploc_force_kernel<<<1, 1, 0, st>>>(nn);
          ploc_flags_kernel<<<gc, kT, 0, st>>>(nn, c, fnew, fkeep);
          VSR_TRY(cudaGetLastError());
          VSR_TRY(cub::DeviceScan::ExclusiveSum(tmp, b1, fnew, snew, c, st));
          made = 1;
        }
        VSR_TRY(cub::DeviceScan::ExclusiveSum(tmp, b2, fkeep, skeep, c, st));
        ploc_apply_kernel<<<gc, kT, 0, st>>>(nn, c, fnew, snew, fkeep, skeep, cl_node[cur],
                                             cl_box[cur], node_base, cl_node[cur ^ 1],
                                             cl_box[cur ^ 1], nchild, nbox);
        VSR_TRY(cudaGetLastError());
        node_base += made;
        c -= made;
        cur ^= 1;
      }
      VSR_TRY(alloc(&pint, m - 1));
      VSR_TRY(alloc(&psize, m - 1));
      VSR_TRY(alloc(&ppos, m));
      VSR_TRY(alloc(&pstart, m - 1));
      VSR_TRY(alloc(&parr, m - 1));
      VSR_TRY(alloc(&order2, m));
      VSR_TRY(cudaMemsetAsync(pint, 0xFF, sizeof(int) * (m - 1), st));
      VSR_TRY(cudaMemsetAsync(parr, 0, sizeof(int) * (m - 1), st));
      ploc_parents_kernel<<<gi, kT, 0, st>>>(nchild, m - 1, pint, parent_leaf);
      ploc_sizes_kernel<<<gl, kT, 0, st>>>(m, nchild, pint, parent_leaf, psize, parr);
      ploc_layout_kernel<<<gl, kT, 0, st>>>(m, order, pint, parent_leaf, nchild, psize, ppos, order2,
                                            pstart);
      ploc_export_kernel<<<gi, kT, 0, st>>>(m, nchild, nbox, psize, pstart, pint, ppos, range, child,
                                            parent_node, node_box);
      VSR_TRY(cudaGetLastError());
      order = order2;
    }
    live_kernel<<<gi, kT, 0, st>>>(range, m, max_leaf, live);
    VSR_TRY(cudaGetLastError());
    VSR_TRY(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, live, newidx, m - 1, st));
    uint32_t last_idx = 0, last_live = 0;
    VSR_TRY(cudaMemcpy(&last_idx, newidx + (m - 2), sizeof last_idx, cudaMemcpyDeviceToHost));
    VSR_TRY(cudaMemcpy(&last_live, live + (m - 2), sizeof last_live, cudaMemcpyDeviceToHost));
    out.num_nodes = last_idx + last_live;
  }
  VSR_TRY(alloc(&out.nodes, out.num_nodes));
  VSR_TRY(alloc(&out.tris, m));
  VSR_TRY(alloc(&out.sides, m));
  VSR_TRY(alloc(&root, 6));
  if (out.num_nodes) {
    write_kernel<<<gi, kT, 0, st>>>(range, child, live, newidx, node_box, box, order, m, out.nodes,
                                    parent_node, counters + 1, counters + 2);
    VSR_TRY(cudaGetLastError());
  }
  gather_kernel<<<gl, kT, 0, st>>>(d_vertices, d_texcoords, d_tri_tex, d_tex, order, m, out.tris,
                                   out.sides);
  VSR_TRY(cudaGetLastError());
  root_box_kernel<<<1, 1, 0, st>>>(box, order, m, node_box, root);
  VSR_TRY(cudaGetLastError());
  uint32_t cnt[3];
  VSR_TRY(cudaMemcpy(cnt, counters, sizeof cnt, cudaMemcpyDeviceToHost));
  VSR_TRY(cudaMemcpy(out.root_lo, root, 3 * sizeof(float), cudaMemcpyDeviceToHost));
  VSR_TRY(cudaMemcpy(out.root_hi, root + 3, 3 * sizeof(float), cudaMemcpyDeviceToHost));
  out.num_tris = m32;
  if (out.num_nodes) {
    out.root_ref = 0;
    out.max_depth = cnt[1];
    out.num_leaves = cnt[2];
  } else {   // m <= max_leaf: one leaf
    out.root_ref = kLeafBit | ((m32 - 1u) << kLeafCountShift);
    out.max_depth = 0;
    out.num_leaves = 1;
  }
  if (out.max_depth > (uint32_t)kMaxStack) {
    e = cudaSuccess;
    return fin(VSR_ERR_BVH_TOO_DEEP, "BVH deeper than 64 levels (traversal stack bound)");
  }
  return fin(VSR_OK, "");
#undef VSR_TRY
}

}  // namespace vsr
