// api_compound.cpp — compound queries of the C ABI (include/vsr.h): lists of
// BVHs (vsr_group_*, vsr_trace_group[_multi]) and two-level instancing
// (vsr_instances_*, vsr_trace_instances[_multi]; reading A27).
#include "api_internal.hpp"

namespace {

// Per-element mask data carrying each element scene's 1-bit alpha plane for a
// threshold (alpha_keep_bits), one device array per threshold seen (≤ 8).
struct PlaneData {
  std::mutex mu;
  uint32_t a_min[vsr_scene::kMaxPlanes] = {};
  IsectData* d[vsr_scene::kMaxPlanes] = {};
  int n = 0;
  void release() {
    for (int i = 0; i < n; ++i) cudaFree(d[i]);
    n = 0;
  }
};

// All-or-nothing: the array for a_min when every element scene has (or can now
// build) its plane, else nullptr (the A8 path runs). Nothing is allocated while
// `stream` is being captured.
const IsectData* compound_planes(PlaneData& pd, const std::vector<vsr_scene*>& scenes,
                                 uint32_t a_min, void* stream) {
  const char* eb = std::getenv("VSR_ALPHA_BITS");
  if (eb && std::strcmp(eb, "0") == 0) return nullptr;
  std::lock_guard<std::mutex> lk(pd.mu);
  for (int i = 0; i < pd.n; ++i)
    if (pd.a_min[i] == a_min) return pd.d[i];
  if (pd.n == vsr_scene::kMaxPlanes) return nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(reinterpret_cast<cudaStream_t>(stream), &cs) != cudaSuccess ||
      cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return nullptr;
  }
  std::vector<IsectData> data(scenes.size());
  for (size_t k = 0; k < scenes.size(); ++k) {
    const uint32_t* b = alpha_plane(scenes[k], a_min, stream);
    if (!b) return nullptr;
    data[k] = IsectData{scenes[k]->d_sides, scenes[k]->d_texdescs, scenes[k]->d_texels, 0u, 0.0f,
                        0.0f, b, scenes[k]->num_texels};
  }
  IsectData* d = nullptr;
  if (cudaMalloc(&d, sizeof(IsectData) * data.size()) != cudaSuccess ||
      cudaMemcpy(d, data.data(), sizeof(IsectData) * data.size(), cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    cudaGetLastError();
    cudaFree(d);
    return nullptr;
  }
  pd.a_min[pd.n] = a_min;
  pd.d[pd.n++] = d;
  return d;
}

}  // namespace

struct vsr_group {
  int device = 0;
  ScratchSet scratch;
  PlaneData planes;   // per-threshold mask data with the elements' 1-bit alpha planes
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
    data[k] = IsectData{scenes[k]->d_sides, scenes[k]->d_texdescs, scenes[k]->d_texels, 0u, 0.0f,
                        0.0f, nullptr, scenes[k]->num_texels};
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
    g->planes.release();
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
                              isect, params, p, false);
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
  if (isect == VSR_ISECT_ALPHA_TEXTURE)
    if (const IsectData* bd = compound_planes(g->planes, g->scenes, p.data.a_min, stream)) {
      p.list_data = bd;
      p.data.bits = alpha_plane(g->scenes[0], p.data.a_min, stream);   // cached: selects the kernel
    }
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
  PlaneData planes;   // per-threshold mask data with the elements' 1-bit alpha planes
  std::vector<vsr_scene*> scenes;
  HostBvh top;                       // host copy of the top-level nodes (export)
  std::vector<Instance> records;     // leaf order (export)
  float r_safe = 0.0f;               // rays with |o|_inf above take the linear path (A27)
  DevScene dev{};                    // top level: nodes, root ref / box
  PairNode* d_nodes = nullptr;
  Instance* d_records = nullptr;
  DevScene* d_list = nullptr;
  IsectData* d_data = nullptr;
  uint32_t* d_grid = nullptr;   // density grid over the instance boxes (order-pass proxy)
};

namespace {

// World box of an instance: the 8 corners of the scene's (padded) root box
// mapped by the fp64 inverse of [A | b], then padded by 2^-10 (diagonal +
// max |coordinate|) and rounded outward (reading A27).  False if A is singular.
bool instance_world_box(const float* m, const float* lo, const float* hi, float* out,
                        double* pad_out = nullptr) {
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
  if (pad_out) *pad_out = pad;
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

// Far-origin bound (reading A27, round 2): the world box above holds the
// instance for a ray whose origin satisfies |o|_inf <= R, where the fp32 ray map
// o' = ((A_i0 o_x + A_i1 o_y) + A_i2 o_z) + b_i, d' = (A d) (3 products, 3 sums)
// errs by |do'| <= g5 (|A||o| + |b|), |dd'| <= g4 |A||d| (componentwise, g_n = n u /
// (1 - n u)).  A point of the mapped ray that reaches the object box is then within
// |A^-1| (|do'| + t |dd'|) of the exact world ray, and t |A||d| <= k t |Ad| <=
// k (mag_obj + |A||o| + |b|) with k = ||A|| ||A^-1|| (inf-norms), so the world-space
// displacement is at most ||A^-1|| [g5 (1 + k)(||A|| R + |b|) + g4 k mag_obj]; the box
// pad P (2^-10 (diagonal + max |coord|)) covers it for R up to the value returned
// (halved for margin; 0 if even R = 0 is not covered).  Rays beyond the minimum of
// this over all instances take the linear path over every instance instead of the
// top-level BVH (trace_instances_kernel), which is the definition itself.
double instance_safe_range(const float* m, const float* obj_lo, const float* obj_hi, double pad) {
  const double a[3][3] = {{m[0], m[1], m[2]}, {m[4], m[5], m[6]}, {m[8], m[9], m[10]}};
  const double bv[3] = {m[3], m[7], m[11]};
  const double det = a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
                     a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
                     a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
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
  double nA = 0.0, nI = 0.0, nb = 0.0, mag = 0.0;
  for (int i = 0; i < 3; ++i) {
    nA = std::max(nA, std::fabs(a[i][0]) + std::fabs(a[i][1]) + std::fabs(a[i][2]));
    nI = std::max(nI, std::fabs(inv[i][0]) + std::fabs(inv[i][1]) + std::fabs(inv[i][2]));
    nb = std::max(nb, std::fabs(bv[i]));
    mag = std::max(mag, std::max(std::fabs((double)obj_lo[i]), std::fabs((double)obj_hi[i])));
  }
  const double u = std::ldexp(1.0, -24), g4 = 4 * u / (1 - 4 * u), g5 = 5 * u / (1 - 5 * u);
  const double k = nA * nI;
  const double r = (pad / nI - g4 * k * mag - g5 * (1.0 + k) * nb) / (g5 * (1.0 + k) * nA);
  return r > 0.0 ? 0.5 * r : 0.0;
}

void free_instances(vsr_instances* I) {
  if (I->device < 0) return;
  DeviceGuard dg(I->device);
  I->scratch.release();
  I->planes.release();
  cudaFree(I->d_nodes);
  cudaFree(I->d_records);
  cudaFree(I->d_list);
  cudaFree(I->d_data);
  cudaFree(I->d_grid);
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
  double r_safe = INFINITY;
  for (uint32_t i = 0; i < num_instances; ++i) {
    const vsr_instance& in = instances[i];
    if (in.bvh >= num_scenes)
      return fail(VSR_ERR_INVALID_ARG, "instance " + std::to_string(i) + ": bvh index out of range");
    for (float x : in.object_from_world)
      if (!std::isfinite(x))
        return fail(VSR_ERR_INVALID_ARG, "instance " + std::to_string(i) + ": non-finite matrix");
    const DevScene& d = scenes[in.bvh]->dev;
    double pad = 0.0;
    if (!instance_world_box(in.object_from_world, d.root_lo, d.root_hi, boxes.data() + 6 * (size_t)i,
                            &pad))
      return fail(VSR_ERR_INVALID_ARG, "instance " + std::to_string(i) + ": singular matrix");
    r_safe = std::min(r_safe, instance_safe_range(in.object_from_world, d.root_lo, d.root_hi, pad));
  }
  vsr_instances* I = new (std::nothrow) vsr_instances();
  if (!I) return fail(VSR_ERR_OOM, "instances allocation");
  I->device = scenes[0]->device;
  I->scenes.assign(scenes, scenes + num_scenes);
  {   // rounded down to fp32: the kernel and walker compare fp32 |o_k| <= r_safe
    float rf = (float)r_safe;
    if ((double)rf > r_safe) rf = std::nextafter(rf, 0.0f);
    I->r_safe = rf;
  }
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
    data[k] = IsectData{scenes[k]->d_sides, scenes[k]->d_texdescs, scenes[k]->d_texels, 0u, 0.0f,
                        0.0f, nullptr, scenes[k]->num_texels};
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
  {   // density grid over the instance world boxes, each weighted by nothing but its presence
      // (order-pass cost proxy VSR_ORDER_PROXY=grid; scheduling only): a box as the triangle
      // (lo, lo + (hi - lo), lo) covers exactly the box's cells
    std::vector<Tri> boxes_as_tris(num_instances);
    for (uint32_t i = 0; i < num_instances; ++i) {
      Tri& t = boxes_as_tris[i];
      std::memset(&t, 0, sizeof t);
      for (int a = 0; a < 3; ++a) {
        t.v0[a] = boxes[6 * (size_t)i + a];
        t.e1[a] = boxes[6 * (size_t)i + 3 + a] - boxes[6 * (size_t)i + a];
      }
    }
    density_grid_dims(I->dev.root_lo, I->dev.root_hi, I->dev.gdim, I->dev.gscale);
    Tri* d_bt = nullptr;
    const size_t words = density_grid_words(I->dev.gdim);
    if ((e = cudaMalloc(&I->d_grid, words * sizeof(uint32_t))) != cudaSuccess ||
        (e = cudaMemset(I->d_grid, 0, words * sizeof(uint32_t))) != cudaSuccess ||
        (e = cudaMalloc(&d_bt, num_instances * sizeof(Tri))) != cudaSuccess ||
        (e = cudaMemcpy(d_bt, boxes_as_tris.data(), num_instances * sizeof(Tri),
                        cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = build_density_grid(d_bt, num_instances, I->dev.root_lo, I->dev.gdim, I->dev.gscale,
                                I->d_grid, nullptr)) != cudaSuccess ||
        (e = cudaDeviceSynchronize()) != cudaSuccess) {
      cudaFree(d_bt);
      free_instances(I);
      delete I;
      return cuda_fail(e, "instances density grid");
    }
    cudaFree(d_bt);
    I->dev.grid = I->d_grid;
  }
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
  v->r_safe = I->r_safe;
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
                              isect, params, p, false);
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
  if (isect == VSR_ISECT_ALPHA_TEXTURE)
    if (const IsectData* bd = compound_planes(I->planes, I->scenes, p.data.a_min, stream)) {
      p.list_data = bd;
      p.data.bits = alpha_plane(I->scenes[0], p.data.a_min, stream);   // cached: selects the kernel
    }
  p.list_count = (uint32_t)I->scenes.size();
  p.instances = I->d_records;
  p.num_instances = (uint32_t)I->records.size();
  p.inst_r_safe = I->r_safe;
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

}  // extern "C"
