// trace.cu — the hot path: per-ray BVH traversal + ray/triangle intersection
// with a compile-time intersector (§3.2).
//
// Traversal: the while-while scheme of Aila & Laine cited by the paper
// (PAPER.md:228-247): an inner-node loop that calls the intersector's box
// hook on both children of a 64-B pair node, then a leaf loop that calls its
// triangle hook on each primitive.  Every decision is a function of the ray
// alone (no warp-voted speculation), so results and the counting
// intersector's numbers do not depend on which lanes share a warp — they are
// deterministic and match the CPU walker bit for bit.
//
// Scheduling (B200), measured in profiles/r01_tuning.md: one thread per ray,
// 128-ray blocks launched longest-first (a small order pass estimates each
// block's cost from its rays' segment inside the root box), so the blocks
// whose single-ray latency would set the tail start first.  A persistent
// dynamic-fetch kernel (warps claim rays from a global counter and refill
// idle lanes) is kept as VSR_SCHED=persistent; it loses on coherent primary
// rays.
//
// This file: the longest-first order pass, the plain / multi-hit / pinhole /
// persistent trace kernels and launch_trace (the one host entry every query
// goes through).  The traversal core is traverse.cuh; lists and instances are
// compound.cu; primitive lists prims.cu.
//
// Build: -gencode arch=compute_100a,code=sm_100a -fmad=false (IEEE fp32
// contract).

#include <algorithm>
#include <mutex>
#include <vector>
#include <cmath>
#include <cstdio>
#include <string>

#include "traverse.cuh"

namespace vsr {

#ifndef VSR_INST_COST
#define VSR_INST_COST 0   // 1: instance-box-count proxy — measured 5-18 % SLOWER (profiles/r02_tuning.md)
#endif
// Cost proxy of an INSTANCED query (p.instances set, p.scene = the top level):
// the number of instance world boxes the ray's [tmin, tmax] segment enters,
// capped at kOrderBuckets - 1.  The length of the segment inside the union of
// all instances (the flat-scene proxy) barely separates a ray that crosses a
// dense cluster of instances from one that crosses open ground, so the
// longest-first order needs the top level itself (measured: the instanced
// forest's tail).  No best_t pruning: this estimates the work.
__device__ uint32_t instance_cost(const TraceParams& p, const RayCtx& r, float tmax) {
  const DevScene& S = p.scene;
  const Aabb root{S.root_lo[0], S.root_lo[1], S.root_lo[2], S.root_hi[0], S.root_hi[1], S.root_hi[2]};
  float tn;
  if (!intersect(r, root, tmax, tn)) return 0u;
  uint32_t stack[kMaxStack];
  int sp = 0;
  uint32_t cur = S.root_ref, cnt = 0;
  const uint32_t cap = kOrderBuckets - 1;
  for (;;) {
    if (cur & kLeafBit) {
      cnt += ((cur >> kLeafCountShift) & 31u) + 1u;
      if (cnt >= cap || sp == 0) break;
      cur = stack[--sp];
      continue;
    }
    const float4* np = reinterpret_cast<const float4*>(S.nodes + cur);
    const BoxPairHit h = intersect(r, AabbPair{__ldg(np), __ldg(np + 1), __ldg(np + 2)}, tmax);
    const float4 nr = __ldg(np + 3);
    const uint32_t r0 = __float_as_uint(nr.x), r1 = __float_as_uint(nr.y);
    if (h.h0 && h.h1) {
      stack[sp++] = r1;
      cur = r0;
    } else if (h.h0 || h.h1) {
      cur = h.h0 ? r0 : r1;
    } else if (sp > 0) {
      cur = stack[--sp];
    } else {
      break;
    }
  }
  return cnt < cap ? cnt : cap;
}

// Density-grid cost proxy (order_proxy 1): the sample ray's [tn, tf] segment
// inside the root box, sampled at kGridSamples evenly spaced points, each
// weighted by the scene's coarse density grid (the number of triangle boxes
// overlapping its cell): a line integral of box density.  The samples' cell
// loads are independent, so they are all in flight at once (a 3D-DDA march
// was measured: its chain of dependent cold loads made the order pass the
// long pole).  Motivation: the rays that skim a dense layer (every billboard
// box reaches down to the ground) cost far more than their segment length
// says (tools/timeline.py: the launch's last warp started 20 us late with an
// 83 us run).  Bucket = 6 log2(1 + integral).
//
// Blended proxy (order_proxy 3, the default for plain scenes): the mean of this
// bucket (4 samples) and the segment-length bucket.  The pure density integral
// mis-ranks terrain scenes (C4 -8 %: every ground cell is dense), the segment
// length mis-ranks the rays that skim a dense layer (C2); the mean measured
// C2 any +1.2 %, closest +0.9 %, C4 any +0.8 %, C5 any -0.2 %.  Four samples
// keep the order pass's grid requests (the cost of the 16-sample form: ~1 M
// requests on a few thousand hot L2 lines) at a quarter.
constexpr int kGridSamples = 16;   // pure density proxy (instanced queries)
#ifndef VSR_MIX_SAMPLES
#define VSR_MIX_SAMPLES 4
#endif
#ifndef VSR_MIX_W
#define VSR_MIX_W 0.5f   // weight of the density bucket in the blend
#endif
constexpr int kMixSamples = VSR_MIX_SAMPLES;   // blended proxy
constexpr int kGridCopies = 32;   // replicas of the grid, one per CTA modulo: spreads the
                                  // order pass's burst of loads over 32x more L2 lines
template <int NS>
__device__ float grid_cost(const DevScene& S, const RayCtx& r, float tn, float tf) {
  const float step = (tf - tn) * (1.0f / NS);
  const uint32_t* grid = S.grid + (uint64_t)(blockIdx.x % kGridCopies) * S.gdim[0] * S.gdim[1] * S.gdim[2];
  float sum = 0.0f;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    const float t = tn + ((float)k + 0.5f) * step;
    int c[3];
    const float pt[3] = {r.ox + t * r.dx, r.oy + t * r.dy, r.oz + t * r.dz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int ca = (int)floorf((pt[a] - S.root_lo[a]) * S.gscale[a]);
      c[a] = ca < 0 ? 0 : (ca >= (int)S.gdim[a] ? (int)S.gdim[a] - 1 : ca);
    }
    sum += (float)__ldg(grid + ((uint64_t)c[2] * S.gdim[1] + c[1]) * S.gdim[0] + c[0]);
  }
  return sum * step * sqrtf(r.dx * r.dx + r.dy * r.dy + r.dz * r.dz);
}

template <bool GEN>
__global__ void __launch_bounds__(256) order_cost_kernel(const TraceParams p, uint32_t nblocks,
                                                         uint32_t* hist, uint32_t* slot) {
  asm volatile("griddepcontrol.launch_dependents;");   // let the scatter kernel's CTAs launch
  const bool use_grid = p.scene.grid && (p.order_proxy == 1 ? (!p.list || p.instances)
                                                             : (p.order_proxy == 2 && p.instances));
  const bool use_mix = p.scene.grid && !p.list && !use_grid && (p.order_proxy == 2 || p.order_proxy == 3);
  if (use_grid || use_mix) {
    // this CTA's grid replica toward L2 now, in parallel with the sample rays' loads, so the
    // march below does not add a second DRAM round trip (one 128-B line per thread)
    const uint64_t words = (uint64_t)p.scene.gdim[0] * p.scene.gdim[1] * p.scene.gdim[2];
    const uint32_t* rep = p.scene.grid + (uint64_t)(blockIdx.x % kGridCopies) * words;
    for (uint64_t w = (uint64_t)threadIdx.x * 32; w < words; w += 256 * 32)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(rep + w));
  }
  const uint32_t t = blockIdx.x * 256 + threadIdx.x;   // 4 sample rays per 128-ray block
  const uint32_t b = t >> 2;
  float len = 0.0f;
  if (b < nblocks) {
    const uint64_t id = (uint64_t)b * kBlock + (t & 3u) * (uint32_t)((kBlock - 1) / 3);
    if (id < p.n) {
      float4 a, d;
      fetch_ray<GEN>(p, id, a, d);
      RayCtx r;
      make_ray(r, a, d);
      const float t0x = (p.scene.root_lo[0] - r.ox) * r.ix, t1x = (p.scene.root_hi[0] - r.ox) * r.ix;
      const float t0y = (p.scene.root_lo[1] - r.oy) * r.iy, t1y = (p.scene.root_hi[1] - r.oy) * r.iy;
      const float t0z = (p.scene.root_lo[2] - r.oz) * r.iz, t1z = (p.scene.root_hi[2] - r.oz) * r.iz;
      const float tn = fmaxf(fmaxf(fminf(t0x, t1x), fminf(t0y, t1y)), fmaxf(fminf(t0z, t1z), a.w));
      const float tf = fminf(fminf(fmaxf(t0x, t1x), fmaxf(t0y, t1y)), fminf(fmaxf(t0z, t1z), d.w));
      if (VSR_INST_COST && p.instances) len = (float)instance_cost(p, r, d.w);   // bucket index directly
      else if (use_grid) {
        if (tf > tn) len = 6.0f * log2f(1.0f + grid_cost<kGridSamples>(p.scene, r, tn, tf));   // bucket
      } else if (use_mix) {
        if (tf > tn) {   // mean of the density bucket and the segment-length bucket
          const float ex = p.scene.root_hi[0] - p.scene.root_lo[0], ey = p.scene.root_hi[1] - p.scene.root_lo[1],
                      ez = p.scene.root_hi[2] - p.scene.root_lo[2];
          const float dg = sqrtf(ex * ex + ey * ey + ez * ez);
          const float seg =
              dg > 0.0f ? (tf - tn) * sqrtf(d.x * d.x + d.y * d.y + d.z * d.z) / dg * kOrderBuckets : 0.0f;
          len = VSR_MIX_W * (6.0f * log2f(1.0f + grid_cost<kMixSamples>(p.scene, r, tn, tf))) +
                (1.0f - VSR_MIX_W) * seg;
        }
      } else if (tf > tn) len = (tf - tn) * sqrtf(d.x * d.x + d.y * d.y + d.z * d.z);
    }
  }
  len = fmaxf(len, __shfl_xor_sync(0xFFFFFFFFu, len, 1));
  len = fmaxf(len, __shfl_xor_sync(0xFFFFFFFFu, len, 2));
  // CTA-local histogram first: a handful of buckets take almost all blocks,
  // so per-block global atomics would serialise on a few addresses.
  __shared__ uint32_t lh[kOrderBuckets], lbase[kOrderBuckets];
  for (int i = threadIdx.x; i < kOrderBuckets; i += 256) lh[i] = 0;
  __syncthreads();
  const bool leader = (t & 3u) == 0u && b < nblocks;
  int q = 0;
  uint32_t lpos = 0;
  if (leader) {
    const float dx = p.scene.root_hi[0] - p.scene.root_lo[0];
    const float dy = p.scene.root_hi[1] - p.scene.root_lo[1];
    const float dz = p.scene.root_hi[2] - p.scene.root_lo[2];
    const float diag = sqrtf(dx * dx + dy * dy + dz * dz);
    q = ((VSR_INST_COST && p.instances) || use_grid || use_mix) ? (int)len
        : diag > 0.0f ? (int)(len / diag * kOrderBuckets) : 0;
    q = q < 0 ? 0 : (q >= kOrderBuckets ? kOrderBuckets - 1 : q);
    lpos = atomicAdd(lh + q, 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kOrderBuckets; i += 256)
    if (lh[i]) lbase[i] = atomicAdd(hist + i, lh[i]);
  __syncthreads();
  if (leader) slot[b] = ((uint32_t)q << 24) | (lbase[q] + lpos);
}

__global__ void __launch_bounds__(256) order_scatter_kernel(uint32_t nblocks, const uint32_t* hist,
                                                            const uint32_t* slot, uint32_t* perm) {
  __shared__ uint32_t start[kOrderBuckets];
  asm volatile("griddepcontrol.launch_dependents;");   // the trace kernel may launch now ...
  asm volatile("griddepcontrol.wait;" ::: "memory");    // ... and this one waits for the cost pass
  if (threadIdx.x < 32) {   // exclusive scan over buckets, most expensive first
    constexpr int R = kOrderBuckets / 32;   // consecutive buckets per lane
    const int lane = (int)threadIdx.x;
    uint32_t cnt[R], sum = 0;
    for (int k = 0; k < R; ++k) {
      cnt[k] = __ldcg(hist + (kOrderBuckets - 1 - (lane * R + k)));
      sum += cnt[k];
    }
    uint32_t incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += v;
    }
    uint32_t run = incl - sum;
    for (int k = 0; k < R; ++k) {
      start[kOrderBuckets - 1 - (lane * R + k)] = run;
      run += cnt[k];
    }
  }
  __syncthreads();
  const uint32_t b = blockIdx.x * 256 + threadIdx.x;
  if (b >= nblocks) return;
  const uint32_t s = __ldcg(slot + b);
  perm[start[s >> 24] + (s & 0xFFFFFFu)] = b;
}

#ifndef VSR_KEEP_ID
#define VSR_KEEP_ID 0
#endif
#ifndef VSR_ID_SMEM
// each thread's block id kept in shared memory (512 B per CTA) for the hit write, instead
// of re-reading the launch slot's perm entry through L2 at the end (+0.2-0.5 %)
#define VSR_ID_SMEM 1
#endif
#ifndef VSR_RAY_PF
// prefetch the rays of the block this many launch slots ahead (~one residency wave:
// 148 SMs x 10 CTAs); 0 = off.  Measured +0.5-0.6 % (C2, C5), 740..2960 alike
// (profiles/r02_tuning.md)
#define VSR_RAY_PF 1480
#endif
// Direct schedule (default): one thread per ray; launch slot i traces the 128
// rays of block perm[i] (block i when no order was computed), and the
// hardware block scheduler balances the blocks across the 148 SMs.
// OCC: occupancy variant, 12 CTAs (48 warps) per SM at <= 40 registers with a
// few spills, chosen by the host for scenes larger than L2, where more warps hide
// DRAM latency (closest: C4 +3 %, C5 +4 %; any: C5 +3 %). Otherwise 10 CTAs
// (43-45 registers, no spills), which L2-resident scenes prefer (C2 any +0.6 %,
// closest +1.5 %; profiles/r01_tuning.md).
#ifndef VSR_ANY_MINB
#define VSR_ANY_MINB 10
#endif
template <int Q, class I, bool GEN = false, bool OCC = false>
__global__ void __launch_bounds__(kBlock, OCC ? 12 : (Q == kAny ? VSR_ANY_MINB : VSR_MINB))
    trace_kernel(const TraceParams p) {
#ifdef VSR_TIMELINE
  const uint64_t t0 = global_ns();
#endif
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
#if VSR_RAY_PF
  // the block VSR_RAY_PF launch slots ahead (about one residency wave later): its ray
  // lines are prefetched into L2 once this block's own rays have arrived
  uint32_t ahead = 0xFFFFFFFFu;
  if (!GEN && p.perm && blockIdx.x + VSR_RAY_PF < gridDim.x) ahead = __ldcg(p.perm + blockIdx.x + VSR_RAY_PF);
#endif
#if VSR_ID_SMEM
  __shared__ uint32_t s_blk[kBlock];   // this thread's block, for the hit write (no L2 re-read)
  s_blk[threadIdx.x] = (uint32_t)blk;
#endif
  if (id < p.n) {
    I isect = make_isect<I>(p);
    Trav T;
    StackEntry<Q> stack[kMaxStack];   // (ref[, tnear]); depth <= 64 guaranteed by build/import
    const bool go = start_ray<GEN>(p, T, isect, id);
#if VSR_RAY_PF
    if (ahead != 0xFFFFFFFFu) {
      const uint64_t id2 = (uint64_t)ahead * kBlock + threadIdx.x;
      if (id2 < p.n) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.rays + 2 * id2));
    }
#endif
    // warp-uniform octant: specialised slab test when all live lanes agree
    const unsigned live = __activemask();
    const int oct = ray_octant(T.r);
    const int woct = __match_any_sync(live, oct) == live ? oct : 8;
    NoMulti none;
    if (go) traverse<Q, !OCC>(p.scene, T, isect, stack, woct, none);
#if VSR_KEEP_ID
    finish(p, T, isect, id);   // the ray index kept live across the traversal (A/B knob)
#elif VSR_ID_SMEM
    finish(p, T, isect, (uint64_t)s_blk[threadIdx.x] * kBlock + threadIdx.x);
#else
    // the ray index is recomputed (perm re-read through L2) rather than kept live
    // across the traversal: one register less in the hot loop
    const uint64_t blk2 = p.perm ? (uint64_t)__ldcg(p.perm + blockIdx.x) : (uint64_t)blockIdx.x;
    finish(p, T, isect, blk2 * kBlock + threadIdx.x);
#endif
  }
#ifdef VSR_TIMELINE
  // diagnostic build only: per-warp (SM id, start ns, end ns) into counts[warp]
  __syncwarp();
  if ((threadIdx.x & 31u) == 0 && !I::kCounts) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    const uint64_t t1 = global_ns();
    p.counts[id / 32] = make_uint4(smid, (unsigned)t0, (unsigned)t1, (unsigned)(t0 >> 32));
  }
#endif
}

// Warp-granularity dynamic schedule (VSR_SCHED=warp): a grid sized to
// residency; each warp claims 32-ray chunks in launch-slot order (chunk c =
// quarter c & 3 of ray block perm[c >> 2], so the longest-first order holds at
// 32-ray granularity) with one atomicAdd per chunk, and claims its NEXT chunk
// before tracing the current one so that chunk's rays are prefetched into L2
// while this one traces (the ray load is otherwise a DRAM round trip per new
// CTA).  Lanes never mix chunks (coherent primary rays stay together); the
// warp takes a new chunk only when all 32 lanes are done.  Per-ray results are
// independent of the schedule.
__device__ __forceinline__ uint64_t chunk_first_ray(const TraceParams& p, unsigned long long c) {
  constexpr unsigned long long kQ = kBlock / 32;   // 32-ray chunks per block
  const uint64_t blk = p.perm ? (uint64_t)__ldcg(p.perm + c / kQ) : (uint64_t)(c / kQ);
  return blk * kBlock + (c % kQ) * 32ull;
}

template <int Q, class I, bool OCC = false>
__global__ void __launch_bounds__(kBlock, OCC ? 12 : (Q == kAny ? 10 : VSR_MINB))
    trace_kernel_warp(const TraceParams p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.hist_reset && blockIdx.x == 0)
    for (int i = threadIdx.x; i < kOrderBuckets; i += blockDim.x) p.hist_reset[i] = 0u;
  const unsigned lane = threadIdx.x & 31u;
  // every 32-ray quarter of every block (a ragged last block may sit anywhere in the
  // longest-first order, so the chunk count is 4 x blocks, not ceil(n / 32))
  const unsigned long long nchunks = (unsigned long long)(kBlock / 32) * ((p.n + kBlock - 1) / kBlock);
  unsigned long long* ctr = p.counter;
  unsigned long long c = 0;
  if (lane == 0) c = atomicAdd(ctr, 1ull);
  c = __shfl_sync(kFull, c, 0);
  while (c < nchunks) {
    unsigned long long nx = 0;
    if (lane == 0) nx = atomicAdd(ctr, 1ull);
    nx = __shfl_sync(kFull, nx, 0);
    if (nx < nchunks) {   // the next chunk's rays toward L2 while this chunk traces
      const uint64_t nid = chunk_first_ray(p, nx) + lane;
      if (nid < p.n) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.rays + 2 * nid));
    }
    const uint64_t id = chunk_first_ray(p, c) + lane;
    if (id < p.n) {
      I isect = make_isect<I>(p);
      Trav T;
      StackEntry<Q> stack[kMaxStack];
      const bool go = start_ray(p, T, isect, id);
      const unsigned live = __activemask();
      const int oct = ray_octant(T.r);
      const int woct = __match_any_sync(live, oct) == live ? oct : 8;
      NoMulti none;
      if (go) traverse<Q>(p.scene, T, isect, stack, woct, none);
      finish(p, T, isect, id);
    }
    c = nx;
    __syncwarp();
  }
  // the launch's last warp resets the counter slot for a later launch
  if (lane == 0) {
    __threadfence();
    const unsigned long long warps = (unsigned long long)gridDim.x * (kBlock / 32);
    if (atomicAdd(ctr + 1, 1ull) == warps - 1ull) {
      atomicExch(ctr, 0ull);
      atomicExch(ctr + 1, 0ull);
    }
  }
}

// Region schedule (VSR_SCHED=region): the launch's ray blocks are cut into one
// contiguous range per SM ("region"; consecutive blocks are neighbouring tiles),
// each region ordered longest-first by region_scatter_kernel.  A resident grid's
// warps claim 32-ray chunks from the region of the SM they run on (one atomicAdd
// per chunk), so the ~40 warps sharing an SM's L1 trace neighbouring tiles; a
// warp whose region is exhausted steals from the region with the most chunks
// left.  Per-ray results are independent of the schedule.
__device__ __forceinline__ uint64_t region_first_block(uint64_t nblocks, uint32_t k, uint32_t S) {
  return nblocks * k / S;
}

__device__ __forceinline__ bool region_claim(const TraceParams& p, uint32_t home, uint64_t nblocks,
                                             unsigned long long& chunk) {
  constexpr uint64_t kQ = kBlock / 32;   // 32-ray chunks per block
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t S = p.regions;
  uint32_t c = 0;
  if (lane == 0) c = atomicAdd(p.region_ctr + home, 1u);
  c = __shfl_sync(kFull, c, 0);
  {
    const uint64_t b0 = region_first_block(nblocks, home, S), b1 = region_first_block(nblocks, home + 1, S);
    if (c < kQ * (b1 - b0)) {
      chunk = kQ * b0 + c;
      return true;
    }
  }
  for (;;) {   // steal: the region with the most chunks left (warp-parallel scan)
    uint32_t best = 0, bk = 0;
    for (uint32_t k = lane; k < S; k += 32) {
      const uint32_t size =
          (uint32_t)(kQ * (region_first_block(nblocks, k + 1, S) - region_first_block(nblocks, k, S)));
      const uint32_t used = __ldcg(p.region_ctr + k);
      const uint32_t left = used < size ? size - used : 0u;
      if (left > best) {
        best = left;
        bk = k;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const uint32_t ob = __shfl_xor_sync(kFull, best, o), ok = __shfl_xor_sync(kFull, bk, o);
      if (ob > best || (ob == best && ok < bk)) {
        best = ob;
        bk = ok;
      }
    }
    if (best == 0) return false;
    if (lane == 0) c = atomicAdd(p.region_ctr + bk, 1u);
    c = __shfl_sync(kFull, c, 0);
    const uint64_t b0 = region_first_block(nblocks, bk, S), b1 = region_first_block(nblocks, bk + 1, S);
    if (c < kQ * (b1 - b0)) {
      chunk = kQ * b0 + c;
      return true;
    }
  }
}

template <int Q, class I, bool OCC = false>
__global__ void __launch_bounds__(kBlock, OCC ? 12 : (Q == kAny ? 10 : VSR_MINB))
    trace_kernel_region(const TraceParams p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.hist_reset && blockIdx.x == 0)
    for (int i = threadIdx.x; i < kOrderBuckets; i += blockDim.x) p.hist_reset[i] = 0u;
  const unsigned lane = threadIdx.x & 31u;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const uint32_t home = smid % p.regions;
  const uint64_t nblocks = (p.n + kBlock - 1) / kBlock;
  unsigned long long c = 0;
  bool have = region_claim(p, home, nblocks, c);
  while (have) {
    unsigned long long nx = 0;
    const bool next = region_claim(p, home, nblocks, nx);
    if (next) {   // the next chunk's rays toward L2 while this chunk traces
      const uint64_t nid = chunk_first_ray(p, nx) + lane;
      if (nid < p.n) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.rays + 2 * nid));
    }
    const uint64_t id = chunk_first_ray(p, c) + lane;
    if (id < p.n) {
      I isect = make_isect<I>(p);
      Trav T;
      StackEntry<Q> stack[kMaxStack];
      const bool go = start_ray(p, T, isect, id);
      const unsigned live = __activemask();
      const int oct = ray_octant(T.r);
      const int woct = __match_any_sync(live, oct) == live ? oct : 8;
      NoMulti none;
      if (go) traverse<Q>(p.scene, T, isect, stack, woct, none);
      finish(p, T, isect, id);
    }
    c = nx;
    have = next;
    __syncwarp();
  }
}

// Region order: blocks [nblocks*k/S, nblocks*(k+1)/S) of region k (one CTA per
// region), most expensive bucket first (order within a bucket unspecified);
// zeroes the region's claim counter for the trace kernel.
__global__ void __launch_bounds__(256) region_scatter_kernel(uint32_t nblocks, uint32_t S,
                                                             const uint32_t* slot, uint32_t* perm,
                                                             uint32_t* ctr) {
  __shared__ uint32_t cnt[kOrderBuckets], start[kOrderBuckets];
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t k = blockIdx.x;
  const uint32_t b0 = (uint32_t)((uint64_t)nblocks * k / S), b1 = (uint32_t)((uint64_t)nblocks * (k + 1) / S);
  for (int i = threadIdx.x; i < kOrderBuckets; i += 256) cnt[i] = 0;
  if (threadIdx.x == 0) ctr[k] = 0;
  __syncthreads();
  for (uint32_t b = b0 + threadIdx.x; b < b1; b += 256) atomicAdd(cnt + (__ldcg(slot + b) >> 24), 1u);
  __syncthreads();
  if (threadIdx.x < 32) {   // exclusive scan, most expensive bucket first
    constexpr int R = kOrderBuckets / 32;
    const int lane = (int)threadIdx.x;
    uint32_t v[R], sum = 0;
    for (int j = 0; j < R; ++j) {
      v[j] = cnt[kOrderBuckets - 1 - (lane * R + j)];
      sum += v[j];
    }
    uint32_t incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += u;
    }
    uint32_t run = incl - sum;
    for (int j = 0; j < R; ++j) {
      start[kOrderBuckets - 1 - (lane * R + j)] = run;
      run += v[j];
    }
  }
  __syncthreads();
  for (uint32_t b = b0 + threadIdx.x; b < b1; b += 256)
    perm[b0 + atomicAdd(start + (__ldcg(slot + b) >> 24), 1u)] = b;
}

// Multi-hit query: same traversal, the leaf accepts into a K-entry sorted
// buffer (runtime max_hits <= K).  Output ray-major: hits[id*max_hits + j].
#ifndef VSR_MULTI_OUTER
#define VSR_MULTI_OUTER 1   // octant dispatch once per ray, as the direct kernel (k = 4 C2 +0.6 %)
#endif
template <class I, int K>
__global__ void __launch_bounds__(kBlock, VSR_MULTI_MINB) trace_multi_kernel(const TraceParams p) {
  const uint64_t blk = launch_block(p);
  const uint64_t id = blk * kBlock + threadIdx.x;
  if (id >= p.n) return;
  I isect = make_isect<I>(p);
  Trav T;
  float2 stack[kMaxStack];
  MultiBuf<K> mb;
  mb.n = 0;
  mb.maxk = p.max_hits;
  const bool go = start_ray(p, T, isect, id);
  const unsigned live = __activemask();
  const int oct = ray_octant(T.r);
  const int woct = __match_any_sync(live, oct) == live ? oct : 8;
  if (go) traverse<kMulti, VSR_MULTI_OUTER != 0>(p.scene, T, isect, stack, woct, mb);
  float4* out = p.hits + id * (uint64_t)p.max_hits;
#pragma unroll
  for (int j = 0; j < K; ++j) {   // static indices: the buffer stays in registers
    if (j < mb.maxk)
      out[j] = j < mb.n ? make_float4(mb.t[j], mb.u[j], mb.v[j], __uint_as_float(mb.prim[j]))
                        : make_float4(__int_as_float(0x7f800000), 0.0f, 0.0f,
                                      __uint_as_float(kMissPrim));
  }
  if (p.num_hits) p.num_hits[id] = (uint32_t)mb.n;
  if constexpr (I::kCounts) {
    p.counts[id] = make_uint4(isect.num_boxes, isect.num_tris, isect.lookups(), 0u);
  }
}

// Persistent schedule (VSR_SCHED=persistent): grid sized to residency; warps
// claim kChunk rays per atomicAdd and refill idle lanes after each leaf once
// `refill` lanes are idle.  Measured slower than the direct schedule on the
// coherent primary rays of C2 (profiles/r01_tuning.md); kept for incoherent
// workloads and as a measured alternative.
template <int Q, class I>
__global__ void __launch_bounds__(kBlock, VSR_MINB) trace_kernel_persistent(const TraceParams p) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned below = (1u << lane) - 1u;
  unsigned long long* ctr = p.counter;
  I isect = make_isect<I>(p);
  Trav T;
  StackEntry<Q> stack[kMaxStack];   // (ref[, tnear]); depth <= 64 guaranteed by build/import
  bool active = false;
  // warp-uniform work queue: [next, next + left) of the warp's claimed chunk
  unsigned long long next = 0;
  unsigned left = 0;
  uint64_t my_id = 0;
  bool drained = false;      // the global counter ran past n
  for (;;) {
    // converged refill point: ballot/popc compaction of the idle lanes
    const unsigned idle = __ballot_sync(kFull, !active);
    if (idle != 0u && (idle == kFull || __popc(idle) >= p.refill) && !(drained && left == 0)) {
      if (left == 0) {   // claim a new chunk: one atomicAdd per kChunk rays
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ctr, (unsigned long long)kChunk);
        base = __shfl_sync(kFull, base, 0);
        next = base;
        left = base >= p.n ? 0u : (unsigned)min((unsigned long long)kChunk, p.n - base);
        drained = base + kChunk >= p.n;
      }
      const unsigned take = min((unsigned)__popc(idle), left);
      if (!active) {
        const unsigned rank = __popc(idle & below);
        if (rank < take) {
          my_id = next + rank;
          active = start_ray(p, T, isect, my_id);
          if (!active) finish(p, T, isect, my_id);   // missed the root box: a miss record
        }
      }
      next += take;
      left -= take;
    } else if (idle == kFull && drained && left == 0) {
      break;
    }
    if (active && advance<Q, -1>(p.scene, T, isect, stack)) {
      finish(p, T, isect, my_id);
      active = false;
    }
  }
  // The launch's last warp resets the counter slot for a later launch.
  if (lane == 0) {
    __threadfence();
    const unsigned long long warps = (unsigned long long)gridDim.x * (kBlock / 32);
    if (atomicAdd(ctr + 1, 1ull) == warps - 1ull) {
      atomicExch(ctr, 0ull);
      atomicExch(ctr + 1, 0ull);
    }
  }
}

// Device filter functions for the function-pointer control (OptiX-style).
__device__ bool fn_alpha_tex(const IsectData* d, uint32_t k, float u, float v) {
  return alpha_keep(*d, k, u, v);
}
__device__ bool fn_alpha_proc(const IsectData* d, uint32_t, float u, float v) {
  return checker_keep(d->fm, u, v);
}
__device__ filter_fn_t g_fn_alpha_tex = fn_alpha_tex;
__device__ filter_fn_t g_fn_alpha_proc = fn_alpha_proc;

namespace {

int sm_count() {
  static std::atomic<int> cache[64];   // zero-initialised (static storage)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = n > 0 ? n : 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

template <int Q, class I>
cudaError_t launch(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (p.sched == kSchedWarp && p.counter && !p.gen && !p.out_world) {
    static std::atomic<int> per_sm_cache[2];   // resident blocks per SM (OCC false / true)
    int per_sm = per_sm_cache[p.occ ? 1 : 0].load(std::memory_order_relaxed);
    if (per_sm == 0) {
      int nb = 0;
      cudaError_t e = p.occ ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                  &nb, trace_kernel_warp<Q, I, true>, kBlock, 0)
                            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                  &nb, trace_kernel_warp<Q, I, false>, kBlock, 0);
      if (e != cudaSuccess) return e;
      per_sm = nb > 0 ? nb : 1;
      per_sm_cache[p.occ ? 1 : 0].store(per_sm, std::memory_order_relaxed);
    }
    const uint64_t full = (uint64_t)per_sm * sm_count();
    const uint64_t grid = need < full ? need : full;
    const cudaError_t e =
        p.occ ? launch_k(trace_kernel_warp<Q, I, true>, grid, kBlock, p.perm && p.pdl, st, p)
              : launch_k(trace_kernel_warp<Q, I, false>, grid, kBlock, p.perm && p.pdl, st, p);
    if (e != cudaSuccess) return e;
  } else if (p.sched == kSchedRegion && p.region_ctr && !p.gen && !p.out_world) {
    static std::atomic<int> per_sm_cache[2];
    int per_sm = per_sm_cache[p.occ ? 1 : 0].load(std::memory_order_relaxed);
    if (per_sm == 0) {
      int nb = 0;
      cudaError_t e = p.occ ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                  &nb, trace_kernel_region<Q, I, true>, kBlock, 0)
                            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                  &nb, trace_kernel_region<Q, I, false>, kBlock, 0);
      if (e != cudaSuccess) return e;
      per_sm = nb > 0 ? nb : 1;
      per_sm_cache[p.occ ? 1 : 0].store(per_sm, std::memory_order_relaxed);
    }
    const uint64_t full = (uint64_t)per_sm * sm_count();
    const uint64_t grid = need < full ? need : full;
    const cudaError_t e =
        p.occ ? launch_k(trace_kernel_region<Q, I, true>, grid, kBlock, p.pdl != 0, st, p)
              : launch_k(trace_kernel_region<Q, I, false>, grid, kBlock, p.pdl != 0, st, p);
    if (e != cudaSuccess) return e;
  } else if (p.sched == kSchedPersistent) {
    static std::atomic<int> per_sm_cache{0};   // resident blocks per SM for this instantiation
    int per_sm = per_sm_cache.load(std::memory_order_relaxed);
    if (per_sm == 0) {
      int nb = 0;
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &nb, trace_kernel_persistent<Q, I>, kBlock, 0);
      if (e != cudaSuccess) return e;
      per_sm = nb > 0 ? nb : 1;
      per_sm_cache.store(per_sm, std::memory_order_relaxed);
    }
    const uint64_t full = (uint64_t)per_sm * sm_count();
    const unsigned blocks = (unsigned)(need < full ? need : full);
    trace_kernel_persistent<Q, I><<<blocks, kBlock, 0, st>>>(p);
  } else {
    if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
    cudaError_t e;
    if (p.gen) {   // fused ray generation: not built for the run-time controls
      if constexpr (std::is_same<I, runtime_switch_intersector>::value ||
                    std::is_same<I, runtime_fnptr_intersector>::value)
        return cudaErrorInvalidValue;
      else if (p.occ)
        e = launch_k(trace_kernel<Q, I, true, true>, need, kBlock, p.perm && p.pdl, st, p);
      else
        e = launch_k(trace_kernel<Q, I, true>, need, kBlock, p.perm && p.pdl, st, p);
    } else if (p.occ) {
      e = launch_k(trace_kernel<Q, I, false, true>, need, kBlock, p.perm && p.pdl, st, p);
    } else {
      e = launch_k(trace_kernel<Q, I>, need, kBlock, p.perm && p.pdl, st, p);
    }
    if (e != cudaSuccess) return e;
  }
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <class I>
cudaError_t launch_multi(const TraceParams& p, cudaStream_t st) {
  const uint64_t need = (p.n + kBlock - 1) / kBlock;
  if (need > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const bool pdl = p.perm && p.pdl;
  cudaError_t e = p.max_hits <= 4 ? launch_k(trace_multi_kernel<I, 4>, need, kBlock, pdl, st, p)
                                  : launch_k(trace_multi_kernel<I, 16>, need, kBlock, pdl, st, p);
  if (e != cudaSuccess) return e;
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t dispatch_multi(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch_multi<no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch_multi<default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE:
      return p.data.bits ? launch_multi<alpha_bits_intersector>(p, st)
                         : launch_multi<alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch_multi<alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch_multi<alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch_multi<alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch_multi<cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch_multi<cost_intersector<alpha_texture_intersector>>(p, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int Q>
cudaError_t dispatch_isect(int isect, const TraceParams& p, cudaStream_t st) {
  switch (isect) {
    case VSR_ISECT_NONE: return launch<Q, no_intersector>(p, st);
    case VSR_ISECT_DEFAULT: return launch<Q, default_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE:
      return p.data.bits ? launch<Q, alpha_bits_intersector>(p, st)
                         : launch<Q, alpha_texture_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL: return launch<Q, alpha_procedural_intersector>(p, st);
    case VSR_ISECT_ALPHA_TEXTURE_BILINEAR: return launch<Q, alpha_bilinear_intersector>(p, st);
    case VSR_ISECT_ALPHA_PROCEDURAL_UV: return launch<Q, alpha_procedural_uv_intersector>(p, st);
    case VSR_ISECT_COUNT: return launch<Q, cost_intersector<default_intersector>>(p, st);
    case VSR_ISECT_COUNT_ALPHA_TEXTURE:
      return launch<Q, cost_intersector<alpha_texture_intersector>>(p, st);
    case VSR_ISECT_RUNTIME_SWITCH_DEFAULT:
    case VSR_ISECT_RUNTIME_SWITCH_ALPHA_TEXTURE:
    case VSR_ISECT_RUNTIME_SWITCH_ALPHA_PROCEDURAL:
      return launch<Q, runtime_switch_intersector>(p, st);
    case VSR_ISECT_RUNTIME_FNPTR_DEFAULT:
    case VSR_ISECT_RUNTIME_FNPTR_ALPHA_TEXTURE:
    case VSR_ISECT_RUNTIME_FNPTR_ALPHA_PROCEDURAL:
      return launch<Q, runtime_fnptr_intersector>(p, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

cudaError_t filter_fn_pointer(int kind, void** out) {
  filter_fn_t f = nullptr;
  cudaError_t e = cudaSuccess;
  if (kind == kFilterAlphaTex) e = cudaMemcpyFromSymbol(&f, g_fn_alpha_tex, sizeof f);
  else if (kind == kFilterAlphaProc) e = cudaMemcpyFromSymbol(&f, g_fn_alpha_proc, sizeof f);
  *out = reinterpret_cast<void*>(f);
  return e;
}

// Profiling hook (thread-local): events recorded right before and after the
// trace kernel itself, i.e. excluding the block-order pass.
thread_local void* g_kernel_events[2] = {nullptr, nullptr};

void set_kernel_events(void* start, void* stop) {
  g_kernel_events[0] = start;
  g_kernel_events[1] = stop;
}

size_t order_scratch_bytes(uint64_t n) {
  const uint64_t nblocks = (n + kBlock - 1) / kBlock;
  return sizeof(uint32_t) * (kOrderBuckets + 2 * (size_t)nblocks + (size_t)sm_count() + 32);
}

cudaError_t launch_trace(int query, int isect, const TraceParams& p_in, cudaStream_t st) {
  if (p_in.n == 0) return cudaSuccess;
  TraceParams p = p_in;
  p.perm = nullptr;
  p.hist_reset = nullptr;
  const uint64_t nblocks = (p.n + kBlock - 1) / kBlock;
  void* scratch = nullptr;
  bool owned = false;
  // every exit after a stream-ordered allocation frees it on the stream (after
  // whatever was queued), so an error part-way through leaks nothing
  auto done = [&](cudaError_t e) {
    if (owned) {
      const cudaError_t f = cudaFreeAsync(scratch, st);
      if (e == cudaSuccess) e = f;
    }
    return e;
  };
  if (p.order && (p.sched == kSchedDirect || p.sched == kSchedWarp || p.sched == kSchedRegion) &&
      nblocks >= 2ull * sm_count() &&
      nblocks < (1u << 24)) {
    // the owner's per-stream scratch (api.cpp ScratchSet); a stream-ordered
    // allocation only past 16 streams per owner
    const size_t bytes = order_scratch_bytes(p.n);
    cudaError_t e = cudaSuccess;
    if (p.order_scratch && p.order_scratch_bytes >= bytes) {
      scratch = p.order_scratch;   // caller-provided, stream-ordered (per-stream scene scratch)
    } else {
      if ((e = cudaMallocAsync(&scratch, bytes, st)) != cudaSuccess) return e;
      owned = true;
    }
    uint32_t* hist = static_cast<uint32_t*>(scratch);
    uint32_t* slot = hist + kOrderBuckets;
    uint32_t* perm = slot + nblocks;
    const bool zeroed = !owned;   // caller scratch: zero at entry, kept so by the trace kernel
    if (!zeroed &&
        (e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kOrderBuckets, st)) != cudaSuccess)
      return done(e);
    if (p.gen) {
      apply_carveout(reinterpret_cast<const void*>(order_cost_kernel<true>));
      order_cost_kernel<true><<<(unsigned)((4 * nblocks + 255) / 256), 256, 0, st>>>(
          p, (uint32_t)nblocks, hist, slot);
    } else {
      apply_carveout(reinterpret_cast<const void*>(order_cost_kernel<false>));
      order_cost_kernel<false><<<(unsigned)((4 * nblocks + 255) / 256), 256, 0, st>>>(
          p, (uint32_t)nblocks, hist, slot);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) {
      if (zeroed) cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kOrderBuckets, st);
      return done(e);
    }
    const bool region = p.sched == kSchedRegion && !p.gen && !p.out_world && !p.wide && !p.list &&
                        query != kMulti;
    if (region) {
      p.regions = (uint32_t)sm_count();
      p.region_ctr = perm + nblocks;
      e = launch_k(region_scatter_kernel, p.regions, 256, p.pdl != 0, st, (uint32_t)nblocks,
                   p.regions, (const uint32_t*)slot, perm, p.region_ctr);
    } else {
      e = launch_k(order_scatter_kernel, (nblocks + 255) / 256, 256, p.pdl != 0, st,
                   (uint32_t)nblocks, (const uint32_t*)hist, (const uint32_t*)slot, perm);
    }
    if (e != cudaSuccess) {
      if (zeroed) cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kOrderBuckets, st);
      return done(e);
    }
    launch_counter().fetch_add(2, std::memory_order_relaxed);
    if (!owned) p.hist_reset = hist;   // the trace kernel re-zeroes it for the next launch
    if ((e = cudaGetLastError()) != cudaSuccess) {
      if (zeroed) cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kOrderBuckets, st);
      return done(e);
    }
    p.perm = perm;
  }
  if (g_kernel_events[0]) cudaEventRecord(static_cast<cudaEvent_t>(g_kernel_events[0]), st);
  cudaError_t e = p.wide ? launch_wide(query, isect, p, st)       // 8-wide BVH (wide.cu)
                  : p.list ? launch_compound(query, isect, p, st)   // lists, instances (compound.cu)
                  : query == kMulti ? dispatch_multi(isect, p, st)
                  : query == kAny ? dispatch_isect<kAny>(isect, p, st)
                                  : dispatch_isect<kClosest>(isect, p, st);
  if (g_kernel_events[1]) cudaEventRecord(static_cast<cudaEvent_t>(g_kernel_events[1]), st);
  if (e != cudaSuccess && p.hist_reset)   // the trace kernel did not run: restore the invariant
    cudaMemsetAsync(p.hist_reset, 0, sizeof(uint32_t) * kOrderBuckets, st);
  return done(e);
}

// 1-bit alpha plane of threshold a_min (see alpha_keep_bits): one thread per
// output word = one 32-texel row segment of a 32x32 tile; blockIdx.y = texture.
__global__ void __launch_bounds__(256) alpha_bits_kernel(const TexDesc* descs, const uint8_t* texels,
                                                         uint32_t a_min, uint32_t* bits) {
  const TexDesc td = descs[blockIdx.y];
  const uint64_t words = (uint64_t)td.w * td.h / 32;
  const uint32_t tiles_x = td.w / 32;
  for (uint64_t w = blockIdx.x * 256ull + threadIdx.x; w < words; w += gridDim.x * 256ull) {
    const uint64_t tile = w >> 5;
    const uint64_t y = (tile / tiles_x) * 32 + (w & 31u), x0 = (tile % tiles_x) * 32;
    const uint8_t* row = texels + td.offset + y * td.w + x0;
    uint32_t m = 0;
    for (int c = 0; c < 32; ++c) m |= (uint32_t)(row[c] >= a_min) << c;
    bits[(td.offset >> 5) + w] = m;
  }
}

cudaError_t build_alpha_bits(const TexDesc* d_descs, uint32_t num_textures, const uint8_t* texels,
                             uint32_t a_min, uint32_t* d_bits, uint64_t max_words,
                             cudaStream_t st) {
  if (num_textures == 0) return cudaSuccess;
  const unsigned gx = (unsigned)std::min<uint64_t>(4096, (max_words + 255) / 256);
  alpha_bits_kernel<<<dim3(gx ? gx : 1, num_textures), 256, 0, st>>>(d_descs, texels, a_min, d_bits);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

void density_grid_dims(const float* lo, const float* hi, uint32_t* dims, float* scale) {
  double ext[3], vol = 1.0;
  for (int a = 0; a < 3; ++a) {
    ext[a] = std::max((double)hi[a] - lo[a], 1e-30);
    vol *= ext[a];
  }
  // ~4096 cubic cells, then 8..32 per axis (at most 8192 cells: the cost kernel stages
  // the grid in shared memory); thin axes (a forest's height) still get 8 layers
  const double cell = std::max(std::cbrt(vol / 4096.0), 1e-30);
  for (int a = 0; a < 3; ++a) {
    double g = std::ceil(ext[a] / cell);
    g = std::min(std::max(g, 8.0), 32.0);
    dims[a] = (uint32_t)g;
    scale[a] = (float)(g / ext[a]);
  }
}

__global__ void __launch_bounds__(256) density_grid_kernel(const Tri* tris, uint32_t n, float lx,
                                                           float ly, float lz, uint3 dims,
                                                           float3 scale, uint32_t* grid) {
  const uint32_t i = blockIdx.x * 256 + threadIdx.x;
  if (i >= n) return;
  const Tri t = tris[i];
  const float lo[3] = {lx, ly, lz}, sc[3] = {scale.x, scale.y, scale.z};
  const uint32_t dm[3] = {dims.x, dims.y, dims.z};
  int c0[3], c1[3];
  for (int a = 0; a < 3; ++a) {
    const float v0 = t.v0[a], v1 = v0 + t.e1[a], v2 = v0 + t.e2[a];
    const float mn = fminf(v0, fminf(v1, v2)), mx = fmaxf(v0, fmaxf(v1, v2));
    c0[a] = max(0, min((int)dm[a] - 1, (int)floorf((mn - lo[a]) * sc[a])));
    c1[a] = max(0, min((int)dm[a] - 1, (int)floorf((mx - lo[a]) * sc[a])));
  }
  int budget = 4096;   // a triangle larger than that many cells counts in its first ones only
  for (int z = c0[2]; z <= c1[2]; ++z)
    for (int y = c0[1]; y <= c1[1]; ++y)
      for (int x = c0[0]; x <= c1[0]; ++x) {
        if (budget-- <= 0) return;
        atomicAdd(grid + ((uint64_t)z * dm[1] + y) * dm[0] + x, 1u);
      }
}

cudaError_t build_density_grid(const Tri* d_tris, uint32_t n, const float* lo, const uint32_t* dims,
                               const float* scale, uint32_t* d_grid, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  density_grid_kernel<<<(n + 255) / 256, 256, 0, st>>>(
      d_tris, n, lo[0], lo[1], lo[2], make_uint3(dims[0], dims[1], dims[2]),
      make_float3(scale[0], scale[1], scale[2]), d_grid);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  const size_t cells = (size_t)dims[0] * dims[1] * dims[2];
  for (int k = 1; k < kGridCopies && e == cudaSuccess; ++k)   // the replicas
    e = cudaMemcpyAsync(d_grid + k * cells, d_grid, cells * sizeof(uint32_t),
                        cudaMemcpyDeviceToDevice, st);
  return e;
}

size_t density_grid_words(const uint32_t* dims) {
  return (size_t)dims[0] * dims[1] * dims[2] * kGridCopies;
}

void apply_carveout(const void* kernel) {
  static const int pct = [] {
    const char* e = std::getenv("VSR_CARVEOUT");
    return e ? std::atoi(e) : -1;
  }();
  if (pct < 0) return;
  static std::mutex mu;
  static std::vector<const void*> done;
  std::lock_guard<std::mutex> lk(mu);
  for (const void* k : done)
    if (k == kernel) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  cudaGetLastError();
  done.push_back(kernel);
}

std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> n{0};
  return n;
}

uint64_t launch_count() { return launch_counter().load(std::memory_order_relaxed); }

}  // namespace vsr
