// lt_bvh_gpu.cu -- the reference's binned-SAH BVH build (build_bvh,
// bvh.py:286-298 -> _triangle_bounds_arrays bvh.py:57-77 -> _build_kernel
// bvh.py:85-262) on the GPU, returning the same arrays as the reference and
// as the host restatement lt_build_bvh (lt_bvh_build.cpp).
//
// Why the result can be identical although the GPU does not follow the
// reference's sequential depth-first loop:
//  * every decision of a node (leaf test, split axis, bin of each member,
//    SAH sweep, split plane) depends on the SET of member triangles, not on
//    their order: bin counts are integers and bounds are min / max, both
//    exact under any association.  The float64 arithmetic is the reference's
//    term by term, and this file is compiled with -fmad=false so nothing is
//    contracted into an FMA;
//  * a child's bounds are the union of the parent's bins on its side (the
//    reference recomputes them by scanning the members: the same min / max);
//  * the order of triangles inside a node's range after a split is the
//    result of the reference's in-place two-pointer partition, which has a
//    closed form (proved by exhaustive comparison, tests/test_bvh_gpu.py):
//    with L lefts, front stream F = range[0, L), back stream B = range
//    reversed from the end, X = rights in F, beta_j = back position of the
//    j-th left in B (1-based) and last = beta_X:
//      - F[k] left            -> k
//      - F[k] the j-th right  -> slot k receives the j-th B-left; F[k] goes
//                                to c - 1 - beta_{j-1} (beta_0 = 0)
//      - B right at back position p (range index c - p):
//                                p < last -> c - 1 - p; else index L -> c-1-last,
//                                others shift down by one;
//    so one prefix sum of the left flags per level yields the permutation;
//  * node numbering: the reference allocates the two children of the k-th
//    internal node it pops (depth first, left child first) as ids 2k+1,
//    2k+2; the GPU uses provisional ids and the host replays that order over
//    the finished tree (O(nodes), no geometry).
// The only representable difference: a bound whose extreme value is zero
// with both +0.0 and -0.0 among the members keeps whichever sign the
// sequential scan met first in the reference and the ordered-integer minimum
// here; the values compare equal.
//
// Structure: nodes larger than kSmall (512) are processed level by level by
// the whole GPU (block-privatised bins -> one thread per node SAH ->
// scan-based partition); every smaller subtree is built depth first by one
// 64-thread CTA in shared memory (small CTAs: many subtrees in flight hide
// the per-node barrier / serial-SAH latency; profiles/r01_bvh_variants.log).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <vector>

#include "lt_internal.h"

namespace {

constexpr double kBoundsPadding = 1e-7;  // geometry.py:19
constexpr double kTraversalCost = 1.0;   // bvh.py:24
constexpr double kIntersectCost = 1.0;   // bvh.py:25
constexpr int kDepthCap = 60;            // bvh.py:26
constexpr int kMaxBins = 32;
#ifndef LT_BVH_SMALL
#define LT_BVH_SMALL 512
#endif
#ifndef LT_BVH_SMALL_THREADS
#define LT_BVH_SMALL_THREADS 64
#endif
constexpr int kSmall = LT_BVH_SMALL;      // subtrees up to this size: one CTA each
constexpr int kThreads = 256;
constexpr int kSmallThreads = LT_BVH_SMALL_THREADS;  // CTA width of the subtree kernel
constexpr int kChunk = 4096;             // positions per binning CTA (large nodes)
constexpr unsigned long long kMsb = 0x8000000000000000ull;

enum : int32_t { ST_LEAF = 0, ST_BIN = 1, ST_MEDIAN = 2 };

// A node to process: its range of the order array, depth and the bounds of
// its members (triangle boxes and centroids).
struct Job {
  double lo[3], hi[3], clo[3], chi[3];
  int32_t id, f, c, depth;
};

// Per-level state of a large node.
struct NodeState {
  int32_t state, axis, plane, L;
  double cmin, scale;
  Job kid[2];
};

struct Counters {
  int32_t nodes;       // provisional ids handed out (root = 0)
  int32_t leaves;
  int32_t max_depth;
  int32_t n_next;      // large jobs of the next level
  int32_t n_small;     // subtree jobs
  int32_t error;       // internal consistency failure
};

// doubles as order-preserving unsigned integers (atomicMin / atomicMax)
__device__ __forceinline__ unsigned long long ord_of(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & kMsb) ? ~b : (b | kMsb);
}
__device__ __forceinline__ double val_of(unsigned long long k) {
  const unsigned long long b = (k & kMsb) ? (k & ~kMsb) : ~k;
  return __longlong_as_double((long long)b);
}

__host__ __device__ __forceinline__ double area2(const double *lo, const double *hi) {
  const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  return 2.0 * (dx * dy + dx * dz + dy * dz);  // 2 * _half_area (bvh.py:80-82)
}

// per-triangle record: tb_min[3], tb_max[3], cent[3] (bvh.py:57-77)
__global__ void k_tri_bounds(const double *__restrict__ v0, const double *__restrict__ v1,
                             const double *__restrict__ v2, int64_t n, double *__restrict__ tb) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double lo[3], hi[3], ext = 0.0;
  for (int a = 0; a < 3; ++a) {
    const double x0 = v0[3 * i + a], x1 = v1[3 * i + a], x2 = v2[3 * i + a];
    // Python min / max keep the first argument unless the second is strictly
    // smaller / larger
    const double m12 = x2 < x1 ? x2 : x1;
    lo[a] = m12 < x0 ? m12 : x0;
    const double M12 = x2 > x1 ? x2 : x1;
    hi[a] = M12 > x0 ? M12 : x0;
    if (hi[a] - lo[a] > ext) ext = hi[a] - lo[a];
  }
  const double pad = kBoundsPadding * ext;
  double *o = tb + 9 * i;
  for (int a = 0; a < 3; ++a) {
    const double l = lo[a] - pad, h = hi[a] + pad;
    o[a] = l;
    o[3 + a] = h;
    o[6 + a] = 0.5 * (l + h);
  }
}

// ---------------------------------------------------------------- bins

// 12 ordered values per bin: tb lo[3] (min), tb hi[3] (max), centroid
// lo[3] (min), centroid hi[3] (max); plus a count.
__device__ __forceinline__ void bin_reset(unsigned long long *v) {
  for (int q = 0; q < 12; ++q) v[q] = (q < 3 || (q >= 6 && q < 9)) ? ~0ull : 0ull;
}

__device__ __forceinline__ void bin_add(unsigned long long *v, unsigned int *cnt,
                                        const double *t) {
  atomicAdd(cnt, 1u);
  for (int a = 0; a < 3; ++a) {
    atomicMin(&v[a], ord_of(t[a]));
    atomicMax(&v[3 + a], ord_of(t[3 + a]));
    atomicMin(&v[6 + a], ord_of(t[6 + a]));
    atomicMax(&v[9 + a], ord_of(t[6 + a]));
  }
}

__device__ __forceinline__ int bin_of(const double *t, int axis, double cmin, double scale,
                                      int n_bins) {
  const long long b = (long long)((t[6 + axis] - cmin) * scale);
  return b >= n_bins ? n_bins - 1 : (int)b;
}

// Leaf test, split axis and bin scale of a node (bvh.py:118-175).
__device__ void classify(const Job &j, int leaf_size, int n_bins, int &state, int &axis,
                         double &cmin, double &scale) {
  const double parent_area = area2(j.lo, j.hi);
  if (j.c <= leaf_size || j.depth >= kDepthCap || parent_area <= 0.0) {
    state = ST_LEAF;
    return;
  }
  const double ex = j.chi[0] - j.clo[0], ey = j.chi[1] - j.clo[1], ez = j.chi[2] - j.clo[2];
  axis = 0;
  double ext = ex;
  if (ey > ext) {
    axis = 1;
    ext = ey;
  }
  if (ez > ext) {
    axis = 2;
    ext = ez;
  }
  cmin = j.clo[axis];
  if (ext > 0.0) {
    state = ST_BIN;
    scale = (double)n_bins / ext;
  } else {
    state = ST_MEDIAN;
  }
}

// SAH sweep over the bins (bvh.py:177-240), exactly the reference's float64
// operations; returns the split plane or -1 (leaf), the left count and the
// two children's bounds (unions of the bins on each side).
__device__ int sah_split(const unsigned long long *bins, const unsigned int *cnt, int n_bins,
                         const Job &j, Job &kl, Job &kr, int &L) {
  const double parent_area = area2(j.lo, j.hi);
  double sweep_area[kMaxBins];
  long long sweep_count[kMaxBins];
  double acc_lo[3], acc_hi[3];
  for (int a = 0; a < 3; ++a) {
    acc_lo[a] = INFINITY;
    acc_hi[a] = -INFINITY;
  }
  long long acc_n = 0;
  for (int b = 0; b < n_bins - 1; ++b) {
    if (cnt[b] > 0) {
      for (int a = 0; a < 3; ++a) {
        const double l = val_of(bins[12 * b + a]), h = val_of(bins[12 * b + 3 + a]);
        if (l < acc_lo[a]) acc_lo[a] = l;
        if (h > acc_hi[a]) acc_hi[a] = h;
      }
      acc_n += cnt[b];
    }
    sweep_count[b] = acc_n;
    sweep_area[b] = acc_n > 0 ? area2(acc_lo, acc_hi) : 0.0;
  }
  double best_cost = INFINITY;
  int best_plane = -1;
  for (int a = 0; a < 3; ++a) {
    acc_lo[a] = INFINITY;
    acc_hi[a] = -INFINITY;
  }
  acc_n = 0;
  for (int b = n_bins - 1; b > 0; --b) {
    if (cnt[b] > 0) {
      for (int a = 0; a < 3; ++a) {
        const double l = val_of(bins[12 * b + a]), h = val_of(bins[12 * b + 3 + a]);
        if (l < acc_lo[a]) acc_lo[a] = l;
        if (h > acc_hi[a]) acc_hi[a] = h;
      }
      acc_n += cnt[b];
    }
    const int plane = b - 1;
    const long long ln = sweep_count[plane], rn = acc_n;
    if (ln > 0 && rn > 0) {
      const double right_area = area2(acc_lo, acc_hi);
      const double cost = kTraversalCost + kIntersectCost *
                                               (sweep_area[plane] * (double)ln +
                                                right_area * (double)rn) /
                                               parent_area;
      if (cost < best_cost) {
        best_cost = cost;
        best_plane = plane;
      }
    }
  }
  if (!(best_plane >= 0 && best_cost < kIntersectCost * (double)j.c)) return -1;
  // children: unions of the bins on each side
  for (int a = 0; a < 3; ++a) {
    kl.lo[a] = kr.lo[a] = kl.clo[a] = kr.clo[a] = INFINITY;
    kl.hi[a] = kr.hi[a] = kl.chi[a] = kr.chi[a] = -INFINITY;
  }
  L = 0;
  for (int b = 0; b < n_bins; ++b) {
    if (cnt[b] == 0) continue;
    Job &k = b <= best_plane ? kl : kr;
    if (b <= best_plane) L += (int)cnt[b];
    for (int a = 0; a < 3; ++a) {
      const double l = val_of(bins[12 * b + a]), h = val_of(bins[12 * b + 3 + a]);
      const double cl = val_of(bins[12 * b + 6 + a]), ch = val_of(bins[12 * b + 9 + a]);
      if (l < k.lo[a]) k.lo[a] = l;
      if (h > k.hi[a]) k.hi[a] = h;
      if (cl < k.clo[a]) k.clo[a] = cl;
      if (ch > k.chi[a]) k.chi[a] = ch;
    }
  }
  return best_plane;
}

__device__ void set_children(Job &kl, Job &kr, const Job &j, int L) {
  kl.f = j.f;
  kl.c = L;
  kr.f = j.f + L;
  kr.c = j.c - L;
  kl.depth = kr.depth = j.depth + 1;
}

// Destination (range-relative) of the element at range index k in the
// reference's two-pointer partition, given the flags' exclusive prefix
// (pre(k) = lefts in [0, k)) and the back-left positions beta[] (see the
// header).  Returns -1 for back-lefts (written by their front partner).
struct PartInfo {
  int c, L, last;
};

// ---------------------------------------------------------------- tree

struct Tree {
  double *bmin, *bmax;
  int32_t *left, *right, *first, *count;
};

__device__ void emit_leaf(const Tree &t, const Job &j, Counters *ctr) {
  t.first[j.id] = j.f;
  t.count[j.id] = j.c;
  atomicAdd(&ctr->leaves, 1);
}

__device__ void emit_bounds(const Tree &t, const Job &j, Counters *ctr) {
  for (int a = 0; a < 3; ++a) {
    t.bmin[3 * (int64_t)j.id + a] = j.lo[a];
    t.bmax[3 * (int64_t)j.id + a] = j.hi[a];
  }
  atomicMax(&ctr->max_depth, j.depth);
}

// ---------------------------------------------------------------- root

__global__ void k_root_reduce(const double *__restrict__ tb, int64_t n,
                              unsigned long long *__restrict__ acc) {
  double v[12];
  for (int a = 0; a < 3; ++a) {
    v[a] = v[6 + a] = INFINITY;
    v[3 + a] = v[9 + a] = -INFINITY;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double *t = tb + 9 * i;
    for (int a = 0; a < 3; ++a) {
      if (t[a] < v[a]) v[a] = t[a];
      if (t[3 + a] > v[3 + a]) v[3 + a] = t[3 + a];
      if (t[6 + a] < v[6 + a]) v[6 + a] = t[6 + a];
      if (t[6 + a] > v[9 + a]) v[9 + a] = t[6 + a];
    }
  }
  for (int q = 0; q < 12; ++q) {
    const bool is_min = q < 3 || (q >= 6 && q < 9);
    unsigned long long k = ord_of(v[q]);
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, off);
      k = is_min ? (o < k ? o : k) : (o > k ? o : k);
    }
    if ((threadIdx.x & 31) == 0) {
      if (is_min) atomicMin(&acc[q], k);
      else atomicMax(&acc[q], k);
    }
  }
}

__global__ void k_root_job(const unsigned long long *__restrict__ acc, int64_t n, Job *large,
                           Job *small, Counters *ctr) {
  Job j;
  for (int a = 0; a < 3; ++a) {
    j.lo[a] = val_of(acc[a]);
    j.hi[a] = val_of(acc[3 + a]);
    j.clo[a] = val_of(acc[6 + a]);
    j.chi[a] = val_of(acc[9 + a]);
  }
  j.id = 0;
  j.f = 0;
  j.c = (int32_t)n;
  j.depth = 0;
  ctr->nodes = 1;
  if (n > kSmall) {
    large[0] = j;
    ctr->n_next = 1;
  } else {
    small[0] = j;
    ctr->n_small = 1;
  }
}

// ---------------------------------------------------------------- levels

__global__ void k_prepare(const Job *__restrict__ jobs, int m, int leaf_size, int n_bins,
                          NodeState *__restrict__ st, Tree t, Counters *ctr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const Job j = jobs[i];
  emit_bounds(t, j, ctr);
  NodeState s;
  s.plane = -1;
  s.L = 0;
  s.axis = 0;
  s.cmin = 0.0;
  s.scale = 0.0;
  classify(j, leaf_size, n_bins, s.state, s.axis, s.cmin, s.scale);
  if (s.state == ST_LEAF) emit_leaf(t, j, ctr);
  st[i] = s;
}

__global__ void k_bins_reset(unsigned long long *__restrict__ bins, unsigned int *__restrict__ cnt,
                             int total_bins) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total_bins) return;
  bin_reset(bins + 12 * (int64_t)i);
  cnt[i] = 0;
}

// chunk = (job index, first position, count)
__global__ void __launch_bounds__(kThreads) k_bin_large(
    const int4 *__restrict__ chunks, const Job *__restrict__ jobs,
    const NodeState *__restrict__ st, const int32_t *__restrict__ order,
    const double *__restrict__ tb, int n_bins, unsigned long long *__restrict__ gbins,
    unsigned int *__restrict__ gcnt) {
  __shared__ unsigned long long s_bins[kMaxBins * 12];
  __shared__ unsigned int s_cnt[kMaxBins];
  const int4 ch = chunks[blockIdx.x];
  const NodeState s = st[ch.x];
  for (int q = threadIdx.x; q < n_bins * 12; q += blockDim.x) {
    const int r = q % 12;
    s_bins[q] = (r < 3 || (r >= 6 && r < 9)) ? ~0ull : 0ull;
  }
  for (int b = threadIdx.x; b < n_bins; b += blockDim.x) s_cnt[b] = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < ch.z; k += blockDim.x) {
    const double *t = tb + 9 * (int64_t)order[ch.y + k];
    const int b = bin_of(t, s.axis, s.cmin, s.scale, n_bins);
    bin_add(s_bins + 12 * b, s_cnt + b, t);
  }
  __syncthreads();
  unsigned long long *gb = gbins + (int64_t)ch.x * kMaxBins * 12;
  unsigned int *gc = gcnt + (int64_t)ch.x * kMaxBins;
  for (int q = threadIdx.x; q < n_bins * 12; q += blockDim.x) {
    const int b = q / 12, r = q % 12;
    if (s_cnt[b] == 0) continue;
    if (r < 3 || (r >= 6 && r < 9)) atomicMin(&gb[q], s_bins[q]);
    else atomicMax(&gb[q], s_bins[q]);
  }
  for (int b = threadIdx.x; b < n_bins; b += blockDim.x)
    if (s_cnt[b]) atomicAdd(&gc[b], s_cnt[b]);
}

__global__ void k_sah_large(const Job *__restrict__ jobs, int m, int n_bins,
                            const unsigned long long *__restrict__ gbins,
                            const unsigned int *__restrict__ gcnt, NodeState *__restrict__ st,
                            Tree t, Counters *ctr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || st[i].state != ST_BIN) return;
  const Job j = jobs[i];
  NodeState &s = st[i];
  int L = 0;
  const int plane = sah_split(gbins + (int64_t)i * kMaxBins * 12, gcnt + (int64_t)i * kMaxBins,
                              n_bins, j, s.kid[0], s.kid[1], L);
  if (plane < 0) {
    s.state = ST_LEAF;  // SAH prefers a leaf (bvh.py:239)
    emit_leaf(t, j, ctr);
    return;
  }
  s.plane = plane;
  s.L = L;
  set_children(s.kid[0], s.kid[1], j, L);
}

// coincident centroids: median split of the range (bvh.py:241-243); the
// children's bounds are reductions over each half (one CTA per node)
__device__ void reduce_range_bounds(const int32_t *__restrict__ order,
                                    const double *__restrict__ tb, int f, int c, Job &out,
                                    unsigned long long *s_acc) {
  for (int q = threadIdx.x; q < 12; q += blockDim.x)
    s_acc[q] = (q < 3 || (q >= 6 && q < 9)) ? ~0ull : 0ull;
  __syncthreads();
  for (int k = threadIdx.x; k < c; k += blockDim.x) {
    const double *t = tb + 9 * (int64_t)order[f + k];
    for (int a = 0; a < 3; ++a) {
      atomicMin(&s_acc[a], ord_of(t[a]));
      atomicMax(&s_acc[3 + a], ord_of(t[3 + a]));
      atomicMin(&s_acc[6 + a], ord_of(t[6 + a]));
      atomicMax(&s_acc[9 + a], ord_of(t[6 + a]));
    }
  }
  __syncthreads();
  for (int a = 0; a < 3; ++a) {
    out.lo[a] = val_of(s_acc[a]);
    out.hi[a] = val_of(s_acc[3 + a]);
    out.clo[a] = val_of(s_acc[6 + a]);
    out.chi[a] = val_of(s_acc[9 + a]);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) k_median_large(const Job *__restrict__ jobs,
                                                           NodeState *__restrict__ st,
                                                           const int32_t *__restrict__ order,
                                                           const double *__restrict__ tb) {
  __shared__ unsigned long long s_acc[12];
  const int i = blockIdx.x;
  if (st[i].state != ST_MEDIAN) return;
  const Job j = jobs[i];
  const int L = j.c / 2;
  Job kl, kr;
  reduce_range_bounds(order, tb, j.f, L, kl, s_acc);
  reduce_range_bounds(order, tb, j.f + L, j.c - L, kr, s_acc);
  if (threadIdx.x == 0) {
    set_children(kl, kr, j, L);
    st[i].kid[0] = kl;
    st[i].kid[1] = kr;
    st[i].L = L;
  }
}

__global__ void k_seg(const Job *__restrict__ jobs, int32_t *__restrict__ seg) {
  const Job j = jobs[blockIdx.x];
  for (int k = threadIdx.x; k < j.c; k += blockDim.x) seg[j.f + k] = blockIdx.x;
}

// left flag of every position of a binned split node (0 elsewhere)
__global__ void k_flags(const int32_t *__restrict__ seg, const NodeState *__restrict__ st,
                        const int32_t *__restrict__ order, const double *__restrict__ tb,
                        int64_t n, int n_bins, int32_t *__restrict__ flag) {
  const int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (pos > n) return;
  int32_t lf = 0;
  if (pos < n) {
    const int s = seg[pos];
    if (s >= 0 && st[s].state == ST_BIN) {
      const NodeState &ns = st[s];
      const double *t = tb + 9 * (int64_t)order[pos];
      lf = bin_of(t, ns.axis, ns.cmin, ns.scale, n_bins) <= ns.plane ? 1 : 0;
    }
  }
  flag[pos] = lf;
}

// back-stream lefts: beta[j-1] = back position, belem[j-1] = element
__global__ void k_back_lefts(const int32_t *__restrict__ seg, const NodeState *__restrict__ st,
                             const Job *__restrict__ jobs, const int32_t *__restrict__ order,
                             const int32_t *__restrict__ flag, const int32_t *__restrict__ pre,
                             int64_t n, int32_t *__restrict__ beta, int32_t *__restrict__ belem) {
  const int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const int s = seg[pos];
  if (s < 0 || st[s].state != ST_BIN || !flag[pos]) return;
  const Job &j = jobs[s];
  const int k = (int)(pos - j.f), L = st[s].L;
  if (k < L) return;
  const int jj = 1 + (pre[j.f + j.c] - pre[pos + 1]);
  beta[j.f + jj - 1] = j.c - k;
  belem[j.f + jj - 1] = order[pos];
}

__device__ __forceinline__ void scatter_one(int k, int lf, int32_t x, int c, int L, int last,
                                            int pre_k, const int32_t *beta_r,
                                            const int32_t *belem_r, int32_t *out_r) {
  if (k < L) {
    if (lf) {
      out_r[k] = x;
    } else {
      const int jj = 1 + (k - pre_k);  // rank among the front rights
      out_r[k] = belem_r[jj - 1];
      out_r[c - 1 - (jj >= 2 ? beta_r[jj - 2] : 0)] = x;
    }
  } else if (!lf) {
    const int p = c - k;
    out_r[(p < last) ? k - 1 : (k == L ? c - 1 - last : k - 1)] = x;
  }
}

__global__ void k_permute(const int32_t *__restrict__ seg, const NodeState *__restrict__ st,
                          const Job *__restrict__ jobs, const int32_t *__restrict__ order,
                          const int32_t *__restrict__ flag, const int32_t *__restrict__ pre,
                          const int32_t *__restrict__ beta, const int32_t *__restrict__ belem,
                          int64_t n, int32_t *__restrict__ out) {
  const int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const int s = seg[pos];
  if (s < 0 || st[s].state != ST_BIN) {
    out[pos] = order[pos];
    return;
  }
  const Job &j = jobs[s];
  const int L = st[s].L;
  const int X = L - (pre[j.f + L] - pre[j.f]);
  const int last = X > 0 ? beta[j.f + X - 1] : 0;
  const int k = (int)(pos - j.f);
  scatter_one(k, flag[pos], order[pos], j.c, L, last, pre[pos] - pre[j.f], beta + j.f,
              belem + j.f, out + j.f);
}

__global__ void k_children(const Job *__restrict__ jobs, int m, NodeState *__restrict__ st,
                           Tree t, Counters *ctr, Job *__restrict__ next, Job *__restrict__ small) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int state = st[i].state;
  if (state == ST_LEAF) return;
  const Job &j = jobs[i];
  const int id = atomicAdd(&ctr->nodes, 2);
  t.left[j.id] = id;
  t.right[j.id] = id + 1;
  for (int s = 0; s < 2; ++s) {
    Job k = st[i].kid[s];
    k.id = id + s;
    if (k.c > kSmall) next[atomicAdd(&ctr->n_next, 1)] = k;
    else small[atomicAdd(&ctr->n_small, 1)] = k;
  }
}

// ---------------------------------------------------------------- subtrees

struct SmallSmem {
  unsigned long long bins[kMaxBins * 12];
  unsigned int cnt[kMaxBins];
  Job stack[kDepthCap + 8];
  Job cur, kid[2];
  int sp, done, state, axis, plane, L, total;
  double cmin, scale;
  int warp_sum[kSmallThreads / 32];
  int32_t ord[kSmall];
  int32_t pre[kSmall + 1];
  int32_t beta[kSmall];
  int32_t belem[kSmall];
  uint8_t flag[kSmall];
};

__global__ void __launch_bounds__(kSmallThreads) k_small(const Job *__restrict__ jobs,
                                                    int32_t *__restrict__ order,
                                                    const double *__restrict__ tb, int leaf_size,
                                                    int n_bins, Tree t, Counters *ctr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmallSmem &S = *reinterpret_cast<SmallSmem *>(smem_raw);
  const int tid = threadIdx.x;
  if (tid == 0) {
    S.stack[0] = jobs[blockIdx.x];
    S.sp = 1;
  }
  __syncthreads();
  while (true) {
    __syncthreads();  // every thread is done with the previous node's shared state
    if (tid == 0) {
      S.done = S.sp == 0;
      if (!S.done) {
        S.cur = S.stack[--S.sp];
        emit_bounds(t, S.cur, ctr);
        int state, axis = 0;
        double cmin = 0.0, scale = 0.0;
        classify(S.cur, leaf_size, n_bins, state, axis, cmin, scale);
        S.state = state;
        S.axis = axis;
        S.cmin = cmin;
        S.scale = scale;
        if (state == ST_LEAF) emit_leaf(t, S.cur, ctr);
      }
    }
    __syncthreads();
    if (S.done) break;
    if (S.state == ST_LEAF) continue;  // (every thread reads S.state after the barrier)
    const Job J = S.cur;
    if (S.state == ST_BIN) {
      for (int q = tid; q < n_bins * 12; q += kSmallThreads) {
        const int r = q % 12;
        S.bins[q] = (r < 3 || (r >= 6 && r < 9)) ? ~0ull : 0ull;
      }
      for (int b = tid; b < n_bins; b += kSmallThreads) S.cnt[b] = 0;
      __syncthreads();
      const int axis = S.axis;
      const double cmin = S.cmin, scale = S.scale;
      for (int k = tid; k < J.c; k += kSmallThreads) {
        const int32_t ti = order[J.f + k];
        S.ord[k] = ti;
        const double *tt = tb + 9 * (int64_t)ti;
        const int b = bin_of(tt, axis, cmin, scale, n_bins);
        bin_add(S.bins + 12 * b, S.cnt + b, tt);
      }
      __syncthreads();
      if (tid == 0) {
        int L = 0;
        const int plane = sah_split(S.bins, S.cnt, n_bins, J, S.kid[0], S.kid[1], L);
        S.plane = plane;
        S.L = L;
        if (plane < 0) {
          S.state = ST_LEAF;
          emit_leaf(t, J, ctr);
        } else {
          set_children(S.kid[0], S.kid[1], J, L);
        }
      }
      __syncthreads();
      if (S.state == ST_LEAF) continue;
      // left flags and their exclusive prefix (contiguous segment per thread)
      const int plane = S.plane;
      const int per = (J.c + kSmallThreads - 1) / kSmallThreads;
      const int k0 = min(J.c, tid * per), k1 = min(J.c, k0 + per);
      int cnt = 0;
      for (int k = k0; k < k1; ++k) {
        const double *tt = tb + 9 * (int64_t)S.ord[k];
        const uint8_t lf = bin_of(tt, axis, cmin, scale, n_bins) <= plane ? 1 : 0;
        S.flag[k] = lf;
        cnt += lf;
      }
      int incl = cnt;
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if ((tid & 31) >= off) incl += o;
      }
      if ((tid & 31) == 31) S.warp_sum[tid >> 5] = incl;
      __syncthreads();
      if (tid == 0) {
        int run = 0;
        for (int w = 0; w < kSmallThreads / 32; ++w) {
          const int v = S.warp_sum[w];
          S.warp_sum[w] = run;
          run += v;
        }
        S.total = run;
      }
      __syncthreads();
      int base = S.warp_sum[tid >> 5] + incl - cnt;
      for (int k = k0; k < k1; ++k) {
        S.pre[k] = base;
        base += S.flag[k];
      }
      if (tid == 0) {
        S.pre[J.c] = S.total;
        if (S.total != S.L) atomicExch(&ctr->error, 1);
      }
      __syncthreads();
      const int L = S.L, c = J.c;
      for (int k = tid; k < c; k += kSmallThreads) {
        if (k >= L && S.flag[k]) {
          const int jj = 1 + (S.pre[c] - S.pre[k + 1]);
          S.beta[jj - 1] = c - k;
          S.belem[jj - 1] = S.ord[k];
        }
      }
      __syncthreads();
      const int X = L - S.pre[L];
      const int last = X > 0 ? S.beta[X - 1] : 0;
      for (int k = tid; k < c; k += kSmallThreads)
        scatter_one(k, S.flag[k], S.ord[k], c, L, last, S.pre[k], S.beta, S.belem,
                    order + J.f);
      __syncthreads();
    } else {  // ST_MEDIAN
      const int L = J.c / 2;
      reduce_range_bounds(order, tb, J.f, L, S.kid[0], S.bins);
      reduce_range_bounds(order, tb, J.f + L, J.c - L, S.kid[1], S.bins);
      if (tid == 0) set_children(S.kid[0], S.kid[1], J, L);
      __syncthreads();
    }
    if (tid == 0) {
      const int id = atomicAdd(&ctr->nodes, 2);
      t.left[J.id] = id;
      t.right[J.id] = id + 1;
      Job kl = S.kid[0], kr = S.kid[1];
      kl.id = id;
      kr.id = id + 1;
      S.stack[S.sp++] = kr;
      S.stack[S.sp++] = kl;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- host

// LT_VERBOSE=1: wall-clock phase times on stderr
struct BuildTimer {
  bool on = std::getenv("LT_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char *what, cudaStream_t st) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[luxb200 bvh-gpu] %-28s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Stream-ordered scratch from the device's default memory pool (kept mapped
// between builds by the pool's release threshold, as the scene buffers).
struct DevMem {
  void *p = nullptr;
  cudaStream_t st = nullptr;
  ~DevMem() {
    if (p) cudaFreeAsync(p, st);
  }
  template <class T>
  T *as() const {
    return static_cast<T *>(p);
  }
};

__global__ void k_iota(int32_t *__restrict__ o, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) o[i] = (int32_t)i;
}

#define GCK(call)                                                                        \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return lt_fail(LT_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));      \
  } while (0)

static thread_local cudaStream_t g_alloc_stream = nullptr;  // the calling thread's build stream

static int alloc(DevMem &m, size_t bytes) {
  m.st = g_alloc_stream;
  cudaError_t e = cudaMallocAsync(&m.p, std::max<size_t>(bytes, 16), m.st);
  if (e != cudaSuccess)
    return lt_fail(LT_ERR_NOMEM, "cudaMallocAsync(%zu) failed: %s", bytes, cudaGetErrorString(e));
  return LT_OK;
}

#define GRET(x)                      \
  do {                               \
    int rc_ = (x);                   \
    if (rc_ != LT_OK) return rc_;    \
  } while (0)

// Device-resident result of a build: provisional node ids (root = 0), the
// final triangle order, counters.
struct TreeOut {
  DevMem tree_b, tree_i, order;
  Tree t;
  Counters ctr{};
};

// The build on device-resident vertices (float64 (n,3) arrays); the tree
// stays on the device.
static int build_tree(const double *dv0, const double *dv1, const double *dv2, int64_t n,
                      int leaf_size, int n_bins, cudaStream_t st, TreeOut &out) {
  BuildTimer bt;
  const int64_t max_nodes = 2 * n;
  DevMem d_tb, d_order[2], d_seg, d_flag, d_pre, d_beta, d_belem, d_ctr, d_acc, d_jobs[2],
      d_small, d_state, d_bins, d_cnt, d_chunks, d_scan_tmp;
  DevMem &d_tree_b = out.tree_b, &d_tree_i = out.tree_i;
  GRET(alloc(d_tb, 9 * n * sizeof(double)));
  for (auto &o : d_order) GRET(alloc(o, n * sizeof(int32_t)));
  GRET(alloc(d_seg, n * sizeof(int32_t)));
  GRET(alloc(d_flag, (n + 1) * sizeof(int32_t)));
  GRET(alloc(d_pre, (n + 1) * sizeof(int32_t)));
  GRET(alloc(d_beta, n * sizeof(int32_t)));
  GRET(alloc(d_belem, n * sizeof(int32_t)));
  GRET(alloc(d_tree_b, 6 * max_nodes * sizeof(double)));
  GRET(alloc(d_tree_i, 4 * max_nodes * sizeof(int32_t)));
  GRET(alloc(d_ctr, sizeof(Counters)));
  GRET(alloc(d_acc, 12 * sizeof(unsigned long long)));
  const int64_t max_large = n / kSmall + 2;
  for (auto &j : d_jobs) GRET(alloc(j, 2 * max_large * sizeof(Job)));
  GRET(alloc(d_small, 2 * (2 * max_large + 2) * sizeof(Job)));
  GRET(alloc(d_state, 2 * max_large * sizeof(NodeState)));
  GRET(alloc(d_bins, 2 * max_large * kMaxBins * 12 * sizeof(unsigned long long)));
  GRET(alloc(d_cnt, 2 * max_large * kMaxBins * sizeof(unsigned int)));

  bt.mark("allocations", st);
  Tree &t = out.t;
  t.bmin = d_tree_b.as<double>();
  t.bmax = t.bmin + 3 * max_nodes;
  t.left = d_tree_i.as<int32_t>();
  t.right = t.left + max_nodes;
  t.first = t.right + max_nodes;
  t.count = t.first + max_nodes;
  GCK(cudaMemsetAsync(t.left, 0xff, 2 * max_nodes * sizeof(int32_t), st));  // -1
  GCK(cudaMemsetAsync(t.first, 0, 2 * max_nodes * sizeof(int32_t), st));
  GCK(cudaMemsetAsync(d_ctr.p, 0, sizeof(Counters), st));
  const unsigned blocks_n = (unsigned)((n + kThreads - 1) / kThreads);
  k_iota<<<blocks_n, kThreads, 0, st>>>(d_order[0].as<int32_t>(), n);
  k_tri_bounds<<<blocks_n, kThreads, 0, st>>>(dv0, dv1, dv2, n, d_tb.as<double>());
  {
    unsigned long long init[12];
    for (int q = 0; q < 12; ++q) init[q] = (q < 3 || (q >= 6 && q < 9)) ? ~0ull : 0ull;
    GCK(cudaMemcpyAsync(d_acc.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    k_root_reduce<<<std::min<unsigned>(blocks_n, 1184), kThreads, 0, st>>>(
        d_tb.as<double>(), n, d_acc.as<unsigned long long>());
    k_root_job<<<1, 1, 0, st>>>(d_acc.as<unsigned long long>(), n, d_jobs[0].as<Job>(),
                                d_small.as<Job>(), d_ctr.as<Counters>());
    GCK(cudaStreamSynchronize(st));  // init leaves scope
  }
  size_t scan_bytes = 0;
  GCK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, d_flag.as<int32_t>(),
                                    d_pre.as<int32_t>(), (int)(n + 1), st));
  GRET(alloc(d_scan_tmp, scan_bytes));

  bt.mark("triangle bounds + root", st);
  int cur = 0;  // order buffer holding the current permutation
  int levels = 0;
  int jl = 0;   // job list of the current level
  while (true) {
    Counters c;
    GCK(cudaMemcpyAsync(&c, d_ctr.p, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    GCK(cudaStreamSynchronize(st));
    const int m = c.n_next;
    if (m == 0) break;
    // reset the next-level counter (this level's jobs live in d_jobs[jl])
    {
      const int zero = 0;
      GCK(cudaMemcpyAsync(&d_ctr.as<Counters>()->n_next, &zero, sizeof(int),
                          cudaMemcpyHostToDevice, st));
      GCK(cudaStreamSynchronize(st));
    }
    const Job *jobs = d_jobs[jl].as<Job>();
    NodeState *nst = d_state.as<NodeState>();
    const unsigned bm = (unsigned)((m + 127) / 128);
    k_prepare<<<bm, 128, 0, st>>>(jobs, m, leaf_size, n_bins, nst, t, d_ctr.as<Counters>());
    // chunk table for the binned nodes
    std::vector<Job> hj(m);
    std::vector<NodeState> hs(m);
    GCK(cudaMemcpyAsync(hj.data(), jobs, m * sizeof(Job), cudaMemcpyDeviceToHost, st));
    GCK(cudaMemcpyAsync(hs.data(), nst, m * sizeof(NodeState), cudaMemcpyDeviceToHost, st));
    GCK(cudaStreamSynchronize(st));
    std::vector<int4> chunks;
    for (int i = 0; i < m; ++i)
      if (hs[i].state == ST_BIN)
        for (int s = 0; s < hj[i].c; s += kChunk)
          chunks.push_back(make_int4(i, hj[i].f + s, std::min(kChunk, hj[i].c - s), 0));
    if (!chunks.empty()) {
      if (d_chunks.p) {
        cudaFreeAsync(d_chunks.p, st);
        d_chunks.p = nullptr;
      }
      GRET(alloc(d_chunks, chunks.size() * sizeof(int4)));
      GCK(cudaMemcpyAsync(d_chunks.p, chunks.data(), chunks.size() * sizeof(int4),
                          cudaMemcpyHostToDevice, st));
      const int total_bins = m * kMaxBins;
      k_bins_reset<<<(total_bins + 255) / 256, 256, 0, st>>>(
          d_bins.as<unsigned long long>(), d_cnt.as<unsigned int>(), total_bins);
      k_bin_large<<<(unsigned)chunks.size(), kThreads, 0, st>>>(
          d_chunks.as<int4>(), jobs, nst, d_order[cur].as<int32_t>(), d_tb.as<double>(), n_bins,
          d_bins.as<unsigned long long>(), d_cnt.as<unsigned int>());
      k_sah_large<<<bm, 128, 0, st>>>(jobs, m, n_bins, d_bins.as<unsigned long long>(),
                                      d_cnt.as<unsigned int>(), nst, t, d_ctr.as<Counters>());
    }
    k_median_large<<<m, kThreads, 0, st>>>(jobs, nst, d_order[cur].as<int32_t>(),
                                           d_tb.as<double>());
    GCK(cudaMemsetAsync(d_seg.p, 0xff, n * sizeof(int32_t), st));
    k_seg<<<m, kThreads, 0, st>>>(jobs, d_seg.as<int32_t>());
    const unsigned bn1 = (unsigned)((n + 1 + kThreads - 1) / kThreads);
    k_flags<<<bn1, kThreads, 0, st>>>(d_seg.as<int32_t>(), nst, d_order[cur].as<int32_t>(),
                                      d_tb.as<double>(), n, n_bins, d_flag.as<int32_t>());
    GCK(cub::DeviceScan::ExclusiveSum(d_scan_tmp.p, scan_bytes, d_flag.as<int32_t>(),
                                      d_pre.as<int32_t>(), (int)(n + 1), st));
    k_back_lefts<<<blocks_n, kThreads, 0, st>>>(d_seg.as<int32_t>(), nst, jobs,
                                                d_order[cur].as<int32_t>(), d_flag.as<int32_t>(),
                                                d_pre.as<int32_t>(), n, d_beta.as<int32_t>(),
                                                d_belem.as<int32_t>());
    k_permute<<<blocks_n, kThreads, 0, st>>>(d_seg.as<int32_t>(), nst, jobs,
                                             d_order[cur].as<int32_t>(), d_flag.as<int32_t>(),
                                             d_pre.as<int32_t>(), d_beta.as<int32_t>(),
                                             d_belem.as<int32_t>(), n,
                                             d_order[cur ^ 1].as<int32_t>());
    cur ^= 1;
    k_children<<<bm, 128, 0, st>>>(jobs, m, nst, t, d_ctr.as<Counters>(),
                                   d_jobs[jl ^ 1].as<Job>(), d_small.as<Job>());
    jl ^= 1;
    ++levels;
    GCK(cudaGetLastError());
  }
  bt.mark("large-node levels", st);
  // every remaining subtree: one CTA each
  Counters c;
  GCK(cudaMemcpyAsync(&c, d_ctr.p, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  GCK(cudaStreamSynchronize(st));
  if (c.n_small > 0) {
    const size_t smem = sizeof(SmallSmem);
    GCK(cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_small<<<c.n_small, kSmallThreads, smem, st>>>(d_small.as<Job>(), d_order[cur].as<int32_t>(),
                                               d_tb.as<double>(), leaf_size, n_bins, t,
                                               d_ctr.as<Counters>());
    GCK(cudaGetLastError());
  }
  bt.mark("subtree kernel", st);
  if (bt.on) std::fprintf(stderr, "[luxb200 bvh-gpu] %d large levels, %d subtree jobs\n", levels, c.n_small);
  GCK(cudaMemcpyAsync(&out.ctr, d_ctr.p, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  GCK(cudaStreamSynchronize(st));
  if (out.ctr.error) return lt_fail(LT_ERR_CUDA, "GPU BVH build: partition count mismatch");
  std::swap(out.order.p, d_order[cur].p);  // the final permutation outlives the scratch
  std::swap(out.order.st, d_order[cur].st);
  return LT_OK;
}

// Host arrays in, provisional-id tree + order out (for lt_build_bvh_device).
static int build_on_device(const double *v0, const double *v1, const double *v2, int64_t n,
                           int leaf_size, int n_bins, cudaStream_t st,
                           std::vector<double> &tbmin, std::vector<double> &tbmax,
                           std::vector<int32_t> &tleft, std::vector<int32_t> &tright,
                           std::vector<int32_t> &tfirst, std::vector<int32_t> &tcount,
                           int32_t *order_out, Counters &ctr_h) {
  BuildTimer bt;
  DevMem d_v;
  GRET(alloc(d_v, 3 * 3 * n * sizeof(double)));
  GCK(cudaMemcpyAsync(d_v.as<double>(), v0, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
  GCK(cudaMemcpyAsync(d_v.as<double>() + 3 * n, v1, 3 * n * sizeof(double),
                      cudaMemcpyHostToDevice, st));
  GCK(cudaMemcpyAsync(d_v.as<double>() + 6 * n, v2, 3 * n * sizeof(double),
                      cudaMemcpyHostToDevice, st));
  bt.mark("vertex upload", st);
  TreeOut out;
  GRET(build_tree(d_v.as<double>(), d_v.as<double>() + 3 * n, d_v.as<double>() + 6 * n, n,
                  leaf_size, n_bins, st, out));
  ctr_h = out.ctr;
  const Tree &t = out.t;
  const int64_t nn = ctr_h.nodes;
  tbmin.resize(3 * nn);
  tbmax.resize(3 * nn);
  tleft.resize(nn);
  tright.resize(nn);
  tfirst.resize(nn);
  tcount.resize(nn);
  GCK(cudaMemcpyAsync(tbmin.data(), t.bmin, 3 * nn * sizeof(double), cudaMemcpyDeviceToHost, st));
  GCK(cudaMemcpyAsync(tbmax.data(), t.bmax, 3 * nn * sizeof(double), cudaMemcpyDeviceToHost, st));
  GCK(cudaMemcpyAsync(tleft.data(), t.left, nn * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GCK(cudaMemcpyAsync(tright.data(), t.right, nn * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GCK(cudaMemcpyAsync(tfirst.data(), t.first, nn * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GCK(cudaMemcpyAsync(tcount.data(), t.count, nn * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GCK(cudaMemcpyAsync(order_out, out.order.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GCK(cudaStreamSynchronize(st));
  bt.mark("tree + order download", st);
  return LT_OK;
}

}  // namespace

// Device-resident build for lt_scene_create (no host round trip): the
// reference's tree with provisional ids (root 0).  `stream` is a cudaStream_t.
extern int lt_gpu_tree_build(const double *dv0, const double *dv1, const double *dv2, int64_t n,
                             int32_t leaf_size, int32_t bins, void *stream, lt_gpu_tree *out) {
  if (n <= 0) return lt_fail(LT_ERR_INVALID, "empty scene");
  if (bins > kMaxBins || bins < 2 || leaf_size < 1)
    return lt_fail(LT_ERR_INVALID, "unsupported BVH build parameters");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  g_alloc_stream = st;
  auto *to = new TreeOut;
  const int rc = build_tree(dv0, dv1, dv2, n, leaf_size, bins, st, *to);
  if (rc != LT_OK) {
    delete to;
    return rc;
  }
  const int64_t max_nodes = 2 * n;
  (void)max_nodes;
  out->bmin = to->t.bmin;
  out->bmax = to->t.bmax;
  out->left = to->t.left;
  out->right = to->t.right;
  out->first = to->t.first;
  out->count = to->t.count;
  out->order = to->order.as<int32_t>();
  out->n_nodes = to->ctr.nodes;
  out->n_leaves = to->ctr.leaves;
  out->max_depth = to->ctr.max_depth;
  out->impl = to;
  return LT_OK;
}

void lt_gpu_tree_free(lt_gpu_tree *t) {
  if (t && t->impl) {
    delete static_cast<TreeOut *>(t->impl);  // frees stream-ordered on the build stream
    t->impl = nullptr;
  }
}

// The reference's numbering: pop depth first (left child first); the k-th
// internal node popped allocates its children as the next two ids.
extern "C" int lt_build_bvh_device(int32_t device, const double *v0, const double *v1,
                                   const double *v2, int64_t n, int32_t leaf_size,
                                   int32_t bins, double *bounds_min, double *bounds_max,
                                   int32_t *left_child, int32_t *right_child,
                                   int32_t *first_triangle, int32_t *triangle_count,
                                   int32_t *triangle_order, int64_t *n_nodes,
                                   int64_t *leaf_count, int64_t *max_depth) {
  if (!v0 || !v1 || !v2 || !bounds_min || !bounds_max || !left_child || !right_child ||
      !first_triangle || !triangle_count || !triangle_order || !n_nodes || !leaf_count ||
      !max_depth)
    return lt_fail(LT_ERR_INVALID, "lt_build_bvh_device: null pointer");
  if (n <= 0) return lt_fail(LT_ERR_INVALID, "empty scene");
  if (leaf_size < 1 || bins < 2) return lt_fail(LT_ERR_INVALID, "leaf_size >= 1 and bins >= 2 required");
  if (bins > kMaxBins)
    return lt_fail(LT_ERR_INVALID, "GPU BVH build supports at most %d bins", kMaxBins);
  if (n > (int64_t)1 << 30) return lt_fail(LT_ERR_INVALID, "too many triangles for the GPU build");
  int prev = 0;
  cudaGetDevice(&prev);
  GCK(cudaSetDevice(device));
  cudaStream_t st;
  GCK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX, cur = 0;
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &cur);
      if (cur < keep) cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  g_alloc_stream = st;
  std::vector<double> tbmin, tbmax;
  std::vector<int32_t> tl, tr, tf, tc;
  Counters ctr{};
  const int rc = build_on_device(v0, v1, v2, n, leaf_size, bins, st, tbmin, tbmax, tl, tr, tf,
                                 tc, triangle_order, ctr);
  cudaStreamSynchronize(st);  // the scratch frees are enqueued on st
  cudaStreamDestroy(st);
  cudaSetDevice(prev);
  if (rc != LT_OK) return rc;
  // replay the reference's allocation order over the finished tree
  const int64_t nn = ctr.nodes;
  for (int64_t k = 0; k < 2 * n; ++k) {
    left_child[k] = -1;
    right_child[k] = -1;
    first_triangle[k] = 0;
    triangle_count[k] = 0;
  }
  std::vector<std::pair<int32_t, int32_t>> stack;  // (provisional id, reference id)
  stack.reserve(kDepthCap + 8);
  stack.push_back({0, 0});
  int64_t next_id = 1;
  while (!stack.empty()) {
    const auto [p, r] = stack.back();
    stack.pop_back();
    for (int a = 0; a < 3; ++a) {
      bounds_min[3 * (int64_t)r + a] = tbmin[3 * (int64_t)p + a];
      bounds_max[3 * (int64_t)r + a] = tbmax[3 * (int64_t)p + a];
    }
    if (tl[p] < 0) {
      first_triangle[r] = tf[p];
      triangle_count[r] = tc[p];
      continue;
    }
    const int32_t lc = (int32_t)next_id, rcid = (int32_t)next_id + 1;
    next_id += 2;
    left_child[r] = lc;
    right_child[r] = rcid;
    stack.push_back({tr[p], rcid});
    stack.push_back({tl[p], lc});
  }
  if (next_id != nn) return lt_fail(LT_ERR_CUDA, "GPU BVH build: node count mismatch");
  *n_nodes = nn;
  *leaf_count = ctr.leaves;
  *max_depth = ctr.max_depth;
  return LT_OK;
}
