// lt_kernels.cu -- the wavefront pipeline kernels and the scene flattening.
//
// One render batch = raygen -> max_depth x (trace -> shade) -> accumulate.
// Queues are device-resident; every kernel reads its queue length from
// device memory, so a whole batch is issued without a host round trip.
#include <cstdint>

#include "lt_kernels.h"
#include "lt_material.cuh"
#include "lt_traverse.cuh"

namespace lt {

constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ flatten

// Node records from the host BVH (bvh.py:38-50): boxes rounded outward to
// fp32 (the float64 pad of 1e-7*extent is below fp32 resolution), links
// renumbered; leaves become ~first_triangle.
__global__ void k_flatten_nodes(const double *__restrict__ bmin, const double *__restrict__ bmax,
                                const int32_t *__restrict__ left,
                                const int32_t *__restrict__ right,
                                const int32_t *__restrict__ first,
                                const int32_t *__restrict__ count,
                                const int32_t *__restrict__ perm,
                                const int32_t *__restrict__ new_index, int64_t n_internal,
                                float4 *__restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_internal) return;
  const int32_t old = perm[i];
  const int32_t ch[2] = {left[old], right[old]};
  float lo[2][3], hi[2][3];
  int32_t link[2];
  for (int c = 0; c < 2; ++c) {
    const int32_t x = ch[c];
    for (int a = 0; a < 3; ++a) {
      lo[c][a] = __double2float_rd(bmin[3 * (int64_t)x + a]);
      hi[c][a] = __double2float_ru(bmax[3 * (int64_t)x + a]);
    }
    link[c] = count[x] > 0 ? ~first[x] : new_index[x];
  }
  out[4 * i + 0] = make_float4(lo[0][0], hi[0][0], lo[0][1], hi[0][1]);
  out[4 * i + 1] = make_float4(lo[1][0], hi[1][0], lo[1][1], hi[1][1]);
  out[4 * i + 2] = make_float4(lo[0][2], hi[0][2], lo[1][2], hi[1][2]);
  out[4 * i + 3] = make_float4(__int_as_float(link[0]), __int_as_float(link[1]), 0.f, 0.f);
}

// BVH4 records: node i gathers the reference nodes children[4 i .. 4 i + 3]
// (-1 = empty slot) chosen by the host collapse; boxes rounded outward,
// links: leaf -> ~first_triangle, internal -> its wide index.
__global__ void k_flatten_wide(const double *__restrict__ bmin, const double *__restrict__ bmax,
                               const int32_t *__restrict__ first,
                               const int32_t *__restrict__ count,
                               const int32_t *__restrict__ children,
                               const int32_t *__restrict__ wide_of, int64_t n_wide,
                               float4 *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_wide) return;
  float lo[3][4], hi[3][4];
  int32_t link[4];
  for (int c = 0; c < 4; ++c) {
    const int32_t x = children[4 * i + c];
    if (x < 0) {
      // empty slot: an inverted infinite box, which the near/far slab test
      // rejects by construction (the min/max form also checks the link)
      for (int a = 0; a < 3; ++a) {
        lo[a][c] = __int_as_float(0x7f800000);
        hi[a][c] = __int_as_float(0xff800000);
      }
      link[c] = LT_LINK_EXIT;
      continue;
    }
    for (int a = 0; a < 3; ++a) {
      lo[a][c] = __double2float_rd(bmin[3 * (int64_t)x + a]);
      hi[a][c] = __double2float_ru(bmax[3 * (int64_t)x + a]);
    }
    link[c] = count[x] > 0 ? ~first[x] : wide_of[x];
  }
  float4 *o = out + LT_NODE_F4 * i;
  for (int a = 0; a < 3; ++a) {
    const float4 l4 = make_float4(lo[a][0], lo[a][1], lo[a][2], lo[a][3]);
    const float4 h4 = make_float4(hi[a][0], hi[a][1], hi[a][2], hi[a][3]);
    o[4 * a] = l4;      // (near, far) for a positive inverse direction
    o[4 * a + 1] = h4;
    o[4 * a + 2] = h4;  // (near, far) for a negative one
    o[4 * a + 3] = l4;
  }
  o[LT_NODE_LINKS + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  o[LT_NODE_LINKS] = make_float4(__int_as_float(link[0]), __int_as_float(link[1]),
                                 __int_as_float(link[2]), __int_as_float(link[3]));
}

// End-of-leaf flags of the leaf-ordered triangle stream.
__global__ void k_leaf_end(const int32_t *__restrict__ first, const int32_t *__restrict__ count,
                           int64_t n_nodes, uint8_t *__restrict__ leaf_end) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_nodes) return;
  const int32_t c = count[i];
  if (c > 0) leaf_end[(int64_t)first[i] + c - 1] = 1;
}

// Triangles in leaf order k (triangle_order[k]); e1/e2 from float64
// differences rounded once; shading normals + material index alongside.
__global__ void k_flatten_tris(const double *__restrict__ v0, const double *__restrict__ v1,
                               const double *__restrict__ v2, const double *__restrict__ n0,
                               const double *__restrict__ n1, const double *__restrict__ n2,
                               const int32_t *__restrict__ mat_index,
                               const int32_t *__restrict__ order,
                               const uint8_t *__restrict__ leaf_end, int64_t n,
                               float4 *__restrict__ tris, float4 *__restrict__ shade) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t ti = order[k];
  const double *a = v0 + 3 * ti, *b = v1 + 3 * ti, *c = v2 + 3 * ti;
  float4 *tr = tris + LT_TRI_F4 * k;
  tr[0] = make_float4((float)a[0], (float)a[1], (float)a[2], __int_as_float((int)ti));
  tr[1] = make_float4((float)(b[0] - a[0]), (float)(b[1] - a[1]), (float)(b[2] - a[2]),
                                __int_as_float(leaf_end[k] ? 1 : 0));
  tr[2] = make_float4((float)(c[0] - a[0]), (float)(c[1] - a[1]), (float)(c[2] - a[2]), 0.f);
  // geometric normal as _hit_frame computes it (geometry.py:217-224), float64
  const double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
  const double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
  double gx = e1y * e2z - e1z * e2y;
  double gy = e1z * e2x - e1x * e2z;
  double gz = e1x * e2y - e1y * e2x;
  const double glen = sqrt(gx * gx + gy * gy + gz * gz);
  if (glen > 0.0) {
    gx /= glen;
    gy /= glen;
    gz /= glen;
  }
  const double *p0 = n0 + 3 * ti, *p1 = n1 + 3 * ti, *p2 = n2 + 3 * ti;
  shade[4 * k + 0] =
      make_float4((float)gx, (float)gy, (float)gz, __int_as_float(mat_index[ti]));
  shade[4 * k + 1] = make_float4((float)p0[0], (float)p0[1], (float)p0[2], 0.f);
  shade[4 * k + 2] = make_float4((float)p1[0], (float)p1[1], (float)p1[2], 0.f);
  shade[4 * k + 3] = make_float4((float)p2[0], (float)p2[1], (float)p2[2], 0.f);
}

// ------------------------------------------------------------------ raygen

// Primary ray of path p = s_local * n_pix + i (sample-major), keyed by the
// GLOBAL pixel index and sample index (integrator.py:253-258): stream seed,
// two jitter draws, float64 pinhole direction; returns the PCG state after
// the two draws.  Raygen writes the ray record the depth-0 trace and shade
// read; the depth-0 shade regenerates only the PCG state (primary_rng).
// seed_stream (rng.py:70-78) from the batch tables: st = 0 -> inc after the
// first step, + init_state, one more step -- the same 64-bit arithmetic
__device__ __forceinline__ void seed_from_tables(const RaygenArgs &ra, int64_t i, int64_t s_local,
                                                 uint64_t &state, uint64_t &inc) {
  inc = __ldg(&ra.inc_tab[i]);
  uint64_t st = inc + __ldg(&ra.init_tab[s_local]);
  (void)pcg_next(st, inc);
  state = st;
}

__device__ __forceinline__ void primary_ray(const RaygenArgs &ra, int64_t p, f3 &o, f3 &d,
                                            uint64_t &state, uint64_t &inc) {
  // batch-local path index and pixel count are < 2^31 (int32 queues): a
  // 32-bit division instead of the 64-bit software routine
  const int64_t s_local = (int64_t)((uint32_t)p / (uint32_t)ra.n_pix);
  const int64_t i = p - s_local * ra.n_pix;
  const int64_t pix = ra.pix_list ? (int64_t)ra.pix_list[ra.pix_offset + i] : ra.pix_offset + i;
  const int64_t sample = ra.sample_base + s_local;
  // (pixel indices are < 2^31: a 32-bit division, not the 64-bit routine)
  const int64_t py = (int64_t)((uint32_t)pix / (uint32_t)ra.width);
  const int64_t px = pix - py * ra.width;
  if (ra.inc_tab)
    seed_from_tables(ra, i, s_local, state, inc);
  else
    seed_stream((uint64_t)pix, (uint64_t)sample, ra.seed, state, inc);
  const double jx = unit_f64(state, inc);
  const double jy = unit_f64(state, inc);
  d = camera_dir(ra.cam, (double)px, (double)py, jx, jy, ra.width, ra.height);
  o = f3{(float)ra.cam[0], (float)ra.cam[1], (float)ra.cam[2]};
}

// The PCG state of path p after its two jitter draws (integer only): the
// depth-0 shade launch regenerates it instead of reading it back.
__device__ __forceinline__ void primary_rng(const RaygenArgs &ra, int64_t p, uint64_t &state,
                                            uint64_t &inc) {
  const int64_t s_local = (int64_t)((uint32_t)p / (uint32_t)ra.n_pix);
  const int64_t i = p - s_local * ra.n_pix;
  if (ra.inc_tab) {
    seed_from_tables(ra, i, s_local, state, inc);
  } else {
    const int64_t pix =
        ra.pix_list ? (int64_t)ra.pix_list[ra.pix_offset + i] : ra.pix_offset + i;
    seed_stream((uint64_t)pix, (uint64_t)(ra.sample_base + s_local), ra.seed, state, inc);
  }
  (void)pcg_next(state, inc);
  (void)pcg_next(state, inc);
}

// Pixel of render path p (the batch's sample-major path numbering) and its
// PCG increment, seed_stream's (mix64(pixel) << 1) | 1 (rng.py:70-78).
__device__ __forceinline__ uint64_t path_inc(const RaygenArgs &ra, int64_t p) {
  const int64_t s_local = (int64_t)((uint32_t)p / (uint32_t)ra.n_pix);
  const int64_t i = p - s_local * ra.n_pix;
  // (not ra.inc_tab: a random 8 B table load measured slower here than the
  // hash, profiles/r02_rng_tables3.jsonl)
  const int64_t pix = ra.pix_list ? (int64_t)ra.pix_list[ra.pix_offset + i] : ra.pix_offset + i;
  return (mix64((uint64_t)pix) << 1) | 1ULL;
}

// The 32 B path record: one 256-bit streaming load / store.
__device__ __forceinline__ void ld_path(const float4 *__restrict__ S, int64_t p, float4 &T,
                                        float4 &L, uint64_t &state) {
  float4 a, b;
  asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                 "=f"(b.w)
               : "l"(S + 2 * p));
  T = make_float4(a.x, a.y, a.z, 0.f);
  L = make_float4(a.w, b.x, b.y, 0.f);
  state = ((uint64_t)__float_as_uint(b.w) << 32) | __float_as_uint(b.z);
}
__device__ __forceinline__ void st_path(float4 *__restrict__ S, int64_t p, const float4 &T,
                                        const float4 &L, uint64_t state) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(S + 2 * p),
               "f"(T.x), "f"(T.y), "f"(T.z), "f"(L.x), "f"(L.y), "f"(L.z),
               "f"(__uint_as_float((uint32_t)state)), "f"(__uint_as_float((uint32_t)(state >> 32)))
               : "memory");
}

__global__ void k_rng_tables(RaygenArgs ra, int64_t n_samples, uint64_t *__restrict__ inc_tab,
                             uint64_t *__restrict__ init_tab) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < ra.n_pix) {
    const int64_t pix =
        ra.pix_list ? (int64_t)ra.pix_list[ra.pix_offset + t] : ra.pix_offset + t;
    inc_tab[t] = (mix64((uint64_t)pix) << 1) | 1ULL;
  }
  if (t < n_samples) init_tab[t] = mix64(ra.seed ^ mix64((uint64_t)(ra.sample_base + t)));
}

// Primary rays of a render batch: only the 16 B direction record is written
// (the origin is the camera, the path id the queue slot); the throughput
// (1), radiance (0) and PCG state are implied / regenerated by the depth-0
// shade launch.
__global__ void k_raygen(RaygenArgs ra, PathArrays pa, float4 *__restrict__ q_o,
                         float4 *__restrict__ q_d, int32_t *__restrict__ count0) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p == 0) *count0 = (int32_t)ra.n_paths;
  if (p >= ra.n_paths) return;
  f3 o, d;
  uint64_t state, inc;
  primary_ray(ra, p, o, d, state, inc);
  (void)q_o;  // a primary ray's origin is the camera and its path id its slot
  __stcs(&q_d[p], make_float4(d.x, d.y, d.z, ra.t_min));
}

// Explicit rays with caller-supplied PCG state (trace_radiance,
// integrator.py:294-307).
__global__ void k_raygen_explicit(const double *__restrict__ o, const double *__restrict__ d,
                                  const uint64_t *__restrict__ state,
                                  const uint64_t *__restrict__ inc, int64_t n, float t_min,
                                  PathArrays pa,
                                  float4 *__restrict__ q_o, float4 *__restrict__ q_d,
                                  int32_t *__restrict__ count0) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p == 0) *count0 = (int32_t)n;
  if (p >= n) return;
  q_o[p] = make_float4((float)o[3 * p], (float)o[3 * p + 1], (float)o[3 * p + 2],
                       __int_as_float((int32_t)p));
  q_d[p] = make_float4((float)d[3 * p], (float)d[3 * p + 1], (float)d[3 * p + 2], t_min);
  st_path(pa.S, p, make_float4(1.f, 1.f, 1.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f), state[p]);
  pa.inc[p] = inc[p];
}

__global__ void k_gather_explicit(PathArrays pa, int64_t n, double *__restrict__ rgb,
                                  uint64_t *__restrict__ state_out) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  float4 T, L;
  uint64_t st;
  ld_path(pa.S, p, T, L, st);
  rgb[3 * p + 0] = L.x;
  rgb[3 * p + 1] = L.y;
  rgb[3 * p + 2] = L.z;
  state_out[p] = st;
}

// ------------------------------------------------------------------ trace

// Persistent closest-hit kernel (the render path).
//  * grid = SMs x resident CTAs; each lane owns one ray at a time and, when
//    it finishes, the warp refills its idle lanes from the queue with one
//    atomic (ballot + popc ranks) once >= sc.refill_min lanes are idle, so
//    short rays do not leave lanes dark while long ones finish;
//  * one loop iteration = refill check, up to LT_NODE_STEPS inner-node
//    visits per lane, then the leaf phase: lanes that reached a leaf wait
//    until >= sc.leaf_min of the warp have (or no lane is left at an inner
//    node) and test their triangles together.  The classic while-while form
//    (leaves only once every lane has one) left ~12 of 32 lanes active in
//    the node visits (profiles/r01_v16_trace_source.txt);
//  * traversal stack: the first kShortStack entries of every lane live in
//    shared memory, laid out [depth][thread] (conflict-free), deeper ones in
//    local memory;
//  * queue reads / hit writes are streaming (__ldcs / __stcs) so they do not
//    evict the scene from L2.
// ray_ctr[0] += queue length; with COUNT also ray_ctr[1] += slab tests and
// ray_ctr[2] += triangle tests.
template <bool COUNT>
__global__ void __launch_bounds__(kTraceThreads, LT_TRACE_MIN_BLOCKS)
    k_trace(SceneView sc, const float4 *__restrict__ q_o, const float4 *__restrict__ q_d,
            const int32_t *__restrict__ count, int32_t *__restrict__ fetch,
            float4 *__restrict__ hits, unsigned long long *__restrict__ ray_ctr, float4 cam_o) {
  extern __shared__ float4 s_mem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const unsigned lanes_below = (1u << lane) - 1u;
  // stack entry = (node, entry t) in one 64-bit word: one STS.64 / LDS.64
  uint2 *const s_stk = reinterpret_cast<uint2 *>(s_mem) + tid;
  uint2 l_stk[LT_STACK - kShortStack];

  const int n = *count;
  if (blockIdx.x == 0 && tid == 0) atomicAdd(ray_ctr, (unsigned long long)n);

  int q = -1;
  bool exhausted = false;  // warp-uniform: the queue is drained
  f3 o{0.f, 0.f, 0.f}, d{0.f, 0.f, 1.f};
  RaySlab rs{};
  float t_min = 0.f;
  HitRec best{0.f, 0.f, 0.f, -1};
  int32_t best_orig = 0x7fffffff;
  int sp = 0;
  int32_t node = LT_LINK_EXIT;
  int nn = 0, nt = 0;

  while (true) {
    // ---- refill idle lanes
    const unsigned idle = __ballot_sync(kFull, q < 0);
    if (!exhausted && __popc(idle) >= sc.refill_min) {
      const int cnt = __popc(idle);
      const int leader = __ffs(idle) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(fetch, cnt);
      base = __shfl_sync(kFull, base, leader);
      exhausted = base + cnt >= n;
      if (q < 0) {
        const int r = base + __popc(idle & lanes_below);
        if (r < n) {
          q = r;
          // (primary rays, q_o NULL: the origin is the camera)
          const float4 ro = q_o ? __ldcs(&q_o[r]) : cam_o;
          const float4 rd = __ldcs(&q_d[r]);
          t_min = rd.w;
          rs = ray_slab(mk(ro.x, ro.y, ro.z), mk(rd.x, rd.y, rd.z));
          best = HitRec{__int_as_float(0x7f800000), 0.f, 0.f, -1};
          best_orig = 0x7fffffff;
          o = mk(ro.x, ro.y, ro.z);
          d = mk(rd.x, rd.y, rd.z);
          sp = 0;
          if (COUNT) ++nn;
          float t_root;
          node = slab(rs, sc.root_lo[0], sc.root_hi[0], sc.root_lo[1], sc.root_hi[1],
                      sc.root_lo[2], sc.root_hi[2], t_min, best.t, t_root)
                     ? sc.wroot_link
                     : LT_LINK_EXIT;
        }
      }
    }
    if (__ballot_sync(kFull, q >= 0) == 0) {
      if (exhausted) break;
      continue;
    }
    // pop the next stack entry not culled by the current best t (bvh.py:389)
    auto pop = [&]() -> int32_t {
      const float cull = cull_dist(best.t);
      while (sp > 0) {
        --sp;
        const uint2 e = sp < kShortStack ? s_stk[sp * kTraceThreads] : l_stk[sp - kShortStack];
        if (!(__uint_as_float(e.y) > cull)) return (int32_t)e.x;
      }
      return LT_LINK_EXIT;
    };
    auto push = [&](int32_t x, float tx) {
      LT_ASSERT(sp < LT_STACK);
      const uint2 e = make_uint2((uint32_t)x, __float_as_uint(tx));
      if (sp < kShortStack)
        s_stk[sp * kTraceThreads] = e;
      else
        l_stk[sp - kShortStack] = e;
      ++sp;
    };
    const float kInf = __int_as_float(0x7f800000);
    // ---- one wide node per active lane: descend nearest-first; the other
    // hit children go on the stack farthest first
#pragma unroll 1
    for (int step = 0; step < LT_NODE_STEPS && q >= 0 && node >= 0; ++step) {
      LT_ASSERT(node < sc.n_wide);
      const Hits4 h = visit4o(sc.wnodes + LT_NODE_F4 * (int64_t)node, rs, t_min, best.t);
      if (COUNT) nn += 4;
      if (sp <= kShortStack - 3) {
        // common case: all three fit in shared memory (predicated stores)
        uint2 *top = s_stk + sp * kTraceThreads;
        if (h.k3 < kInf) { *top = make_uint2((uint32_t)h.l3, __float_as_uint(h.k3)); top += kTraceThreads; ++sp; }
        if (h.k2 < kInf) { *top = make_uint2((uint32_t)h.l2, __float_as_uint(h.k2)); top += kTraceThreads; ++sp; }
        if (h.k1 < kInf) { *top = make_uint2((uint32_t)h.l1, __float_as_uint(h.k1)); top += kTraceThreads; ++sp; }
      } else {
        if (h.k3 < kInf) push(h.l3, h.k3);
        if (h.k2 < kInf) push(h.l2, h.k2);
        if (h.k1 < kInf) push(h.l1, h.k1);
      }
      node = h.k0 < kInf ? h.l0 : pop();
    }
    // ---- leaves: lanes that reached one wait until enough of the warp has
    // (or no lane is still at an inner node), then test their triangles
    // together, so inner-node iterations keep more lanes busy
    const bool at_leaf = q >= 0 && node < 0 && node != LT_LINK_EXIT;
    const unsigned leaf_mask = __ballot_sync(kFull, at_leaf);
    if (leaf_mask && (__popc(leaf_mask) >= sc.leaf_min ||
                      __ballot_sync(kFull, q >= 0 && node >= 0) == 0)) {
      if (at_leaf) {
        leaf_test<COUNT>(sc, ~(uint32_t)node, o, d, t_min, best, best_orig, nt);
        node = pop();
      }
    }
    if (q >= 0 && node == LT_LINK_EXIT) {
      __stcs(&hits[q], make_float4(best.t, best.u, best.v, __int_as_float(best.k)));
      q = -1;
    }
  }
  if (COUNT) {
    for (int off = 16; off > 0; off >>= 1) {
      nn += __shfl_down_sync(kFull, nn, off);
      nt += __shfl_down_sync(kFull, nt, off);
    }
    if (lane == 0) {
      atomicAdd(ray_ctr + 1, (unsigned long long)nn);
      atomicAdd(ray_ctr + 2, (unsigned long long)nt);
    }
  }
}

// Arbitrary rays (intersect_scene_batch): ray (o, d), t_min in q_d.w,
// t_max in q_o.w.  Optionally counts work per ray (traversal_counts_batch).
template <bool COUNT>
__global__ void __launch_bounds__(kTraceThreads)
    k_trace_rays(SceneView sc, const float4 *__restrict__ q_o, const float4 *__restrict__ q_d,
                 int64_t n, float4 *__restrict__ hits, int32_t *__restrict__ nodes,
                 int32_t *__restrict__ tests) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  const float4 ro = q_o[q];
  const float4 rd = q_d[q];
  int nn = 0, nt = 0;
  // closest-hit queries walk the wide layout (as the render path); the
  // counter query walks the reference's binary nodes (its counter semantics)
  const HitRec h = traverse<!COUNT, COUNT>(sc, mk(ro.x, ro.y, ro.z), mk(rd.x, rd.y, rd.z), rd.w,
                                           ro.w, &nn, &nt);
  hits[q] = make_float4(h.t, h.u, h.v, __int_as_float(h.k));
  if (COUNT) {
    nodes[q] = nn;
    tests[q] = nt;
  }
}

// ------------------------------------------------------------------ shade

// Direction octant of a continuation ray (the block-level grouping of the
// append; 24 / 64 finer bins measured +-0 / -1 %, profiles/r01_v12 sweeps).
#define LT_DIR_BINS 8
__device__ __forceinline__ int dir_bin(const float4 &d) {
  return (d.x < 0.f ? 1 : 0) | (d.y < 0.f ? 2 : 0) | (d.z < 0.f ? 4 : 0);
}

// One path segment of _trace (integrator.py:160-226) after its closest-hit
// query h = (t, u, v, k): miss -> environment; hit -> emission; the final
// segment stops; otherwise hit frame, 3 draws, BSDF sample, throughput and
// Russian roulette (4th draw).  Returns true when the path continues with
// the ray (out_o, out_d) and throughput Tn.  `inc_of()` yields the PCG
// increment, asked for only when the segment draws.  Shared by the
// wavefront shade kernel and the fused small-pass kernel, so both round
// identically.
struct Segment {
  bool wrote_l = false;    // L changed and the path ends here
  bool scattered = false;  // the draws ran (state advanced)
  uint64_t st_out;         // PCG state after the segment's draws
  float4 Tn;               // throughput of the continuation
  float4 out_o, out_d;     // the continuation ray (path id / t_min in .w)
  int cls = 0;             // material class (LT_FLAG_COUNT statistics)
};
template <class IncFn>
__device__ __forceinline__ bool shade_segment(const SceneView &sc, int32_t depth,
                                              int32_t max_depth, int32_t rr_start, float t_min,
                                              bool want_cls, int32_t p, const float4 &h, f3 o,
                                              f3 d, const float4 &T, float4 &L, uint64_t state,
                                              IncFn inc_of, Segment &sg) {
  const int32_t k = __float_as_int(h.w);
  sg.st_out = state;
  if (k < 0) {
    const f3 e = env_radiance(sc, d);
    L.x += T.x * e.x;
    L.y += T.y * e.y;
    L.z += T.z * e.z;
    sg.wrote_l = true;
    return false;
  }
  // issue every random load of this hit before using any of them: one
  // 64 B shading record (geometric normal + material, vertex normals)
  LT_ASSERT(k < sc.n_tris);
  const int64_t k4 = 4 * (int64_t)k;
  const bool scatter = depth != max_depth - 1;
  const float4 s0 = __ldg(&sc.shade[k4]);
  float4 s1{}, s2{}, s3{};
  uint64_t inc = 0;
  if (scatter) {
    s1 = __ldg(&sc.shade[k4 + 1]);
    s2 = __ldg(&sc.shade[k4 + 2]);
    s3 = __ldg(&sc.shade[k4 + 3]);
    inc = inc_of();
  }
  const int32_t mi = __float_as_int(s0.w);
  LT_ASSERT(mi >= 0 && mi < sc.n_mats);
  const GpuMaterial &mt = sc.mats[mi];
  if (want_cls)
    sg.cls = !scatter ? 1
                      : (mt.flags & MAT_DIFFUSE_ONLY)
                            ? 2
                            : (mt.flags & (MAT_COAT | MAT_GLASS))
                                  ? 3 + (int)(mt.flags & (MAT_COAT | MAT_GLASS))
                                  : 3;
  if (mt.flags & MAT_EMISSIVE) {
    L.x += T.x * mt.el * mt.ec[0];
    L.y += T.y * mt.el * mt.ec[1];
    L.z += T.z * mt.el * mt.ec[2];
    sg.wrote_l = true;
  }
  if (!scatter) return false;
  f3 g, sn;
  bool front;
  hit_frame(d, mk(s0.x, s0.y, s0.z), mk(s1.x, s1.y, s1.z), mk(s2.x, s2.y, s2.z),
            mk(s3.x, s3.y, s3.z), h.y, h.z, g, sn, front);
  const float u_lobe = unit_f32(state, inc);
  const float u1 = unit_f32(state, inc);
  const float u2 = unit_f32(state, inc);
  f3 wi, w;
  bool alive = sample_material(-d, sn, mt, front, u_lobe, u1, u2, wi, w);
  float4 Tn = T;
  if (alive) {
    Tn.x *= w.x;
    Tn.y *= w.y;
    Tn.z *= w.z;
    if (Tn.x <= 0.f && Tn.y <= 0.f && Tn.z <= 0.f) alive = false;
  }
  if (alive && depth >= rr_start) {
    float pr = fmaxf(fmaxf(Tn.x, Tn.y), Tn.z);
    pr = fminf(fmaxf(pr, LT_RR_MIN_F), 1.f);
    const float u_rr = unit_f32(state, inc);
    if (u_rr >= pr) {
      alive = false;
    } else {
      Tn.x /= pr;
      Tn.y /= pr;
      Tn.z /= pr;
    }
  }
  sg.scattered = true;
  sg.st_out = state;
  if (!alive) return false;
  sg.wrote_l = false;  // (the continuation's record carries L)
  sg.Tn = Tn;
  const float t = h.x;
  sg.out_o = make_float4(o.x + t * d.x, o.y + t * d.y, o.z + t * d.z, __int_as_float(p));
  sg.out_d = make_float4(wi.x, wi.y, wi.z, t_min);
  return true;
}

// One bounce of _trace (integrator.py:160-226) for every queued path:
// miss -> environment; hit -> emission; final segment stops; otherwise hit
// frame, 3 draws, BSDF sample, throughput, Russian roulette (4th draw), and
// the continuation ray is appended to the next queue: one atomic per block
// iteration (LT_SHADE_ITEMS x 128 entries), the block's rays laid out by
// direction octant (with ShadeArgs.octant_sort off, in shading order).
// With ShadeArgs.perm the queue is shaded in material-class order.
__global__ void __launch_bounds__(kShadeThreads, LT_SHADE_MIN_BLOCKS)
    k_shade(SceneView sc, ShadeArgs sa, RaygenArgs ra, PathArrays pa,
            const float4 *__restrict__ q_o, const float4 *__restrict__ q_d,
            const float4 *__restrict__ hits, const int32_t *__restrict__ count_in,
            float4 *__restrict__ n_o, float4 *__restrict__ n_d, int32_t *__restrict__ count_out) {
  // primary launch (depth 0 of a render batch): throughput 1, radiance 0 and
  // the PCG state are regenerated here instead of read back
  const bool primary = sa.primary != 0;
  const int n = *count_in;
  const int lane = threadIdx.x & 31;
  __shared__ int s_cnt[LT_DIR_BINS], s_off[LT_DIR_BINS], s_base;
  // this block iteration's continuation rays, staged for the grouped append
  __shared__ float4 s_ro[LT_SHADE_ITEMS * kShadeThreads], s_rd[LT_SHADE_ITEMS * kShadeThreads];
  for (int b = threadIdx.x; b < LT_DIR_BINS; b += blockDim.x) s_cnt[b] = 0;
  __syncthreads();
  // one queue entry: the segment, its path record, the continuation ray
  auto process = [&](int qi, bool &emit, float4 &out_o, float4 &out_d, int &cls) {
    if (qi < n) {
      const int q = sa.perm ? __ldg(&sa.perm[qi]) : qi;
      // queue entries and path state stream through (evict-first) so the
      // L2 keeps the triangle / shading records
      const float4 h = __ldcs(&hits[q]);
      int32_t p;
      f3 o, d;
      float4 T, L;
      ulonglong2 rs{};
      {
        // the ray record (regenerating the float64 camera ray here instead
        // measured slower: +17 % instructions on an issue-bound launch,
        // profiles/r01_v13_ncu_shade.txt)
        const float4 ro = primary ? make_float4((float)ra.cam[0], (float)ra.cam[1],
                                                (float)ra.cam[2], __int_as_float(q))
                                  : __ldcs(&q_o[q]);
        const float4 rd = __ldcs(&q_d[q]);
        p = __float_as_int(ro.w);
        LT_ASSERT(p >= 0 && p < sa.cap);
        o = mk(ro.x, ro.y, ro.z);
        d = mk(rd.x, rd.y, rd.z);
      }
      if (primary) {
        uint64_t st0, inc0;
        primary_rng(ra, p, st0, inc0);
        rs = make_ulonglong2(st0, inc0);
        T = make_float4(1.f, 1.f, 1.f, 0.f);
        L = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        uint64_t st0;
        ld_path(pa.S, p, T, L, st0);
        rs.x = st0;
      }
      Segment sg;
      emit = shade_segment(
          sc, sa.depth, sa.max_depth, sa.rr_start, sa.t_min, sa.warp_ctr != nullptr, p, h, o, d,
          T, L, rs.x,
          [&]() -> uint64_t {
            return primary ? rs.y : pa.inc ? __ldg(&pa.inc[p]) : path_inc(ra, p);
          },
          sg);
      cls = sg.cls;
      if (emit) {
        st_path(pa.S, p, sg.Tn, L, sg.st_out);
        out_o = sg.out_o;
        out_d = sg.out_d;
      }
      if (!emit && (sg.wrote_l || primary || (sg.scattered && pa.inc)))
        st_path(pa.S, p, T, L, sg.st_out);
    }
  };
  // LT_SHADE_ITEMS consecutive 128-entry ranges per block iteration; their
  // continuation rays are staged in shared memory (8 KB per block at 2, so
  // a shade CTA still fits beside the trace CTAs of the other lane) and
  // appended as one contiguous range of the next queue per block, laid out
  // by direction octant (counting sort), so a trace warp fetches rays with
  // nearby origins and similar directions; with octant_sort off the range
  // keeps shading order.  (s_cnt is zeroed before the loop and re-zeroed by
  // thread 0 once it has read the counts: two barriers per iteration.)
  // One instance of the segment code per kernel: every ordering option
  // runs the same arithmetic.
  const int span = LT_SHADE_ITEMS * kShadeThreads;
  for (int base = blockIdx.x * span; base < n; base += gridDim.x * span) {
    int bins[LT_SHADE_ITEMS], ranks[LT_SHADE_ITEMS];
#pragma unroll 1
    for (int it = 0; it < LT_SHADE_ITEMS; ++it) {
      bool emit = false;
      float4 out_o, out_d;
      int cls = -1;  // material class of the lane's hit (LT_FLAG_COUNT statistics)
      process(base + it * kShadeThreads + threadIdx.x, emit, out_o, out_d, cls);
      if (sa.warp_ctr) {
        // shading divergence: distinct material classes among a warp's lanes
        const unsigned act = __ballot_sync(kFull, cls >= 0);
        if (act) {
          const unsigned same = __match_any_sync(kFull, cls);
          const bool first_of_class = cls >= 0 && __ffs(same & act) - 1 == lane;
          const int distinct = __popc(__ballot_sync(kFull, first_of_class));
          if (lane == __ffs(act) - 1) {
            atomicAdd(&sa.warp_ctr[0], 1ull);
            atomicAdd(&sa.warp_ctr[1], distinct > 1 ? 1ull : 0ull);
            atomicAdd(&sa.warp_ctr[2], (unsigned long long)distinct);
          }
        }
      }
      bins[it] = -1;
      if (emit) {
        bins[it] = sa.octant_sort ? dir_bin(out_d) : 0;
        ranks[it] = atomicAdd(&s_cnt[bins[it]], 1);
        s_ro[it * kShadeThreads + threadIdx.x] = out_o;
        s_rd[it * kShadeThreads + threadIdx.x] = out_d;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int b = 0; b < LT_DIR_BINS; ++b) {
        s_off[b] = run;
        run += s_cnt[b];
        s_cnt[b] = 0;
      }
      s_base = run ? atomicAdd(count_out, run) : 0;
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < LT_SHADE_ITEMS; ++it)
      if (bins[it] >= 0) {
        const int slot = s_base + s_off[bins[it]] + ranks[it];
        LT_ASSERT(slot < sa.cap);
        __stcs(&n_o[slot], s_ro[it * kShadeThreads + threadIdx.x]);
        __stcs(&n_d[slot], s_rd[it * kShadeThreads + threadIdx.x]);
      }
  }
}

// Fused small pass: one thread runs a whole (pixel, sample) path -- the
// camera ray, then per segment the per-thread closest-hit traversal
// (traverse<true>: the wide layout, leaf test and tie rule of k_trace) and
// shade_segment -- and leaves its radiance in the path record for
// k_accumulate.  For passes too small to fill the GPU, where the
// wavefront's two dependent launches per segment are the cost (C1: 16 K
// paths); results are bit-identical to the wavefront path.
__global__ void __launch_bounds__(kShadeThreads)
    k_path_small(SceneView sc, RaygenArgs ra, int32_t max_depth, int32_t rr_start, PathArrays pa,
                 unsigned long long *__restrict__ ray_ctr) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned rays = 0;
  if (p < ra.n_paths) {
    f3 o, d;
    uint64_t state, inc;
    primary_ray(ra, p, o, d, state, inc);
    float4 T = make_float4(1.f, 1.f, 1.f, 0.f), L = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int32_t depth = 0; depth < max_depth; ++depth) {
      const HitRec hr =
          traverse<true, false>(sc, o, d, ra.t_min, __int_as_float(0x7f800000), nullptr, nullptr);
      ++rays;
      const float4 h = make_float4(hr.t, hr.u, hr.v, __int_as_float(hr.k));
      Segment sg;
      const bool cont = shade_segment(sc, depth, max_depth, rr_start, ra.t_min, false,
                                      (int32_t)p, h, o, d, T, L, state,
                                      [&]() -> uint64_t { return inc; }, sg);
      state = sg.st_out;
      if (!cont) break;
      T = sg.Tn;
      o = mk(sg.out_o.x, sg.out_o.y, sg.out_o.z);
      d = mk(sg.out_d.x, sg.out_d.y, sg.out_d.z);
    }
    st_path(pa.S, p, T, L, state);
  }
  // closest-hit queries of the pass (ray_ctr[0], as k_trace counts them)
  for (int off = 16; off > 0; off >>= 1) rays += __shfl_xor_sync(kFull, rays, off);
  if ((threadIdx.x & 31) == 0 && rays) atomicAdd(ray_ctr, (unsigned long long)rays);
}

// ------------------------------------------------------------------ device layout
// Layout of a BVH built on the device (lt_scene_create without host BVH
// arrays): the binary-node list for the counter query and the 4-wide
// collapse, the same greedy largest-area expansion as the host path.

__global__ void k_internal_flags(const int32_t *__restrict__ count, int64_t nn,
                                 int32_t *__restrict__ flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nn) flags[i] = count[i] == 0 ? 1 : 0;
}

__global__ void k_internal_scatter(const int32_t *__restrict__ flags,
                                   const int32_t *__restrict__ scan, int64_t nn,
                                   int32_t *__restrict__ perm, int32_t *__restrict__ new_index) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  if (flags[i]) {
    new_index[i] = scan[i];
    perm[scan[i]] = (int32_t)i;
  } else {
    new_index[i] = -1;
  }
}

__device__ __forceinline__ double node_area(const double *__restrict__ bmin,
                                            const double *__restrict__ bmax, int32_t x) {
  const double *lo = bmin + 3 * (int64_t)x, *hi = bmax + 3 * (int64_t)x;
  const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  return dx * dy + dy * dz + dz * dx;
}

// Greedy largest-area expansion of binary node r into up to four children
// (ch, -1 padded); returns how many of them are internal.
__device__ __forceinline__ int collapse_node(const double *__restrict__ bmin,
                                             const double *__restrict__ bmax,
                                             const int32_t *__restrict__ left,
                                             const int32_t *__restrict__ right,
                                             const int32_t *__restrict__ count, int32_t r,
                                             int32_t (&ch)[4], int (&dep)[4]) {
  ch[0] = left[r];
  ch[1] = right[r];
  ch[2] = ch[3] = -1;
  dep[0] = dep[1] = 1;  // binary levels below r
  dep[2] = dep[3] = 0;
  int nc = 2;
  while (nc < 4) {
    int pick = -1;
    double best_area = -1.0;
    for (int k = 0; k < nc; ++k)
      if (count[ch[k]] == 0) {
        const double a = node_area(bmin, bmax, ch[k]);
        if (a > best_area) {
          best_area = a;
          pick = k;
        }
      }
    if (pick < 0) break;
    const int32_t x = ch[pick];
    const int dx = dep[pick] + 1;
    for (int k = nc; k > pick + 1; --k) {
      ch[k] = ch[k - 1];
      dep[k] = dep[k - 1];
    }
    ch[pick] = left[x];
    ch[pick + 1] = right[x];
    dep[pick] = dep[pick + 1] = dx;
    ++nc;
  }
  int internal = 0;
  for (int k = 0; k < 4; ++k) internal += (ch[k] >= 0 && count[ch[k]] == 0) ? 1 : 0;
  return internal;
}

// The whole collapse in one CTA: a FIFO of binary roots processed 1024 at a
// time (wide node id = FIFO position, i.e. breadth-first, the numbering of
// the level-by-level launches) -- one launch instead of ~4 per level plus a
// host synchronization per level.  Alongside each FIFO entry: its binary
// depth and the traversal-stack entries pending when a ray reaches it (its
// ancestors' hit siblings, at most nchildren - 1 per wide level); out[1] =
// the deepest traversal stack the wide tree can need, out[2] = the binary
// tree's depth (the counter query's stack), both checked against LT_STACK.
__global__ void __launch_bounds__(1024)
    k_collapse_all(const double *__restrict__ bmin, const double *__restrict__ bmax,
                   const int32_t *__restrict__ left, const int32_t *__restrict__ right,
                   const int32_t *__restrict__ count, int32_t *__restrict__ fifo,
                   int32_t *__restrict__ wide_children, int32_t *__restrict__ wide_of,
                   int32_t *__restrict__ out) {
  __shared__ int s_warp[32];
  __shared__ int s_tail;
  __shared__ int s_stack, s_depth;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // fifo layout: [node ids | binary depth | pending stack entries], capacity
  // = internal node count, passed as out[0] on entry
  const int cap = out[0];
  int32_t *f_dep = fifo + cap, *f_pend = fifo + 2 * (int64_t)cap;
  __syncthreads();
  if (tid == 0) {
    fifo[0] = 0;  // the root (binary node 0)
    f_dep[0] = 0;
    f_pend[0] = 0;
    s_tail = 1;
    s_stack = 0;
    s_depth = 0;
  }
  __syncthreads();
  int head = 0;
  int my_stack = 0, my_depth = 0;
  while (head < s_tail) {
    const int tail = s_tail;
    const int i = head + tid;
    int32_t ch[4] = {-1, -1, -1, -1};
    int dep[4] = {0, 0, 0, 0};
    int kids = 0, depth = 0, pend = 0, nch = 0;
    if (i < tail) {
      const int32_t r = fifo[i];
      depth = f_dep[i];
      pend = f_pend[i];
      wide_of[r] = i;
      kids = collapse_node(bmin, bmax, left, right, count, r, ch, dep);
      for (int k = 0; k < 4; ++k) {
        wide_children[4 * (int64_t)i + k] = ch[k];
        if (ch[k] >= 0) {
          ++nch;
          my_depth = max(my_depth, depth + dep[k]);
        }
      }
      my_stack = max(my_stack, pend + nch - 1);
    }
    // block exclusive scan of the internal-children counts
    int x = kids;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int excl = x - kids + (warp ? s_warp[warp - 1] : 0);
    int j = tail + excl;
    for (int k = 0; k < 4; ++k)
      if (ch[k] >= 0 && count[ch[k]] == 0) {
        fifo[j] = ch[k];
        f_dep[j] = depth + dep[k];
        f_pend[j] = pend + nch - 1;
        ++j;
      }
    const int total = s_warp[(blockDim.x >> 5) - 1];
    __syncthreads();
    if (tid == 0) s_tail = tail + total;
    head = min(head + (int)blockDim.x, tail);
    __syncthreads();
  }
  atomicMax(&s_stack, my_stack);
  atomicMax(&s_depth, my_depth);
  __syncthreads();
  if (tid == 0) {
    out[0] = s_tail;
    out[1] = s_stack;
    out[2] = s_depth;
  }
}


void launch_internal_flags(const int32_t *count, int64_t nn, int32_t *flags, cudaStream_t st) {
  if (nn > 0) k_internal_flags<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(count, nn, flags);
}
void launch_internal_scatter(const int32_t *flags, const int32_t *scan, int64_t nn,
                             int32_t *perm, int32_t *new_index, cudaStream_t st) {
  if (nn > 0)
    k_internal_scatter<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(flags, scan, nn, perm,
                                                                      new_index);
}
void launch_collapse_all(const double *bmin, const double *bmax, const int32_t *left,
                         const int32_t *right, const int32_t *count, int32_t *fifo,
                         int32_t *wide_children, int32_t *wide_of, int32_t *n_wide,
                         cudaStream_t st) {
  k_collapse_all<<<1, 1024, 0, st>>>(bmin, bmax, left, right, count, fifo, wide_children,
                                     wide_of, n_wide);
}

// ------------------------------------------------------------------ env map

__global__ void k_expand_rgb(const float *__restrict__ rgb, int64_t n, float4 *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_float4(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], 0.f);
}

void launch_expand_rgb(const float *rgb, int64_t n, float4 *out, cudaStream_t st) {
  if (n > 0) k_expand_rgb<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rgb, n, out);
}

// ------------------------------------------------------------------ pixel order

__global__ void k_pixel_list(int32_t W, int32_t H, int32_t T, int32_t rank, int32_t n_ranks,
                             const int32_t *__restrict__ tile_start, int32_t *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)W * H) return;
  const int32_t y = (int32_t)(i / W), x = (int32_t)(i - (int64_t)y * W);
  const int32_t ntx = (W + T - 1) / T;
  const int32_t tx = x / T, ty = y / T;
  const int32_t tile = ty * ntx + tx;
  if (tile % n_ranks != rank) return;
  const int32_t w = min(W, (tx + 1) * T) - tx * T;
  out[tile_start[tile / n_ranks] + (y - ty * T) * w + (x - tx * T)] = (int32_t)i;
}

void launch_pixel_list(int32_t width, int32_t height, int32_t tile, int32_t rank, int32_t n_ranks,
                       const int32_t *tile_start, int32_t *out, cudaStream_t st) {
  const int64_t n = (int64_t)width * height;
  if (n <= 0) return;
  k_pixel_list<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(width, height, tile, rank, n_ranks,
                                                            tile_start, out);
}

// ------------------------------------------------------------------ accumulate

// Per-pixel sum of the batch's finite samples in sample order, plus valid /
// invalid counts (integrator.py:266-272; the mean is sum / valid).
__global__ void k_accumulate(AccumArgs aa, const float4 *__restrict__ S,
                             float *__restrict__ accum, uint32_t *__restrict__ valid,
                             uint32_t *__restrict__ invalid) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= aa.n_pix) return;
  const int64_t pix =
      aa.pix_list ? (int64_t)aa.pix_list[aa.pix_offset + i] : aa.pix_offset + i;
  float r = accum[3 * pix + 0], g = accum[3 * pix + 1], b = accum[3 * pix + 2];
  uint32_t nv = valid[pix], ni = invalid[pix];
  for (int64_t s = 0; s < aa.n_samples; ++s) {
    const int64_t p = s * aa.n_pix + i;
    const float4 sa = __ldcs(&S[2 * p]), sb = __ldcs(&S[2 * p + 1]);
    const float3 x = make_float3(sa.w, sb.x, sb.y);
    if (isfinite(x.x) && isfinite(x.y) && isfinite(x.z)) {
      r += x.x;
      g += x.y;
      b += x.z;
      ++nv;
    } else {
      ++ni;
    }
  }
  accum[3 * pix + 0] = r;
  accum[3 * pix + 1] = g;
  accum[3 * pix + 2] = b;
  valid[pix] = nv;
  invalid[pix] = ni;
}

// ------------------------------------------------------------------ ray I/O

__global__ void k_pack_rays_f32(const float *__restrict__ o, const float *__restrict__ d,
                                int64_t n, float t_min, float t_max, float4 *__restrict__ q_o,
                                float4 *__restrict__ q_d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  q_o[i] = make_float4(o[3 * i], o[3 * i + 1], o[3 * i + 2], t_max);
  q_d[i] = make_float4(d[3 * i], d[3 * i + 1], d[3 * i + 2], t_min);
}

__global__ void k_pack_rays_f64(const double *__restrict__ o, const double *__restrict__ d,
                                int64_t n, float t_min, float t_max, float4 *__restrict__ q_o,
                                float4 *__restrict__ q_d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  q_o[i] = make_float4((float)o[3 * i], (float)o[3 * i + 1], (float)o[3 * i + 2], t_max);
  q_d[i] = make_float4((float)d[3 * i], (float)d[3 * i + 1], (float)d[3 * i + 2], t_min);
}

__global__ void k_unpack_hits(SceneView sc, const float4 *__restrict__ hits, int64_t n,
                              int32_t *__restrict__ idx32, float *__restrict__ t32,
                              int64_t *__restrict__ idx64, double *__restrict__ t64,
                              double *__restrict__ uv64) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 h = hits[i];
  const int32_t k = __float_as_int(h.w);
  const int32_t orig = k >= 0 ? __float_as_int(__ldg(&sc.tris[LT_TRI_F4 * (int64_t)k]).w) : -1;
  const float t = k >= 0 ? h.x : __int_as_float(0x7f800000);
  if (idx32) idx32[i] = orig;
  if (t32) t32[i] = t;
  if (idx64) idx64[i] = orig;
  if (t64) t64[i] = (double)t;
  if (uv64) {
    uv64[2 * i] = k >= 0 ? (double)h.y : 0.0;
    uv64[2 * i + 1] = k >= 0 ? (double)h.z : 0.0;
  }
}

// Exhaustive closest hit (brute_force_intersect_batch, bvh.py:586-610,
// 694-701) with the traversal's own fp32 Moller-Trumbore and (t, original
// index) tie rule: one ray per thread, the leaf-ordered triangles streamed
// through shared memory a block-sized tile at a time.  Its result equals the
// BVH traversal's exactly (the closest hit is a lexicographic minimum and
// the traversal's boxes are conservative) -- the GPU twin of the
// reference's test_bvh.py:91-100 check.
__global__ void __launch_bounds__(128)
    k_brute_force(SceneView sc, int64_t n_tris, const float4 *__restrict__ q_o,
                  const float4 *__restrict__ q_d, int64_t n, float4 *__restrict__ hits) {
  __shared__ float4 tile[3 * 128];
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = q < n;
  const float4 ro = live ? q_o[q] : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 rd = live ? q_d[q] : make_float4(0.f, 0.f, 1.f, 0.f);
  const f3 o = mk(ro.x, ro.y, ro.z), d = mk(rd.x, rd.y, rd.z);
  HitRec best{ro.w, 0.f, 0.f, -1};
  int32_t best_orig = 0x7fffffff;
  for (int64_t base = 0; base < n_tris; base += 128) {
    const int64_t k = base + threadIdx.x;
    __syncthreads();
    if (k < n_tris)
      for (int c = 0; c < 3; ++c) tile[3 * threadIdx.x + c] = __ldg(&sc.tris[LT_TRI_F4 * k + c]);
    __syncthreads();
    const int cnt = n_tris - base < 128 ? (int)(n_tris - base) : 128;
    if (live)
      for (int j = 0; j < cnt; ++j)
        mt_test(o, d, rd.w, tile[3 * j], tile[3 * j + 1], tile[3 * j + 2], (int32_t)(base + j),
                best, best_orig);
  }
  if (live) hits[q] = make_float4(best.t, best.u, best.v, __int_as_float(best.k));
}

void launch_brute_force(const SceneView &sc, int64_t n_tris, const float4 *q_o,
                        const float4 *q_d, int64_t n, float4 *hits, cudaStream_t st) {
  if (n > 0)
    k_brute_force<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(sc, n_tris, q_o, q_d, n, hits);
}

// ------------------------------------------------------------------ display

// tonemap.py:18-61 (PBR Neutral -> sRGB -> half-up u8), float64 arithmetic
__global__ void k_tonemap_u8(const float *__restrict__ lin, int64_t n_pixels,
                             uint8_t *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_pixels) return;
  const double kStart = 0.8 - 0.04, kDesat = 0.15;
  double c[3] = {lin[3 * i], lin[3 * i + 1], lin[3 * i + 2]};
  const double x = fmin(c[0], fmin(c[1], c[2]));
  const double offset = x < 0.08 ? x - 6.25 * x * x : 0.04;
  for (int k = 0; k < 3; ++k) c[k] -= offset;
  const double peak = fmax(c[0], fmax(c[1], c[2]));
  const double dd = 1.0 - kStart;
  const double new_peak = 1.0 - dd * dd / (peak + dd - kStart);
  const bool compress = peak > kStart;
  const double gg = compress ? 1.0 - 1.0 / (kDesat * (peak - new_peak) + 1.0) : 0.0;
  for (int k = 0; k < 3; ++k) {
    double v = c[k];
    if (compress) v = (v * (new_peak / peak)) * (1.0 - gg) + new_peak * gg;
    v = fmin(fmax(v, 0.0), 1.0);
    v = v <= 0.0031308 ? 12.92 * v : 1.055 * pow(v, 1.0 / 2.4) - 0.055;
    v = floor(255.0 * fmin(fmax(v, 0.0), 1.0) + 0.5);
    out[3 * i + k] = (uint8_t)v;
  }
}

// ------------------------------------------------------------------ BSDF / any-hit queries

__device__ __forceinline__ f3 load3(const double *a, int64_t i) {
  return f3{(float)a[3 * i], (float)a[3 * i + 1], (float)a[3 * i + 2]};
}

// eval_bsdf / pdf_bsdf (material.py:389-407) with the shade kernel's code
__global__ void k_bsdf_eval(const GpuMaterial *__restrict__ mats, const double *__restrict__ wo,
                            const double *__restrict__ wi, const double *__restrict__ nrm,
                            const int32_t *__restrict__ front, int64_t n, double *__restrict__ f,
                            double *__restrict__ pdf) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const GpuMaterial mt = mats[i];
  f3 v;
  float p;
  eval_material(load3(wo, i), load3(wi, i), load3(nrm, i), mt, front ? front[i] != 0 : true, v,
                p);
  f[3 * i] = v.x;
  f[3 * i + 1] = v.y;
  f[3 * i + 2] = v.z;
  pdf[i] = p;
}

// sample_bsdf (material.py:410-426): the draws are rounded toward zero to
// fp32 as the shade kernel's unit_f32 does
__global__ void k_bsdf_sample(const GpuMaterial *__restrict__ mats, const double *__restrict__ wo,
                              const double *__restrict__ nrm, const double *__restrict__ u,
                              const int32_t *__restrict__ front, int64_t n,
                              int32_t *__restrict__ ok, double *__restrict__ wi,
                              double *__restrict__ wgt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const GpuMaterial mt = mats[i];
  f3 w{0.f, 0.f, 0.f}, g{0.f, 0.f, 0.f};
  const bool r = sample_material(load3(wo, i), load3(nrm, i), mt, front ? front[i] != 0 : true,
                                 __double2float_rz(u[3 * i]), __double2float_rz(u[3 * i + 1]),
                                 __double2float_rz(u[3 * i + 2]), w, g);
  ok[i] = r ? 1 : 0;
  wi[3 * i] = r ? w.x : 0.0;
  wi[3 * i + 1] = r ? w.y : 0.0;
  wi[3 * i + 2] = r ? w.z : 0.0;
  wgt[3 * i] = r ? g.x : 0.0;
  wgt[3 * i + 1] = r ? g.y : 0.0;
  wgt[3 * i + 2] = r ? g.z : 0.0;
}

__global__ void k_occluded(SceneView sc, const float4 *__restrict__ q_o,
                           const float4 *__restrict__ q_d, int64_t n,
                           int32_t *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 ro = q_o[i], rd = q_d[i];
  out[i] = occluded(sc, mk(ro.x, ro.y, ro.z), mk(rd.x, rd.y, rd.z), rd.w, ro.w) ? 1 : 0;
}

void launch_bsdf_eval(const GpuMaterial *mats, const double *wo, const double *wi,
                      const double *nrm, const int32_t *front, int64_t n, double *f, double *pdf,
                      cudaStream_t st) {
  if (n > 0)
    k_bsdf_eval<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(mats, wo, wi, nrm, front, n, f, pdf);
}

void launch_bsdf_sample(const GpuMaterial *mats, const double *wo, const double *nrm,
                        const double *u, const int32_t *front, int64_t n, int32_t *ok, double *wi,
                        double *wgt, cudaStream_t st) {
  if (n > 0)
    k_bsdf_sample<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(mats, wo, nrm, u, front, n, ok, wi,
                                                               wgt);
}

void launch_occluded(const SceneView &sc, const float4 *q_o, const float4 *q_d, int64_t n,
                     int32_t *out, cudaStream_t st) {
  if (n > 0) k_occluded<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(sc, q_o, q_d, n, out);
}

// ------------------------------------------------------------------ probe

// Streaming read of `n4` float4 (grid-stride, 4 independent loads in flight
// per thread); the bandwidth probe behind lt_read_bandwidth.
__global__ void k_read_probe(const float4 *__restrict__ src, int64_t n4, int passes,
                             float *__restrict__ sink) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int pass = 0; pass < passes; ++pass) {
    // rotate the starting block per pass so each pass reads other lines
    int64_t i = ((blockIdx.x + pass * 37) % gridDim.x) * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
      const float4 a = __ldcg(src + i), b = __ldcg(src + i + stride);
      const float4 c = __ldcg(src + i + 2 * stride), d = __ldcg(src + i + 3 * stride);
      acc += a.x + a.w + b.y + b.z + c.x + c.w + d.y + d.z;
    }
    for (; i < n4; i += stride) {
      const float4 a = __ldcg(src + i);
      acc += a.x + a.w;
    }
  }
  if (acc == 123.456f) sink[threadIdx.x] = acc;  // keeps the loads alive
}

void launch_read_probe(const float4 *src, int64_t n4, int passes, float *sink, int grid,
                       cudaStream_t st) {
  k_read_probe<<<grid, 512, 0, st>>>(src, n4, passes, sink);
}

// ------------------------------------------------------------------ launchers

const void *trace_kernel_ptr(bool count) {
  return count ? (const void *)k_trace<true> : (const void *)k_trace<false>;
}
const void *shade_kernel_ptr() { return (const void *)k_shade; }

void launch_flatten_nodes(const double *bmin, const double *bmax, const int32_t *left,
                          const int32_t *right, const int32_t *first, const int32_t *count,
                          const int32_t *perm, const int32_t *new_index, int64_t n_internal,
                          float4 *out, cudaStream_t st) {
  if (n_internal <= 0) return;
  k_flatten_nodes<<<(unsigned)((n_internal + 255) / 256), 256, 0, st>>>(
      bmin, bmax, left, right, first, count, perm, new_index, n_internal, out);
}

void launch_flatten_wide(const double *bmin, const double *bmax, const int32_t *first,
                         const int32_t *count, const int32_t *children, const int32_t *wide_of,
                         int64_t n_wide, float4 *out, cudaStream_t st) {
  if (n_wide <= 0) return;
  k_flatten_wide<<<(unsigned)((n_wide + 255) / 256), 256, 0, st>>>(bmin, bmax, first, count,
                                                                   children, wide_of, n_wide, out);
}

void launch_leaf_end(const int32_t *first, const int32_t *count, int64_t n_nodes,
                     uint8_t *leaf_end, cudaStream_t st) {
  if (n_nodes <= 0) return;
  k_leaf_end<<<(unsigned)((n_nodes + 255) / 256), 256, 0, st>>>(first, count, n_nodes, leaf_end);
}

void launch_flatten_tris(const double *v0, const double *v1, const double *v2, const double *n0,
                         const double *n1, const double *n2, const int32_t *mat_index,
                         const int32_t *order, const uint8_t *leaf_end, int64_t n, float4 *tris,
                         float4 *shade, cudaStream_t st) {
  k_flatten_tris<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v0, v1, v2, n0, n1, n2, mat_index,
                                                              order, leaf_end, n, tris, shade);
}

void launch_rng_tables(const RaygenArgs &ra, int64_t n_samples, uint64_t *inc_tab,
                       uint64_t *init_tab, cudaStream_t st) {
  const int64_t n = ra.n_pix > n_samples ? ra.n_pix : n_samples;
  if (n <= 0) return;
  k_rng_tables<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ra, n_samples, inc_tab, init_tab);
}

void launch_raygen(const RaygenArgs &ra, const PathArrays &pa, float4 *q_o, float4 *q_d,
                   int32_t *count0, cudaStream_t st) {
  const int64_t n = ra.n_paths > 0 ? ra.n_paths : 1;
  k_raygen<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ra, pa, q_o, q_d, count0);
}

void launch_raygen_explicit(const double *o, const double *d, const uint64_t *state,
                            const uint64_t *inc, int64_t n, float t_min, const PathArrays &pa,
                            float4 *q_o, float4 *q_d, int32_t *count0, cudaStream_t st) {
  const int64_t m = n > 0 ? n : 1;
  k_raygen_explicit<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(o, d, state, inc, n, t_min, pa,
                                                                 q_o, q_d, count0);
}

void launch_gather_explicit(const PathArrays &pa, int64_t n, double *rgb, uint64_t *state_out,
                            cudaStream_t st) {
  if (n <= 0) return;
  k_gather_explicit<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pa, n, rgb, state_out);
}

size_t trace_smem_bytes() { return (size_t)kShortStack * kTraceThreads * 8; }

cudaError_t launch_trace(const SceneView &sc, bool count_work, int grid,
                         const cudaAccessPolicyWindow *window, const float4 *q_o,
                         const float4 *q_d, const int32_t *count, int32_t *fetch, float4 *hits,
                         unsigned long long *ray_ctr, float4 cam_o, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTraceThreads);
  cfg.dynamicSmemBytes = trace_smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (window) {
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow = *window;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  if (count_work)
    return cudaLaunchKernelEx(&cfg, k_trace<true>, sc, q_o, q_d, count, fetch, hits, ray_ctr,
                              cam_o);
  return cudaLaunchKernelEx(&cfg, k_trace<false>, sc, q_o, q_d, count, fetch, hits, ray_ctr,
                            cam_o);
}

void launch_trace_rays(const SceneView &sc, const float4 *q_o, const float4 *q_d, int64_t n,
                       float4 *hits, int32_t *nodes, int32_t *tests, cudaStream_t st) {
  if (n <= 0) return;
  const unsigned grid = (unsigned)((n + kTraceThreads - 1) / kTraceThreads);
  if (nodes)
    k_trace_rays<true><<<grid, kTraceThreads, 0, st>>>(sc, q_o, q_d, n, hits, nodes, tests);
  else
    k_trace_rays<false><<<grid, kTraceThreads, 0, st>>>(sc, q_o, q_d, n, hits, nullptr, nullptr);
}

cudaError_t launch_shade(const SceneView &sc, const ShadeArgs &sa, const PathArrays &pa, int grid,
                         const cudaAccessPolicyWindow *window, const RaygenArgs *rargs,
                         bool primary, const float4 *q_o, const float4 *q_d, const float4 *hits,
                         const int32_t *count_in, float4 *n_o, float4 *n_d, int32_t *count_out,
                         cudaStream_t st) {
  const RaygenArgs ra = rargs ? *rargs : RaygenArgs{};
  ShadeArgs s2 = sa;
  s2.primary = primary && rargs ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kShadeThreads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (window) {
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow = *window;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, k_shade, sc, s2, ra, pa, q_o, q_d, hits, count_in, n_o, n_d,
                            count_out);
}

void launch_path_small(const SceneView &sc, const RaygenArgs &ra, int32_t max_depth,
                       int32_t rr_start, const PathArrays &pa, unsigned long long *ray_ctr,
                       cudaStream_t st) {
  if (ra.n_paths <= 0) return;
  const int grid = (int)((ra.n_paths + kShadeThreads - 1) / kShadeThreads);
  k_path_small<<<grid, kShadeThreads, 0, st>>>(sc, ra, max_depth, rr_start, pa, ray_ctr);
}

void launch_accumulate(const AccumArgs &aa, const float4 *S, float *accum, uint32_t *valid,
                       uint32_t *invalid, cudaStream_t st) {
  if (aa.n_pix <= 0) return;
  k_accumulate<<<(unsigned)((aa.n_pix + 255) / 256), 256, 0, st>>>(aa, S, accum, valid, invalid);
}

void launch_pack_rays_f32(const float *o, const float *d, int64_t n, float t_min, float t_max,
                          float4 *q_o, float4 *q_d, cudaStream_t st) {
  if (n <= 0) return;
  k_pack_rays_f32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(o, d, n, t_min, t_max, q_o, q_d);
}

void launch_pack_rays_f64(const double *o, const double *d, int64_t n, float t_min, float t_max,
                          float4 *q_o, float4 *q_d, cudaStream_t st) {
  if (n <= 0) return;
  k_pack_rays_f64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(o, d, n, t_min, t_max, q_o, q_d);
}

void launch_unpack_hits(const SceneView &sc, const float4 *hits, int64_t n, int32_t *idx32,
                        float *t32, int64_t *idx64, double *t64, double *uv64, cudaStream_t st) {
  if (n <= 0) return;
  k_unpack_hits<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sc, hits, n, idx32, t32, idx64, t64,
                                                             uv64);
}

// Shading class of queue entry q (k_shade's divergence classes).
__device__ __forceinline__ int shade_class(const SceneView &sc, const float4 *__restrict__ hits,
                                           int q, bool scatter) {
  const int32_t k = __float_as_int(__ldg(&hits[q]).w);
  if (k < 0) return 0;
  if (!scatter) return 1;
  const uint32_t f = sc.mats[__float_as_int(__ldg(&sc.shade[4 * (int64_t)k]).w)].flags;
  if (f & MAT_DIFFUSE_ONLY) return 2;
  const uint32_t cg = f & (MAT_COAT | MAT_GLASS);
  return cg == 0 ? 3 : cg == MAT_COAT ? 4 : cg == MAT_GLASS ? 5 : 6;
}

__global__ void __launch_bounds__(256)
    k_class_count(SceneView sc, const float4 *__restrict__ hits, const int32_t *__restrict__ count,
                  int scatter, uint8_t *__restrict__ cls, int32_t *__restrict__ totals) {
  __shared__ int s_h[kShadeClasses];
  if (threadIdx.x < kShadeClasses) s_h[threadIdx.x] = 0;
  __syncthreads();
  const int n = *count;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int c = shade_class(sc, hits, q, scatter != 0);
    cls[q] = (uint8_t)c;
    atomicAdd(&s_h[c], 1);
  }
  __syncthreads();
  if (threadIdx.x < kShadeClasses && s_h[threadIdx.x])
    atomicAdd(&totals[threadIdx.x], s_h[threadIdx.x]);
}

// perm[class base + cursor] = q, each block reserving one range per class
__global__ void __launch_bounds__(256)
    k_class_scatter(const uint8_t *__restrict__ cls, const int32_t *__restrict__ count,
                    const int32_t *__restrict__ totals, int32_t *__restrict__ cursor,
                    int32_t *__restrict__ perm) {
  __shared__ int s_base[kShadeClasses], s_cnt[kShadeClasses], s_off[kShadeClasses];
  if (threadIdx.x == 0) {
    int run = 0;
    for (int c = 0; c < kShadeClasses; ++c) {
      s_base[c] = run;
      run += totals[c];
    }
  }
  const int n = *count;
  for (int b = blockIdx.x * blockDim.x; b < n; b += gridDim.x * blockDim.x) {
    if (threadIdx.x < kShadeClasses) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int q = b + threadIdx.x;
    int c = 0, r = 0;
    if (q < n) {
      c = cls[q];
      r = atomicAdd(&s_cnt[c], 1);
    }
    __syncthreads();
    if (threadIdx.x < kShadeClasses)
      s_off[threadIdx.x] =
          s_cnt[threadIdx.x] ? atomicAdd(&cursor[threadIdx.x], s_cnt[threadIdx.x]) : 0;
    __syncthreads();
    if (q < n) perm[s_base[c] + s_off[c] + r] = q;
    __syncthreads();
  }
}

void launch_material_sort(const SceneView &sc, const float4 *hits, const int32_t *count,
                          bool scatter, int grid, uint8_t *cls, int32_t *cls_ctr, int32_t *perm,
                          cudaStream_t st) {
  k_class_count<<<grid, 256, 0, st>>>(sc, hits, count, scatter ? 1 : 0, cls, cls_ctr);
  k_class_scatter<<<grid, 256, 0, st>>>(cls, count, cls_ctr, cls_ctr + kShadeClasses, perm);
}

// Final means of an accumulation, as the Python layer's
// sum.double() / max(valid, 1) and invalid as int64, in one pass.
__global__ void k_accum_finish(const float *__restrict__ sum, const uint32_t *__restrict__ valid,
                               const uint32_t *__restrict__ invalid, int64_t n_pix,
                               double *__restrict__ mean, int64_t *__restrict__ inv) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_pix) return;
  const double v = (double)max(valid[i], 1u);
  mean[3 * i + 0] = (double)sum[3 * i + 0] / v;
  mean[3 * i + 1] = (double)sum[3 * i + 1] / v;
  mean[3 * i + 2] = (double)sum[3 * i + 2] / v;
  inv[i] = (int64_t)invalid[i];
}

void launch_accum_finish(const float *sum, const uint32_t *valid, const uint32_t *invalid,
                         int64_t n_pix, double *mean, int64_t *inv, cudaStream_t st) {
  if (n_pix <= 0) return;
  k_accum_finish<<<(unsigned)((n_pix + 255) / 256), 256, 0, st>>>(sum, valid, invalid, n_pix,
                                                                  mean, inv);
}

void launch_tonemap_u8(const float *lin, int64_t n_pixels, uint8_t *out, cudaStream_t st) {
  if (n_pixels <= 0) return;
  k_tonemap_u8<<<(unsigned)((n_pixels + 255) / 256), 256, 0, st>>>(lin, n_pixels, out);
}

}  // namespace lt
