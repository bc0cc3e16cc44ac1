// lt_traverse.cuh -- closest-hit BVH traversal (bvh.py:359-425) in fp32.
//
// Structure: per-thread while-while traversal over the two-boxes-per-node
// layout (lt_device.cuh), near child first, far child pushed with its entry
// distance on a 64-entry per-thread stack, pop-time culling against the
// current best t (bvh.py:389-390).  The top BFS levels of the tree are read
// from shared memory when USE_SMEM.
//
// Semantics kept from the reference:
//   * slab test in compare/select form: an origin on a slab plane with a zero
//     direction component gives 0*inf = NaN, which keeps the running interval
//     (geometry.py:170-207); fminf/fmaxf on the clipped interval reproduce
//     "if t0 > tn: tn = t0" exactly for NaN t0;
//   * zero direction components (either sign) use +inf (bvh.py:367-369);
//   * Moller-Trumbore, double sided, |det| <= 1e-9 rejected, inclusive
//     [t_min, best_t] (geometry.py:138-167);
//   * ties on t go to the lower ORIGINAL triangle index (bvh.py:399), so the
//     result is independent of traversal order.
// Robustness: child exit distances are widened by LT_SLAB_WIDEN (a relative
// 4e-7, far below the 1e-7*extent padding's effect in float64), so fp32
// rounding cannot cull a box the float64 traversal would enter.
#pragma once
#include "lt_device.cuh"

struct HitRec {
  float t, u, v;
  int32_t k;  // leaf-order triangle position, -1 on miss
};

__device__ __forceinline__ void slab_axis(float lo, float hi, float o, float inv, float &tn,
                                          float &tf) {
  const float t0 = (lo - o) * inv;
  const float t1 = (hi - o) * inv;
  const bool sw = t0 > t1;
  const float a = sw ? t1 : t0;
  const float b = sw ? t0 : t1;
  tn = fmaxf(tn, a);  // NaN a keeps tn, as "if t0 > tn"
  tf = fminf(tf, b);  // NaN b keeps tf, as "if t1 < tf"
}

__device__ __forceinline__ bool slab(f3 o, f3 inv, float lox, float hix, float loy, float hiy,
                                     float loz, float hiz, float t_min, float t_max,
                                     float &t_enter) {
  float tn = t_min, tf = t_max;
  slab_axis(lox, hix, o.x, inv.x, tn, tf);
  slab_axis(loy, hiy, o.y, inv.y, tn, tf);
  slab_axis(loz, hiz, o.z, inv.z, tn, tf);
  t_enter = tn;
  return tn <= tf * LT_SLAB_WIDEN;
}

template <bool USE_SMEM, bool COUNT>
__device__ __forceinline__ HitRec traverse(const SceneView &sc, const float4 *top, f3 o, f3 d,
                                           float t_min, float t_max, int *n_nodes,
                                           int *n_tests) {
  const float kInf = __int_as_float(0x7f800000);
  const f3 inv{d.x == 0.f ? kInf : 1.f / d.x, d.y == 0.f ? kInf : 1.f / d.y,
               d.z == 0.f ? kInf : 1.f / d.z};
  HitRec best{t_max, 0.f, 0.f, -1};
  int32_t best_orig = 0x7fffffff;
  int nodes = 1, tests = 0;

  float t_root;
  if (!slab(o, inv, sc.root_lo[0], sc.root_hi[0], sc.root_lo[1], sc.root_hi[1], sc.root_lo[2],
            sc.root_hi[2], t_min, t_max, t_root)) {
    if (COUNT) {
      *n_nodes = nodes;
      *n_tests = tests;
    }
    return best;
  }

  int32_t stk_node[LT_STACK];
  float stk_t[LT_STACK];
  int sp = 0;
  int32_t node = sc.root_link;

  while (true) {
    // ---- internal nodes: descend until a leaf or a dead end
    while (node >= 0) {
      float4 a, b, c, e;
      if (USE_SMEM && node < sc.n_top) {
        const float4 *np = top + 4 * node;
        a = np[0];
        b = np[1];
        c = np[2];
        e = np[3];
      } else {
        const float4 *np = sc.nodes + 4 * (int64_t)node;
        a = __ldg(np + 0);
        b = __ldg(np + 1);
        c = __ldg(np + 2);
        e = __ldg(np + 3);
      }
      if (COUNT) nodes += 2;
      float tl, tr;
      const bool hl = slab(o, inv, a.x, a.y, a.z, a.w, c.x, c.y, t_min, best.t, tl);
      const bool hr = slab(o, inv, b.x, b.y, b.z, b.w, c.z, c.w, t_min, best.t, tr);
      const int32_t lc = __float_as_int(e.x), rc = __float_as_int(e.y);
      if (hl && hr) {
        const bool left_near = tl <= tr;  // bvh.py:414
        stk_node[sp] = left_near ? rc : lc;
        stk_t[sp] = left_near ? tr : tl;
        ++sp;
        node = left_near ? lc : rc;
      } else if (hl) {
        node = lc;
      } else if (hr) {
        node = rc;
      } else {
        node = LT_LINK_EXIT;  // pop below
        break;
      }
    }
    // ---- leaf: test its triangles (the last one carries the end flag)
    if (node != LT_LINK_EXIT) {
      int64_t k = ~node;
      while (true) {
        const float4 t0 = __ldg(&sc.tris[3 * k + 0]);
        const float4 t1 = __ldg(&sc.tris[3 * k + 1]);
        const float4 t2 = __ldg(&sc.tris[3 * k + 2]);
        if (COUNT) ++tests;
        // _mt_intersect, term order of geometry.py:143-166
        const float px = d.y * t2.z - d.z * t2.y;
        const float py = d.z * t2.x - d.x * t2.z;
        const float pz = d.x * t2.y - d.y * t2.x;
        const float det = t1.x * px + t1.y * py + t1.z * pz;
        const float inv_det = 1.f / det;
        const float sx = o.x - t0.x, sy = o.y - t0.y, sz = o.z - t0.z;
        const float u = (sx * px + sy * py + sz * pz) * inv_det;
        const float qx = sy * t1.z - sz * t1.y;
        const float qy = sz * t1.x - sx * t1.z;
        const float qz = sx * t1.y - sy * t1.x;
        const float v = (d.x * qx + d.y * qy + d.z * qz) * inv_det;
        const float t = (t2.x * qx + t2.y * qy + t2.z * qz) * inv_det;
        const bool det_ok = !(det >= -LT_DET_EPS_F && det <= LT_DET_EPS_F);
        const bool hit = det_ok && !(u < 0.f || u > 1.f) && !(v < 0.f || u + v > 1.f) &&
                         !(t < t_min || t > best.t);
        const int32_t orig = __float_as_int(t0.w);
        if (hit && (t < best.t || (t == best.t && orig < best_orig) || best.k < 0)) {
          best.t = t;
          best.u = u;
          best.v = v;
          best.k = (int32_t)k;
          best_orig = orig;
        }
        if (__float_as_int(t1.w) != 0) break;
        ++k;
      }
    }
    // ---- pop the next entry not culled by the current best t (bvh.py:389)
    const float cull = best.t * LT_SLAB_WIDEN;
    node = LT_LINK_EXIT;
    while (sp > 0) {
      --sp;
      if (!(stk_t[sp] > cull)) {
        node = stk_node[sp];
        break;
      }
    }
    if (node == LT_LINK_EXIT) break;
  }
  if (COUNT) {
    *n_nodes = nodes;
    *n_tests = tests;
  }
  return best;
}
