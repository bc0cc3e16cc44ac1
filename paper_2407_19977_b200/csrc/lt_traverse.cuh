// lt_traverse.cuh -- closest-hit BVH traversal (bvh.py:359-425) in fp32.
//
// Semantics kept from the reference:
//   * slab test (geometry.py:170-207): a zero direction component gives an
//     "infinite" inverse (bvh.py:367-369).  The reference's compare/select
//     form keeps the running interval when 0*inf = NaN (origin exactly on a
//     slab plane); here the inverse is clamped to +-2^64 instead, so that
//     product is an exact 0 and the plain min/max form yields the same
//     decision (inside-or-on-the-slab passes, outside misses) with no NaN --
//     identical except for origins within ~1e-20 of a plane;
//   * Moller-Trumbore, double sided, |det| <= 1e-9 rejected, inclusive
//     [t_min, best_t] (geometry.py:138-167), reference term order;
//   * ties on t go to the lower ORIGINAL triangle index (bvh.py:399), so the
//     result is independent of traversal order.
// Robustness: child exit distances are widened by LT_SLAB_WIDEN (relative
// 4e-7) so fp32 rounding cannot cull a box the float64 traversal enters.
#pragma once
#include "lt_device.cuh"

struct HitRec {
  float t, u, v;
  int32_t k;  // leaf-order triangle position, -1 on miss
};

#define LT_INV_CLAMP 1.8446744e19f  // 2^64

__device__ __forceinline__ float fmin3f(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ f3 ray_inverse(f3 d) {
  return f3{fminf(fmaxf(1.f / d.x, -LT_INV_CLAMP), LT_INV_CLAMP),
            fminf(fmaxf(1.f / d.y, -LT_INV_CLAMP), LT_INV_CLAMP),
            fminf(fmaxf(1.f / d.z, -LT_INV_CLAMP), LT_INV_CLAMP)};
}

// _slab_intersect with a clipped interval [t_min, t_max]
__device__ __forceinline__ bool slab(f3 o, f3 inv, float lox, float hix, float loy, float hiy,
                                     float loz, float hiz, float t_min, float t_max,
                                     float &t_enter) {
  const float t0x = (lox - o.x) * inv.x, t1x = (hix - o.x) * inv.x;
  const float t0y = (loy - o.y) * inv.y, t1y = (hiy - o.y) * inv.y;
  const float t0z = (loz - o.z) * inv.z, t1z = (hiz - o.z) * inv.z;
  const float tn = fmax3f(fminf(t0x, t1x), fminf(t0y, t1y), fmaxf(fminf(t0z, t1z), t_min));
  const float tf = fmin3f(fmaxf(t0x, t1x), fmaxf(t0y, t1y), fminf(fmaxf(t0z, t1z), t_max));
  t_enter = tn;
  return tn <= tf * LT_SLAB_WIDEN;
}

// _mt_intersect (geometry.py:138-167) against the leaf-ordered record
// (v0, e1, e2); updates `best` with the reference's acceptance rule.
__device__ __forceinline__ void mt_test(f3 o, f3 d, float t_min, float4 t0, float4 t1, float4 t2,
                                        int32_t k, HitRec &best, int32_t &best_orig) {
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
    best.k = k;
    best_orig = orig;
  }
}

// Simple per-thread traversal with a local-memory stack: the query kernel
// (intersect_scene_batch / traversal counts).  The render path uses the
// persistent kernel in lt_kernels.cu.
template <bool COUNT>
__device__ __forceinline__ HitRec traverse(const SceneView &sc, f3 o, f3 d, float t_min,
                                           float t_max, int *n_nodes, int *n_tests) {
  const f3 inv = ray_inverse(d);
  HitRec best{t_max, 0.f, 0.f, -1};
  int32_t best_orig = 0x7fffffff;
  int nodes = 1, tests = 0;
  float t_root;
  if (slab(o, inv, sc.root_lo[0], sc.root_hi[0], sc.root_lo[1], sc.root_hi[1], sc.root_lo[2],
           sc.root_hi[2], t_min, t_max, t_root)) {
    int32_t stk_node[LT_STACK];
    float stk_t[LT_STACK];
    int sp = 0;
    int32_t node = sc.root_link;
    while (true) {
      while (node >= 0) {
        const float4 *np = sc.nodes + 4 * (int64_t)node;
        const float4 a = __ldg(np + 0), b = __ldg(np + 1), c = __ldg(np + 2), e = __ldg(np + 3);
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
          node = LT_LINK_EXIT;
        }
      }
      if (node != LT_LINK_EXIT) {
        int64_t k = ~node;
        while (true) {
          const float4 t0 = __ldg(&sc.tris[3 * k]), t1 = __ldg(&sc.tris[3 * k + 1]),
                       t2 = __ldg(&sc.tris[3 * k + 2]);
          if (COUNT) ++tests;
          mt_test(o, d, t_min, t0, t1, t2, (int32_t)k, best, best_orig);
          if (__float_as_int(t1.w) != 0) break;
          ++k;
        }
      }
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
  }
  if (COUNT) {
    *n_nodes = nodes;
    *n_tests = tests;
  }
  return best;
}
