// lt_traverse.cuh -- closest-hit BVH traversal (bvh.py:359-425) in fp32.
//
// Two node layouts of the same host-built tree (lt_device.cuh):
//   * BVH2 records (the reference's nodes, children boxes in the parent):
//     used by the counter query so `traversal_counts_batch` keeps the
//     reference's per-node semantics;
//   * BVH4 records: the reference tree collapsed to 4-wide nodes (the same
//     leaves and boxes; intermediate levels skipped), used by the render and
//     closest-hit kernels.  The closest hit is a lexicographic minimum over
//     (t, original triangle index), so the grouping changes work, not
//     results.
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
//   * ties on t go to the lower ORIGINAL triangle index (bvh.py:399).
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

// Per-ray constants of the slab test: `inv` is the clamped inverse
// direction; `nx/ny/nz` index the wide node's (near, far) plane pair per
// axis in float4 units: the record stores [lo, hi, hi, lo] per axis a, and
// the pair starts at 4a + 2 sign(inv_a).
struct RaySlab {
  f3 o, inv;
  int nx, ny, nz;
};

__device__ __forceinline__ RaySlab ray_slab(f3 o, f3 d) {
  RaySlab r;
  r.o = o;
  r.inv = f3{fminf(fmaxf(1.f / d.x, -LT_INV_CLAMP), LT_INV_CLAMP),
             fminf(fmaxf(1.f / d.y, -LT_INV_CLAMP), LT_INV_CLAMP),
             fminf(fmaxf(1.f / d.z, -LT_INV_CLAMP), LT_INV_CLAMP)};
  r.nx = 2 * (int)(__float_as_uint(r.inv.x) >> 31);
  r.ny = 4 + 2 * (int)(__float_as_uint(r.inv.y) >> 31);
  r.nz = 8 + 2 * (int)(__float_as_uint(r.inv.z) >> 31);
  return r;
}

// _slab_intersect with a clipped interval [t_min, t_max] (min/max form)
__device__ __forceinline__ bool slab(const RaySlab &r, float lox, float hix, float loy, float hiy,
                                     float loz, float hiz, float t_min, float t_max,
                                     float &t_enter) {
  const float t0x = (lox - r.o.x) * r.inv.x, t1x = (hix - r.o.x) * r.inv.x;
  const float t0y = (loy - r.o.y) * r.inv.y, t1y = (hiy - r.o.y) * r.inv.y;
  const float t0z = (loz - r.o.z) * r.inv.z, t1z = (hiz - r.o.z) * r.inv.z;
  const float tn = fmax3f(fminf(t0x, t1x), fminf(t0y, t1y), fmaxf(fminf(t0z, t1z), t_min));
  const float tf = fmin3f(fmaxf(t0x, t1x), fmaxf(t0y, t1y), fminf(fmaxf(t0z, t1z), t_max));
  t_enter = tn;
  return tn <= tf * LT_SLAB_WIDEN;
}

// Two adjacent float4s with one 256-bit load (sm_100: LDG.E.256; the
// address is 32 B aligned).  Per lane a 32 B access costs ~1.3 L1
// wavefronts against 1 per 16 B access (tools/micro/ldg256.cu: 1.47x the
// record rate of 16 B loads on random 128 B records).
__device__ __forceinline__ void ldg_pair(const float4 *__restrict__ p, float4 &a, float4 &b) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
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

// All triangles of the leaf starting at leaf-order position `first` (the
// last one carries the end-of-leaf flag).
template <bool COUNT>
__device__ __forceinline__ void leaf_test(const SceneView &sc, uint32_t k, f3 o, f3 d, float t_min,
                                          HitRec &best, int32_t &best_orig, int &tests) {
  while (true) {
    LT_ASSERT(k < (uint32_t)sc.n_tris);
    const float4 t0 = __ldg(&sc.tris[LT_TRI_F4 * (size_t)k]);
    const float4 t1 = __ldg(&sc.tris[LT_TRI_F4 * (size_t)k + 1]);
    const float4 t2 = __ldg(&sc.tris[LT_TRI_F4 * (size_t)k + 2]);
    if (COUNT) ++tests;
    mt_test(o, d, t_min, t0, t1, t2, (int32_t)k, best, best_orig);
    if (__float_as_int(t1.w) != 0) break;
    ++k;
  }
}

__device__ __forceinline__ void cswap(float &ka, int32_t &la, float &kb, int32_t &lb) {
  const bool s = kb < ka;
  const float tk = s ? kb : ka;
  const int32_t tl = s ? lb : la;
  kb = s ? ka : kb;
  lb = s ? la : lb;
  ka = tk;
  la = tl;
}

// One BVH4 node visit: the four child boxes against [t_min, best_t], the
// hits sorted by entry distance (5-comparator network), returned nearest
// first in (l0..l3) with +inf keys for misses / empty slots.
struct Hits4 {
  float k0, k1, k2, k3;
  int32_t l0, l1, l2, l3;
};

// The ray's direction signs pick the near and far plane arrays, so each
// child needs no per-axis min/max: for a box with lo <= hi, (lo - o) * inv
// and (hi - o) * inv are ordered by the sign of inv (rounding is
// monotonic), so the entry / exit distances equal the min/max form's
// exactly.  Empty slots hold inverted infinite boxes and miss without a
// link check.
// (p0 - o) * inv and (p1 - o) * inv as one FADD2 + one FMUL2.
__device__ __forceinline__ void plane2(float p0, float p1, float o, float inv, float &t0,
                                       float &t1) {
  unsigned long long p, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(p0), "f"(p1));
  asm("{\n\t.reg .b64 ob, ib, d;\n\t"
      "mov.b64 ob, {%2, %2};\n\t"
      "mov.b64 ib, {%3, %3};\n\t"
      "sub.rn.f32x2 d, %1, ob;\n\t"
      "mul.rn.f32x2 %0, d, ib;\n\t}"
      : "=l"(r) : "l"(p), "f"(o), "f"(inv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(t0), "=f"(t1) : "l"(r));
}

// (a * s, b * s) as one FMUL2.
__device__ __forceinline__ void scale2(float a, float b, float sc, float &ra, float &rb) {
  unsigned long long p, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(a), "f"(b));
  asm("{\n\t.reg .b64 sb;\n\t"
      "mov.b64 sb, {%2, %2};\n\t"
      "mul.rn.f32x2 %0, %1, sb;\n\t}"
      : "=l"(r) : "l"(p), "f"(sc));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(ra), "=f"(rb) : "l"(r));
}

// The four child boxes of a wide node against [t_min, t_max] for one ray:
// entry distances in node (slot) order, +inf for misses / empty slots, and
// the node's links.
__device__ __forceinline__ void visit4_keys(const float4 *__restrict__ np, const RaySlab &rs,
                                            float t_min, float t_max, float (&key)[4],
                                            int4 &ln) {
  const float kInf = __int_as_float(0x7f800000);
  float4 nx, fx, ny, fy, nz, fz;
  ldg_pair(np + rs.nx, nx, fx);
  ldg_pair(np + rs.ny, ny, fy);
  ldg_pair(np + rs.nz, nz, fz);
  ln = __ldg(reinterpret_cast<const int4 *>(np + LT_NODE_LINKS));
  // sm_100 packed fp32 (FADD2 / FMUL2, one issue slot per two children;
  // the scalar origin / inverse are broadcast operands): same IEEE roundings
  // as the scalar form.
  float a0x, a1x, a2x, a3x, b0x, b1x, b2x, b3x;
  float a0y, a1y, a2y, a3y, b0y, b1y, b2y, b3y;
  float a0z, a1z, a2z, a3z, b0z, b1z, b2z, b3z;
  plane2(nx.x, nx.y, rs.o.x, rs.inv.x, a0x, a1x);
  plane2(nx.z, nx.w, rs.o.x, rs.inv.x, a2x, a3x);
  plane2(fx.x, fx.y, rs.o.x, rs.inv.x, b0x, b1x);
  plane2(fx.z, fx.w, rs.o.x, rs.inv.x, b2x, b3x);
  plane2(ny.x, ny.y, rs.o.y, rs.inv.y, a0y, a1y);
  plane2(ny.z, ny.w, rs.o.y, rs.inv.y, a2y, a3y);
  plane2(fy.x, fy.y, rs.o.y, rs.inv.y, b0y, b1y);
  plane2(fy.z, fy.w, rs.o.y, rs.inv.y, b2y, b3y);
  plane2(nz.x, nz.y, rs.o.z, rs.inv.z, a0z, a1z);
  plane2(nz.z, nz.w, rs.o.z, rs.inv.z, a2z, a3z);
  plane2(fz.x, fz.y, rs.o.z, rs.inv.z, b0z, b1z);
  plane2(fz.z, fz.w, rs.o.z, rs.inv.z, b2z, b3z);
  const float tn0 = fmax3f(a0x, a0y, fmaxf(a0z, t_min));
  const float tn1 = fmax3f(a1x, a1y, fmaxf(a1z, t_min));
  const float tn2 = fmax3f(a2x, a2y, fmaxf(a2z, t_min));
  const float tn3 = fmax3f(a3x, a3y, fmaxf(a3z, t_min));
  float tf0, tf1, tf2, tf3;
  scale2(fmin3f(b0x, b0y, fminf(b0z, t_max)), fmin3f(b1x, b1y, fminf(b1z, t_max)),
         LT_SLAB_WIDEN, tf0, tf1);
  scale2(fmin3f(b2x, b2y, fminf(b2z, t_max)), fmin3f(b3x, b3y, fminf(b3z, t_max)),
         LT_SLAB_WIDEN, tf2, tf3);
  key[0] = tn0 <= tf0 ? tn0 : kInf;
  key[1] = tn1 <= tf1 ? tn1 : kInf;
  key[2] = tn2 <= tf2 ? tn2 : kInf;
  key[3] = tn3 <= tf3 ? tn3 : kInf;
}

__device__ __forceinline__ Hits4 visit4o(const float4 *__restrict__ np, const RaySlab &rs,
                                         float t_min, float t_max) {
  float key[4];
  int4 ln;
  visit4_keys(np, rs, t_min, t_max, key, ln);
  Hits4 h;
  h.k0 = key[0];
  h.k1 = key[1];
  h.k2 = key[2];
  h.k3 = key[3];
  h.l0 = ln.x;
  h.l1 = ln.y;
  h.l2 = ln.z;
  h.l3 = ln.w;
  cswap(h.k0, h.l0, h.k1, h.l1);
  cswap(h.k2, h.l2, h.k3, h.l3);
  cswap(h.k0, h.l0, h.k2, h.l2);
  cswap(h.k1, h.l1, h.k3, h.l3);
  cswap(h.k1, h.l1, h.k2, h.l2);
  return h;
}

// Pop-time cull distance for the current best t: a stacked entry whose entry
// distance exceeds it cannot hold a closer hit (bvh.py:389), with the same
// error allowance as the slab test.
__device__ __forceinline__ float cull_dist(float best_t) { return best_t * LT_SLAB_WIDEN; }

// Any-hit occlusion (_traverse_any, bvh.py:511-551): true as soon as any
// triangle is hit within [t_min, t_max]; wide layout, no ordering needed.
__device__ __forceinline__ bool occluded(const SceneView &sc, f3 o, f3 d, float t_min,
                                         float t_max) {
  const float kInf = __int_as_float(0x7f800000);
  const RaySlab rs = ray_slab(o, d);
  float t_root;
  if (!slab(rs, sc.root_lo[0], sc.root_hi[0], sc.root_lo[1], sc.root_hi[1], sc.root_lo[2],
            sc.root_hi[2], t_min, t_max, t_root))
    return false;
  int32_t stk[LT_STACK];
  int sp = 0;
  int32_t node = sc.wroot_link;
  HitRec best{t_max, 0.f, 0.f, -1};
  int32_t best_orig = 0x7fffffff;
  while (true) {
    while (node >= 0) {
      LT_ASSERT(node < sc.n_wide && sp + 3 <= LT_STACK);
      const Hits4 h = visit4o(sc.wnodes + LT_NODE_F4 * (int64_t)node, rs, t_min, t_max);
      if (h.k3 < kInf) stk[sp++] = h.l3;
      if (h.k2 < kInf) stk[sp++] = h.l2;
      if (h.k1 < kInf) stk[sp++] = h.l1;
      node = h.k0 < kInf ? h.l0 : LT_LINK_EXIT;
      if (node == LT_LINK_EXIT && sp > 0) node = stk[--sp];
    }
    if (node == LT_LINK_EXIT) return false;
    int tests = 0;
    leaf_test<false>(sc, ~(uint32_t)node, o, d, t_min, best, best_orig, tests);
    if (best.k >= 0) return true;
    if (sp == 0) return false;
    node = stk[--sp];
  }
}

// Per-thread traversal with a local-memory stack for the query kernels.
// WIDE: the BVH4 layout (closest-hit queries); otherwise the BVH2 layout
// with the reference's counters (traversal_counts_batch).
template <bool WIDE, bool COUNT>
__device__ __forceinline__ HitRec traverse(const SceneView &sc, f3 o, f3 d, float t_min,
                                           float t_max, int *n_nodes, int *n_tests) {
  const float kInf = __int_as_float(0x7f800000);
  const RaySlab rs = ray_slab(o, d);
  HitRec best{t_max, 0.f, 0.f, -1};
  int32_t best_orig = 0x7fffffff;
  int nodes = 1, tests = 0;
  float t_root;
  if (slab(rs,sc.root_lo[0], sc.root_hi[0], sc.root_lo[1], sc.root_hi[1], sc.root_lo[2],
           sc.root_hi[2], t_min, t_max, t_root)) {
    int32_t stk_node[LT_STACK];
    float stk_t[LT_STACK];
    int sp = 0;
    int32_t node = WIDE ? sc.wroot_link : sc.root_link;
    while (true) {
      while (node >= 0) {
        if (WIDE) {
          LT_ASSERT(node < sc.n_wide && sp + 3 <= LT_STACK);
          const Hits4 h = visit4o(sc.wnodes + LT_NODE_F4 * (int64_t)node, rs, t_min, best.t);
          if (COUNT) nodes += 4;
          if (h.k3 < kInf) { stk_node[sp] = h.l3; stk_t[sp] = h.k3; ++sp; }
          if (h.k2 < kInf) { stk_node[sp] = h.l2; stk_t[sp] = h.k2; ++sp; }
          if (h.k1 < kInf) { stk_node[sp] = h.l1; stk_t[sp] = h.k1; ++sp; }
          node = h.k0 < kInf ? h.l0 : LT_LINK_EXIT;
        } else {
          LT_ASSERT(sp + 1 <= LT_STACK);
          const float4 *np = sc.nodes + 4 * (int64_t)node;
          const float4 a = __ldg(np + 0), b = __ldg(np + 1), c = __ldg(np + 2), e = __ldg(np + 3);
          if (COUNT) nodes += 2;
          float tl, tr;
          const bool hl = slab(rs,a.x, a.y, a.z, a.w, c.x, c.y, t_min, best.t, tl);
          const bool hr = slab(rs,b.x, b.y, b.z, b.w, c.z, c.w, t_min, best.t, tr);
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
      }
      if (node != LT_LINK_EXIT) leaf_test<COUNT>(sc, ~(uint32_t)node, o, d, t_min, best,
                                                 best_orig, tests);
      const float cull = cull_dist(best.t);
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
