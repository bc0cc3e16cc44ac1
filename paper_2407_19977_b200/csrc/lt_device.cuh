// lt_device.cuh -- device data layout and scalar device functions.
//
// HBM layout (all 16-byte aligned):
//   wnodes : LT_NODE_F4 x float4 per node of the host BVH collapsed to
//            4-wide (each wide node absorbs the largest-area internal
//            children of its binary node until it has 4 children); default
//            (224 B): per axis a = x, y, z the float4s
//            [4a .. 4a+3] = lo[4], hi[4], hi[4], lo[4] (the (near, far) pair
//            for a positive / negative inverse direction), f4[12] = 4 child
//            links (>= 0 wide node, < 0 leaf = ~first, INT_MIN empty slot),
//            f4[13] unused.  Boxes are the reference's float64 boxes rounded
//            outward; empty slots carry inverted infinite boxes.
//   nodes  : 4 x float4 per INTERNAL node of the host BVH; a node holds the
//            fp32 boxes of both children (rounded outward) and their links.
//              n0 = (L.lo.x, L.hi.x, L.lo.y, L.hi.y)
//              n1 = (R.lo.x, R.hi.x, R.lo.y, R.hi.y)
//              n2 = (L.lo.z, L.hi.z, R.lo.z, R.hi.z)
//              n3 = (link L, link R, -, -)   link >= 0: internal node,
//                                            link < 0: leaf, first = ~link
//            Internal nodes in the order of their index in the source
//            tree (the reference's numbering, or the device build's).
//   tris   : LT_TRI_F4 (3) x float4 per triangle in LEAF order (triangle_order)
//              (v0.xyz, original index), (e1.xyz, last-in-leaf flag),
//              (e2.xyz, 0); e1/e2 are rounded from the float64 differences.
//   shade  : 4 x float4 (64 B, one aligned half line) per triangle in leaf
//            order: (g.xyz = float64 normalize(e1 x e2), material index),
//            (n0.xyz, 0), (n1.xyz, 0), (n2.xyz, 0)
//   mats   : 128-byte GpuMaterial records, derived constants precomputed in
//            float64 on the host and rounded once.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// -DLT_CHECKS (the checked build, tools/checked_tests.sh): device asserts on
// every index the hot kernels derive (node / triangle / material ids, stack
// depth, queue slots, pixels); compiled out otherwise.
#ifdef LT_CHECKS
#include <cassert>
#define LT_ASSERT(c) assert(c)
#else
#define LT_ASSERT(c) ((void)0)
#endif

#define LT_PI_F 3.14159265358979323846f
#define LT_INV_PI_F 0.318309886183790671538f
#define LT_DET_EPS_F 1e-9f      // geometry.py:17
#define LT_RR_MIN_F 0.05f       // integrator.py:34
// traversal stack entries: a 4-wide visit leaves up to 3 siblings pending
// per level, so a tree the reference builds (depth cap 60, bvh.py:26) needs
// up to 3 * 60 + 1; scene creation rejects trees that could need more
// (k_collapse_all measures it).  Entries past the shared-memory part live in
// local memory, touched only by the deepest rays.
#define LT_STACK 192
#define LT_LINK_EXIT ((int32_t)0x80000000)
// Wide-node record, in float4 units (224 B): every axis stored as
// [lo, hi, hi, lo] so the ray's direction octant selects a 32 B-aligned
// (near, far) pair that one 256-bit load fetches (+4.5 % on C4 over the
// 128 B [lo, hi] record, profiles/r01_trace_variants.txt); f4[12] = links.
// Leaf-ordered triangle record in float4 units: (v0, orig), (e1, leaf-end),
// (e2, 0) = 48 B.
#define LT_TRI_F4 3
#define LT_NODE_F4 14
#define LT_NODE_LINKS 12
// robustness: child exit distances are widened by 1 + 2*gamma(3) so fp32
// rounding in the slab test never culls a box the float64 reference keeps
#define LT_SLAB_WIDEN 1.0000004f

enum : uint32_t {
  MAT_DIFFUSE_ONLY = 1u,  // m <= 0 and sw <= 0 (material.py:304-315 fast path)
  MAT_COAT = 2u,          // extension
  MAT_GLASS = 4u,         // extension
  MAT_EMISSIVE = 8u,
  MAT_CLASS_MASK = 7u,
};

struct __align__(16) GpuMaterial {
  float bw, bc[3];            // base_weight, base_color
  float m, sw, alpha, f0d;    // metalness, specular_weight, alpha_of(rough), f0_from_ior
  float sc[3], diff;          // specular_color, bw/pi (1 - avg Fresnel)
  float el, ec[3];            // emission luminance / color
  float cw, calpha, f0c, rsv;    // coat extension (rsv: unused)
  float cc[3], tw;            // coat color, transmission weight
  float tc[3], ior;           // transmission color, specular ior
  uint32_t flags;
  float a2, ca2, fdavg;       // alpha^2, coat alpha^2, avg dielectric Fresnel
};
static_assert(sizeof(GpuMaterial) == 128, "material record is 128 bytes");

struct SceneView {
  const float4 *__restrict__ wnodes;   // BVH4: 8 x float4 per node (render / queries)
  int32_t wroot_link;
  const float4 *__restrict__ nodes;    // BVH2 (reference counters)
  const float4 *__restrict__ tris;
  const float4 *__restrict__ shade;
  const GpuMaterial *__restrict__ mats;
  const float4 *__restrict__ env_map;  // (h, w) RGB + pad
  int32_t root_link;
  int32_t refill_min;   // idle lanes that trigger a warp refill in k_trace
  int32_t leaf_min;     // lanes at a leaf that trigger the warp's leaf tests
  float root_lo[3], root_hi[3];
  int32_t env_kind;
  int32_t env_w, env_h;
  float env_scale;
  float env_a[3], env_b[3];
  int32_t n_wide, n_tris, n_mats;  // bounds for the checked build
};

// --------------------------------------------------------------- PCG32
// rng.py:37-85; integer arithmetic, bit-exact with the reference.

__device__ __forceinline__ uint32_t pcg_next(uint64_t &state, uint64_t inc) {
  uint64_t old = state;
  state = old * 6364136223846793005ULL + inc;
  uint32_t x = (uint32_t)(((old >> 18) ^ old) >> 27);
  uint32_t r = (uint32_t)(old >> 59);
  return __funnelshift_r(x, x, r);  // rotate right
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void seed_stream(uint64_t pixel, uint64_t sample, uint64_t seed,
                                            uint64_t &state, uint64_t &inc) {
  const uint64_t init_state = mix64(seed ^ mix64(sample));
  inc = (mix64(pixel) << 1) | 1ULL;
  uint64_t st = 0;
  (void)pcg_next(st, inc);
  st += init_state;
  (void)pcg_next(st, inc);
  state = st;
}

// u32 * 2^-32 as float64: exact, identical to _next_unit
__device__ __forceinline__ double unit_f64(uint64_t &state, uint64_t inc) {
  return (double)pcg_next(state, inc) * (1.0 / 4294967296.0);
}
// float32 draw: round toward zero so the value stays < 1 (2^32 - 128 and up
// would round to 1.0f); differs from the f64 draw by < 2^-24 relative
__device__ __forceinline__ float unit_f32(uint64_t &state, uint64_t inc) {
  return __uint2float_rz(pcg_next(state, inc)) * 2.3283064365386963e-10f;
}

// --------------------------------------------------------------- vectors
struct f3 {
  float x, y, z;
};
__device__ __forceinline__ f3 mk(float x, float y, float z) { return f3{x, y, z}; }
__device__ __forceinline__ float dot(f3 a, f3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ f3 operator-(f3 a) { return f3{-a.x, -a.y, -a.z}; }

// --------------------------------------------------------------- camera
// _camera_dir (integrator.py:86-98), evaluated in float64 then rounded once
__device__ __forceinline__ f3 camera_dir(const double *cam, double px, double py, double jx,
                                         double jy, int width, int height) {
  double sx = 2.0 * (px + jx) / (double)width - 1.0;
  double sy = 1.0 - 2.0 * (py + jy) / (double)height;
  double hx = cam[12] * cam[13] * sx;
  double hy = cam[12] * sy;
  double dx = cam[3] + cam[6] * hx + cam[9] * hy;
  double dy = cam[4] + cam[7] * hx + cam[10] * hy;
  double dz = cam[5] + cam[8] * hx + cam[11] * hy;
  double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
  return f3{(float)(dx * inv), (float)(dy * inv), (float)(dz * inv)};
}

// --------------------------------------------------------------- environment
// _env_radiance (integrator.py:124-136); LT_ENV_LATLONG is the extension
__device__ __forceinline__ f3 env_radiance(const SceneView &sc, f3 d) {
  if (sc.env_kind == 0) return f3{sc.env_a[0], sc.env_a[1], sc.env_a[2]};
  if (sc.env_kind == 1) {
    float t = d.y;
    if (t < 0.f) t = 0.f;
    else if (t > 1.f) t = 1.f;
    return f3{sc.env_b[0] + (sc.env_a[0] - sc.env_b[0]) * t,
              sc.env_b[1] + (sc.env_a[1] - sc.env_b[1]) * t,
              sc.env_b[2] + (sc.env_a[2] - sc.env_b[2]) * t};
  }
  float y = fminf(fmaxf(d.y, -1.f), 1.f);
  float u = 0.5f + atan2f(d.x, -d.z) * (0.5f * LT_INV_PI_F);
  float v = acosf(y) * LT_INV_PI_F;
  float fx = u * (float)sc.env_w - 0.5f, fy = v * (float)sc.env_h - 0.5f;
  float x0f = floorf(fx), y0f = floorf(fy);
  float ax = fx - x0f, ay = fy - y0f;
  int x0 = (int)x0f, y0 = (int)y0f;
  int x1 = x0 + 1, y1 = y0 + 1;
  // wrap around the seam: u in [0, 1] puts x0 in [-1, w - 1] and x1 in
  // [0, w]; the integer modulo (~20 instructions each) only for anything else
  x0 += x0 < 0 ? sc.env_w : 0;
  x1 -= x1 >= sc.env_w ? sc.env_w : 0;
  if ((unsigned)x0 >= (unsigned)sc.env_w) x0 = ((x0 % sc.env_w) + sc.env_w) % sc.env_w;
  if ((unsigned)x1 >= (unsigned)sc.env_w) x1 = ((x1 % sc.env_w) + sc.env_w) % sc.env_w;
  y0 = min(max(y0, 0), sc.env_h - 1);
  y1 = min(max(y1, 0), sc.env_h - 1);
  float4 c00 = __ldg(&sc.env_map[y0 * sc.env_w + x0]);
  float4 c10 = __ldg(&sc.env_map[y0 * sc.env_w + x1]);
  float4 c01 = __ldg(&sc.env_map[y1 * sc.env_w + x0]);
  float4 c11 = __ldg(&sc.env_map[y1 * sc.env_w + x1]);
  auto lerp2 = [&](float a00, float a10, float a01, float a11) {
    float top = a00 + (a10 - a00) * ax;
    float bot = a01 + (a11 - a01) * ax;
    return (top + (bot - top) * ay) * sc.env_scale;
  };
  return f3{lerp2(c00.x, c10.x, c01.x, c11.x), lerp2(c00.y, c10.y, c01.y, c11.y),
            lerp2(c00.z, c10.z, c01.z, c11.z)};
}

// --------------------------------------------------------------- hit frame
// _hit_frame (geometry.py:210-241).  The unit geometric normal g0 =
// normalize(e1 x e2) is precomputed per triangle in float64 at upload (the
// reference's float64 value, rounded once); orientation, interpolation of
// the vertex normals and the hemisphere flip happen here per hit.
__device__ __forceinline__ void hit_frame(f3 d, f3 g0, f3 n0, f3 n1, f3 n2, float u, float v,
                                          f3 &g, f3 &s, bool &front) {
  float gx = g0.x, gy = g0.y, gz = g0.z;
  front = (gx * d.x + gy * d.y + gz * d.z) < 0.f;
  if (!front) {
    gx = -gx;
    gy = -gy;
    gz = -gz;
  }
  float w = 1.f - u - v;
  float sx = w * n0.x + u * n1.x + v * n2.x;
  float sy = w * n0.y + u * n1.y + v * n2.y;
  float sz = w * n0.z + u * n1.z + v * n2.z;
  float slen = sqrtf(sx * sx + sy * sy + sz * sz);
  if (slen > 0.f) {
    // one reciprocal, three products (<= 1 ulp from the quotients): an IEEE
    // quotient with an exactly-zero numerator (axis-aligned normals) takes
    // the division slow path
    const float r = 1.f / slen;
    sx *= r;
    sy *= r;
    sz *= r;
  } else {
    sx = gx;
    sy = gy;
    sz = gz;
  }
  if (sx * gx + sy * gy + sz * gz < 0.f) {
    sx = -sx;
    sy = -sy;
    sz = -sz;
  }
  g = f3{gx, gy, gz};
  s = f3{sx, sy, sz};
}
