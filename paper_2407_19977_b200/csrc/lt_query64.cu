// lt_query64.cu -- the reference's scalar query API in float64 on the device.
//
// The render path is fp32 (lt_kernels.cu); the public single-object queries
// of the drop-in API -- ray_triangle_intersect / ray_aabb_intersect / the
// hit frame (geometry.py:138-248, 255-295), eval_bsdf / pdf_bsdf /
// sample_bsdf and the microfacet helpers (material.py:99-351, 366-426) and
// the display transform (tonemap.py:18-61) -- are batch kernels here in
// float64 with the reference's operation order, compiled with -fmad=false
// (no contraction, as numba compiles the reference), so a caller of these
// helpers gets the reference's numbers (transcendentals: CUDA's
// correctly-rounded-to-1-ulp sin / cos / pow against the host libm).
#include <cstdint>

#include <math_constants.h>

#include "lt_kernels.h"

namespace lt {
namespace q64 {

constexpr double kPi = 3.141592653589793;
constexpr double kInvPi = 1.0 / 3.141592653589793;
constexpr double kDetEps = 1e-9;    // geometry.py:17
constexpr double kAlphaMin = 1e-4;  // material.py:21

struct V {
  double x, y, z;
};

__device__ __forceinline__ V ld(const double *p, int64_t i) {
  return V{p[3 * i], p[3 * i + 1], p[3 * i + 2]};
}
__device__ __forceinline__ void st(double *p, int64_t i, V v) {
  p[3 * i] = v.x;
  p[3 * i + 1] = v.y;
  p[3 * i + 2] = v.z;
}

// _mt_intersect (geometry.py:138-167)
__device__ bool mt(V o, V d, V a, V b, V c, double t_min, double t_max, double &t, double &u,
                   double &v) {
  const double e1x = b.x - a.x, e1y = b.y - a.y, e1z = b.z - a.z;
  const double e2x = c.x - a.x, e2y = c.y - a.y, e2z = c.z - a.z;
  const double px = d.y * e2z - d.z * e2y;
  const double py = d.z * e2x - d.x * e2z;
  const double pz = d.x * e2y - d.y * e2x;
  const double det = e1x * px + e1y * py + e1z * pz;
  if (-kDetEps <= det && det <= kDetEps) return false;
  const double inv_det = 1.0 / det;
  const double sx = o.x - a.x, sy = o.y - a.y, sz = o.z - a.z;
  u = (sx * px + sy * py + sz * pz) * inv_det;
  if (u < 0.0 || u > 1.0) return false;
  const double qx = sy * e1z - sz * e1y;
  const double qy = sz * e1x - sx * e1z;
  const double qz = sx * e1y - sy * e1x;
  v = (d.x * qx + d.y * qy + d.z * qz) * inv_det;
  if (v < 0.0 || u + v > 1.0) return false;
  t = (e2x * qx + e2y * qy + e2z * qz) * inv_det;
  if (t < t_min || t > t_max) return false;
  return true;
}

// _inv_component (geometry.py:244-248): +inf for any zero component
__device__ __forceinline__ double inv_component(double d) { return d == 0.0 ? CUDART_INF : 1.0 / d; }

// _slab_intersect (geometry.py:170-207), compare / select form: a 0 * inf
// NaN fails every comparison and keeps the running interval
__device__ bool slab(V o, V inv, V lo, V hi, double t_min, double t_max, double &tn, double &tf) {
  tn = t_min;
  tf = t_max;
  const double ov[3] = {o.x, o.y, o.z}, iv[3] = {inv.x, inv.y, inv.z};
  const double lv[3] = {lo.x, lo.y, lo.z}, hv[3] = {hi.x, hi.y, hi.z};
  for (int a = 0; a < 3; ++a) {
    double t0 = (lv[a] - ov[a]) * iv[a];
    double t1 = (hv[a] - ov[a]) * iv[a];
    if (t0 > t1) {
      const double s = t0;
      t0 = t1;
      t1 = s;
    }
    if (t0 > tn) tn = t0;
    if (t1 < tf) tf = t1;
  }
  return tn <= tf;
}

// _hit_frame (geometry.py:210-241)
__device__ void hit_frame(V d, V a, V b, V c, V n0, V n1, V n2, double u, double v, V &g, V &s,
                          bool &front) {
  const double e1x = b.x - a.x, e1y = b.y - a.y, e1z = b.z - a.z;
  const double e2x = c.x - a.x, e2y = c.y - a.y, e2z = c.z - a.z;
  double gx = e1y * e2z - e1z * e2y;
  double gy = e1z * e2x - e1x * e2z;
  double gz = e1x * e2y - e1y * e2x;
  const double glen = sqrt(gx * gx + gy * gy + gz * gz);
  if (glen > 0.0) {
    gx /= glen;
    gy /= glen;
    gz /= glen;
  }
  front = (gx * d.x + gy * d.y + gz * d.z) < 0.0;
  if (!front) {
    gx = -gx;
    gy = -gy;
    gz = -gz;
  }
  const double w = 1.0 - u - v;
  double sx = w * n0.x + u * n1.x + v * n2.x;
  double sy = w * n0.y + u * n1.y + v * n2.y;
  double sz = w * n0.z + u * n1.z + v * n2.z;
  const double slen = sqrt(sx * sx + sy * sy + sz * sz);
  if (slen > 0.0) {
    sx /= slen;
    sy /= slen;
    sz /= slen;
  } else {
    sx = gx;
    sy = gy;
    sz = gz;
  }
  if (sx * gx + sy * gy + sz * gz < 0.0) {
    sx = -sx;
    sy = -sy;
    sz = -sz;
  }
  g = V{gx, gy, gz};
  s = V{sx, sy, sz};
}

// ---- material.py:99-351

struct Mat {  // the reference's 11 material scalars (pack order)
  double bw, bc[3], m, sw, sc[3], rough, ior;
};

__device__ __forceinline__ Mat ld_mat(const double *p, int64_t i) {
  const double *q = p + 11 * i;
  return Mat{q[0], {q[1], q[2], q[3]}, q[4], q[5], {q[6], q[7], q[8]}, q[9], q[10]};
}

__device__ __forceinline__ double alpha_of(double r) {
  double a = r * r;
  if (a < kAlphaMin) a = kAlphaMin;
  return a;
}

__device__ __forceinline__ double ggx_ndf(double nh, double alpha) {
  if (nh <= 0.0) return 0.0;
  const double a2 = alpha * alpha;
  const double t = nh * nh * a2 + (1.0 - nh) * (1.0 + nh);
  return a2 / (kPi * t * t);
}

__device__ __forceinline__ double smith_g2(double no, double ni, double alpha) {
  const double a2 = alpha * alpha;
  const double lo = ni * sqrt(a2 + (1.0 - a2) * no * no);
  const double li = no * sqrt(a2 + (1.0 - a2) * ni * ni);
  const double denom = lo + li;
  if (denom <= 0.0) return 0.0;
  return 2.0 * no * ni / denom;
}

__device__ __forceinline__ double pow5(double x) {
  const double x2 = x * x;
  return x2 * x2 * x;
}

__device__ __forceinline__ double f0_from_ior(double ior) {
  const double r = (ior - 1.0) / (ior + 1.0);
  return r * r;
}

__device__ __forceinline__ double diel_fresnel(double c, double f0d, double sw) {
  return sw * (f0d + (1.0 - f0d) * pow5(1.0 - c));
}

__device__ __forceinline__ double diel_fresnel_avg(double f0d, double sw) {
  return sw * (f0d + (1.0 - f0d) / 21.0);
}

__device__ V eval_core(V wo, V wi, V n, const Mat &mt) {
  const double no = n.x * wo.x + n.y * wo.y + n.z * wo.z;
  const double ni = n.x * wi.x + n.y * wi.y + n.z * wi.z;
  if (no <= 0.0 || ni <= 0.0) return V{0.0, 0.0, 0.0};
  double hx = wo.x + wi.x, hy = wo.y + wi.y, hz = wo.z + wi.z;
  const double hl = sqrt(hx * hx + hy * hy + hz * hz);
  if (hl <= 0.0) return V{0.0, 0.0, 0.0};
  hx /= hl;
  hy /= hl;
  hz /= hl;
  const double nh = n.x * hx + n.y * hy + n.z * hz;
  const double oh = wo.x * hx + wo.y * hy + wo.z * hz;
  if (oh <= 0.0) return V{0.0, 0.0, 0.0};
  const double alpha = alpha_of(mt.rough);
  const double spec_common = ggx_ndf(nh, alpha) * smith_g2(no, ni, alpha) / (4.0 * no * ni);
  double f[3] = {0.0, 0.0, 0.0};
  if (mt.m < 1.0) {
    const double f0d = f0_from_ior(mt.ior);
    const double diff = mt.bw * kInvPi * (1.0 - diel_fresnel_avg(f0d, mt.sw));
    const double fd = diel_fresnel(oh, f0d, mt.sw) * spec_common;
    const double w = 1.0 - mt.m;
    for (int k = 0; k < 3; ++k) f[k] += w * (diff * mt.bc[k] + fd);
  }
  if (mt.m > 0.0) {
    const double s = pow5(1.0 - oh);
    for (int k = 0; k < 3; ++k) {
      const double f0 = mt.bw * mt.bc[k];
      f[k] += mt.m * spec_common * (f0 + (mt.sc[k] - f0) * s);
    }
  }
  return V{f[0], f[1], f[2]};
}

__device__ __forceinline__ double p_spec_select(double no, const Mat &mt, double f0d) {
  const bool has_diff = mt.bw > 0.0, has_spec = mt.sw > 0.0;
  if (has_diff && has_spec) {
    double p = diel_fresnel(no, f0d, mt.sw);
    if (p < 0.05) p = 0.05;
    else if (p > 0.95) p = 0.95;
    return p;
  }
  if (has_spec) return 1.0;
  if (has_diff) return 0.0;
  return -1.0;
}

__device__ double pdf_core(V wo, V wi, V n, const Mat &mt) {
  const double no = n.x * wo.x + n.y * wo.y + n.z * wo.z;
  const double ni = n.x * wi.x + n.y * wi.y + n.z * wi.z;
  if (no <= 0.0 || ni <= 0.0) return 0.0;
  double hx = wo.x + wi.x, hy = wo.y + wi.y, hz = wo.z + wi.z;
  const double hl = sqrt(hx * hx + hy * hy + hz * hz);
  if (hl <= 0.0) return 0.0;
  hx /= hl;
  hy /= hl;
  hz /= hl;
  const double nh = n.x * hx + n.y * hy + n.z * hz;
  const double oh = wo.x * hx + wo.y * hy + wo.z * hz;
  const double alpha = alpha_of(mt.rough);
  double pdf_ggx = 0.0;
  if (oh > 0.0 && nh > 0.0) pdf_ggx = ggx_ndf(nh, alpha) * nh / (4.0 * oh);
  const double pdf_cos = ni * kInvPi;
  double pdf = mt.m * pdf_ggx;
  if (mt.m < 1.0) {
    const double p_spec = p_spec_select(no, mt, f0_from_ior(mt.ior));
    if (p_spec >= 0.0) pdf += (1.0 - mt.m) * (p_spec * pdf_ggx + (1.0 - p_spec) * pdf_cos);
  }
  return pdf;
}

__device__ void onb(V n, V &t, V &b) {
  double ax, ay, az;
  if (fabs(n.x) > 0.9) {
    ax = 0.0;
    ay = 1.0;
    az = 0.0;
  } else {
    ax = 1.0;
    ay = 0.0;
    az = 0.0;
  }
  double tx = ay * n.z - az * n.y;
  double ty = az * n.x - ax * n.z;
  double tz = ax * n.y - ay * n.x;
  const double tl = sqrt(tx * tx + ty * ty + tz * tz);
  tx /= tl;
  ty /= tl;
  tz /= tl;
  t = V{tx, ty, tz};
  b = V{n.y * tz - n.z * ty, n.z * tx - n.x * tz, n.x * ty - n.y * tx};
}

__device__ V cosine_sample(V n, double u1, double u2) {
  V t, b;
  onb(n, t, b);
  const double r = sqrt(u1);
  const double phi = 2.0 * kPi * u2;
  const double x = r * cos(phi), y = r * sin(phi);
  const double z = sqrt(fmax(0.0, 1.0 - u1));
  return V{x * t.x + y * b.x + z * n.x, x * t.y + y * b.y + z * n.y, x * t.z + y * b.z + z * n.z};
}

__device__ V ggx_sample_half(V n, double alpha, double u1, double u2) {
  V t, b;
  onb(n, t, b);
  const double a2 = alpha * alpha;
  const double ct = sqrt((1.0 - u1) / (1.0 + (a2 - 1.0) * u1));
  const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
  const double phi = 2.0 * kPi * u2;
  const double x = st * cos(phi), y = st * sin(phi);
  return V{x * t.x + y * b.x + ct * n.x, x * t.y + y * b.y + ct * n.y,
           x * t.z + y * b.z + ct * n.z};
}

// _sample_core (material.py:293-351)
__device__ bool sample_core(V wo, V n, const Mat &mt, double u_lobe, double u1, double u2, V &wi,
                            V &wgt, double &pdf, bool &spike) {
  const double alpha = alpha_of(mt.rough);
  const double f0d = f0_from_ior(mt.ior);
  const double no = n.x * wo.x + n.y * wo.y + n.z * wo.z;
  spike = false;
  if (mt.m <= 0.0 && mt.sw <= 0.0) {
    if (mt.bw <= 0.0 || no <= 0.0) return false;
    wi = cosine_sample(n, u1, u2);
    const double ni = n.x * wi.x + n.y * wi.y + n.z * wi.z;
    if (ni <= 0.0) return false;
    pdf = ni * kInvPi;
    if (pdf <= 0.0) return false;
    wgt = V{mt.bw * mt.bc[0], mt.bw * mt.bc[1], mt.bw * mt.bc[2]};
    return true;
  }
  bool use_ggx = false;
  if (u_lobe < mt.m) {
    use_ggx = true;
  } else {
    const double p_spec = p_spec_select(no, mt, f0d);
    if (p_spec < 0.0) return false;
    const double u_d = mt.m < 1.0 ? (u_lobe - mt.m) / (1.0 - mt.m) : 0.0;
    use_ggx = u_d < p_spec;
  }
  if (use_ggx) {
    const V h = ggx_sample_half(n, alpha, u1, u2);
    const double oh = wo.x * h.x + wo.y * h.y + wo.z * h.z;
    if (oh <= 0.0) return false;
    wi = V{2.0 * oh * h.x - wo.x, 2.0 * oh * h.y - wo.y, 2.0 * oh * h.z - wo.z};
  } else {
    wi = cosine_sample(n, u1, u2);
  }
  const double ni = n.x * wi.x + n.y * wi.y + n.z * wi.z;
  if (ni <= 0.0) return false;
  pdf = pdf_core(wo, wi, n, mt);
  if (pdf <= 0.0 || !isfinite(pdf)) return false;
  const V f = eval_core(wo, wi, n, mt);
  const double scale = ni / pdf;
  wgt = V{f.x * scale, f.y * scale, f.z * scale};
  spike = use_ggx && alpha <= kAlphaMin;
  return true;
}

// ---- tonemap.py:18-61
__device__ void pbr_neutral(const double *in, double *out) {
  const double kStart = 0.8 - 0.04, kDesat = 0.15;
  double c[3] = {in[0], in[1], in[2]};
  const double x = fmin(c[0], fmin(c[1], c[2]));
  const double offset = x < 0.08 ? x - 6.25 * x * x : 0.04;
  for (int k = 0; k < 3; ++k) c[k] = c[k] - offset;
  const double peak = fmax(c[0], fmax(c[1], c[2]));
  const double d = 1.0 - kStart;
  const double new_peak = 1.0 - d * d / (peak + d - kStart);
  const bool compress = peak > kStart;
  if (!compress) {
    for (int k = 0; k < 3; ++k) out[k] = c[k];
    return;
  }
  const double g = 1.0 - 1.0 / (kDesat * (peak - new_peak) + 1.0);
  for (int k = 0; k < 3; ++k) out[k] = c[k] * (new_peak / peak) * (1.0 - g) + new_peak * g;
}

}  // namespace q64

// ------------------------------------------------------------------ kernels

__global__ void k_ray_triangle64(const double *__restrict__ o, const double *__restrict__ d,
                                 const double *__restrict__ tmin, const double *__restrict__ tmax,
                                 const double *__restrict__ v0, const double *__restrict__ v1,
                                 const double *__restrict__ v2, const double *__restrict__ n0,
                                 const double *__restrict__ n1, const double *__restrict__ n2,
                                 int64_t n, int32_t *__restrict__ ok, double *__restrict__ tuv,
                                 double *__restrict__ g, double *__restrict__ s,
                                 int32_t *__restrict__ front) {
  using namespace q64;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t = 0.0, u = 0.0, v = 0.0;
  const V dd = ld(d, i);
  const bool hit = mt(ld(o, i), dd, ld(v0, i), ld(v1, i), ld(v2, i), tmin[i], tmax[i], t, u, v);
  ok[i] = hit ? 1 : 0;
  tuv[3 * i] = hit ? t : 0.0;
  tuv[3 * i + 1] = hit ? u : 0.0;
  tuv[3 * i + 2] = hit ? v : 0.0;
  V gg{0.0, 0.0, 0.0}, ss{0.0, 0.0, 0.0};
  bool fr = false;
  if (hit) hit_frame(dd, ld(v0, i), ld(v1, i), ld(v2, i), ld(n0, i), ld(n1, i), ld(n2, i), u, v,
                     gg, ss, fr);
  st(g, i, gg);
  st(s, i, ss);
  front[i] = fr ? 1 : 0;
}

__global__ void k_hit_frame64(const double *__restrict__ d, const double *__restrict__ v0,
                              const double *__restrict__ v1, const double *__restrict__ v2,
                              const double *__restrict__ n0, const double *__restrict__ n1,
                              const double *__restrict__ n2, const double *__restrict__ uv,
                              int64_t n, double *__restrict__ g, double *__restrict__ s,
                              int32_t *__restrict__ front) {
  using namespace q64;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  V gg, ss;
  bool fr;
  hit_frame(ld(d, i), ld(v0, i), ld(v1, i), ld(v2, i), ld(n0, i), ld(n1, i), ld(n2, i),
            uv[2 * i], uv[2 * i + 1], gg, ss, fr);
  st(g, i, gg);
  st(s, i, ss);
  front[i] = fr ? 1 : 0;
}

__global__ void k_ray_aabb64(const double *__restrict__ o, const double *__restrict__ d,
                             const double *__restrict__ tmin, const double *__restrict__ tmax,
                             const double *__restrict__ lo, const double *__restrict__ hi,
                             int64_t n, int32_t *__restrict__ ok, double *__restrict__ tnf) {
  using namespace q64;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const V dd = ld(d, i);
  const V inv{inv_component(dd.x), inv_component(dd.y), inv_component(dd.z)};
  double tn, tf;
  ok[i] = slab(ld(o, i), inv, ld(lo, i), ld(hi, i), tmin[i], tmax[i], tn, tf) ? 1 : 0;
  tnf[2 * i] = tn;
  tnf[2 * i + 1] = tf;
}

__global__ void k_bsdf64(int mode, const double *__restrict__ params,
                         const double *__restrict__ wo, const double *__restrict__ wi,
                         const double *__restrict__ nrm, const double *__restrict__ u, int64_t n,
                         int32_t *__restrict__ ok, double *__restrict__ out3a,
                         double *__restrict__ out3b, double *__restrict__ out1,
                         int32_t *__restrict__ flag) {
  using namespace q64;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Mat mt = ld_mat(params, i);
  if (mode == 0) {  // eval + pdf
    st(out3a, i, eval_core(ld(wo, i), ld(wi, i), ld(nrm, i), mt));
    out1[i] = pdf_core(ld(wo, i), ld(wi, i), ld(nrm, i), mt);
    return;
  }
  V w{0.0, 0.0, 0.0}, g{0.0, 0.0, 0.0};
  double pdf = 0.0;
  bool spike = false;
  const bool r = sample_core(ld(wo, i), ld(nrm, i), mt, u[3 * i], u[3 * i + 1], u[3 * i + 2], w,
                             g, pdf, spike);
  ok[i] = r ? 1 : 0;
  st(out3a, i, r ? w : V{0.0, 0.0, 0.0});
  st(out3b, i, r ? g : V{0.0, 0.0, 0.0});
  out1[i] = r ? pdf : 0.0;
  flag[i] = r && spike ? 1 : 0;
}

// microfacet helpers: op 0 ggx_ndf(a, b), 1 smith_g2(a, b, c), 2
// cosine_sample(nrm, a, b), 3 ggx_sample_half(nrm, c, a, b)
__global__ void k_microfacet64(int op, const double *__restrict__ a, const double *__restrict__ b,
                               const double *__restrict__ c, const double *__restrict__ nrm,
                               int64_t n, double *__restrict__ out) {
  using namespace q64;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (op == 0) out[i] = ggx_ndf(a[i], b[i]);
  else if (op == 1) out[i] = smith_g2(a[i], b[i], c[i]);
  else if (op == 2) st(out, i, cosine_sample(ld(nrm, i), a[i], b[i]));
  else st(out, i, ggx_sample_half(ld(nrm, i), c[i], a[i], b[i]));
}

// display transform: op 0 pbr_neutral_tonemap (per rgb triple), 1
// linear_to_srgb, 2 srgb_to_linear, 3 quantize_to_u8 (per value)
__global__ void k_display64(int op, const double *__restrict__ in, int64_t n,
                            double *__restrict__ out, uint8_t *__restrict__ out8) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (op == 0) {
    q64::pbr_neutral(in + 3 * i, out + 3 * i);
    return;
  }
  const double x = in[i];
  if (op == 1) {
    const double c = fmin(fmax(x, 0.0), 1.0);
    out[i] = c <= 0.0031308 ? 12.92 * c : 1.055 * pow(c, 1.0 / 2.4) - 0.055;
  } else if (op == 2) {
    out[i] = x <= 0.04045 ? x / 12.92 : pow((x + 0.055) / 1.055, 2.4);
  } else {
    const double c = fmin(fmax(x, 0.0), 1.0);
    out8[i] = (uint8_t)floor(255.0 * c + 0.5);
  }
}

static unsigned blocks(int64_t n) { return (unsigned)((n + 127) / 128); }

void launch_ray_triangle64(const double *o, const double *d, const double *tmin,
                           const double *tmax, const double *v0, const double *v1,
                           const double *v2, const double *n0, const double *n1,
                           const double *n2, int64_t n, int32_t *ok, double *tuv, double *g,
                           double *s, int32_t *front, cudaStream_t st) {
  if (n > 0)
    k_ray_triangle64<<<blocks(n), 128, 0, st>>>(o, d, tmin, tmax, v0, v1, v2, n0, n1, n2, n, ok,
                                                tuv, g, s, front);
}

void launch_hit_frame64(const double *d, const double *v0, const double *v1, const double *v2,
                        const double *n0, const double *n1, const double *n2, const double *uv,
                        int64_t n, double *g, double *s, int32_t *front, cudaStream_t st) {
  if (n > 0)
    k_hit_frame64<<<blocks(n), 128, 0, st>>>(d, v0, v1, v2, n0, n1, n2, uv, n, g, s, front);
}

void launch_ray_aabb64(const double *o, const double *d, const double *tmin, const double *tmax,
                       const double *lo, const double *hi, int64_t n, int32_t *ok, double *tnf,
                       cudaStream_t st) {
  if (n > 0) k_ray_aabb64<<<blocks(n), 128, 0, st>>>(o, d, tmin, tmax, lo, hi, n, ok, tnf);
}

void launch_bsdf64(int mode, const double *params, const double *wo, const double *wi,
                   const double *nrm, const double *u, int64_t n, int32_t *ok, double *out3a,
                   double *out3b, double *out1, int32_t *flag, cudaStream_t st) {
  if (n > 0)
    k_bsdf64<<<blocks(n), 128, 0, st>>>(mode, params, wo, wi, nrm, u, n, ok, out3a, out3b, out1,
                                        flag);
}

void launch_microfacet64(int op, const double *a, const double *b, const double *c,
                         const double *nrm, int64_t n, double *out, cudaStream_t st) {
  if (n > 0) k_microfacet64<<<blocks(n), 128, 0, st>>>(op, a, b, c, nrm, n, out);
}

void launch_display64(int op, const double *in, int64_t n, double *out, uint8_t *out8,
                      cudaStream_t st) {
  if (n > 0) k_display64<<<blocks(n), 128, 0, st>>>(op, in, n, out, out8);
}

}  // namespace lt

// ------------------------------------------------------------------ C-ABI
// Host-buffer entry points (include/luxb200.h).  Every call stages its
// arrays through one per-device scratch buffer (grow-only, serialized by a
// mutex) and runs synchronously on a per-device non-blocking stream, so a
// query never waits for (or blocks) render work on other streams.

#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "lt_internal.h"

#include "lt_staged.h"

using namespace lt;
using lt_staged::Staged;

extern "C" int lt_ray_triangle_batch(const double *origins, const double *dirs,
                                     const double *t_min, const double *t_max, const double *v0,
                                     const double *v1, const double *v2, const double *n0,
                                     const double *n1, const double *n2, int64_t n, int32_t *ok,
                                     double *tuv, double *geo_normal, double *shading_normal,
                                     int32_t *front) {
  if (n < 0) return lt_fail(LT_ERR_INVALID, "negative count");
  if (n == 0) return LT_OK;
  if (!origins || !dirs || !t_min || !t_max || !v0 || !v1 || !v2 || !n0 || !n1 || !n2 || !ok ||
      !tuv || !geo_normal || !shading_normal || !front)
    return lt_fail(LT_ERR_INVALID, "null buffer");
  Staged s;
  const size_t v3 = 24 * (size_t)n;
  const int io = s.add(origins, nullptr, v3), id = s.add(dirs, nullptr, v3);
  const int i0 = s.add(t_min, nullptr, 8 * n), i1 = s.add(t_max, nullptr, 8 * n);
  int iv[6];
  const double *vs[6] = {v0, v1, v2, n0, n1, n2};
  for (int k = 0; k < 6; ++k) iv[k] = s.add(vs[k], nullptr, v3);
  const int iok = s.add(nullptr, ok, 4 * n), it = s.add(nullptr, tuv, v3);
  const int ig = s.add(nullptr, geo_normal, v3), isn = s.add(nullptr, shading_normal, v3);
  const int ifr = s.add(nullptr, front, 4 * n);
  Q_RET(s.begin());
  launch_ray_triangle64(s.dev<double>(io), s.dev<double>(id), s.dev<double>(i0),
                        s.dev<double>(i1), s.dev<double>(iv[0]), s.dev<double>(iv[1]),
                        s.dev<double>(iv[2]), s.dev<double>(iv[3]), s.dev<double>(iv[4]),
                        s.dev<double>(iv[5]), n, s.dev<int32_t>(iok), s.dev<double>(it),
                        s.dev<double>(ig), s.dev<double>(isn), s.dev<int32_t>(ifr), s.stream());
  return s.finish();
}

extern "C" int lt_hit_frame_batch(const double *dirs, const double *v0, const double *v1,
                                  const double *v2, const double *n0, const double *n1,
                                  const double *n2, const double *uv, int64_t n,
                                  double *geo_normal, double *shading_normal, int32_t *front) {
  if (n < 0) return lt_fail(LT_ERR_INVALID, "negative count");
  if (n == 0) return LT_OK;
  if (!dirs || !v0 || !v1 || !v2 || !n0 || !n1 || !n2 || !uv || !geo_normal || !shading_normal ||
      !front)
    return lt_fail(LT_ERR_INVALID, "null buffer");
  Staged s;
  const size_t v3 = 24 * (size_t)n;
  const int id = s.add(dirs, nullptr, v3);
  int iv[6];
  const double *vs[6] = {v0, v1, v2, n0, n1, n2};
  for (int k = 0; k < 6; ++k) iv[k] = s.add(vs[k], nullptr, v3);
  const int iuv = s.add(uv, nullptr, 16 * n);
  const int ig = s.add(nullptr, geo_normal, v3), isn = s.add(nullptr, shading_normal, v3);
  const int ifr = s.add(nullptr, front, 4 * n);
  Q_RET(s.begin());
  launch_hit_frame64(s.dev<double>(id), s.dev<double>(iv[0]), s.dev<double>(iv[1]),
                     s.dev<double>(iv[2]), s.dev<double>(iv[3]), s.dev<double>(iv[4]),
                     s.dev<double>(iv[5]), s.dev<double>(iuv), n, s.dev<double>(ig),
                     s.dev<double>(isn), s.dev<int32_t>(ifr), s.stream());
  return s.finish();
}

extern "C" int lt_ray_aabb_batch(const double *origins, const double *dirs, const double *t_min,
                                 const double *t_max, const double *box_min,
                                 const double *box_max, int64_t n, int32_t *ok,
                                 double *t_enter_exit) {
  if (n < 0) return lt_fail(LT_ERR_INVALID, "negative count");
  if (n == 0) return LT_OK;
  if (!origins || !dirs || !t_min || !t_max || !box_min || !box_max || !ok || !t_enter_exit)
    return lt_fail(LT_ERR_INVALID, "null buffer");
  Staged s;
  const size_t v3 = 24 * (size_t)n;
  const int io = s.add(origins, nullptr, v3), id = s.add(dirs, nullptr, v3);
  const int i0 = s.add(t_min, nullptr, 8 * n), i1 = s.add(t_max, nullptr, 8 * n);
  const int il = s.add(box_min, nullptr, v3), ih = s.add(box_max, nullptr, v3);
  const int iok = s.add(nullptr, ok, 4 * n), it = s.add(nullptr, t_enter_exit, 16 * n);
  Q_RET(s.begin());
  launch_ray_aabb64(s.dev<double>(io), s.dev<double>(id), s.dev<double>(i0), s.dev<double>(i1),
                    s.dev<double>(il), s.dev<double>(ih), n, s.dev<int32_t>(iok),
                    s.dev<double>(it), s.stream());
  return s.finish();
}

extern "C" int lt_bsdf64_eval_batch(const double *params, const double *wo, const double *wi,
                                    const double *normal, int64_t n, double *f, double *pdf) {
  if (n < 0) return lt_fail(LT_ERR_INVALID, "negative count");
  if (n == 0) return LT_OK;
  if (!params || !wo || !wi || !normal || !f || !pdf) return lt_fail(LT_ERR_INVALID, "null buffer");
  Staged s;
  const size_t v3 = 24 * (size_t)n;
  const int ip = s.add(params, nullptr, 88 * n);
  const int io = s.add(wo, nullptr, v3), ii = s.add(wi, nullptr, v3), in = s.add(normal, nullptr, v3);
  const int iff = s.add(nullptr, f, v3), ipdf = s.add(nullptr, pdf, 8 * n);
  Q_RET(s.begin());
  launch_bsdf64(0, s.dev<double>(ip), s.dev<double>(io), s.dev<double>(ii), s.dev<double>(in),
                nullptr, n, nullptr, s.dev<double>(iff), nullptr, s.dev<double>(ipdf), nullptr,
                s.stream());
  return s.finish();
}

extern "C" int lt_bsdf64_sample_batch(const double *params, const double *wo,
                                      const double *normal, const double *u, int64_t n,
                                      int32_t *ok, double *wi, double *weight, double *pdf,
                                      int32_t *spike) {
  if (n < 0) return lt_fail(LT_ERR_INVALID, "negative count");
  if (n == 0) return LT_OK;
  if (!params || !wo || !normal || !u || !ok || !wi || !weight || !pdf || !spike)
    return lt_fail(LT_ERR_INVALID, "null buffer");
  Staged s;
  const size_t v3 = 24 * (size_t)n;
  const int ip = s.add(params, nullptr, 88 * n);
  const int io = s.add(wo, nullptr, v3), in = s.add(normal, nullptr, v3), iu = s.add(u, nullptr, v3);
  const int iok = s.add(nullptr, ok, 4 * n), iwi = s.add(nullptr, wi, v3);
  const int iw = s.add(nullptr, weight, v3), ipdf = s.add(nullptr, pdf, 8 * n);
  const int isp = s.add(nullptr, spike, 4 * n);
  Q_RET(s.begin());
  launch_bsdf64(1, s.dev<double>(ip), s.dev<double>(io), nullptr, s.dev<double>(in),
                s.dev<double>(iu), n, s.dev<int32_t>(iok), s.dev<double>(iwi), s.dev<double>(iw),
                s.dev<double>(ipdf), s.dev<int32_t>(isp), s.stream());
  return s.finish();
}

extern "C" int lt_microfacet_batch(int32_t op, const double *a, const double *b, const double *c,
                                   const double *normal, int64_t n, double *out) {
  if (n < 0 || op < 0 || op > 3) return lt_fail(LT_ERR_INVALID, "invalid microfacet query");
  if (n == 0) return LT_OK;
  const bool needs_n = op >= 2, needs_c = op == 1 || op == 3;
  if (!a || !b || !out || (needs_n && !normal) || (needs_c && !c))
    return lt_fail(LT_ERR_INVALID, "null buffer");
  Staged s;
  const int ia = s.add(a, nullptr, 8 * n), ib = s.add(b, nullptr, 8 * n);
  const int ic = needs_c ? s.add(c, nullptr, 8 * n) : -1;
  const int in = needs_n ? s.add(normal, nullptr, 24 * n) : -1;
  const int iout = s.add(nullptr, out, (needs_n ? 24 : 8) * (size_t)n);
  Q_RET(s.begin());
  launch_microfacet64(op, s.dev<double>(ia), s.dev<double>(ib),
                      ic >= 0 ? s.dev<double>(ic) : nullptr, in >= 0 ? s.dev<double>(in) : nullptr,
                      n, s.dev<double>(iout), s.stream());
  return s.finish();
}

extern "C" int lt_display_batch(int32_t op, const double *in, int64_t n, double *out,
                                uint8_t *out_u8) {
  if (n < 0 || op < 0 || op > 3) return lt_fail(LT_ERR_INVALID, "invalid display transform");
  if (n == 0) return LT_OK;
  if (!in || (op < 3 && !out) || (op == 3 && !out_u8)) return lt_fail(LT_ERR_INVALID, "null buffer");
  const int64_t vals = op == 0 ? 3 * n : n;
  Staged s;
  const int ii = s.add(in, nullptr, 8 * vals);
  const int io = op < 3 ? s.add(nullptr, out, 8 * vals) : s.add(nullptr, out_u8, vals);
  Q_RET(s.begin());
  launch_display64(op, s.dev<double>(ii), n, op < 3 ? s.dev<double>(io) : nullptr,
                   op == 3 ? s.dev<uint8_t>(io) : nullptr, s.stream());
  return s.finish();
}
