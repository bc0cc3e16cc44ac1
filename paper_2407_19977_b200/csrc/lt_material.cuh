// lt_material.cuh -- OpenPBR-subset BSDF in fp32 (material.py:99-351) plus
// the coat and transmission extension lobes (no reference; parity unpinned).
// Term order follows the reference so fp32 results track the float64 ones;
// the material record carries the float64-derived constants (alpha, a2, f0,
// the diffuse factor) rounded once on the host.
#pragma once
#include "lt_device.cuh"

__device__ __forceinline__ float pow5f(float x) {
  float x2 = x * x;
  return x2 * x2 * x;
}

// _ggx_ndf (material.py:107-114), cancellation-safe form
__device__ __forceinline__ float ggx_ndf(float nh, float a2) {
  if (nh <= 0.f) return 0.f;
  float t = nh * nh * a2 + (1.f - nh) * (1.f + nh);
  return a2 / (LT_PI_F * t * t);
}

// _smith_g2 (material.py:117-126)
__device__ __forceinline__ float smith_g2(float no, float ni, float a2) {
  float lo = ni * sqrtf(a2 + (1.f - a2) * no * no);
  float li = no * sqrtf(a2 + (1.f - a2) * ni * ni);
  float denom = lo + li;
  if (denom <= 0.f) return 0.f;
  return 2.f * no * ni / denom;
}

// _diel_fresnel (material.py:141-145)
__device__ __forceinline__ float diel_fresnel(float c, float f0d, float sw) {
  return sw * (f0d + (1.f - f0d) * pow5f(1.f - c));
}

// _onb (material.py:246-261)
__device__ __forceinline__ void onb(f3 n, f3 &t, f3 &b) {
  float ax, ay, az;
  if (fabsf(n.x) > 0.9f) {
    ax = 0.f; ay = 1.f; az = 0.f;
  } else {
    ax = 1.f; ay = 0.f; az = 0.f;
  }
  float tx = ay * n.z - az * n.y;
  float ty = az * n.x - ax * n.z;
  float tz = ax * n.y - ay * n.x;
  // reciprocal once (tl >= 0.43): the tangent always has an exactly-zero
  // component, whose IEEE quotient would take the division slow path
  const float rl = 1.f / sqrtf(tx * tx + ty * ty + tz * tz);
  tx *= rl;
  ty *= rl;
  tz *= rl;
  t = f3{tx, ty, tz};
  b = f3{n.y * tz - n.z * ty, n.z * tx - n.x * tz, n.x * ty - n.y * tx};
}

// The sampling frame shared by every lobe of one scatter: the tangent frame
// of n (_onb) and sincos(2 pi u2) -- computed once, before the lobe branch,
// so a warp whose lanes pick different lobes runs them convergently.
struct SampleFrame {
  f3 t, b;
  float sphi, cphi;
};

__device__ __forceinline__ SampleFrame sample_frame(f3 n, float u2) {
  SampleFrame F;
  onb(n, F.t, F.b);
  sincospif(2.f * u2, &F.sphi, &F.cphi);  // sincospi(2u) == sincos(2 pi u)
  return F;
}

// _cosine_sample (material.py:264-274)
__device__ __forceinline__ f3 cosine_sample(const SampleFrame &F, f3 n, float u1) {
  float r = sqrtf(u1);
  float x = r * F.cphi, y = r * F.sphi;
  float z = sqrtf(fmaxf(0.f, 1.f - u1));
  return f3{x * F.t.x + y * F.b.x + z * n.x, x * F.t.y + y * F.b.y + z * n.y,
            x * F.t.z + y * F.b.z + z * n.z};
}

// _ggx_sample_half (material.py:277-290).  The reference's
// ct = sqrt((1-u1)/(1+(a2-1)u1)) is exact in float64 but cancels in fp32
// (a2-1 rounds to -1 for a2 < 2^-25, and 1-ct^2 loses the tangent near the
// mirror direction); the same angle through tan^2 = a2 u1/(1-u1) has no
// cancellation (1-u1 is exact for u1 >= 0.5 by Sterbenz).
__device__ __forceinline__ f3 ggx_sample_half(const SampleFrame &F, f3 n, float a2, float u1) {
  float t2 = a2 * u1 / (1.f - u1);
  float ct = 1.f / sqrtf(1.f + t2);
  float st = sqrtf(t2) * ct;
  float x = st * F.cphi, y = st * F.sphi;
  return f3{x * F.t.x + y * F.b.x + ct * n.x, x * F.t.y + y * F.b.y + ct * n.y,
            x * F.t.z + y * F.b.z + ct * n.z};
}

// _p_spec_select (material.py:196-213)
__device__ __forceinline__ float p_spec_select(float no, const GpuMaterial &mt) {
  bool has_diff = mt.bw > 0.f, has_spec = mt.sw > 0.f;
  if (has_diff && has_spec) {
    float p = diel_fresnel(no, mt.f0d, mt.sw);
    return fminf(fmaxf(p, 0.05f), 0.95f);
  }
  if (has_spec) return 1.f;
  if (has_diff) return 0.f;
  return -1.f;
}

// _eval_core (material.py:155-193); `opaque` scales the dielectric side for
// the transmission extension (exactly 1 for reference materials)
__device__ __forceinline__ f3 eval_core(f3 wo, f3 wi, f3 n, const GpuMaterial &mt,
                                        float opaque) {
  float no = dot(n, wo), ni = dot(n, wi);
  f3 f{0.f, 0.f, 0.f};
  if (no <= 0.f || ni <= 0.f) return f;
  float hx = wo.x + wi.x, hy = wo.y + wi.y, hz = wo.z + wi.z;
  float hl = sqrtf(hx * hx + hy * hy + hz * hz);
  if (hl <= 0.f) return f;
  const float rh = 1.f / hl;
  hx *= rh;
  hy *= rh;
  hz *= rh;
  float nh = n.x * hx + n.y * hy + n.z * hz;
  float oh = wo.x * hx + wo.y * hy + wo.z * hz;
  if (oh <= 0.f) return f;
  float spec_common = ggx_ndf(nh, mt.a2) * smith_g2(no, ni, mt.a2) / (4.f * no * ni);
  if (mt.m < 1.f) {
    float fd = diel_fresnel(oh, mt.f0d, mt.sw) * spec_common;
    float w = (1.f - mt.m) * opaque;
    f.x += w * (mt.diff * mt.bc[0] + fd);
    f.y += w * (mt.diff * mt.bc[1] + fd);
    f.z += w * (mt.diff * mt.bc[2] + fd);
  }
  if (mt.m > 0.f) {
    float s5 = pow5f(1.f - oh);
    float f0r = mt.bw * mt.bc[0], f0g = mt.bw * mt.bc[1], f0b = mt.bw * mt.bc[2];
    float ms = mt.m * spec_common;
    f.x += ms * (f0r + (mt.sc[0] - f0r) * s5);
    f.y += ms * (f0g + (mt.sc[1] - f0g) * s5);
    f.z += ms * (f0b + (mt.sc[2] - f0b) * s5);
  }
  return f;
}

// _pdf_core (material.py:216-243)
__device__ __forceinline__ float pdf_core(f3 wo, f3 wi, f3 n, const GpuMaterial &mt,
                                          float opaque) {
  float no = dot(n, wo), ni = dot(n, wi);
  if (no <= 0.f || ni <= 0.f) return 0.f;
  float hx = wo.x + wi.x, hy = wo.y + wi.y, hz = wo.z + wi.z;
  float hl = sqrtf(hx * hx + hy * hy + hz * hz);
  if (hl <= 0.f) return 0.f;
  const float rh = 1.f / hl;
  hx *= rh;
  hy *= rh;
  hz *= rh;
  float nh = n.x * hx + n.y * hy + n.z * hz;
  float oh = wo.x * hx + wo.y * hy + wo.z * hz;
  float pdf_ggx = 0.f;
  if (oh > 0.f && nh > 0.f) pdf_ggx = ggx_ndf(nh, mt.a2) * nh / (4.f * oh);
  float pdf_cos = ni * LT_INV_PI_F;
  float pdf = mt.m * pdf_ggx;
  if (mt.m < 1.f) {
    float p_spec = p_spec_select(no, mt);
    if (p_spec >= 0.f)
      pdf += (1.f - mt.m) * opaque * (p_spec * pdf_ggx + (1.f - p_spec) * pdf_cos);
  }
  return pdf;
}

// reference branch of _sample_core (material.py:293-351)
__device__ __forceinline__ bool sample_reference(f3 wo, f3 n, const GpuMaterial &mt,
                                                 float opaque, float u_lobe, float u1,
                                                 const SampleFrame &F, f3 &wi, f3 &wgt) {
  float no = dot(n, wo);
  if ((mt.flags & MAT_DIFFUSE_ONLY) && opaque == 1.f) {
    // diffuse-only: f cos / pdf collapses to the albedo exactly
    if (mt.bw <= 0.f || no <= 0.f) return false;
    wi = cosine_sample(F, n, u1);
    float ni = dot(n, wi);
    if (ni <= 0.f) return false;
    wgt = f3{mt.bw * mt.bc[0], mt.bw * mt.bc[1], mt.bw * mt.bc[2]};
    return true;
  }
  bool use_ggx;
  if (u_lobe < mt.m) {
    use_ggx = true;
  } else {
    float p_spec = p_spec_select(no, mt);
    if (p_spec < 0.f) return false;
    float u_d = mt.m < 1.f ? (u_lobe - mt.m) / (1.f - mt.m) : 0.f;
    use_ggx = u_d < p_spec;
  }
  if (use_ggx) {
    f3 h = ggx_sample_half(F, n, mt.a2, u1);
    float oh = dot(wo, h);
    if (oh <= 0.f) return false;
    float k = 2.f * oh;
    wi = f3{k * h.x - wo.x, k * h.y - wo.y, k * h.z - wo.z};
  } else {
    wi = cosine_sample(F, n, u1);
  }
  float ni = dot(n, wi);
  if (ni <= 0.f) return false;
  float pdf = pdf_core(wo, wi, n, mt, opaque);
  if (!(pdf > 0.f) || !isfinite(pdf)) return false;
  f3 f = eval_core(wo, wi, n, mt, opaque);
  float scale = ni / pdf;
  wgt = f3{f.x * scale, f.y * scale, f.z * scale};
  return true;
}

// extension: rough dielectric interface (see oracle oc_sample_glass)
__device__ __forceinline__ bool sample_glass(f3 wo, f3 n, const GpuMaterial &mt, bool front,
                                             float u_sel, float u1, const SampleFrame &fr, f3 &wi,
                                             f3 &wgt) {
  f3 h = ggx_sample_half(fr, n, mt.a2, u1);
  float c = dot(wo, h), no = dot(n, wo), nh = dot(n, h);
  if (c <= 0.f || no <= 0.f || nh <= 0.f) return false;
  float eta = front ? 1.f / mt.ior : mt.ior;
  float sin2t = eta * eta * (1.f - c * c);
  float F, cos_t = 0.f;
  if (sin2t >= 1.f) {
    F = 1.f;
  } else {
    cos_t = sqrtf(1.f - sin2t);
    float rs = (eta * c - cos_t) / (eta * c + cos_t);
    float rp = (c - eta * cos_t) / (c + eta * cos_t);
    F = 0.5f * (rs * rs + rp * rp);
  }
  f3 tint{1.f, 1.f, 1.f};
  bool reflect = u_sel < F;
  if (reflect) {
    float k = 2.f * c;
    wi = f3{k * h.x - wo.x, k * h.y - wo.y, k * h.z - wo.z};
  } else {
    float k = eta * c - cos_t;
    wi = f3{-eta * wo.x + k * h.x, -eta * wo.y + k * h.y, -eta * wo.z + k * h.z};
    tint = f3{mt.tc[0], mt.tc[1], mt.tc[2]};
  }
  float ni = dot(n, wi);
  if (reflect ? ni <= 0.f : ni >= 0.f) return false;
  float g = smith_g2(no, fabsf(ni), mt.a2);
  float w = c * g / (no * nh);
  if (!(w > 0.f) || !isfinite(w)) return false;
  wgt = f3{w * tint.x, w * tint.y, w * tint.z};
  return true;
}

// extension: clear-coat GGX lobe (see oracle oc_sample_coat)
__device__ __forceinline__ bool sample_coat(f3 wo, f3 n, const GpuMaterial &mt, float p_coat,
                                            float u1, const SampleFrame &F, f3 &wi, f3 &wgt) {
  f3 h = ggx_sample_half(F, n, mt.ca2, u1);
  float oh = dot(wo, h);
  if (oh <= 0.f) return false;
  float k = 2.f * oh;
  wi = f3{k * h.x - wo.x, k * h.y - wo.y, k * h.z - wo.z};
  float no = dot(n, wo), ni = dot(n, wi), nh = dot(n, h);
  if (no <= 0.f || ni <= 0.f || nh <= 0.f) return false;
  float Fc = mt.f0c + (1.f - mt.f0c) * pow5f(1.f - oh);
  float D = ggx_ndf(nh, mt.ca2);
  float pdf = D * nh / (4.f * oh);
  float f = mt.cw * Fc * D * smith_g2(no, ni, mt.ca2) / (4.f * no * ni);
  float w = f * ni / (p_coat * pdf);
  if (!(pdf > 0.f) || !isfinite(w)) return false;
  wgt = f3{w, w, w};
  return true;
}

// _sample_core with the extension chain on the same lobe draw:
// coat -> [metal | glass | reference dielectric]; reduces exactly to the
// reference for materials without coat/transmission.  The coat is a GGX
// interface of Schlick reflectance F (f0 from coat_ior) picked with
// probability cw F(no); the light that reaches the base crosses it twice
// and keeps (1 - cw F(no)) (1 - cw F(|ni|)) -- reciprocal, and energy
// conserving up to the coat's own masking (white furnace <= 1).
__device__ __forceinline__ bool sample_material(f3 wo, f3 n, const GpuMaterial &mt, bool front,
                                                float u_lobe, float u1, float u2, f3 &wi,
                                                f3 &wgt) {
  const SampleFrame F = sample_frame(n, u2);
  if (!(mt.flags & (MAT_COAT | MAT_GLASS)))
    return sample_reference(wo, n, mt, 1.f, u_lobe, u1, F, wi, wgt);
  float under = 1.f;
  if (mt.flags & MAT_COAT) {
    float no = dot(n, wo);
    if (no <= 0.f) return false;
    const float fo = mt.f0c + (1.f - mt.f0c) * pow5f(1.f - no);
    float p_coat = mt.cw * fminf(fmaxf(fo, 0.05f), 0.95f);
    if (u_lobe < p_coat) return sample_coat(wo, n, mt, p_coat, u1, F, wi, wgt);
    u_lobe = (u_lobe - p_coat) / (1.f - p_coat);
    under = (1.f - mt.cw * fo) / (1.f - p_coat);
  }
  bool ok;
  if (mt.flags & MAT_GLASS) {
    float lo = mt.m, hi = mt.m + (1.f - mt.m) * mt.tw;
    if (u_lobe >= lo && u_lobe < hi) {
      ok = sample_glass(wo, n, mt, front, (u_lobe - lo) / (hi - lo), u1, F, wi, wgt);
    } else {
      float u_ref = u_lobe;
      if (u_lobe >= hi) u_ref = fmaxf(mt.m + (u_lobe - hi) / (1.f - hi) * (1.f - mt.m), mt.m);
      ok = sample_reference(wo, n, mt, 1.f - mt.tw, u_ref, u1, F, wi, wgt);
    }
  } else {
    ok = sample_reference(wo, n, mt, 1.f, u_lobe, u1, F, wi, wgt);
  }
  if (ok && (mt.flags & MAT_COAT)) {
    // light crosses the coat twice: (1 - cw F(no)) (1 - cw F(|ni|))
    const float fi = mt.f0c + (1.f - mt.f0c) * pow5f(1.f - fabsf(dot(n, wi)));
    under *= 1.f - mt.cw * fi;
    wgt.x *= under * (1.f + (mt.cc[0] - 1.f) * mt.cw);
    wgt.y *= under * (1.f + (mt.cc[1] - 1.f) * mt.cw);
    wgt.z *= under * (1.f + (mt.cc[2] - 1.f) * mt.cw);
  }
  return ok;
}

// ---- the effective BSDF of the extension estimator (no reference; checked
// by furnace, reciprocity and chi-square tests, tests/test_gpu_functions.py)
//
// sample_material draws one lobe per scatter; the value and density that
// sampler realizes are:
//   f   = f_coat + (1 - cw F(no)) (1 - cw F(|ni|)) * tint_c * f_under
//   pdf = p_coat * pdf_coat + (1 - p_coat) * pdf_under
//   f_under   = f_ref(opaque = 1 - tw) + (1 - m) * tw * f_glass
//   pdf_under = pdf_ref(opaque)        + (1 - m) * tw * pdf_glass
// with the rough-dielectric interface of Walter et al. 2007 for the glass
// lobe (h ~ D(h) n.h, reflection with probability F):
//   reflection   f = F D G / (4 no |ni|),            pdf = F D nh / (4 wo.h)
//   transmission f = (1-F) D G (wo.h)|wi.h| / (no |ni| (eta wo.h + wi.h)^2) * tint_t,
//                pdf = (1-F) D nh |wi.h| / (eta wo.h + wi.h)^2
// (eta = eta_wo / eta_wi); every sample weight equals f |ni| / (lobe pdf).

__device__ __forceinline__ void eval_glass(f3 wo, f3 wi, f3 n, const GpuMaterial &mt, bool front,
                                           f3 &f, float &pdf) {
  f = f3{0.f, 0.f, 0.f};
  pdf = 0.f;
  const float no = dot(n, wo), ni = dot(n, wi);
  if (no <= 0.f || ni == 0.f) return;
  const float eta = front ? 1.f / mt.ior : mt.ior;
  const bool reflect = ni > 0.f;
  float hx, hy, hz;
  if (reflect) {
    hx = wo.x + wi.x;
    hy = wo.y + wi.y;
    hz = wo.z + wi.z;
  } else {  // wi = -eta wo + k h  =>  h ~ wi + eta wo
    hx = wi.x + eta * wo.x;
    hy = wi.y + eta * wo.y;
    hz = wi.z + eta * wo.z;
  }
  const float hl = sqrtf(hx * hx + hy * hy + hz * hz);
  if (!(hl > 0.f)) return;
  float s = 1.f / hl;
  if (n.x * hx + n.y * hy + n.z * hz < 0.f) s = -s;
  const f3 h{hx * s, hy * s, hz * s};
  const float c = dot(wo, h), ih = dot(wi, h), nh = dot(n, h);
  if (c <= 0.f || nh <= 0.f) return;
  const float sin2t = eta * eta * (1.f - c * c);
  float F = 1.f;
  if (sin2t < 1.f) {
    const float cos_t = sqrtf(1.f - sin2t);
    const float rs = (eta * c - cos_t) / (eta * c + cos_t);
    const float rp = (c - eta * cos_t) / (c + eta * cos_t);
    F = 0.5f * (rs * rs + rp * rp);
  }
  const float D = ggx_ndf(nh, mt.a2);
  const float G = smith_g2(no, fabsf(ni), mt.a2);
  if (reflect) {
    const float v = F * D * G / (4.f * no * ni);
    f = f3{v, v, v};
    pdf = F * D * nh / (4.f * c);
  } else {
    if (ih >= 0.f || F >= 1.f) return;  // not reachable by refraction
    const float den = eta * c + ih;
    const float q = (1.f - F) * D / (den * den);
    const float v = q * G * c * fabsf(ih) / (no * fabsf(ni));
    f = f3{v * mt.tc[0], v * mt.tc[1], v * mt.tc[2]};
    pdf = q * nh * fabsf(ih);
  }
}

__device__ __forceinline__ void eval_material(f3 wo, f3 wi, f3 n, const GpuMaterial &mt,
                                              bool front, f3 &f, float &pdf) {
  if (!(mt.flags & (MAT_COAT | MAT_GLASS))) {
    f = eval_core(wo, wi, n, mt, 1.f);
    pdf = pdf_core(wo, wi, n, mt, 1.f);
    return;
  }
  const float opaque = (mt.flags & MAT_GLASS) ? 1.f - mt.tw : 1.f;
  f3 fu = eval_core(wo, wi, n, mt, opaque);
  float pu = pdf_core(wo, wi, n, mt, opaque);
  if (mt.flags & MAT_GLASS) {
    f3 fg;
    float pg;
    eval_glass(wo, wi, n, mt, front, fg, pg);
    const float sg = (1.f - mt.m) * mt.tw;
    fu = f3{fu.x + sg * fg.x, fu.y + sg * fg.y, fu.z + sg * fg.z};
    pu += sg * pg;
  }
  if (!(mt.flags & MAT_COAT)) {
    f = fu;
    pdf = pu;
    return;
  }
  f = f3{0.f, 0.f, 0.f};
  pdf = 0.f;
  const float no = dot(n, wo), ni = dot(n, wi);
  if (no <= 0.f) return;
  const float fo = mt.f0c + (1.f - mt.f0c) * pow5f(1.f - no);
  const float p_coat = mt.cw * fminf(fmaxf(fo, 0.05f), 0.95f);
  float fc = 0.f, pc = 0.f;
  if (ni > 0.f) {
    float hx = wo.x + wi.x, hy = wo.y + wi.y, hz = wo.z + wi.z;
    const float hl = sqrtf(hx * hx + hy * hy + hz * hz);
    if (hl > 0.f) {
      const float r = 1.f / hl;
      const f3 h{hx * r, hy * r, hz * r};
      const float oh = dot(wo, h), nh = dot(n, h);
      if (oh > 0.f && nh > 0.f) {
        const float D = ggx_ndf(nh, mt.ca2);
        fc = mt.cw * (mt.f0c + (1.f - mt.f0c) * pow5f(1.f - oh)) * D *
             smith_g2(no, ni, mt.ca2) / (4.f * no * ni);
        pc = D * nh / (4.f * oh);
      }
    }
  }
  const float under = (1.f - mt.cw * fo) *
                      (1.f - mt.cw * (mt.f0c + (1.f - mt.f0c) * pow5f(1.f - fabsf(ni))));
  f = f3{fc + under * (1.f + (mt.cc[0] - 1.f) * mt.cw) * fu.x,
         fc + under * (1.f + (mt.cc[1] - 1.f) * mt.cw) * fu.y,
         fc + under * (1.f + (mt.cc[2] - 1.f) * mt.cw) * fu.z};
  pdf = p_coat * pc + (1.f - p_coat) * pu;
}
