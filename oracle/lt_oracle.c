/*
 * lt_oracle.c -- CPU fp64 restatement of the luxtrace reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (the parity checker and the CPU baseline; see
 * lt_oracle.h).  Each function names the reference function it restates,
 * as file:line under /root/reference/pkg/src/luxtrace/.  Operation order is
 * kept term-for-term so that, compiled with -ffp-contract=off, results are
 * bit-identical to the numba reference (pinned by tests/golden/).
 *
 * Extension lobes (coat, transmission) and the HDR environment have no
 * reference implementation: PARITY UNPINNED.  They are gated on non-zero
 * weights so reference materials never touch them.
 */
#include "lt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OC_PI 3.141592653589793
#define OC_INV_PI (1.0 / 3.141592653589793)
#define OC_DET_EPSILON 1e-9   /* geometry.py:17 */
#define OC_ALPHA_MIN 1e-4     /* material.py:21 */
#define OC_RR_MIN 0.05        /* integrator.py:34 */
#define OC_STACK 64           /* bvh.py:27 */

static void oc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------ rng.py */

/* _pcg_next, rng.py:37-47: XSH-RR output of the OLD state, then LCG step */
uint32_t oc_pcg_next(uint64_t *state, uint64_t inc) {
  uint64_t old = *state;
  *state = old * 6364136223846793005ULL + inc;
  uint32_t x = (uint32_t)(((old >> 18) ^ old) >> 27);
  uint32_t r = (uint32_t)(old >> 59);
  return (x >> r) | (x << ((32u - r) & 31u));
}

/* _pcg_seed, rng.py:50-58 */
void oc_pcg_seed(uint64_t init_state, uint64_t init_seq, uint64_t *state, uint64_t *inc) {
  uint64_t c = (init_seq << 1) | 1ULL;
  uint64_t st = 0;
  (void)oc_pcg_next(&st, c);
  st += init_state;
  (void)oc_pcg_next(&st, c);
  *state = st;
  *inc = c;
}

/* _mix64, rng.py:61-67 (splitmix64 finalizer) */
uint64_t oc_mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* _seed_stream, rng.py:70-78 */
void oc_seed_stream(uint64_t pixel, uint64_t sample, uint64_t seed, uint64_t *state,
                    uint64_t *inc) {
  oc_pcg_seed(oc_mix64(seed ^ oc_mix64(sample)), oc_mix64(pixel), state, inc);
}

/* _next_unit, rng.py:81-85 */
static inline double oc_unit(uint64_t *state, uint64_t inc) {
  return (double)oc_pcg_next(state, inc) * (1.0 / 4294967296.0);
}

/* ------------------------------------------------------------ geometry.py */

/* _mt_intersect, geometry.py:138-167 (double sided, |det| <= 1e-9 rejected) */
int oc_mt_intersect(const double o[3], const double d[3], const double a[3],
                    const double b[3], const double c[3], double t_min, double t_max,
                    double *t_out, double *u_out, double *v_out) {
  double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
  double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
  double px = d[1] * e2z - d[2] * e2y;
  double py = d[2] * e2x - d[0] * e2z;
  double pz = d[0] * e2y - d[1] * e2x;
  double det = e1x * px + e1y * py + e1z * pz;
  if (-OC_DET_EPSILON <= det && det <= OC_DET_EPSILON) return 0;
  double inv_det = 1.0 / det;
  double sx = o[0] - a[0], sy = o[1] - a[1], sz = o[2] - a[2];
  double u = (sx * px + sy * py + sz * pz) * inv_det;
  if (u < 0.0 || u > 1.0) return 0;
  double qx = sy * e1z - sz * e1y;
  double qy = sz * e1x - sx * e1z;
  double qz = sx * e1y - sy * e1x;
  double v = (d[0] * qx + d[1] * qy + d[2] * qz) * inv_det;
  if (v < 0.0 || u + v > 1.0) return 0;
  double t = (e2x * qx + e2y * qy + e2z * qz) * inv_det;
  if (t < t_min || t > t_max) return 0;
  *t_out = t;
  *u_out = u;
  *v_out = v;
  return 1;
}

/* _slab_intersect, geometry.py:170-207: compare/select form, NaN keeps the
 * running interval (0 * inf for an origin on a slab plane) */
int oc_slab_intersect(const double o[3], const double inv[3], const double bmin[3],
                      const double bmax[3], double t_min, double t_max,
                      double *t_enter, double *t_exit) {
  double tn = t_min, tf = t_max;
  for (int k = 0; k < 3; ++k) {
    double t0 = (bmin[k] - o[k]) * inv[k];
    double t1 = (bmax[k] - o[k]) * inv[k];
    if (t0 > t1) {
      double tmp = t0;
      t0 = t1;
      t1 = tmp;
    }
    if (t0 > tn) tn = t0;
    if (t1 < tf) tf = t1;
  }
  *t_enter = tn;
  *t_exit = tf;
  return tn <= tf;
}

/* _hit_frame, geometry.py:210-241 */
static void oc_hit_frame(const double d[3], const double *a, const double *b,
                         const double *c, const double *n0, const double *n1,
                         const double *n2, double u, double v, double g[3], double s[3],
                         int *front) {
  double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
  double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
  double gx = e1y * e2z - e1z * e2y;
  double gy = e1z * e2x - e1x * e2z;
  double gz = e1x * e2y - e1y * e2x;
  double glen = sqrt(gx * gx + gy * gy + gz * gz);
  if (glen > 0.0) {
    gx /= glen;
    gy /= glen;
    gz /= glen;
  }
  int fr = (gx * d[0] + gy * d[1] + gz * d[2]) < 0.0;
  if (!fr) {
    gx = -gx;
    gy = -gy;
    gz = -gz;
  }
  double w = 1.0 - u - v;
  double sx = w * n0[0] + u * n1[0] + v * n2[0];
  double sy = w * n0[1] + u * n1[1] + v * n2[1];
  double sz = w * n0[2] + u * n1[2] + v * n2[2];
  double slen = sqrt(sx * sx + sy * sy + sz * sz);
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
  g[0] = gx; g[1] = gy; g[2] = gz;
  s[0] = sx; s[1] = sy; s[2] = sz;
  *front = fr;
}

/* ----------------------------------------------------------------- bvh.py */

#define V3(arr, i) (&(arr)[3 * (int64_t)(i)])

/* _traverse_impl / _traverse_counted, bvh.py:359-425 / 439-508 */
int64_t oc_traverse(const oc_scene *s, const double o[3], const double d[3], double t_min,
                    double t_max, double *t_out, double *u_out, double *v_out,
                    int64_t *nodes_visited, int64_t *tri_tests) {
  double inv[3];
  for (int k = 0; k < 3; ++k) inv[k] = (d[k] == 0.0) ? INFINITY : 1.0 / d[k];
  int64_t nv = 1, tt = 0;
  double enter, ex;
  int64_t best_i = -1;
  double best_t = t_max, best_u = 0.0, best_v = 0.0;
  int ok = oc_slab_intersect(o, inv, V3(s->bmin, 0), V3(s->bmax, 0), t_min, t_max, &enter,
                             &ex);
  if (ok) {
    int32_t stack_node[OC_STACK];
    double stack_t[OC_STACK];
    int sp = 0;
    stack_node[sp] = 0;
    stack_t[sp] = enter;
    ++sp;
    while (sp > 0) {
      --sp;
      int32_t node = stack_node[sp];
      if (stack_t[sp] > best_t) continue;
      if (s->count[node] > 0) {
        int32_t f = s->first[node], c = s->count[node];
        for (int32_t k = f; k < f + c; ++k) {
          int32_t ti = s->order[k];
          double t, u, v;
          ++tt;
          if (oc_mt_intersect(o, d, V3(s->v0, ti), V3(s->v1, ti), V3(s->v2, ti), t_min, best_t,
                              &t, &u, &v) &&
              (t < best_t || (t == best_t && ti < best_i) || best_i < 0)) {
            best_t = t;
            best_i = ti;
            best_u = u;
            best_v = v;
          }
        }
      } else {
        int32_t lc = s->left[node], rc = s->right[node];
        double el, er, dummy;
        nv += 2;
        int okl = oc_slab_intersect(o, inv, V3(s->bmin, lc), V3(s->bmax, lc), t_min, best_t,
                                    &el, &dummy);
        int okr = oc_slab_intersect(o, inv, V3(s->bmin, rc), V3(s->bmax, rc), t_min, best_t,
                                    &er, &dummy);
        if (okl && okr) {
          if (el <= er) {
            stack_node[sp] = rc; stack_t[sp] = er; ++sp;
            stack_node[sp] = lc; stack_t[sp] = el; ++sp;
          } else {
            stack_node[sp] = lc; stack_t[sp] = el; ++sp;
            stack_node[sp] = rc; stack_t[sp] = er; ++sp;
          }
        } else if (okl) {
          stack_node[sp] = lc; stack_t[sp] = el; ++sp;
        } else if (okr) {
          stack_node[sp] = rc; stack_t[sp] = er; ++sp;
        }
      }
    }
  }
  if (nodes_visited) *nodes_visited = nv;
  if (tri_tests) *tri_tests = tt;
  *t_out = best_t;
  *u_out = best_u;
  *v_out = best_v;
  return best_i;
}

/* _traverse_batch, bvh.py:554-567 */
void oc_intersect_batch(const oc_scene *s, const double *origins, const double *dirs,
                        int64_t n, double t_min, double t_max, int64_t *idx, double *tout,
                        int n_threads) {
  oc_set_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t r = 0; r < n; ++r) {
    double t, u, v;
    int64_t i = oc_traverse(s, &origins[3 * r], &dirs[3 * r], t_min, t_max, &t, &u, &v, NULL,
                            NULL);
    idx[r] = i;
    tout[r] = i >= 0 ? t : INFINITY;
  }
}

/* _traverse_batch_counted, bvh.py:570-583 */
void oc_traversal_counts_batch(const oc_scene *s, const double *origins, const double *dirs,
                               int64_t n, double t_min, double t_max, int64_t *nodes,
                               int64_t *tests, int n_threads) {
  oc_set_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t r = 0; r < n; ++r) {
    double t, u, v;
    (void)oc_traverse(s, &origins[3 * r], &dirs[3 * r], t_min, t_max, &t, &u, &v, &nodes[r],
                      &tests[r]);
  }
}

/* _brute_force_batch, bvh.py:586-610 */
void oc_brute_force_batch(const oc_scene *s, const double *origins, const double *dirs,
                          int64_t n, double t_min, double t_max, int64_t *idx, double *tout,
                          int n_threads) {
  oc_set_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < n; ++r) {
    int64_t best_i = -1;
    double best_t = t_max;
    for (int64_t ti = 0; ti < s->n_tris; ++ti) {
      double t, u, v;
      if (oc_mt_intersect(&origins[3 * r], &dirs[3 * r], V3(s->v0, ti), V3(s->v1, ti),
                          V3(s->v2, ti), t_min, best_t, &t, &u, &v) &&
          (t < best_t || best_i < 0)) {
        best_t = t;
        best_i = ti;
      }
    }
    idx[r] = best_i;
    tout[r] = best_i >= 0 ? best_t : INFINITY;
  }
}

/* ------------------------------------------------------------ material.py */

typedef struct {
  double bw, bc[3], m, sw, sc[3], rough, ior;
  double cw, crough, cior, cc[3];  /* extension: coat */
  double tw, tc[3];                /* extension: transmission */
} oc_mat;

static void oc_mat_from_params(const double *p, oc_mat *mt) {
  mt->bw = p[0];
  mt->bc[0] = p[1]; mt->bc[1] = p[2]; mt->bc[2] = p[3];
  mt->m = p[4];
  mt->sw = p[5];
  mt->sc[0] = p[6]; mt->sc[1] = p[7]; mt->sc[2] = p[8];
  mt->rough = p[9];
  mt->ior = p[10];
  mt->cw = p[11];
  mt->crough = p[12];
  mt->cior = p[13];
  mt->cc[0] = p[14]; mt->cc[1] = p[15]; mt->cc[2] = p[16];
  mt->tw = p[17];
  mt->tc[0] = p[18]; mt->tc[1] = p[19]; mt->tc[2] = p[20];
}

static void oc_mat_from_scene(const oc_scene *s, int32_t mi, oc_mat *mt) {
  mt->bw = s->bw[mi];
  mt->m = s->metal[mi];
  mt->sw = s->sw[mi];
  mt->rough = s->rough[mi];
  mt->ior = s->ior[mi];
  for (int k = 0; k < 3; ++k) {
    mt->bc[k] = s->bc[3 * mi + k];
    mt->sc[k] = s->sc[3 * mi + k];
  }
  mt->cw = s->coat_w ? s->coat_w[mi] : 0.0;
  mt->crough = s->coat_rough ? s->coat_rough[mi] : 0.0;
  mt->cior = s->coat_ior ? s->coat_ior[mi] : 1.5;
  mt->tw = s->tr_w ? s->tr_w[mi] : 0.0;
  for (int k = 0; k < 3; ++k) {
    mt->cc[k] = s->coat_color ? s->coat_color[3 * mi + k] : 1.0;
    mt->tc[k] = s->tr_color ? s->tr_color[3 * mi + k] : 1.0;
  }
}

/* _alpha_of, material.py:99-104 */
static inline double oc_alpha_of(double r) {
  double a = r * r;
  if (a < OC_ALPHA_MIN) a = OC_ALPHA_MIN;
  return a;
}

/* _ggx_ndf, material.py:107-114 (cancellation-safe form) */
static inline double oc_ggx_ndf(double nh, double alpha) {
  if (nh <= 0.0) return 0.0;
  double a2 = alpha * alpha;
  double t = nh * nh * a2 + (1.0 - nh) * (1.0 + nh);
  return a2 / (OC_PI * t * t);
}

/* _smith_g2, material.py:117-126 */
static inline double oc_smith_g2(double no, double ni, double alpha) {
  double a2 = alpha * alpha;
  double lo = ni * sqrt(a2 + (1.0 - a2) * no * no);
  double li = no * sqrt(a2 + (1.0 - a2) * ni * ni);
  double denom = lo + li;
  if (denom <= 0.0) return 0.0;
  return 2.0 * no * ni / denom;
}

/* _pow5, material.py:129-132 */
static inline double oc_pow5(double x) {
  double x2 = x * x;
  return x2 * x2 * x;
}

/* _f0_from_ior, material.py:135-138 */
static inline double oc_f0_from_ior(double ior) {
  double r = (ior - 1.0) / (ior + 1.0);
  return r * r;
}

/* _diel_fresnel / _diel_fresnel_avg, material.py:141-152 */
static inline double oc_diel_fresnel(double c, double f0d, double sw) {
  return sw * (f0d + (1.0 - f0d) * oc_pow5(1.0 - c));
}
static inline double oc_diel_fresnel_avg(double f0d, double sw) {
  return sw * (f0d + (1.0 - f0d) / 21.0);
}

static inline double dot3(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/* _eval_core, material.py:155-193.  `opaque` scales the dielectric side for
 * the transmission extension (1.0 exactly for reference materials, where the
 * scaling branch is skipped altogether). */
static void oc_eval_core(const double wo[3], const double wi[3], const double n[3],
                         const oc_mat *mt, double opaque, double f[3]) {
  f[0] = f[1] = f[2] = 0.0;
  double no = n[0] * wo[0] + n[1] * wo[1] + n[2] * wo[2];
  double ni = n[0] * wi[0] + n[1] * wi[1] + n[2] * wi[2];
  if (no <= 0.0 || ni <= 0.0) return;
  double hx = wo[0] + wi[0], hy = wo[1] + wi[1], hz = wo[2] + wi[2];
  double hl = sqrt(hx * hx + hy * hy + hz * hz);
  if (hl <= 0.0) return;
  hx /= hl;
  hy /= hl;
  hz /= hl;
  double nh = n[0] * hx + n[1] * hy + n[2] * hz;
  double oh = wo[0] * hx + wo[1] * hy + wo[2] * hz;
  if (oh <= 0.0) return;
  double alpha = oc_alpha_of(mt->rough);
  double spec_common = oc_ggx_ndf(nh, alpha) * oc_smith_g2(no, ni, alpha) / (4.0 * no * ni);
  double fr = 0.0, fg = 0.0, fb = 0.0;
  if (mt->m < 1.0) {
    double f0d = oc_f0_from_ior(mt->ior);
    double diff = mt->bw * OC_INV_PI * (1.0 - oc_diel_fresnel_avg(f0d, mt->sw));
    double fd = oc_diel_fresnel(oh, f0d, mt->sw) * spec_common;
    double w = 1.0 - mt->m;
    if (opaque != 1.0) w = w * opaque; /* transmission extension only */
    fr += w * (diff * mt->bc[0] + fd);
    fg += w * (diff * mt->bc[1] + fd);
    fb += w * (diff * mt->bc[2] + fd);
  }
  if (mt->m > 0.0) {
    double s5 = oc_pow5(1.0 - oh);
    double f0r = mt->bw * mt->bc[0], f0g = mt->bw * mt->bc[1], f0b = mt->bw * mt->bc[2];
    fr += mt->m * spec_common * (f0r + (mt->sc[0] - f0r) * s5);
    fg += mt->m * spec_common * (f0g + (mt->sc[1] - f0g) * s5);
    fb += mt->m * spec_common * (f0b + (mt->sc[2] - f0b) * s5);
  }
  f[0] = fr;
  f[1] = fg;
  f[2] = fb;
}

/* _p_spec_select, material.py:196-213 */
static inline double oc_p_spec_select(double no, double bw, double sw, double f0d) {
  int has_diff = bw > 0.0, has_spec = sw > 0.0;
  if (has_diff && has_spec) {
    double p = oc_diel_fresnel(no, f0d, sw);
    if (p < 0.05) p = 0.05;
    else if (p > 0.95) p = 0.95;
    return p;
  }
  if (has_spec) return 1.0;
  if (has_diff) return 0.0;
  return -1.0;
}

/* _pdf_core, material.py:216-243 (`opaque` as in oc_eval_core) */
static double oc_pdf_core(const double wo[3], const double wi[3], const double n[3],
                          const oc_mat *mt, double opaque) {
  double no = n[0] * wo[0] + n[1] * wo[1] + n[2] * wo[2];
  double ni = n[0] * wi[0] + n[1] * wi[1] + n[2] * wi[2];
  if (no <= 0.0 || ni <= 0.0) return 0.0;
  double hx = wo[0] + wi[0], hy = wo[1] + wi[1], hz = wo[2] + wi[2];
  double hl = sqrt(hx * hx + hy * hy + hz * hz);
  if (hl <= 0.0) return 0.0;
  hx /= hl;
  hy /= hl;
  hz /= hl;
  double nh = n[0] * hx + n[1] * hy + n[2] * hz;
  double oh = wo[0] * hx + wo[1] * hy + wo[2] * hz;
  double alpha = oc_alpha_of(mt->rough);
  double pdf_ggx = 0.0;
  if (oh > 0.0 && nh > 0.0) pdf_ggx = oc_ggx_ndf(nh, alpha) * nh / (4.0 * oh);
  double pdf_cos = ni * OC_INV_PI;
  double pdf = mt->m * pdf_ggx;
  if (mt->m < 1.0) {
    double p_spec = oc_p_spec_select(no, mt->bw, mt->sw, oc_f0_from_ior(mt->ior));
    if (p_spec >= 0.0) {
      double w = 1.0 - mt->m;
      if (opaque != 1.0) w = w * opaque;
      pdf += w * (p_spec * pdf_ggx + (1.0 - p_spec) * pdf_cos);
    }
  }
  return pdf;
}

/* _onb, material.py:246-261 */
static void oc_onb(const double n[3], double t[3], double b[3]) {
  double ax, ay, az;
  if (fabs(n[0]) > 0.9) {
    ax = 0.0; ay = 1.0; az = 0.0;
  } else {
    ax = 1.0; ay = 0.0; az = 0.0;
  }
  double tx = ay * n[2] - az * n[1];
  double ty = az * n[0] - ax * n[2];
  double tz = ax * n[1] - ay * n[0];
  double tl = sqrt(tx * tx + ty * ty + tz * tz);
  tx /= tl;
  ty /= tl;
  tz /= tl;
  t[0] = tx; t[1] = ty; t[2] = tz;
  b[0] = n[1] * tz - n[2] * ty;
  b[1] = n[2] * tx - n[0] * tz;
  b[2] = n[0] * ty - n[1] * tx;
}

/* _cosine_sample, material.py:264-274 */
static void oc_cosine_sample(const double n[3], double u1, double u2, double w[3]) {
  double t[3], b[3];
  oc_onb(n, t, b);
  double r = sqrt(u1);
  double phi = 2.0 * OC_PI * u2;
  double x = r * cos(phi);
  double y = r * sin(phi);
  double zz = 1.0 - u1;
  double z = sqrt(zz > 0.0 ? zz : 0.0);
  for (int k = 0; k < 3; ++k) w[k] = x * t[k] + y * b[k] + z * n[k];
}

/* _ggx_sample_half, material.py:277-290 */
static void oc_ggx_sample_half(const double n[3], double alpha, double u1, double u2,
                               double h[3]) {
  double t[3], b[3];
  oc_onb(n, t, b);
  double a2 = alpha * alpha;
  double ct = sqrt((1.0 - u1) / (1.0 + (a2 - 1.0) * u1));
  double q = 1.0 - ct * ct;
  double st = sqrt(q > 0.0 ? q : 0.0);
  double phi = 2.0 * OC_PI * u2;
  double x = st * cos(phi);
  double y = st * sin(phi);
  for (int k = 0; k < 3; ++k) h[k] = x * t[k] + y * b[k] + ct * n[k];
}

/* exact dielectric Fresnel for the transmission extension; eta = eta_i/eta_t */
static double oc_fresnel_dielectric(double c, double eta, double *cos_t) {
  double sin2t = eta * eta * (1.0 - c * c);
  if (sin2t >= 1.0) {
    *cos_t = 0.0;
    return 1.0;
  }
  double ct = sqrt(1.0 - sin2t);
  double rs = (eta * c - ct) / (eta * c + ct);
  double rp = (c - eta * ct) / (c + eta * ct);
  *cos_t = ct;
  return 0.5 * (rs * rs + rp * rp);
}

/* Reference branch of _sample_core (material.py:293-351) with lobe draw u.
 * `opaque` = 1 - transmission weight (exactly 1 for reference materials). */
static int oc_sample_reference(const double wo[3], const double n[3], const oc_mat *mt,
                               double opaque, double u_lobe, double u1, double u2,
                               double wi[3], double wgt[3], double *pdf_out, int *spike) {
  double alpha = oc_alpha_of(mt->rough);
  double f0d = oc_f0_from_ior(mt->ior);
  double no = n[0] * wo[0] + n[1] * wo[1] + n[2] * wo[2];
  if (mt->m <= 0.0 && mt->sw <= 0.0 && opaque == 1.0) {
    /* diffuse-only material: f cos / pdf collapses to the albedo exactly */
    if (mt->bw <= 0.0 || no <= 0.0) return 0;
    oc_cosine_sample(n, u1, u2, wi);
    double ni = n[0] * wi[0] + n[1] * wi[1] + n[2] * wi[2];
    if (ni <= 0.0) return 0;
    double pdf = ni * OC_INV_PI;
    if (pdf <= 0.0) return 0;
    wgt[0] = mt->bw * mt->bc[0];
    wgt[1] = mt->bw * mt->bc[1];
    wgt[2] = mt->bw * mt->bc[2];
    *pdf_out = pdf;
    *spike = 0;
    return 1;
  }
  int use_ggx = 0;
  if (u_lobe < mt->m) {
    use_ggx = 1;
  } else {
    double p_spec = oc_p_spec_select(no, mt->bw, mt->sw, f0d);
    if (p_spec < 0.0) return 0;
    double u_d = mt->m < 1.0 ? (u_lobe - mt->m) / (1.0 - mt->m) : 0.0;
    use_ggx = u_d < p_spec;
  }
  if (use_ggx) {
    double h[3];
    oc_ggx_sample_half(n, alpha, u1, u2, h);
    double oh = wo[0] * h[0] + wo[1] * h[1] + wo[2] * h[2];
    if (oh <= 0.0) return 0;
    for (int k = 0; k < 3; ++k) wi[k] = 2.0 * oh * h[k] - wo[k];
  } else {
    oc_cosine_sample(n, u1, u2, wi);
  }
  double ni = n[0] * wi[0] + n[1] * wi[1] + n[2] * wi[2];
  if (ni <= 0.0) return 0;
  double pdf = oc_pdf_core(wo, wi, n, mt, opaque);
  if (pdf <= 0.0 || !isfinite(pdf)) return 0;
  double f[3];
  oc_eval_core(wo, wi, n, mt, opaque, f);
  double scale = ni / pdf;
  wgt[0] = f[0] * scale;
  wgt[1] = f[1] * scale;
  wgt[2] = f[2] * scale;
  *pdf_out = pdf;
  *spike = use_ggx && alpha <= OC_ALPHA_MIN;
  return 1;
}

/* Extension: rough dielectric interface (transmission lobe), GGX half-vector
 * sampling with D(h)(n.h); reflect with probability F, else refract.  The
 * Fresnel term cancels against the selection probability, so both branches
 * carry |wo.h| G2 / (|wo.n| |n.h|).  PARITY UNPINNED. */
static int oc_sample_glass(const double wo[3], const double n[3], const oc_mat *mt,
                           int front, double u_sel, double u1, double u2, double wi[3],
                           double wgt[3], double *pdf_out, int *spike) {
  double alpha = oc_alpha_of(mt->rough);
  double h[3];
  oc_ggx_sample_half(n, alpha, u1, u2, h);
  double c = dot3(wo, h);
  double no = dot3(n, wo);
  double nh = dot3(n, h);
  if (c <= 0.0 || no <= 0.0 || nh <= 0.0) return 0;
  double eta = front ? 1.0 / mt->ior : mt->ior;
  double cos_t;
  double F = oc_fresnel_dielectric(c, eta, &cos_t);
  double D = oc_ggx_ndf(nh, alpha);
  double tint[3] = {1.0, 1.0, 1.0};
  double pdf;
  if (u_sel < F) {
    for (int k = 0; k < 3; ++k) wi[k] = 2.0 * c * h[k] - wo[k];
    pdf = F * D * nh / (4.0 * c);
  } else {
    for (int k = 0; k < 3; ++k) wi[k] = -eta * wo[k] + (eta * c - cos_t) * h[k];
    for (int k = 0; k < 3; ++k) tint[k] = mt->tc[k];
    double ih = dot3(wi, h);
    double den = eta * c + ih; /* (eta_i (o.h) + eta_t (i.h)) / eta_t, i.h < 0 */
    pdf = (1.0 - F) * D * nh * fabs(ih) / (den * den);
  }
  double ni = dot3(n, wi);
  int reflected = u_sel < F;
  if (reflected ? ni <= 0.0 : ni >= 0.0) return 0;
  double g = oc_smith_g2(no, fabs(ni), alpha);
  double w = c * g / (no * nh);
  if (!(w > 0.0) || !isfinite(w) || !(pdf > 0.0)) return 0;
  for (int k = 0; k < 3; ++k) wgt[k] = w * tint[k];
  *pdf_out = pdf;
  *spike = alpha <= OC_ALPHA_MIN;
  return 1;
}

/* Extension: clear-coat GGX lobe on top of the base, picked with probability
 * cw F(no); the base's light crosses the coat twice, (1 - cw F(no)) (1 - cw
 * F(|ni|)) -- the estimator of csrc/lt_material.cuh.  PARITY UNPINNED. */
static int oc_sample_coat(const double wo[3], const double n[3], const oc_mat *mt,
                          double p_coat, double u1, double u2, double wi[3], double wgt[3],
                          double *pdf_out, int *spike) {
  double alpha = oc_alpha_of(mt->crough);
  double h[3];
  oc_ggx_sample_half(n, alpha, u1, u2, h);
  double oh = dot3(wo, h);
  if (oh <= 0.0) return 0;
  for (int k = 0; k < 3; ++k) wi[k] = 2.0 * oh * h[k] - wo[k];
  double no = dot3(n, wo), ni = dot3(n, wi), nh = dot3(n, h);
  if (no <= 0.0 || ni <= 0.0 || nh <= 0.0) return 0;
  double f0c = oc_f0_from_ior(mt->cior);
  double Fc = f0c + (1.0 - f0c) * oc_pow5(1.0 - oh);
  double D = oc_ggx_ndf(nh, alpha);
  double pdf = D * nh / (4.0 * oh);
  double f = mt->cw * Fc * D * oc_smith_g2(no, ni, alpha) / (4.0 * no * ni);
  double w = f * ni / (p_coat * pdf);
  if (!(pdf > 0.0) || !isfinite(w)) return 0;
  wgt[0] = wgt[1] = wgt[2] = w;
  *pdf_out = p_coat * pdf;
  *spike = alpha <= OC_ALPHA_MIN;
  return 1;
}

/* _sample_core, material.py:293-351, plus the extension chain on the same
 * lobe draw (coat -> [metal | glass | reference dielectric]).  For reference
 * materials (coat and transmission weights 0) this is exactly _sample_core. */
static int oc_sample_material(const double wo[3], const double n[3], const oc_mat *mt,
                              int front, double u_lobe, double u1, double u2, double wi[3],
                              double wgt[3], double *pdf, int *spike) {
  double under = 1.0, f0c = 0.0;
  if (mt->cw > 0.0) {
    double no = dot3(n, wo);
    if (no <= 0.0) return 0;
    f0c = oc_f0_from_ior(mt->cior);
    double fo = f0c + (1.0 - f0c) * oc_pow5(1.0 - no);
    double fc = fo;
    if (fc < 0.05) fc = 0.05;
    else if (fc > 0.95) fc = 0.95;
    double p_coat = mt->cw * fc;
    if (u_lobe < p_coat) return oc_sample_coat(wo, n, mt, p_coat, u1, u2, wi, wgt, pdf, spike);
    u_lobe = (u_lobe - p_coat) / (1.0 - p_coat);
    under = (1.0 - mt->cw * fo) / (1.0 - p_coat);
  }
  int ok;
  if (mt->tw > 0.0 && mt->m < 1.0) {
    /* glass is selected inside the dielectric branch: u in [m, m + (1-m) tw) */
    double p_glass_lo = mt->m, p_glass_hi = mt->m + (1.0 - mt->m) * mt->tw;
    if (u_lobe >= p_glass_lo && u_lobe < p_glass_hi) {
      double u_sel = (u_lobe - p_glass_lo) / (p_glass_hi - p_glass_lo);
      ok = oc_sample_glass(wo, n, mt, front, u_sel, u1, u2, wi, wgt, pdf, spike);
    } else {
      /* the remaining lobes, re-normalized: metal keeps u < m; the dielectric
       * draw is remapped over the opaque part of [m, 1) */
      double u_ref = u_lobe;
      if (u_lobe >= p_glass_hi) {
        u_ref = mt->m + (u_lobe - p_glass_hi) / (1.0 - p_glass_hi) * (1.0 - mt->m);
        if (u_ref < mt->m) u_ref = mt->m;
      }
      /* eval and pdf scale the dielectric side by (1 - tw): the pdf is then
       * the joint density of "non-glass lobe and this direction", which is
       * exactly the one-sample estimator for the non-glass part of f */
      double opaque = 1.0 - mt->tw;
      ok = oc_sample_reference(wo, n, mt, opaque, u_ref, u1, u2, wi, wgt, pdf, spike);
    }
  } else {
    ok = oc_sample_reference(wo, n, mt, 1.0, u_lobe, u1, u2, wi, wgt, pdf, spike);
  }
  if (ok && mt->cw > 0.0) {
    /* the light that reaches the base crosses the coat twice */
    double fi = f0c + (1.0 - f0c) * oc_pow5(1.0 - fabs(dot3(n, wi)));
    under = under * (1.0 - mt->cw * fi);
    for (int k = 0; k < 3; ++k) {
      double tint = 1.0 + (mt->cc[k] - 1.0) * mt->cw;
      wgt[k] = wgt[k] * under * tint;
    }
  }
  return ok;
}

/* public checked-free wrappers (eval_bsdf / pdf_bsdf / sample_bsdf) */
void oc_eval_bsdf(const double wo[3], const double wi[3], const double n[3],
                  const double *params, double f[3]) {
  oc_mat mt;
  oc_mat_from_params(params, &mt);
  oc_eval_core(wo, wi, n, &mt, 1.0, f);
}

double oc_pdf_bsdf(const double wo[3], const double wi[3], const double n[3],
                   const double *params) {
  oc_mat mt;
  oc_mat_from_params(params, &mt);
  return oc_pdf_core(wo, wi, n, &mt, 1.0);
}

int oc_sample_bsdf(const double wo[3], const double n[3], const double *params,
                   double u_lobe, double u1, double u2, int front, double wi[3],
                   double weight[3], double *pdf, int *spike) {
  oc_mat mt;
  oc_mat_from_params(params, &mt);
  *pdf = 0.0;
  *spike = 0;
  int ok = oc_sample_material(wo, n, &mt, front, u_lobe, u1, u2, wi, weight, pdf, spike);
  if (!ok) {
    wi[0] = wi[1] = wi[2] = 0.0;
    weight[0] = weight[1] = weight[2] = 0.0;
  }
  return ok;
}

/* ---------------------------------------------------------- integrator.py */

/* _camera_dir, integrator.py:86-98 */
void oc_camera_dir(const double cam[14], double px, double py, double jx, double jy,
                   int32_t width, int32_t height, double d[3]) {
  double sx = 2.0 * (px + jx) / (double)width - 1.0;
  double sy = 1.0 - 2.0 * (py + jy) / (double)height;
  double hx = cam[12] * cam[13] * sx;
  double hy = cam[12] * sy;
  double dx = cam[3] + cam[6] * hx + cam[9] * hy;
  double dy = cam[4] + cam[7] * hx + cam[10] * hy;
  double dz = cam[5] + cam[8] * hx + cam[11] * hy;
  double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
  d[0] = dx * inv;
  d[1] = dy * inv;
  d[2] = dz * inv;
}

/* _env_radiance, integrator.py:124-136; kind 2 = HDR lat-long map
 * (extension, bilinear, PARITY UNPINNED) */
void oc_env_radiance(const oc_scene *s, const double d[3], double out[3]) {
  if (s->env_kind == 0) {
    out[0] = s->env_a[0];
    out[1] = s->env_a[1];
    out[2] = s->env_a[2];
    return;
  }
  if (s->env_kind == 1) {
    double t = d[1];
    if (t < 0.0) t = 0.0;
    else if (t > 1.0) t = 1.0;
    for (int k = 0; k < 3; ++k) out[k] = s->env_b[k] + (s->env_a[k] - s->env_b[k]) * t;
    return;
  }
  /* lat-long: u = 0.5 + atan2(x, -z)/(2 pi), v = acos(y)/pi */
  double y = d[1] < -1.0 ? -1.0 : (d[1] > 1.0 ? 1.0 : d[1]);
  double u = 0.5 + atan2(d[0], -d[2]) * (0.5 / OC_PI);
  double v = acos(y) * (1.0 / OC_PI);
  double fx = u * s->env_w - 0.5, fy = v * s->env_h - 0.5;
  double x0f = floor(fx), y0f = floor(fy);
  double ax = fx - x0f, ay = fy - y0f;
  int64_t x0 = (int64_t)x0f, y0 = (int64_t)y0f;
  int64_t x1 = x0 + 1, y1 = y0 + 1;
  x0 = ((x0 % s->env_w) + s->env_w) % s->env_w;
  x1 = ((x1 % s->env_w) + s->env_w) % s->env_w;
  if (y0 < 0) y0 = 0;
  if (y1 < 0) y1 = 0;
  if (y0 > s->env_h - 1) y0 = s->env_h - 1;
  if (y1 > s->env_h - 1) y1 = s->env_h - 1;
  for (int k = 0; k < 3; ++k) {
    double c00 = s->env_map[(y0 * s->env_w + x0) * 3 + k];
    double c10 = s->env_map[(y0 * s->env_w + x1) * 3 + k];
    double c01 = s->env_map[(y1 * s->env_w + x0) * 3 + k];
    double c11 = s->env_map[(y1 * s->env_w + x1) * 3 + k];
    double top = c00 + (c10 - c00) * ax;
    double bot = c01 + (c11 - c01) * ax;
    out[k] = (top + (bot - top) * ay) * s->env_scale;
  }
}

/* _trace, integrator.py:149-227.  Returns the number of segments traced. */
int oc_trace(const oc_scene *s, const double o_in[3], const double d_in[3], uint64_t *state,
             uint64_t inc, int32_t max_depth, int32_t rr_start, double t_min,
             double rgb[3]) {
  double o[3] = {o_in[0], o_in[1], o_in[2]};
  double d[3] = {d_in[0], d_in[1], d_in[2]};
  double lr = 0.0, lg = 0.0, lb = 0.0;
  double tr = 1.0, tg = 1.0, tb = 1.0;
  int segments = 0;
  for (int32_t depth = 0; depth < max_depth; ++depth) {
    double t, u, v;
    ++segments;
    int64_t ti = oc_traverse(s, o, d, t_min, INFINITY, &t, &u, &v, NULL, NULL);
    if (ti < 0) {
      double e[3];
      oc_env_radiance(s, d, e);
      lr += tr * e[0];
      lg += tg * e[1];
      lb += tb * e[2];
      break;
    }
    int32_t mi = s->mat_index[ti];
    double el = s->el[mi];
    if (el > 0.0) {
      lr += tr * el * s->ec[3 * mi + 0];
      lg += tg * el * s->ec[3 * mi + 1];
      lb += tb * el * s->ec[3 * mi + 2];
    }
    if (depth == max_depth - 1) break; /* segment budget spent */
    double g[3], sn[3];
    int front;
    oc_hit_frame(d, V3(s->v0, ti), V3(s->v1, ti), V3(s->v2, ti), V3(s->n0, ti), V3(s->n1, ti),
                 V3(s->n2, ti), u, v, g, sn, &front);
    double u_lobe = oc_unit(state, inc);
    double u1 = oc_unit(state, inc);
    double u2 = oc_unit(state, inc);
    oc_mat mt;
    oc_mat_from_scene(s, mi, &mt);
    double wo[3] = {-d[0], -d[1], -d[2]};
    double wi[3], w[3], pdf;
    int spike;
    if (!oc_sample_material(wo, sn, &mt, front, u_lobe, u1, u2, wi, w, &pdf, &spike)) break;
    tr *= w[0];
    tg *= w[1];
    tb *= w[2];
    if (tr <= 0.0 && tg <= 0.0 && tb <= 0.0) break;
    if (depth >= rr_start) {
      double p = tr;
      if (tg > p) p = tg;
      if (tb > p) p = tb;
      if (p > 1.0) p = 1.0;
      else if (p < OC_RR_MIN) p = OC_RR_MIN;
      double u_rr = oc_unit(state, inc);
      if (u_rr >= p) break;
      tr /= p;
      tg /= p;
      tb /= p;
    }
    o[0] = o[0] + t * d[0];
    o[1] = o[1] + t * d[1];
    o[2] = o[2] + t * d[2];
    d[0] = wi[0];
    d[1] = wi[1];
    d[2] = wi[2];
  }
  rgb[0] = lr;
  rgb[1] = lg;
  rgb[2] = lb;
  return segments;
}

static void oc_primary(int64_t pix, int64_t sample, const double cam[14], int32_t width,
                       int32_t height, uint64_t seed, uint64_t *state, uint64_t *inc,
                       double d[3]) {
  int64_t py = pix / width;
  int64_t px = pix - py * width;
  oc_seed_stream((uint64_t)pix, (uint64_t)sample, seed, state, inc);
  double jx = oc_unit(state, *inc);
  double jy = oc_unit(state, *inc);
  oc_camera_dir(cam, (double)px, (double)py, jx, jy, width, height, d);
}

/* _render_pass, integrator.py:230-277 */
void oc_render_pass(const oc_scene *s, double *accum, int64_t *valid, int64_t *invalid,
                    int64_t sample_start, int64_t sample_count, const double cam[14],
                    int32_t width, int32_t height, uint64_t seed, int32_t max_depth,
                    int32_t rr_start, double t_min, int n_threads, int64_t *segments) {
  int64_t n_pixels = (int64_t)width * height;
  int64_t seg_total = 0;
  oc_set_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : seg_total)
  for (int64_t pix = 0; pix < n_pixels; ++pix) {
    double mr = accum[3 * pix + 0], mg = accum[3 * pix + 1], mb = accum[3 * pix + 2];
    int64_t nv = valid[pix], ni = invalid[pix];
    for (int64_t smp = sample_start; smp < sample_start + sample_count; ++smp) {
      uint64_t state, inc;
      double d[3], rgb[3];
      oc_primary(pix, smp, cam, width, height, seed, &state, &inc, d);
      seg_total += oc_trace(s, cam, d, &state, inc, max_depth, rr_start, t_min, rgb);
      if (isfinite(rgb[0]) && isfinite(rgb[1]) && isfinite(rgb[2])) {
        nv += 1;
        mr += (rgb[0] - mr) / (double)nv;
        mg += (rgb[1] - mg) / (double)nv;
        mb += (rgb[2] - mb) / (double)nv;
      } else {
        ni += 1;
      }
    }
    accum[3 * pix + 0] = mr;
    accum[3 * pix + 1] = mg;
    accum[3 * pix + 2] = mb;
    valid[pix] = nv;
    invalid[pix] = ni;
  }
  if (segments) *segments = seg_total;
}

void oc_sample_values(const oc_scene *s, const int64_t *pixels, int64_t n, int64_t sample,
                      const double cam[14], int32_t width, int32_t height, uint64_t seed,
                      int32_t max_depth, int32_t rr_start, double t_min, double *rgb,
                      int32_t *segments, int n_threads) {
  oc_set_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t state, inc;
    double d[3];
    oc_primary(pixels[i], sample, cam, width, height, seed, &state, &inc, d);
    int sg = oc_trace(s, cam, d, &state, inc, max_depth, rr_start, t_min, &rgb[3 * i]);
    if (segments) segments[i] = sg;
  }
}

void oc_primary_rays(const int64_t *pixels, int64_t n, int64_t sample, const double cam[14],
                     int32_t width, int32_t height, uint64_t seed, double *origins,
                     double *dirs) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t state, inc;
    oc_primary(pixels[i], sample, cam, width, height, seed, &state, &inc, &dirs[3 * i]);
    origins[3 * i + 0] = cam[0];
    origins[3 * i + 1] = cam[1];
    origins[3 * i + 2] = cam[2];
  }
}

/* ---------------------------------------------------------- bvh.py build */

/* _triangle_bounds_arrays (bvh.py:57-77) + _build_kernel (bvh.py:85-262):
 * the reference's single-threaded binned-SAH build restated in C so the CPU
 * baseline (bench.py --impl reference) builds its tree without the product
 * library.  Output arrays are caller-owned, sized for 2n nodes; returns the
 * node count, or -1 on an allocation failure. */
static double oc_half_area(double dx, double dy, double dz) { return dx * dy + dx * dz + dy * dz; }

#define OC_BOUNDS_PADDING 1e-7  /* geometry.py:19 */
#define OC_MAX_TREE_DEPTH 60    /* bvh.py:26 */

int64_t oc_build_bvh(const double *v0, const double *v1, const double *v2, int64_t n,
                     int32_t leaf_size, int32_t n_bins, double *bmin, double *bmax,
                     int32_t *left, int32_t *right, int32_t *first, int32_t *count,
                     int32_t *order, int64_t *leaf_count_out, int64_t *max_depth_out) {
  double *tb_min = malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  double *tb_max = malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  double *cent = malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  int64_t *bin_count = malloc(sizeof(int64_t) * (size_t)n_bins);
  double *bin_min = malloc(sizeof(double) * 3 * (size_t)n_bins);
  double *bin_max = malloc(sizeof(double) * 3 * (size_t)n_bins);
  double *sweep_area = malloc(sizeof(double) * (size_t)n_bins);
  int64_t *sweep_count = malloc(sizeof(int64_t) * (size_t)n_bins);
  int64_t (*stack)[4] = malloc(sizeof(int64_t) * 4 * (OC_MAX_TREE_DEPTH + 8));
  int64_t n_nodes = -1;
  if (!tb_min || !tb_max || !cent || !bin_count || !bin_min || !bin_max || !sweep_area ||
      !sweep_count || !stack)
    goto done;
  for (int64_t i = 0; i < n; ++i) {
    double ext = 0.0;
    for (int a = 0; a < 3; ++a) {
      double p = v0[3 * i + a], q = v1[3 * i + a], r = v2[3 * i + a];
      double lo = p < (q < r ? q : r) ? p : (q < r ? q : r);
      double hi = p > (q > r ? q : r) ? p : (q > r ? q : r);
      tb_min[3 * i + a] = lo;
      tb_max[3 * i + a] = hi;
      if (hi - lo > ext) ext = hi - lo;
    }
    double pad = OC_BOUNDS_PADDING * ext;
    for (int a = 0; a < 3; ++a) {
      tb_min[3 * i + a] -= pad;
      tb_max[3 * i + a] += pad;
      cent[3 * i + a] = 0.5 * (tb_min[3 * i + a] + tb_max[3 * i + a]);
    }
  }
  for (int64_t i = 0; i < 2 * n; ++i) {
    left[i] = -1;
    right[i] = -1;
    first[i] = 0;
    count[i] = 0;
  }
  for (int64_t i = 0; i < n; ++i) order[i] = (int32_t)i;
  int64_t sp = 0, leaf_count = 0, max_depth = 0;
  stack[0][0] = 0; stack[0][1] = 0; stack[0][2] = n; stack[0][3] = 0;
  sp = 1;
  n_nodes = 1;
  while (sp > 0) {
    --sp;
    const int64_t node = stack[sp][0], f = stack[sp][1], c = stack[sp][2], depth = stack[sp][3];
    if (depth > max_depth) max_depth = depth;
    double nmin[3] = {INFINITY, INFINITY, INFINITY}, nmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t k = f; k < f + c; ++k) {
      const int64_t ti = order[k];
      for (int a = 0; a < 3; ++a) {
        if (tb_min[3 * ti + a] < nmin[a]) nmin[a] = tb_min[3 * ti + a];
        if (tb_max[3 * ti + a] > nmax[a]) nmax[a] = tb_max[3 * ti + a];
      }
    }
    for (int a = 0; a < 3; ++a) {
      bmin[3 * node + a] = nmin[a];
      bmax[3 * node + a] = nmax[a];
    }
    const double parent_area =
        2.0 * oc_half_area(nmax[0] - nmin[0], nmax[1] - nmin[1], nmax[2] - nmin[2]);
    int make_leaf = c <= leaf_size || depth >= OC_MAX_TREE_DEPTH || parent_area <= 0.0;
    int64_t mid = -1;
    if (!make_leaf) {
      double cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int64_t k = f; k < f + c; ++k) {
        const int64_t ti = order[k];
        for (int a = 0; a < 3; ++a) {
          if (cent[3 * ti + a] < cmin[a]) cmin[a] = cent[3 * ti + a];
          if (cent[3 * ti + a] > cmax[a]) cmax[a] = cent[3 * ti + a];
        }
      }
      int axis = 0;
      double ext = cmax[0] - cmin[0];
      if (cmax[1] - cmin[1] > ext) { axis = 1; ext = cmax[1] - cmin[1]; }
      if (cmax[2] - cmin[2] > ext) { axis = 2; ext = cmax[2] - cmin[2]; }
      const double cmin_axis = cmin[axis];
      if (ext > 0.0) {
        const double scale = n_bins / ext;
        for (int b = 0; b < n_bins; ++b) {
          bin_count[b] = 0;
          for (int a = 0; a < 3; ++a) {
            bin_min[3 * b + a] = INFINITY;
            bin_max[3 * b + a] = -INFINITY;
          }
        }
        for (int64_t k = f; k < f + c; ++k) {
          const int64_t ti = order[k];
          int64_t b = (int64_t)((cent[3 * ti + axis] - cmin_axis) * scale);
          if (b >= n_bins) b = n_bins - 1;
          bin_count[b] += 1;
          for (int a = 0; a < 3; ++a) {
            if (tb_min[3 * ti + a] < bin_min[3 * b + a]) bin_min[3 * b + a] = tb_min[3 * ti + a];
            if (tb_max[3 * ti + a] > bin_max[3 * b + a]) bin_max[3 * b + a] = tb_max[3 * ti + a];
          }
        }
        double a0[3] = {INFINITY, INFINITY, INFINITY}, a1[3] = {-INFINITY, -INFINITY, -INFINITY};
        int64_t acc_n = 0;
        for (int b = 0; b < n_bins - 1; ++b) {
          if (bin_count[b] > 0) {
            for (int a = 0; a < 3; ++a) {
              if (bin_min[3 * b + a] < a0[a]) a0[a] = bin_min[3 * b + a];
              if (bin_max[3 * b + a] > a1[a]) a1[a] = bin_max[3 * b + a];
            }
            acc_n += bin_count[b];
          }
          sweep_count[b] = acc_n;
          sweep_area[b] = acc_n > 0 ? 2.0 * oc_half_area(a1[0] - a0[0], a1[1] - a0[1], a1[2] - a0[2])
                                    : 0.0;
        }
        double best_cost = INFINITY;
        int best_plane = -1;
        for (int a = 0; a < 3; ++a) {
          a0[a] = INFINITY;
          a1[a] = -INFINITY;
        }
        acc_n = 0;
        for (int b = n_bins - 1; b > 0; --b) {
          if (bin_count[b] > 0) {
            for (int a = 0; a < 3; ++a) {
              if (bin_min[3 * b + a] < a0[a]) a0[a] = bin_min[3 * b + a];
              if (bin_max[3 * b + a] > a1[a]) a1[a] = bin_max[3 * b + a];
            }
            acc_n += bin_count[b];
          }
          const int plane = b - 1;
          const int64_t ln = sweep_count[plane], rn = acc_n;
          if (ln > 0 && rn > 0) {
            const double right_area = 2.0 * oc_half_area(a1[0] - a0[0], a1[1] - a0[1], a1[2] - a0[2]);
            /* TRAVERSAL_COST + INTERSECT_COST * (...) / parent_area, both costs 1.0 */
            const double cost = 1.0 + 1.0 * (sweep_area[plane] * (double)ln + right_area * (double)rn) /
                                          parent_area;
            if (cost < best_cost) {
              best_cost = cost;
              best_plane = plane;
            }
          }
        }
        if (best_plane >= 0 && best_cost < 1.0 * (double)c) {
          int64_t i = f, j = f + c - 1;
          while (i <= j) {
            const int64_t ti = order[i];
            int64_t b = (int64_t)((cent[3 * ti + axis] - cmin_axis) * scale);
            if (b >= n_bins) b = n_bins - 1;
            if (b <= best_plane) {
              ++i;
            } else {
              const int32_t tmp = order[i];
              order[i] = order[j];
              order[j] = tmp;
              --j;
            }
          }
          mid = i;
          if (mid <= f || mid >= f + c) mid = f + c / 2;
        } else {
          make_leaf = 1;
        }
      } else {
        mid = f + c / 2;
      }
    }
    if (make_leaf) {
      first[node] = (int32_t)f;
      count[node] = (int32_t)c;
      ++leaf_count;
      continue;
    }
    const int64_t lchild = n_nodes, rchild = n_nodes + 1;
    n_nodes += 2;
    left[node] = (int32_t)lchild;
    right[node] = (int32_t)rchild;
    stack[sp][0] = rchild; stack[sp][1] = mid; stack[sp][2] = f + c - mid; stack[sp][3] = depth + 1;
    ++sp;
    stack[sp][0] = lchild; stack[sp][1] = f; stack[sp][2] = mid - f; stack[sp][3] = depth + 1;
    ++sp;
  }
  if (leaf_count_out) *leaf_count_out = leaf_count;
  if (max_depth_out) *max_depth_out = max_depth;
done:
  free(tb_min); free(tb_max); free(cent); free(bin_count); free(bin_min); free(bin_max);
  free(sweep_area); free(sweep_count); free(stack);
  return n_nodes;
}

/* _hit_frame (geometry.py:210-241) for the query-kernel checks */
void oc_hit_frame_api(const double d[3], const double a[3], const double b[3], const double c[3],
                      const double n0[3], const double n1[3], const double n2[3], double u,
                      double v, double g[3], double sh[3], int *front) {
  oc_hit_frame(d, a, b, c, n0, n1, n2, u, v, g, sh, front);
}
