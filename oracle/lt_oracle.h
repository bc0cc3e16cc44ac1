/*
 * lt_oracle.h -- CPU fp64 restatement of the luxtrace reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker and the CPU
 * baseline.  Only tests/, __graft_entry__.smoke() and bench.py (its
 * cpu_baseline leg and `--impl reference`) may load it.  The product path
 * (paper_2407_19977_b200) never links or calls it.
 *
 * Every function follows a reference function file:line under
 * /root/reference/pkg/src/luxtrace/ (cited in lt_oracle.c).  The pinned part
 * (base / dielectric specular / metal / emission, uniform + gradient
 * environments) is checked against golden vectors produced by the reference
 * itself (tests/golden/make_golden.py).  The extension lobes (coat,
 * transmission) and the HDR environment have no reference implementation:
 * PARITY UNPINNED for those; they default to zero weight so reference
 * materials reduce to the reference arithmetic exactly.
 */
#ifndef LT_ORACLE_H
#define LT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  /* BVH exactly as luxtrace.bvh.Bvh (bvh.py:38-50) */
  int64_t n_nodes;
  const double *bmin, *bmax;           /* (n_nodes,3) */
  const int32_t *left, *right, *first, *count;
  const int32_t *order;                /* (n_tris,) */
  /* triangles exactly as luxtrace.geometry.TriangleBuffer (geometry.py:88-131) */
  int64_t n_tris;
  const double *v0, *v1, *v2, *n0, *n1, *n2;   /* (n_tris,3) */
  const int32_t *mat_index;
  /* materials as luxtrace.material.pack_materials (material.py:68-92) */
  int32_t n_mats;
  const double *bw, *bc, *metal, *sw, *sc, *rough, *ior, *el, *ec; /* bc/sc/ec are (k,3) */
  /* extensions, may be NULL (= zero weight): PARITY UNPINNED */
  const double *coat_w, *coat_rough, *coat_ior, *coat_color; /* coat_color (k,3) */
  const double *tr_w, *tr_color;                             /* tr_color (k,3) */
  /* environment (integrator.py:118-136); kind 2 = HDR lat-long map (extension) */
  int32_t env_kind;
  double env_a[3], env_b[3];
  int32_t env_w, env_h;
  const float *env_map;                /* (env_h, env_w, 3) */
  double env_scale;
} oc_scene;

/* ---- rng.py ---- */
uint32_t oc_pcg_next(uint64_t *state, uint64_t inc);
void oc_pcg_seed(uint64_t init_state, uint64_t init_seq, uint64_t *state, uint64_t *inc);
uint64_t oc_mix64(uint64_t x);
void oc_seed_stream(uint64_t pixel, uint64_t sample, uint64_t seed, uint64_t *state, uint64_t *inc);

/* ---- geometry.py / bvh.py ---- */
int oc_mt_intersect(const double o[3], const double d[3], const double a[3],
                    const double b[3], const double c[3], double t_min, double t_max,
                    double *t, double *u, double *v);
int oc_slab_intersect(const double o[3], const double inv[3], const double bmin[3],
                      const double bmax[3], double t_min, double t_max,
                      double *t_enter, double *t_exit);
void oc_hit_frame_api(const double d[3], const double a[3], const double b[3], const double c[3],
                      const double n0[3], const double n1[3], const double n2[3], double u,
                      double v, double g[3], double sh[3], int *front);
int64_t oc_traverse(const oc_scene *s, const double o[3], const double d[3],
                    double t_min, double t_max, double *t, double *u, double *v,
                    int64_t *nodes_visited, int64_t *tri_tests);
void oc_intersect_batch(const oc_scene *s, const double *origins, const double *dirs,
                        int64_t n, double t_min, double t_max, int64_t *idx, double *t,
                        int n_threads);
void oc_traversal_counts_batch(const oc_scene *s, const double *origins, const double *dirs,
                               int64_t n, double t_min, double t_max, int64_t *nodes,
                               int64_t *tests, int n_threads);
void oc_brute_force_batch(const oc_scene *s, const double *origins, const double *dirs,
                          int64_t n, double t_min, double t_max, int64_t *idx, double *t,
                          int n_threads);

/* ---- bvh.py build: _triangle_bounds_arrays + _build_kernel (bvh.py:57-262);
 * node arrays sized 2n (bounds 2n*3), order n; returns the node count ---- */
int64_t oc_build_bvh(const double *v0, const double *v1, const double *v2, int64_t n,
                     int32_t leaf_size, int32_t n_bins, double *bmin, double *bmax,
                     int32_t *left, int32_t *right, int32_t *first, int32_t *count,
                     int32_t *order, int64_t *leaf_count, int64_t *max_depth);

/* ---- material.py ---- */
/* params: [bw, bcr, bcg, bcb, m, sw, scr, scg, scb, rough, ior,
 *          coat_w, coat_rough, coat_ior, ccr, ccg, ccb, tr_w, tcr, tcg, tcb] (21) */
void oc_eval_bsdf(const double wo[3], const double wi[3], const double n[3],
                  const double *params, double f[3]);
double oc_pdf_bsdf(const double wo[3], const double wi[3], const double n[3],
                   const double *params);
int oc_sample_bsdf(const double wo[3], const double n[3], const double *params,
                   double u_lobe, double u1, double u2, int front,
                   double wi[3], double weight[3], double *pdf, int *spike);

/* ---- integrator.py ---- */
void oc_camera_dir(const double cam[14], double px, double py, double jx, double jy,
                   int32_t width, int32_t height, double d[3]);
void oc_env_radiance(const oc_scene *s, const double d[3], double out[3]);
/* one path; returns segments traced (closest-hit queries) */
int oc_trace(const oc_scene *s, const double o[3], const double d[3], uint64_t *state,
             uint64_t inc, int32_t max_depth, int32_t rr_start, double t_min,
             double rgb[3]);
/* _render_pass (integrator.py:230-277): running mean in f64, counts in i64 */
void oc_render_pass(const oc_scene *s, double *accum, int64_t *valid, int64_t *invalid,
                    int64_t sample_start, int64_t sample_count, const double cam[14],
                    int32_t width, int32_t height, uint64_t seed, int32_t max_depth,
                    int32_t rr_start, double t_min, int n_threads, int64_t *segments);
/* the radiance of sample `sample` for each listed pixel (no accumulation);
 * rgb (n,3), segments (n,) -- the matched-stream per-sample oracle */
void oc_sample_values(const oc_scene *s, const int64_t *pixels, int64_t n, int64_t sample,
                      const double cam[14], int32_t width, int32_t height, uint64_t seed,
                      int32_t max_depth, int32_t rr_start, double t_min, double *rgb,
                      int32_t *segments, int n_threads);
/* primary rays for (pixel, sample) exactly as _render_pass builds them */
void oc_primary_rays(const int64_t *pixels, int64_t n, int64_t sample, const double cam[14],
                     int32_t width, int32_t height, uint64_t seed, double *origins,
                     double *dirs);

#ifdef __cplusplus
}
#endif
#endif
