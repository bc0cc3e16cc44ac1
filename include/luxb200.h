/*
 * luxb200.h -- C-ABI of the B200-native path tracer (the drop-in boundary).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (`void *stream` is a cudaStream_t, NULL = the legacy default stream).
 * Every entry point returns an int status (LT_OK = 0) and leaves a
 * thread-local message for lt_last_error().  Non-finite path samples are
 * counted, never raised (integrator.py:266-272).
 *
 * Each entry point names the reference interface it replaces, as file:line
 * under /root/reference/pkg/src/luxtrace/.  The Python mirror
 * (paper_2407_19977_b200/) binds these with ctypes; INTEGRATION.md shows the
 * binding a luxtrace maintainer would add on the reference side.
 */
#ifndef LUXB200_H
#define LUXB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LT_ABI_VERSION 2

/* status codes */
#define LT_OK 0
#define LT_ERR_INVALID 1   /* bad argument: the Python mirror raises ValueError */
#define LT_ERR_CUDA 2      /* CUDA runtime failure: RuntimeError */
#define LT_ERR_NOMEM 3     /* allocation failure: MemoryError */
#define LT_ERR_UNSUPPORTED 4

/* environment kinds: _ENV_UNIFORM / _ENV_GRADIENT (integrator.py:37-38);
 * LT_ENV_LATLONG is the synthetic-HDR extension (no reference, parity unpinned) */
#define LT_ENV_UNIFORM 0
#define LT_ENV_GRADIENT 1
#define LT_ENV_LATLONG 2

/* lt_render_params.flags */
#define LT_FLAG_SORT_MATERIALS 1u   /* shade every bounce in material-class order: a
                                       classify + counting-sort pass groups the hit queue
                                       by class (miss, final segment, diffuse-only, GGX,
                                       coat, glass, coat + glass) and the shade kernel
                                       reads it through that permutation; results are
                                       unchanged (off by default) */
#define LT_FLAG_PROFILE 4u          /* time every trace launch with CUDA events */
#define LT_FLAG_COUNT 8u            /* count slab / triangle tests in the trace kernel */

typedef struct lt_scene lt_scene;

/* Scene description: the arrays `_scene_arrays` packs for `_render_pass`
 * (integrator.py:284-291), all host pointers, row-major, reference dtypes. */
typedef struct lt_scene_desc {
  /* TriangleBuffer (geometry.py:88-131): (n,3) float64 each, (n,) int32 */
  int64_t n_triangles;
  const double *v0, *v1, *v2, *n0, *n1, *n2;
  const int32_t *material_index;
  /* Bvh (bvh.py:38-50), the host-built tree, consumed unchanged.  n_nodes
   * = 0 with all seven BVH pointers NULL: the scene builds the reference's
   * tree itself on the device (build_bvh defaults: leaf size 4, 12 bins),
   * without a host round trip (render_progressive(scene, settings) with no
   * BVH, integrator.py:321-326). */
  int64_t n_nodes;
  const double *bounds_min, *bounds_max;            /* (n_nodes,3) */
  const int32_t *left_child, *right_child;          /* (n_nodes,) -1 at leaves */
  const int32_t *first_triangle, *triangle_count;   /* (n_nodes,) leaf iff count > 0 */
  const int32_t *triangle_order;                    /* (n,) */
  /* pack_materials (material.py:68-92): (k,) or (k,3) float64 */
  int32_t n_materials;
  const double *base_weight, *base_color, *base_metalness, *specular_weight;
  const double *specular_color, *specular_roughness, *specular_ior;
  const double *emission_luminance, *emission_color;
  /* extension lobes (no reference; NULL = zero weight = reference material) */
  const double *coat_weight, *coat_roughness, *coat_ior, *coat_color;
  const double *transmission_weight, *transmission_color;
  /* _environment_pack (integrator.py:118-121) */
  int32_t env_kind;
  double env_a[3], env_b[3];
  /* LT_ENV_LATLONG: (env_height, env_width, 3) float32 radiance, times env_scale */
  int32_t env_width, env_height;
  const float *env_texels;
  double env_scale;
} lt_scene_desc;

typedef struct lt_scene_info {
  int32_t device;
  int64_t n_triangles, n_nodes, n_internal;
  int64_t device_bytes;         /* resident scene bytes in HBM */
  int32_t sm_count;
  int64_t n_wide;               /* 4-wide nodes of the render layout */
  int64_t l2_persist_bytes;     /* persisting-L2 limit set for the scene (0: none) */
  int64_t l2_window_bytes;      /* access-policy window of the trace launches */
  int64_t default_batch_paths;  /* paths per wavefront batch when not overridden */
} lt_scene_info;

/* One render pass: `_render_pass(..., sample_start, sample_count, cam, width,
 * height, ..., seed, max_depth, rr_start, t_min)` (integrator.py:230-237). */
typedef struct lt_render_params {
  double camera[14];            /* _camera_pack (integrator.py:75-83) */
  int32_t width, height;
  int64_t sample_start, sample_count;
  uint64_t seed;
  int32_t max_depth, rr_start;
  double t_min;
  /* image sharding: square tiles of tile_size, tile k (raster order) is
   * rendered by rank k % n_ranks.  n_ranks <= 1 renders every pixel.
   * RNG streams stay keyed by the GLOBAL pixel index, so any sharding yields
   * the same per-pixel values as one GPU. */
  int32_t tile_size, rank, n_ranks;
  uint32_t flags;
  int64_t max_batch_paths;      /* 0 = library default */
} lt_render_params;

typedef struct lt_render_stats {
  int64_t paths;                /* (pixel, sample) paths traced */
  int64_t rays;                 /* closest-hit queries (primary + continuation) */
  int64_t batches;
  int64_t kernel_launches;
  int64_t trace_launches;       /* trace kernel launches in the pass */
  int64_t slab_tests;           /* child-box tests incl. root (LT_FLAG_COUNT only) */
  int64_t tri_tests;            /* triangle tests (LT_FLAG_COUNT only) */
  double trace_ms;              /* sum of CUDA-event times of the trace launches
                                   (LT_FLAG_PROFILE only, else 0) */
  /* LT_FLAG_COUNT only: shade warps, warps whose active lanes span more than
   * one material class (miss / last segment / diffuse-only / full BSDF /
   * coat / glass), and the sum of distinct classes per warp */
  int64_t shade_warps, shade_mixed_warps, shade_warp_classes;
} lt_render_stats;

/* ---- library ---- */
int lt_abi_version(void);
const char *lt_last_error(void);
int lt_device_count(int32_t *count);

/* ---- host BVH build: build_bvh (bvh.py:286-298), same binned SAH
 * (bvh.py:85-262), bit-identical arrays.  Output buffers are caller-owned:
 * node arrays sized 2n (bounds 2n*3), order sized n. ---- */
int lt_build_bvh(const double *v0, const double *v1, const double *v2, int64_t n,
                 int32_t leaf_size, int32_t bins, double *bounds_min, double *bounds_max,
                 int32_t *left_child, int32_t *right_child, int32_t *first_triangle,
                 int32_t *triangle_count, int32_t *triangle_order, int64_t *n_nodes,
                 int64_t *leaf_count, int64_t *max_depth);

/* ---- GPU BVH build: build_bvh (bvh.py:286-298) on `device`; the same
 * arrays as lt_build_bvh / the reference (split decisions, bounds, the
 * two-pointer partition order and the node numbering reproduced; see
 * csrc/lt_bvh_gpu.cu).  Host buffers as lt_build_bvh; bins <= 32. ---- */
int lt_build_bvh_device(int32_t device, const double *v0, const double *v1, const double *v2,
                        int64_t n, int32_t leaf_size, int32_t bins, double *bounds_min,
                        double *bounds_max, int32_t *left_child, int32_t *right_child,
                        int32_t *first_triangle, int32_t *triangle_count,
                        int32_t *triangle_order, int64_t *n_nodes, int64_t *leaf_count,
                        int64_t *max_depth);

/* ---- scene residency: replaces the per-call `_scene_arrays` packing
 * (integrator.py:284-291); flattens the host BVH into the HBM layout ---- */
int lt_scene_create(const lt_scene_desc *desc, int32_t device, lt_scene **out);

/* ---- glTF ingest on the device: flatten_scene (scene.py:519-596) fed from
 * the GLB's own float32 / integer accessors, uploaded as raw bytes (the GLB
 * stores float32, procgen.py:123) instead of the host's float64 world-space
 * soup.  The host keeps the cheap part -- JSON, accessor validation, the node
 * walk and its 4x4 products, material resolution (scene.py:251-490) -- and
 * hands over one record per primitive and one per (node, primitive)
 * instance in flatten_scene's visit order.  The device decodes the
 * accessors, generates smooth normals where NORMAL is absent
 * (scene.py:493-508: the per-vertex sums in np.add.at's order), applies the
 * transforms with the rounding numpy's BLAS product uses (one fused
 * multiply-add chain per output, k = 0, 1, 2), computes the extent, drops
 * degenerate triangles and normalises the normals -- the reference's
 * float64 arithmetic step for step, so the arrays are bit-identical to
 * load_scene's. ---- */
typedef struct lt_gltf_primitive {
  /* POSITION: float32 VEC3 at buffers[pos_buffer] + pos_offset, pos_stride bytes apart */
  int32_t pos_buffer, pos_stride;
  int64_t pos_offset, n_vertices;
  /* NORMAL: float32 VEC3; nrm_buffer = -1: none (smooth normals are generated) */
  int32_t nrm_buffer, nrm_stride;
  int64_t nrm_offset;
  /* indices: idx_bytes = 1 / 2 / 4 (u8 / u16 / u32); idx_buffer = -1: 0..n_indices-1 */
  int32_t idx_buffer, idx_stride, idx_bytes, reserved;
  int64_t idx_offset, n_indices;  /* n_indices % 3 == 0, every index < n_vertices */
} lt_gltf_primitive;

typedef struct lt_gltf_instance {
  int32_t primitive, material;    /* material: slot in the scene's material table */
  double linear[9];               /* world[:3, :3], row-major */
  double translation[3];          /* world[:3, 3] */
  double normal_matrix[9];        /* np.linalg.inv(linear).T, row-major */
} lt_gltf_instance;

typedef struct lt_gltf_desc {
  int32_t n_buffers;
  const uint8_t *const *buffers;  /* host bytes of each glTF buffer */
  const int64_t *buffer_bytes;
  int32_t n_primitives;
  const lt_gltf_primitive *primitives;
  int32_t n_instances;
  const lt_gltf_instance *instances;
} lt_gltf_desc;

/* flatten_scene on `device` with the arrays copied back: v0..n2 (cap,3)
 * float64 and material_index (cap,), cap >= the instances' total triangle
 * count; *n_kept / *n_dropped as SceneDescription.degenerate_dropped.  An
 * all-degenerate scene returns LT_ERR_INVALID "empty scene". */
int lt_gltf_flatten(const lt_gltf_desc *gltf, int32_t device, int64_t cap, double *v0,
                    double *v1, double *v2, double *n0, double *n1, double *n2,
                    int32_t *material_index, int64_t *n_kept, int64_t *n_dropped);
/* the same flatten feeding lt_scene_create without leaving the device: the
 * triangle arrays never exist on the host, the BVH is built on the device.
 * `scene` supplies the materials and environment; its triangle and BVH
 * fields must be 0 / NULL. */
int lt_scene_create_gltf(const lt_gltf_desc *gltf, const lt_scene_desc *scene, int32_t device,
                         lt_scene **out, int64_t *n_kept, int64_t *n_dropped);
int lt_scene_destroy(lt_scene *scene);
int lt_scene_info_get(const lt_scene *scene, lt_scene_info *info);

/* ---- closest hit: intersect_scene_batch (bvh.py:667-677) / _traverse_batch
 * (bvh.py:554-567).  Device pointers: origins/dirs (n,3) float32; outputs
 * idx (n,) int32 (-1 on miss), t (n,) float32 (+inf on miss). ---- */
int lt_intersect_batch(lt_scene *scene, const float *origins, const float *dirs, int64_t n,
                       float t_min, float t_max, int32_t *idx, float *t, void *stream);
/* Host-buffer twin with the reference dtypes: float64 rays, int64 idx,
 * float64 t (the fp32 result widened). */
int lt_intersect_batch_host(lt_scene *scene, const double *origins, const double *dirs,
                            int64_t n, double t_min, double t_max, int64_t *idx, double *t);
/* The same with the barycentrics of each hit: uv (n,2) float64 (0 on a miss);
 * the scalar intersect_scene (bvh.py:632-641) builds its Hit from them. */
int lt_intersect_hits_host(lt_scene *scene, const double *origins, const double *dirs,
                           int64_t n, double t_min, double t_max, int64_t *idx, double *t,
                           double *uv);
/* Exhaustive closest hit: brute_force_intersect_batch (bvh.py:694-701,
 * _brute_force_batch bvh.py:586-610), every triangle against every ray with
 * the traversal's fp32 arithmetic and tie rule, so it equals
 * lt_intersect_batch_host exactly (test_bvh.py:91-100). */
int lt_brute_force_batch_host(lt_scene *scene, const double *origins, const double *dirs,
                              int64_t n, double t_min, double t_max, int64_t *idx, double *t);
/* Work counters: traversal_counts_batch (bvh.py:680-691), host buffers.
 * nodes = child-box tests + 1 (root), tests = triangle tests. */
int lt_traversal_counts_host(lt_scene *scene, const double *origins, const double *dirs,
                             int64_t n, double t_min, double t_max, int64_t *nodes,
                             int64_t *tests);

/* ---- the operator: _render_pass (integrator.py:230-277).
 * Device pointers: accum_sum (h*w*3) float32 per-pixel SUM of finite
 * samples, valid/invalid (h*w) uint32 counts; all updated in place.
 * Samples of a pixel are added in sample-index order. ---- */
int lt_render_pass(lt_scene *scene, const lt_render_params *params, float *accum_sum,
                   uint32_t *valid, uint32_t *invalid, void *stream);
/* Host-buffer drop-in with the reference's exact in/out contract:
 * accum (h,w,3) float64 running MEAN, valid/invalid (h,w) int64, updated in
 * place with samples [sample_start, sample_start + sample_count). */
int lt_render_pass_host(lt_scene *scene, const lt_render_params *params, double *accum_mean,
                        int64_t *valid, int64_t *invalid);
int lt_render_stats_get(const lt_scene *scene, lt_render_stats *stats);

/* ---- single paths with caller-supplied PCG state: trace_radiance
 * (integrator.py:294-307) batched.  Host buffers: origins/dirs (n,3) f64,
 * state/inc (n,) u64 in, rgb (n,3) f64 out, state_out (n,) u64. ---- */
int lt_trace_paths_host(lt_scene *scene, const double *origins, const double *dirs,
                        const uint64_t *state, const uint64_t *inc, int64_t n,
                        int32_t max_depth, int32_t rr_start, double t_min, double *rgb,
                        uint64_t *state_out);

/* ---- result of a device accumulation (lt_render_pass buffers) as the
 * reference's RenderResult arrays (integrator.py:62-68): per pixel
 * mean = sum / max(valid, 1) in float64 (h*w*3) and invalid as int64, on
 * the device, one launch on `stream` ---- */
int lt_accum_finish(const float *accum_sum, const uint32_t *valid, const uint32_t *invalid,
                    int64_t n_pixels, double *mean, int64_t *invalid_out, void *stream);

/* ---- display transform (tonemap.py:18-61, the §8(f) next row): linear
 * (h*w*3) float32 device -> sRGB u8 (h*w*3) device ---- */
int lt_tonemap_u8(const float *linear, int64_t n_pixels, uint8_t *out, void *stream);

/* ---- BSDF kernels on caller inputs (material.py:389-426: eval_bsdf,
 * pdf_bsdf, sample_bsdf), the device code the shade kernel runs, in fp32.
 * Host buffers; params (n,21) float64 per case:
 *   [bw, bc.rgb, metalness, sw, sc.rgb, roughness, ior,
 *    coat_w, coat_rough, coat_ior, coat_color.rgb, transmission_w, transmission_color.rgb]
 * wo, wi, normal (n,3) unit float64; u (n,3) the three lobe / direction
 * draws; front (n,) geometric-side flag (transmission only). ---- */
int lt_bsdf_eval_batch(const double *params, const double *wo, const double *wi,
                       const double *normal, int64_t n, double *f, double *pdf);
/* The same with the effective BSDF of the extension estimator for coat /
 * transmission materials (the value and density sample_bsdf realizes; see
 * csrc/lt_material.cuh eval_material): front (n,) geometric side (NULL =
 * outside), for the dielectric interface's eta.  lt_bsdf_eval_batch = this
 * with front NULL.  Extension: no reference (parity unpinned). */
int lt_bsdf_eval_ext_batch(const double *params, const double *wo, const double *wi,
                           const double *normal, const int32_t *front, int64_t n, double *f,
                           double *pdf);
int lt_bsdf_sample_batch(const double *params, const double *wo, const double *normal,
                         const double *u, const int32_t *front, int64_t n, int32_t *ok,
                         double *wi, double *weight);

/* ---- any-hit occlusion: intersect_any (bvh.py:658-664) / _traverse_any
 * (bvh.py:511-551), host buffers; occluded (n,) 1 if any triangle is hit
 * within [t_min, t_max]. ---- */
int lt_occluded_batch_host(lt_scene *scene, const double *origins, const double *dirs,
                           int64_t n, double t_min, double t_max, int32_t *occluded);

/* ---- the reference's scalar query API in float64 on the device
 * (csrc/lt_query64.cu, the reference's operation order, no FMA contraction).
 * Host buffers; (n,3) arrays row-major. ---- */
/* ray_triangle_intersect (geometry.py:255-278): per case a ray (origin,
 * dir, t_min, t_max) and a triangle (v0..v2, n0..n2); ok, tuv (n,3) =
 * (t, u, v), the hit frame of _hit_frame (geometry.py:210-241). */
int lt_ray_triangle_batch(const double *origins, const double *dirs, const double *t_min,
                          const double *t_max, const double *v0, const double *v1,
                          const double *v2, const double *n0, const double *n1, const double *n2,
                          int64_t n, int32_t *ok, double *tuv, double *geo_normal,
                          double *shading_normal, int32_t *front);
/* _hit_frame (geometry.py:210-241) at given barycentrics uv (n,2). */
int lt_hit_frame_batch(const double *dirs, const double *v0, const double *v1, const double *v2,
                       const double *n0, const double *n1, const double *n2, const double *uv,
                       int64_t n, double *geo_normal, double *shading_normal, int32_t *front);
/* ray_aabb_intersect (geometry.py:281-295): _inv_component + the
 * compare/select _slab_intersect; t_enter_exit (n,2). */
int lt_ray_aabb_batch(const double *origins, const double *dirs, const double *t_min,
                      const double *t_max, const double *box_min, const double *box_max,
                      int64_t n, int32_t *ok, double *t_enter_exit);
/* eval_bsdf / pdf_bsdf / sample_bsdf (material.py:389-426) on the reference
 * materials: params (n,11) = [bw, bc.rgb, m, sw, sc.rgb, roughness, ior]. */
int lt_bsdf64_eval_batch(const double *params, const double *wo, const double *wi,
                         const double *normal, int64_t n, double *f, double *pdf);
int lt_bsdf64_sample_batch(const double *params, const double *wo, const double *normal,
                           const double *u, int64_t n, int32_t *ok, double *wi, double *weight,
                           double *pdf, int32_t *spike);
/* microfacet helpers (material.py:107-126, 264-290, 371-386): op 0
 * ggx_ndf(a = n.h, b = alpha) -> out (n,); 1 smith_g2(a = n.o, b = n.i,
 * c = alpha); 2 cosine_sample_hemisphere(normal, a = u1, b = u2) -> out
 * (n,3); 3 ggx_sample_half_vector(normal, c = alpha, a = u1, b = u2). */
int lt_microfacet_batch(int32_t op, const double *a, const double *b, const double *c,
                        const double *normal, int64_t n, double *out);
/* display transform (tonemap.py:18-61): op 0 pbr_neutral_tonemap (n rgb
 * triples -> out (n,3)), 1 linear_to_srgb, 2 srgb_to_linear (n values ->
 * out), 3 quantize_to_u8 (n values -> out_u8). */
int lt_display_batch(int32_t op, const double *in, int64_t n, double *out, uint8_t *out_u8);

/* ---- measurement helper (not on the render path): streaming-read
 * bandwidth of a `bytes` device buffer, `iters` passes, CUDA events.  A
 * buffer smaller than L2 measures L2 bandwidth (the roofline denominator for
 * the L2-resident traversal set), a large one HBM. ---- */
int lt_read_bandwidth(int32_t device, int64_t bytes, int32_t iters, double *gbps);

#ifdef __cplusplus
}
#endif
#endif
