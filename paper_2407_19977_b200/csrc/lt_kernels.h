// lt_kernels.h -- kernel argument structs and launchers (host <-> device).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lt_device.cuh"

namespace lt {

#ifndef LT_TRACE_THREADS
#define LT_TRACE_THREADS 128
#endif
constexpr int kTraceThreads = LT_TRACE_THREADS;
#ifndef LT_SHADE_THREADS
#define LT_SHADE_THREADS 128
#endif
constexpr int kShadeThreads = LT_SHADE_THREADS;
#ifndef LT_SHORT_STACK
#define LT_SHORT_STACK 16
#endif
// resident CTAs per SM the register allocation must allow (occupancy)
#ifndef LT_TRACE_MIN_BLOCKS
#define LT_TRACE_MIN_BLOCKS 9
#endif
// inner-node visits per lane between two leaf phases of k_trace
#ifndef LT_NODE_STEPS
#define LT_NODE_STEPS 3
#endif
// queue entries per shade thread and block iteration: their continuation
// rays are appended as one octant-grouped range of LT_SHADE_ITEMS x 128
// (2: -3.8 % C4 step time, the next trace gains from the wider grouping;
// profiles/r02_shade_items2.jsonl)
#ifndef LT_SHADE_ITEMS
#define LT_SHADE_ITEMS 2
#endif
#ifndef LT_SHADE_MIN_BLOCKS
#define LT_SHADE_MIN_BLOCKS 8
#endif
constexpr int kShortStack = LT_SHORT_STACK;  // per-lane traversal stack entries in shared memory

// Per-path state, 32 B: S[2p] = (throughput.rgb, radiance.r), S[2p + 1] =
// (radiance.gb, PCG state low / high words).  The PCG increment of a
// rendered path is recomputed from its pixel (seed_stream's mix64), so it
// is stored only for explicit paths (trace_radiance): inc (NULL in renders).
struct PathArrays {
  float4 *S;
  uint64_t *inc;
};

struct RaygenArgs {
  double cam[14];
  int32_t width, height;
  uint64_t seed;
  int64_t sample_base;   // sample index of s_local = 0
  int64_t n_pix;         // pixels in this batch
  int64_t pix_offset;    // first local pixel of this batch
  const int32_t *pix_list;  // local -> global pixel (NULL: identity)
  int64_t n_paths;       // n_pix * samples in this batch
  float t_min;
  // optional per-batch tables (launch_rng_tables): the PCG increment of
  // batch pixel i and the seeding term mix64(seed ^ mix64(sample)) of
  // batch sample s -- the same values seed_stream derives per path
  const uint64_t *inc_tab;
  const uint64_t *init_tab;
};

struct ShadeArgs {
  int32_t depth, max_depth, rr_start;
  float t_min;
  int32_t primary;  // depth-0 launch of a render batch: rays from RaygenArgs
  int32_t octant_sort;  // append continuation rays grouped by direction octant
  // LT_FLAG_SORT_MATERIALS: queue entry i is shaded from slot perm[i] (slots
  // grouped by material class); nullptr = queue order
  const int32_t *perm;
  // LT_FLAG_COUNT: [warps, warps whose active lanes span > 1 material class,
  // sum over warps of the distinct classes] (shading divergence evidence)
  unsigned long long *warp_ctr;
  int64_t cap;  // path / queue capacity of the lane (checked build)
};

struct AccumArgs {
  int64_t n_pix, pix_offset, n_samples;
  const int32_t *pix_list;
};

const void *trace_kernel_ptr(bool count);
const void *shade_kernel_ptr();

void launch_flatten_nodes(const double *bmin, const double *bmax, const int32_t *left,
                          const int32_t *right, const int32_t *first, const int32_t *count,
                          const int32_t *perm, const int32_t *new_index, int64_t n_internal,
                          float4 *out, cudaStream_t st);
// leaf_end[first + count - 1] = 1 for every leaf node (flags pre-zeroed)
void launch_leaf_end(const int32_t *first, const int32_t *count, int64_t n_nodes,
                     uint8_t *leaf_end, cudaStream_t st);
void launch_flatten_wide(const double *bmin, const double *bmax, const int32_t *first,
                         const int32_t *count, const int32_t *children, const int32_t *wide_of,
                         int64_t n_wide, float4 *out, cudaStream_t st);
void launch_flatten_tris(const double *v0, const double *v1, const double *v2, const double *n0,
                         const double *n1, const double *n2, const int32_t *mat_index,
                         const int32_t *order, const uint8_t *leaf_end, int64_t n, float4 *tris,
                         float4 *shade, cudaStream_t st);
// fill ra.inc_tab[0 .. n_pix) and ra.init_tab[0 .. n_samples) for a batch
void launch_rng_tables(const RaygenArgs &ra, int64_t n_samples, uint64_t *inc_tab,
                       uint64_t *init_tab, cudaStream_t st);
void launch_raygen(const RaygenArgs &ra, const PathArrays &pa, float4 *q_o, float4 *q_d,
                   int32_t *count0, cudaStream_t st);
void launch_raygen_explicit(const double *o, const double *d, const uint64_t *state,
                            const uint64_t *inc, int64_t n, float t_min, const PathArrays &pa,
                            float4 *q_o, float4 *q_d, int32_t *count0, cudaStream_t st);
void launch_gather_explicit(const PathArrays &pa, int64_t n, double *rgb, uint64_t *state_out,
                            cudaStream_t st);
size_t trace_smem_bytes();
// q_o NULL: primary rays (origin cam_o.xyz, path id = queue slot)
cudaError_t launch_trace(const SceneView &sc, bool count_work, int grid,
                         const cudaAccessPolicyWindow *window, const float4 *q_o,
                         const float4 *q_d, const int32_t *count, int32_t *fetch, float4 *hits,
                         unsigned long long *ray_ctr, float4 cam_o, cudaStream_t st);
void launch_trace_rays(const SceneView &sc, const float4 *q_o, const float4 *q_d, int64_t n,
                       float4 *hits, int32_t *nodes, int32_t *tests, cudaStream_t st);
// `ra`: the batch's RaygenArgs (render paths: pixel of a path id, the
// depth-0 launch regenerates the primary state) or NULL for explicit paths;
// `primary`: the depth-0 launch of a render batch.
cudaError_t launch_shade(const SceneView &sc, const ShadeArgs &sa, const PathArrays &pa, int grid,
                         const cudaAccessPolicyWindow *window, const RaygenArgs *ra, bool primary,
                         const float4 *q_o, const float4 *q_d, const float4 *hits,
                         const int32_t *count_in, float4 *n_o, float4 *n_d, int32_t *count_out,
                         cudaStream_t st);
// tile-ordered local pixel list: tiles k = rank, rank + n_ranks, ... of the
// T x T tiling (row-major tiles, row-major pixels inside a tile)
void launch_pixel_list(int32_t width, int32_t height, int32_t tile, int32_t rank, int32_t n_ranks,
                       const int32_t *tile_start, int32_t *out, cudaStream_t st);
// rgb float3 texels -> float4 records (environment map upload)
void launch_expand_rgb(const float *rgb, int64_t n, float4 *out, cudaStream_t st);
// device layout of a GPU-built BVH (see lt_kernels.cu "device layout")
void launch_internal_flags(const int32_t *count, int64_t nn, int32_t *flags, cudaStream_t st);
void launch_internal_scatter(const int32_t *flags, const int32_t *scan, int64_t nn,
                             int32_t *perm, int32_t *new_index, cudaStream_t st);
// the whole breadth-first collapse in one single-CTA launch; *n_wide (device)
// receives the wide-node count
void launch_collapse_all(const double *bmin, const double *bmax, const int32_t *left,
                         const int32_t *right, const int32_t *count, int32_t *fifo,
                         int32_t *wide_children, int32_t *wide_of, int32_t *n_wide,
                         cudaStream_t st);
// a whole render batch in one launch (small passes): path records for
// launch_accumulate, closest-hit count into ray_ctr[0]
void launch_path_small(const SceneView &sc, const RaygenArgs &ra, int32_t max_depth,
                       int32_t rr_start, const PathArrays &pa, unsigned long long *ray_ctr,
                       cudaStream_t st);
void launch_accumulate(const AccumArgs &aa, const float4 *S, float *accum, uint32_t *valid,
                       uint32_t *invalid, cudaStream_t st);
void launch_pack_rays_f32(const float *o, const float *d, int64_t n, float t_min, float t_max,
                          float4 *q_o, float4 *q_d, cudaStream_t st);
void launch_pack_rays_f64(const double *o, const double *d, int64_t n, float t_min, float t_max,
                          float4 *q_o, float4 *q_d, cudaStream_t st);
void launch_unpack_hits(const SceneView &sc, const float4 *hits, int64_t n, int32_t *idx32,
                        float *t32, int64_t *idx64, double *t64, double *uv64, cudaStream_t st);
void launch_tonemap_u8(const float *lin, int64_t n_pixels, uint8_t *out, cudaStream_t st);
// material-class grouping of a hit queue (LT_FLAG_SORT_MATERIALS): per
// entry class (miss, final segment, diffuse-only, reference GGX, coat,
// glass, coat + glass), then perm = the queue slots grouped by class.
// cls_ctr: 16 zeroed ints (class totals, class cursors).
constexpr int kShadeClasses = 8;
void launch_material_sort(const SceneView &sc, const float4 *hits, const int32_t *count,
                          bool scatter, int grid, uint8_t *cls, int32_t *cls_ctr, int32_t *perm,
                          cudaStream_t st);
void launch_accum_finish(const float *sum, const uint32_t *valid, const uint32_t *invalid,
                         int64_t n_pix, double *mean, int64_t *inv, cudaStream_t st);
void launch_bsdf_eval(const GpuMaterial *mats, const double *wo, const double *wi,
                      const double *nrm, const int32_t *front, int64_t n, double *f, double *pdf,
                      cudaStream_t st);
void launch_bsdf_sample(const GpuMaterial *mats, const double *wo, const double *nrm,
                        const double *u, const int32_t *front, int64_t n, int32_t *ok, double *wi,
                        double *wgt, cudaStream_t st);
void launch_occluded(const SceneView &sc, const float4 *q_o, const float4 *q_d, int64_t n,
                     int32_t *out, cudaStream_t st);
void launch_read_probe(const float4 *src, int64_t n4, int passes, float *sink, int grid,
                       cudaStream_t st);
// exhaustive closest hit over the leaf-ordered triangles (the traversal's
// fp32 Moller-Trumbore and tie rule, no BVH): hits as k_trace_rays writes them
void launch_brute_force(const SceneView &sc, int64_t n_tris, const float4 *q_o,
                        const float4 *q_d, int64_t n, float4 *hits, cudaStream_t st);

// ---- float64 query kernels (lt_query64.cu, the reference's arithmetic)
void launch_ray_triangle64(const double *o, const double *d, const double *tmin,
                           const double *tmax, const double *v0, const double *v1,
                           const double *v2, const double *n0, const double *n1,
                           const double *n2, int64_t n, int32_t *ok, double *tuv, double *g,
                           double *s, int32_t *front, cudaStream_t st);
void launch_hit_frame64(const double *d, const double *v0, const double *v1, const double *v2,
                        const double *n0, const double *n1, const double *n2, const double *uv,
                        int64_t n, double *g, double *s, int32_t *front, cudaStream_t st);
void launch_ray_aabb64(const double *o, const double *d, const double *tmin, const double *tmax,
                       const double *lo, const double *hi, int64_t n, int32_t *ok, double *tnf,
                       cudaStream_t st);
void launch_bsdf64(int mode, const double *params, const double *wo, const double *wi,
                   const double *nrm, const double *u, int64_t n, int32_t *ok, double *out3a,
                   double *out3b, double *out1, int32_t *flag, cudaStream_t st);
void launch_microfacet64(int op, const double *a, const double *b, const double *c,
                         const double *nrm, int64_t n, double *out, cudaStream_t st);
void launch_display64(int op, const double *in, int64_t n, double *out, uint8_t *out8,
                      cudaStream_t st);

}  // namespace lt
