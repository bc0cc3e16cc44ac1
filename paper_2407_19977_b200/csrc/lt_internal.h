// lt_internal.h -- shared host-side declarations of the luxb200 library.
#pragma once
#include <cstdint>

#include "luxb200.h"

// Sets the thread-local last error and returns `code`.
int lt_fail(int code, const char *fmt, ...);

int lt_build_bvh_impl(const double *v0, const double *v1, const double *v2, int64_t n,
                      int32_t leaf_size, int32_t n_bins, double *bmin, double *bmax,
                      int32_t *left, int32_t *right, int32_t *first, int32_t *count,
                      int32_t *order, int64_t *n_nodes_out, int64_t *leaf_count_out,
                      int64_t *max_depth_out);

// A BVH built on the device (lt_bvh_gpu.cu): the reference's tree with
// provisional node ids (root 0; children of node i are left[i] / right[i],
// -1 at leaves), bounds (n_nodes, 3) float64, leaf ranges into `order`.
// All pointers are device memory owned by `impl`.
struct lt_gpu_tree {
  double *bmin, *bmax;
  int32_t *left, *right, *first, *count, *order;
  int64_t n_nodes, n_leaves, max_depth;
  void *impl;
};
// dv0/dv1/dv2: device float64 (n,3) vertex arrays; stream: cudaStream_t.
int lt_gpu_tree_build(const double *dv0, const double *dv1, const double *dv2, int64_t n,
                      int32_t leaf_size, int32_t bins, void *stream, lt_gpu_tree *out);
void lt_gpu_tree_free(lt_gpu_tree *t);

// glTF ingest on the device (lt_ingest.cu): flatten_scene's triangle soup in
// one stream-ordered allocation `mem` (v[0..5] (n_kept,3) float64, mat).
struct lt_ingest_out {
  double *v[6];
  int32_t *mat;
  int64_t n_total, n_kept, n_dropped;
  void *mem;
};
// Structural checks of a description (ranges inside their buffers, ids,
// counts); n_materials <= 0 skips the material-slot check.  *n_out_tris =
// the instances' total triangle count.
int lt_ingest_check(const lt_gltf_desc *g, int32_t n_materials, int64_t *n_out_tris);
// d_raw: the glTF buffers on the device, buffer b at d_raw + buf_at[b].
int lt_ingest_run(const lt_gltf_desc *g, const uint8_t *d_raw, const int64_t *buf_at,
                  void *stream, lt_ingest_out *out);
void lt_ingest_free(lt_ingest_out *o, void *stream);
