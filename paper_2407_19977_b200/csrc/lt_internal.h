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
