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
