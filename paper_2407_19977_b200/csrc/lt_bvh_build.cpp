// lt_bvh_build.cpp -- host binned-SAH BVH build, bit-identical to the
// reference `build_bvh` (bvh.py:286-298 -> _triangle_bounds_arrays
// bvh.py:57-77 -> _build_kernel bvh.py:85-262).
//
// The north star keeps the reference's host-built tree unchanged as the
// upload input; this restatement exists so the product can produce that same
// tree where the reference is not installed (the GPU box).  Compiled with
// -ffp-contract=off so every float64 operation rounds exactly as numba's.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#include "lt_internal.h"

namespace {

constexpr double kBoundsPadding = 1e-7;  // geometry.py:19
constexpr double kTraversalCost = 1.0;   // bvh.py:24
constexpr double kIntersectCost = 1.0;   // bvh.py:25
constexpr int kDepthCap = 60;            // bvh.py:26

inline double half_area(double dx, double dy, double dz) { return dx * dy + dx * dz + dy * dz; }

struct Box {
  double lo[3], hi[3];
  void reset() {
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::numeric_limits<double>::infinity();
      hi[a] = -std::numeric_limits<double>::infinity();
    }
  }
  void grow_min(const double *p) {
    for (int a = 0; a < 3; ++a)
      if (p[a] < lo[a]) lo[a] = p[a];
  }
  void grow_max(const double *p) {
    for (int a = 0; a < 3; ++a)
      if (p[a] > hi[a]) hi[a] = p[a];
  }
  double area2() const { return 2.0 * half_area(hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]); }
};

struct Job {
  int64_t node, first, count, depth;
};

}  // namespace

int lt_build_bvh_impl(const double *v0, const double *v1, const double *v2, int64_t n,
                      int32_t leaf_size, int32_t n_bins, double *bmin, double *bmax,
                      int32_t *left, int32_t *right, int32_t *first, int32_t *count,
                      int32_t *order, int64_t *n_nodes_out, int64_t *leaf_count_out,
                      int64_t *max_depth_out) {
  if (n <= 0) return lt_fail(LT_ERR_INVALID, "empty scene");
  if (leaf_size < 1 || n_bins < 2) return lt_fail(LT_ERR_INVALID, "leaf_size >= 1 and bins >= 2 required");

  // triangle bounds padded by 1e-7 * max extent, centroids of the padded box
  std::vector<double> tbmin(3 * n), tbmax(3 * n), cent(3 * n);
  for (int64_t i = 0; i < n; ++i) {
    double ext = 0.0;
    for (int a = 0; a < 3; ++a) {
      double x0 = v0[3 * i + a], x1 = v1[3 * i + a], x2 = v2[3 * i + a];
      // Python min/max keep the first argument unless the second is strictly
      // smaller/larger (matters only for the sign of zero)
      double m12 = x2 < x1 ? x2 : x1;
      double lo = m12 < x0 ? m12 : x0;
      double M12 = x2 > x1 ? x2 : x1;
      double hi = M12 > x0 ? M12 : x0;
      tbmin[3 * i + a] = lo;
      tbmax[3 * i + a] = hi;
      if (hi - lo > ext) ext = hi - lo;
    }
    double pad = kBoundsPadding * ext;
    for (int a = 0; a < 3; ++a) {
      tbmin[3 * i + a] -= pad;
      tbmax[3 * i + a] += pad;
      cent[3 * i + a] = 0.5 * (tbmin[3 * i + a] + tbmax[3 * i + a]);
    }
  }

  const int64_t max_nodes = 2 * n;
  for (int64_t k = 0; k < max_nodes; ++k) {
    left[k] = -1;
    right[k] = -1;
    first[k] = 0;
    count[k] = 0;
  }
  for (int64_t k = 0; k < n; ++k) order[k] = (int32_t)k;

  std::vector<int64_t> bin_count(n_bins), sweep_count(n_bins);
  std::vector<Box> bins(n_bins);
  std::vector<double> sweep_area(n_bins);
  std::vector<Job> stack;
  stack.reserve(kDepthCap + 8);
  stack.push_back({0, 0, n, 0});
  int64_t n_nodes = 1, leaf_count = 0, max_depth = 0;

  while (!stack.empty()) {
    Job job = stack.back();
    stack.pop_back();
    const int64_t node = job.node, f = job.first, c = job.count, depth = job.depth;
    if (depth > max_depth) max_depth = depth;

    Box nb;
    nb.reset();
    for (int64_t k = f; k < f + c; ++k) {
      const int64_t ti = order[k];
      nb.grow_min(&tbmin[3 * ti]);
      nb.grow_max(&tbmax[3 * ti]);
    }
    for (int a = 0; a < 3; ++a) {
      bmin[3 * node + a] = nb.lo[a];
      bmax[3 * node + a] = nb.hi[a];
    }
    const double parent_area = nb.area2();

    bool make_leaf = c <= leaf_size || depth >= kDepthCap || parent_area <= 0.0;
    int64_t mid = -1;

    if (!make_leaf) {
      Box cb;
      cb.reset();
      for (int64_t k = f; k < f + c; ++k) {
        const double *p = &cent[3 * (int64_t)order[k]];
        cb.grow_min(p);
        cb.grow_max(p);
      }
      double ex = cb.hi[0] - cb.lo[0], ey = cb.hi[1] - cb.lo[1], ez = cb.hi[2] - cb.lo[2];
      int axis = 0;
      double ext = ex;
      if (ey > ext) {
        axis = 1;
        ext = ey;
      }
      if (ez > ext) {
        axis = 2;
        ext = ez;
      }
      const double cmin_axis = cb.lo[axis];

      if (ext > 0.0) {
        const double scale = (double)n_bins / ext;
        auto bin_of = [&](int64_t ti) {
          int64_t b = (int64_t)((cent[3 * ti + axis] - cmin_axis) * scale);
          return b >= n_bins ? (int64_t)(n_bins - 1) : b;
        };
        for (int b = 0; b < n_bins; ++b) {
          bin_count[b] = 0;
          bins[b].reset();
        }
        for (int64_t k = f; k < f + c; ++k) {
          const int64_t ti = order[k];
          const int64_t b = bin_of(ti);
          bin_count[b] += 1;
          bins[b].grow_min(&tbmin[3 * ti]);
          bins[b].grow_max(&tbmax[3 * ti]);
        }
        // prefix sweep: left side of the plane after bin b
        Box acc;
        acc.reset();
        int64_t acc_n = 0;
        for (int b = 0; b < n_bins - 1; ++b) {
          if (bin_count[b] > 0) {
            acc.grow_min(bins[b].lo);
            acc.grow_max(bins[b].hi);
            acc_n += bin_count[b];
          }
          sweep_count[b] = acc_n;
          sweep_area[b] = acc_n > 0 ? acc.area2() : 0.0;
        }
        // suffix sweep + SAH cost; lowest plane index wins ties
        double best_cost = std::numeric_limits<double>::infinity();
        int best_plane = -1;
        acc.reset();
        acc_n = 0;
        for (int b = n_bins - 1; b > 0; --b) {
          if (bin_count[b] > 0) {
            acc.grow_min(bins[b].lo);
            acc.grow_max(bins[b].hi);
            acc_n += bin_count[b];
          }
          const int plane = b - 1;
          const int64_t ln = sweep_count[plane], rn = acc_n;
          if (ln > 0 && rn > 0) {
            const double right_area = acc.area2();
            const double cost =
                kTraversalCost + kIntersectCost * (sweep_area[plane] * (double)ln +
                                                   right_area * (double)rn) /
                                     parent_area;
            if (cost < best_cost) {
              best_cost = cost;
              best_plane = plane;
            }
          }
        }
        if (best_plane >= 0 && best_cost < kIntersectCost * (double)c) {
          int64_t i = f, j = f + c - 1;
          while (i <= j) {
            if (bin_of(order[i]) <= best_plane) {
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
          make_leaf = true;
        }
      } else {
        mid = f + c / 2;  // coincident centroids: median split of the range
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
    stack.push_back({rchild, mid, f + c - mid, depth + 1});
    stack.push_back({lchild, f, mid - f, depth + 1});
  }
  *n_nodes_out = n_nodes;
  *leaf_count_out = leaf_count;
  *max_depth_out = max_depth;
  return LT_OK;
}
