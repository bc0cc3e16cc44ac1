// lt_ingest.cu -- flatten_scene (scene.py:519-596) on the device, fed from
// the GLB's raw accessor bytes (include/luxb200.h, lt_gltf_desc).
//
// Compiled with -fmad=false: every float64 operation rounds separately, as
// numpy's elementwise ufuncs do; the one place numpy fuses -- the BLAS
// product `positions @ linear.T` (OpenBLAS dgemm: one FMA chain over k = 0,
// 1, 2 per output, first product rounded) -- is written out with __fma_rn.
//
// Data flow (all on one stream):
//   raw bytes -> k_decode_idx   global vertex id per index position
//             -> k_decode_vtx   float64 positions / given normals per vertex
//   smooth normals (primitives without NORMAL, scene.py:493-508):
//             -> k_contrib      (vertex, triangle) pairs in np.add.at order
//                               (pass k = 0, 1, 2, triangles ascending)
//             -> stable radix sort by vertex; k_segments; k_smooth sums each
//                vertex's faces in that order from +0.0
//   instances (one per node x primitive, flatten_scene's visit order):
//             -> k_extent       world corners -> per-axis min / max
//             -> k_keep         area > 1e-12 * extent^2
//             -> exclusive scan -> k_emit: kept triangles, unit normals
// World corners are recomputed by each pass instead of stored (3 x 72 B per
// triangle of HBM traffic saved; the arithmetic is identical every time).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "lt_internal.h"

namespace {

struct DPrim {
  int64_t pos_at, nrm_at, idx_at;  // device byte offsets into the raw buffer
  int32_t pos_stride, nrm_stride, idx_stride, idx_bytes;
  int64_t vtx_off, n_vertices;     // global vertex range
  int64_t tri_off, n_tris;         // global primitive-triangle range
  int32_t has_nrm, has_idx;
};

struct DInst {
  int64_t tri_off;                 // first output (pre-filter) triangle
  int32_t prim, material;
  double L[9], T[3], N[9];
};

__device__ __forceinline__ float ld_f32(const uint8_t *p) {
  float f;
  memcpy(&f, p, 4);  // accessor offsets need not be 4-aligned in a foreign file
  return f;
}

template <class T>
__device__ __forceinline__ int64_t upper_index(const T *arr, int64_t n, int64_t key,
                                               int64_t (*get)(const T &)) {
  // last i with get(arr[i]) <= key
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (get(arr[mid]) <= key) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ int64_t prim_tri(const DPrim &p) { return p.tri_off; }
__device__ int64_t prim_vtx(const DPrim &p) { return p.vtx_off; }
__device__ int64_t inst_tri(const DInst &p) { return p.tri_off; }

__global__ void k_decode_idx(const uint8_t *raw, const DPrim *prims, int32_t n_prims,
                             int64_t n_pos, int32_t *gidx, int32_t *bad) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_pos) return;
  const int64_t t = q / 3;
  const DPrim &p = prims[upper_index(prims, n_prims, t, prim_tri)];
  const int64_t local = q - 3 * p.tri_off;
  int64_t v = local;
  if (p.has_idx) {
    const uint8_t *s = raw + p.idx_at + local * p.idx_stride;
    v = p.idx_bytes == 4 ? (int64_t)(uint32_t)(s[0] | s[1] << 8 | s[2] << 16 | (uint32_t)s[3] << 24)
        : p.idx_bytes == 2 ? (int64_t)(s[0] | s[1] << 8)
                           : (int64_t)s[0];
  }
  if (v >= p.n_vertices) {
    atomicMin(bad, (int32_t)(&p - prims));
    v = 0;
  }
  gidx[q] = (int32_t)(p.vtx_off + v);
}

__global__ void k_decode_vtx(const uint8_t *raw, const DPrim *prims, int32_t n_prims,
                             int64_t n_vtx, double *pos, double *nrm) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n_vtx) return;
  const DPrim &p = prims[upper_index(prims, n_prims, v, prim_vtx)];
  const int64_t local = v - p.vtx_off;
  const uint8_t *s = raw + p.pos_at + local * p.pos_stride;
  for (int a = 0; a < 3; ++a) pos[3 * v + a] = (double)ld_f32(s + 4 * a);
  if (p.has_nrm) {
    const uint8_t *q = raw + p.nrm_at + local * p.nrm_stride;
    for (int a = 0; a < 3; ++a) nrm[3 * v + a] = (double)ld_f32(q + 4 * a);
  }
}

// np.cross (numeric.py): each component a product difference, rounded twice
__device__ __forceinline__ void cross64(const double a[3], const double b[3], double c[3]) {
  c[0] = __dmul_rn(a[1], b[2]) - __dmul_rn(a[2], b[1]);
  c[1] = __dmul_rn(a[2], b[0]) - __dmul_rn(a[0], b[2]);
  c[2] = __dmul_rn(a[0], b[1]) - __dmul_rn(a[1], b[0]);
}

// np.linalg.norm(x, axis=1) on (n, 3): sqrt((x0^2 + x1^2) + x2^2)
__device__ __forceinline__ double norm3(const double c[3]) {
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(c[0], c[0]), __dmul_rn(c[1], c[1])),
                        __dmul_rn(c[2], c[2])));
}

// face normal of primitive triangle t: cross(b - a, c - a) (scene.py:493-508)
__device__ __forceinline__ void face64(const double *pos, const int32_t *gidx, int64_t t,
                                       double f[3]) {
  const double *a = pos + 3 * (int64_t)gidx[3 * t];
  const double *b = pos + 3 * (int64_t)gidx[3 * t + 1];
  const double *c = pos + 3 * (int64_t)gidx[3 * t + 2];
  double e1[3], e2[3];
  for (int k = 0; k < 3; ++k) {
    e1[k] = b[k] - a[k];
    e2[k] = c[k] - a[k];
  }
  cross64(e1, e2, f);
}

// one (vertex, triangle) pair per index position of the smooth-normal
// primitives, laid out pass-major: np.add.at(acc, indices[k::3], face) runs
// pass k = 0, 1, 2, each over the triangles in order
__global__ void k_contrib(const DPrim *prims, int32_t n_prims, const int32_t *gidx,
                          int64_t n_tris, uint32_t sentinel, uint32_t *key, uint32_t *val) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_tris) return;
  const DPrim &p = prims[upper_index(prims, n_prims, t, prim_tri)];
  const int64_t local = t - p.tri_off;
  for (int k = 0; k < 3; ++k) {
    const int64_t slot = 3 * p.tri_off + k * p.n_tris + local;
    key[slot] = p.has_nrm ? sentinel : (uint32_t)gidx[3 * t + k];
    val[slot] = (uint32_t)t;
  }
}

__global__ void k_segments(const uint32_t *key, int64_t n, uint32_t sentinel, int32_t *start,
                           int32_t *end) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t k = key[i];
  if (k == sentinel) return;
  if (i == 0 || key[i - 1] != k) start[k] = (int32_t)i;
  if (i == n - 1 || key[i + 1] != k) end[k] = (int32_t)(i + 1);
}

__global__ void k_smooth(const DPrim *prims, int32_t n_prims, const double *pos,
                         const int32_t *gidx, const uint32_t *val, const int32_t *start,
                         const int32_t *end, int64_t n_vtx, double *nrm) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n_vtx) return;
  const DPrim &p = prims[upper_index(prims, n_prims, v, prim_vtx)];
  if (p.has_nrm) return;
  double acc[3] = {0.0, 0.0, 0.0};  // np.zeros_like(positions)
  for (int32_t i = start[v]; i < end[v]; ++i) {
    double f[3];
    face64(pos, gidx, val[i], f);
    for (int k = 0; k < 3; ++k) acc[k] = __dadd_rn(acc[k], f[k]);
  }
  double len = norm3(acc);
  if (len == 0.0) {
    acc[0] = 0.0;
    acc[1] = 0.0;
    acc[2] = 1.0;
    len = 1.0;
  }
  for (int k = 0; k < 3; ++k) nrm[3 * v + k] = acc[k] / len;
}

// positions @ linear.T + translation: OpenBLAS's dgemm accumulates k = 0, 1,
// 2 in one FMA chain whose first product is rounded; the translation is a
// separate numpy add
__device__ __forceinline__ void xform(const double *M, const double x[3], double out[3]) {
  for (int j = 0; j < 3; ++j)
    out[j] = __fma_rn(x[2], M[3 * j + 2], __fma_rn(x[1], M[3 * j + 1], __dmul_rn(x[0], M[3 * j])));
}

struct Corners {
  double v[3][3];
};

__device__ __forceinline__ const DInst &inst_of(const DInst *inst, int32_t n_inst, int64_t j) {
  return inst[upper_index(inst, n_inst, j, inst_tri)];
}

__device__ __forceinline__ void world_corners(const DInst &I, const DPrim *prims,
                                              const double *pos, const int32_t *gidx,
                                              int64_t j, Corners &c, int64_t &pt) {
  const DPrim &p = prims[I.prim];
  pt = p.tri_off + (j - I.tri_off);
  for (int k = 0; k < 3; ++k) {
    const double *x = pos + 3 * (int64_t)gidx[3 * pt + k];
    double w[3];
    xform(I.L, x, w);
    for (int a = 0; a < 3; ++a) c.v[k][a] = __dadd_rn(w[a], I.T[a]);
  }
}

// order-preserving uint64 image of a double (min / max by integer atomics)
__device__ __forceinline__ unsigned long long ord64(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double unord64(unsigned long long u) {
  const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
  double d;
  memcpy(&d, &b, 8);
  return d;
}

// ext[0..2] = ord(min) per axis, ext[3..5] = ord(max), ext[6] = NaN seen
__global__ void k_extent(const DInst *inst, int32_t n_inst, const DPrim *prims,
                         const double *pos, const int32_t *gidx, int64_t n,
                         unsigned long long *ext) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long lo[3], hi[3], nan = 0;
  for (int a = 0; a < 3; ++a) {
    lo[a] = ~0ull;
    hi[a] = 0;
  }
  if (j < n) {
    Corners c;
    int64_t pt;
    world_corners(inst_of(inst, n_inst, j), prims, pos, gidx, j, c, pt);
    for (int k = 0; k < 3; ++k)
      for (int a = 0; a < 3; ++a) {
        const double x = c.v[k][a];
        if (isnan(x)) nan = 1;
        const unsigned long long u = ord64(x);
        lo[a] = u < lo[a] ? u : lo[a];
        hi[a] = u > hi[a] ? u : hi[a];
      }
  }
  for (int o = 16; o > 0; o >>= 1) {
    for (int a = 0; a < 3; ++a) {
      const unsigned long long l = __shfl_xor_sync(0xffffffffu, lo[a], o);
      const unsigned long long h = __shfl_xor_sync(0xffffffffu, hi[a], o);
      lo[a] = l < lo[a] ? l : lo[a];
      hi[a] = h > hi[a] ? h : hi[a];
    }
    nan |= __shfl_xor_sync(0xffffffffu, nan, o);
  }
  if ((threadIdx.x & 31) == 0) {
    for (int a = 0; a < 3; ++a) {
      atomicMin(&ext[a], lo[a]);
      atomicMax(&ext[3 + a], hi[a]);
    }
    if (nan) atomicMax(&ext[6], 1ull);
  }
}

// extent = max over axes of (max - min), NaN-propagating like np.max;
// threshold = DEGENERATE_AREA_SCALE * extent * extent (scene.py:29, 578)
__device__ __forceinline__ double area_threshold(const unsigned long long *ext) {
  double e = 0.0;
  bool nan = ext[6] != 0;
  for (int a = 0; a < 3; ++a) {
    const double d = unord64(ext[3 + a]) - unord64(ext[a]);
    if (isnan(d)) nan = true;
    e = a == 0 ? d : (d > e ? d : e);
  }
  if (nan) e = __longlong_as_double(0x7ff8000000000000ll);
  return __dmul_rn(__dmul_rn(1e-12, e), e);
}

__device__ __forceinline__ double tri_area(const Corners &c) {
  double e1[3], e2[3], x[3];
  for (int a = 0; a < 3; ++a) {
    e1[a] = c.v[1][a] - c.v[0][a];
    e2[a] = c.v[2][a] - c.v[0][a];
  }
  cross64(e1, e2, x);
  return __dmul_rn(0.5, norm3(x));
}

__global__ void k_keep(const DInst *inst, int32_t n_inst, const DPrim *prims, const double *pos,
                       const int32_t *gidx, int64_t n, const unsigned long long *ext,
                       int32_t *keep) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  Corners c;
  int64_t pt;
  world_corners(inst_of(inst, n_inst, j), prims, pos, gidx, j, c, pt);
  keep[j] = tri_area(c) > area_threshold(ext) ? 1 : 0;
}

// unit_rows (scene.py:585-589): zero-length rows are left as they are
__device__ __forceinline__ void unit_row(double x[3]) {
  double len = norm3(x);
  if (len == 0.0) len = 1.0;
  for (int a = 0; a < 3; ++a) x[a] = x[a] / len;
}

__global__ void k_emit(const DInst *inst, int32_t n_inst, const DPrim *prims, const double *pos,
                       const double *nrm, const int32_t *gidx, int64_t n, const int32_t *keep,
                       const int32_t *slot, double *v0, double *v1, double *v2, double *n0,
                       double *n1, double *n2, int32_t *mat) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n || !keep[j]) return;
  const DInst &I = inst_of(inst, n_inst, j);
  Corners c;
  int64_t pt;
  world_corners(I, prims, pos, gidx, j, c, pt);
  const int64_t o = slot[j];
  double *vo[3] = {v0, v1, v2}, *no[3] = {n0, n1, n2};
  for (int k = 0; k < 3; ++k) {
    double w[3];
    xform(I.N, nrm + 3 * (int64_t)gidx[3 * pt + k], w);  // local_n @ to_normals.T
    unit_row(w);
    for (int a = 0; a < 3; ++a) {
      vo[k][3 * o + a] = c.v[k][a];
      no[k][3 * o + a] = w[a];
    }
  }
  mat[o] = I.material;
}

inline unsigned grid(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

#define ICK(call)                                                                  \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return lt_fail(e_ == cudaErrorMemoryAllocation ? LT_ERR_NOMEM : LT_ERR_CUDA, \
                     "ingest: %s failed: %s", #call, cudaGetErrorString(e_));      \
  } while (0)

int lt_ingest_check(const lt_gltf_desc *g, int32_t n_materials, int64_t *n_out_tris) {
  if (!g) return lt_fail(LT_ERR_INVALID, "null glTF description");
  if (g->n_buffers < 0 || (g->n_buffers > 0 && (!g->buffers || !g->buffer_bytes)))
    return lt_fail(LT_ERR_INVALID, "glTF buffers must be non-null");
  if (g->n_primitives < 0 || (g->n_primitives > 0 && !g->primitives) || g->n_instances < 0 ||
      (g->n_instances > 0 && !g->instances))
    return lt_fail(LT_ERR_INVALID, "glTF primitive / instance tables must be non-null");
  for (int32_t b = 0; b < g->n_buffers; ++b)
    if (g->buffer_bytes[b] < 0 || (g->buffer_bytes[b] > 0 && !g->buffers[b]))
      return lt_fail(LT_ERR_INVALID, "buffer %d: null data", b);
  int64_t n_idx = 0, n_vtx = 0;
  auto in_buffer = [&](int32_t buf, int64_t off, int32_t stride, int64_t count, int64_t elem) {
    if (buf < 0 || buf >= g->n_buffers || off < 0 || stride < elem) return false;
    return count == 0 || off + stride * (count - 1) + elem <= g->buffer_bytes[buf];
  };
  for (int32_t i = 0; i < g->n_primitives; ++i) {
    const lt_gltf_primitive &p = g->primitives[i];
    if (p.n_vertices < 0 || p.n_indices < 0 || p.n_indices % 3 != 0)
      return lt_fail(LT_ERR_INVALID, "primitive %d: bad vertex / index count", i);
    if (!in_buffer(p.pos_buffer, p.pos_offset, p.pos_stride, p.n_vertices, 12))
      return lt_fail(LT_ERR_INVALID, "primitive %d: POSITION range outside its buffer", i);
    if (p.nrm_buffer != -1 && !in_buffer(p.nrm_buffer, p.nrm_offset, p.nrm_stride, p.n_vertices, 12))
      return lt_fail(LT_ERR_INVALID, "primitive %d: NORMAL range outside its buffer", i);
    if (p.idx_buffer != -1) {
      if (p.idx_bytes != 1 && p.idx_bytes != 2 && p.idx_bytes != 4)
        return lt_fail(LT_ERR_INVALID, "primitive %d: index size %d", i, p.idx_bytes);
      if (!in_buffer(p.idx_buffer, p.idx_offset, p.idx_stride, p.n_indices, p.idx_bytes))
        return lt_fail(LT_ERR_INVALID, "primitive %d: index range outside its buffer", i);
    } else if (p.n_indices > p.n_vertices) {
      return lt_fail(LT_ERR_INVALID, "primitive %d: index out of range", i);
    }
    n_idx += p.n_indices;
    n_vtx += p.n_vertices;
  }
  if (n_vtx >= (int64_t(1) << 31) - 1 || n_idx >= (int64_t(1) << 31) - 3)
    return lt_fail(LT_ERR_INVALID, "glTF geometry too large for 32-bit ids");
  int64_t n_out = 0;
  for (int32_t i = 0; i < g->n_instances; ++i) {
    const lt_gltf_instance &I = g->instances[i];
    if (I.primitive < 0 || I.primitive >= g->n_primitives)
      return lt_fail(LT_ERR_INVALID, "instance %d: primitive %d out of range", i, I.primitive);
    if (I.material < 0 || (n_materials > 0 && I.material >= n_materials))
      return lt_fail(LT_ERR_INVALID, "instance %d: material %d out of range [0, %d)", i,
                     I.material, n_materials);
    n_out += g->primitives[I.primitive].n_indices / 3;
  }
  if (n_out >= (int64_t(1) << 31) - 1)
    return lt_fail(LT_ERR_INVALID, "too many triangles (%lld)", (long long)n_out);
  *n_out_tris = n_out;
  return LT_OK;
}

void lt_ingest_free(lt_ingest_out *o, void *stream) {
  if (o->mem) cudaFreeAsync(o->mem, (cudaStream_t)stream);
  *o = lt_ingest_out{};
}

int lt_ingest_run(const lt_gltf_desc *g, const uint8_t *d_raw, const int64_t *buf_at,
                  void *stream, lt_ingest_out *out) {
  cudaStream_t st = (cudaStream_t)stream;
  *out = lt_ingest_out{};
  int64_t n_out = 0;
  if (int rc = lt_ingest_check(g, 0, &n_out)) return rc;
  // device tables: primitives with their global vertex / triangle ranges,
  // instances with their output triangle ranges
  std::vector<DPrim> prims(g->n_primitives);
  int64_t n_vtx = 0, n_tris = 0;
  bool any_smooth = false;
  for (int32_t i = 0; i < g->n_primitives; ++i) {
    const lt_gltf_primitive &s = g->primitives[i];
    DPrim &p = prims[i];
    p.pos_at = buf_at[s.pos_buffer] + s.pos_offset;
    p.pos_stride = s.pos_stride;
    p.has_nrm = s.nrm_buffer >= 0;
    p.nrm_at = p.has_nrm ? buf_at[s.nrm_buffer] + s.nrm_offset : 0;
    p.nrm_stride = s.nrm_stride;
    p.has_idx = s.idx_buffer >= 0;
    p.idx_at = p.has_idx ? buf_at[s.idx_buffer] + s.idx_offset : 0;
    p.idx_stride = s.idx_stride;
    p.idx_bytes = s.idx_bytes;
    p.vtx_off = n_vtx;
    p.n_vertices = s.n_vertices;
    p.tri_off = n_tris;
    p.n_tris = s.n_indices / 3;
    n_vtx += s.n_vertices;
    n_tris += p.n_tris;
    any_smooth |= !p.has_nrm && p.n_tris > 0;
  }
  std::vector<DInst> inst(g->n_instances);
  int64_t at = 0;
  for (int32_t i = 0; i < g->n_instances; ++i) {
    const lt_gltf_instance &s = g->instances[i];
    DInst &d = inst[i];
    d.tri_off = at;
    d.prim = s.primitive;
    d.material = s.material;
    memcpy(d.L, s.linear, sizeof d.L);
    memcpy(d.T, s.translation, sizeof d.T);
    memcpy(d.N, s.normal_matrix, sizeof d.N);
    at += g->primitives[s.primitive].n_indices / 3;
  }
  out->n_total = n_out;
  if (n_out == 0) return lt_fail(LT_ERR_INVALID, "empty scene");
  // primitives / instances with no triangles are skipped by the binary
  // searches (equal offsets: the last one wins and owns the range)

  // one allocation for everything that outlives this call (the flattened
  // arrays) and one scratch for the rest
  const int64_t n_pos = 3 * n_tris;
  const uint32_t sentinel = (uint32_t)n_vtx;
  int end_bit = 1;
  while (end_bit < 32 && (uint64_t(1) << end_bit) <= (uint64_t)sentinel) ++end_bit;
  size_t sort_tmp = 0, scan_tmp = 0;
  if (any_smooth)
    ICK(cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (uint32_t *)nullptr,
                                        (uint32_t *)nullptr, (uint32_t *)nullptr,
                                        (uint32_t *)nullptr, (int)n_pos, 0, end_bit, st));
  ICK(cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (int32_t *)nullptr, (int32_t *)nullptr,
                                    (int)n_out, st));
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t out_bytes = 6 * al(24 * (size_t)n_out) + al(4 * (size_t)n_out);
  size_t tmp_bytes = al(sizeof(DPrim) * prims.size()) + al(sizeof(DInst) * inst.size()) +
                     al(4 * (size_t)n_pos) + al(24 * (size_t)n_vtx) * 2 + al(8 * 8) + al(4) +
                     al(4 * (size_t)n_out) * 2 + al(scan_tmp);
  if (any_smooth) tmp_bytes += 4 * al(4 * (size_t)n_pos) + 2 * al(4 * (size_t)n_vtx) + al(sort_tmp);
  void *tmp = nullptr;
  ICK(cudaMallocAsync(&out->mem, out_bytes, st));
  {
    const cudaError_t e = cudaMallocAsync(&tmp, tmp_bytes, st);
    if (e != cudaSuccess) {
      lt_ingest_free(out, st);
      return lt_fail(LT_ERR_NOMEM, "ingest scratch: %s", cudaGetErrorString(e));
    }
  }
  struct TmpGuard {
    void *p;
    cudaStream_t st;
    ~TmpGuard() { cudaFreeAsync(p, st); }
  } tmp_guard{tmp, st};
  char *o = static_cast<char *>(out->mem);
  for (int k = 0; k < 6; ++k, o += al(24 * (size_t)n_out)) out->v[k] = reinterpret_cast<double *>(o);
  out->mat = reinterpret_cast<int32_t *>(o);
  char *t = static_cast<char *>(tmp);
  auto take = [&](size_t b) {
    char *r = t;
    t += al(b);
    return r;
  };
  DPrim *d_prims = reinterpret_cast<DPrim *>(take(sizeof(DPrim) * prims.size()));
  DInst *d_inst = reinterpret_cast<DInst *>(take(sizeof(DInst) * inst.size()));
  int32_t *gidx = reinterpret_cast<int32_t *>(take(4 * (size_t)n_pos));
  double *pos = reinterpret_cast<double *>(take(24 * (size_t)n_vtx));
  double *nrm = reinterpret_cast<double *>(take(24 * (size_t)n_vtx));
  unsigned long long *ext = reinterpret_cast<unsigned long long *>(take(64));
  int32_t *bad = reinterpret_cast<int32_t *>(take(4));
  int32_t *keep = reinterpret_cast<int32_t *>(take(4 * (size_t)n_out));
  int32_t *slot = reinterpret_cast<int32_t *>(take(4 * (size_t)n_out));
  void *scan_buf = take(scan_tmp);
  const int B = 256;
  int rc = LT_OK;
  do {
    cudaError_t e;
    const int32_t np = g->n_primitives, ni = g->n_instances;
#define ISTEP(call)                                                                 \
  if ((e = (call)) != cudaSuccess) {                                                \
    rc = lt_fail(e == cudaErrorMemoryAllocation ? LT_ERR_NOMEM : LT_ERR_CUDA,      \
                 "ingest: %s failed: %s", #call, cudaGetErrorString(e));            \
    break;                                                                          \
  }
    // the tables are staged in pageable host vectors: synchronous copies
    ISTEP(cudaMemcpyAsync(d_prims, prims.data(), sizeof(DPrim) * prims.size(),
                          cudaMemcpyHostToDevice, st));
    ISTEP(cudaMemcpyAsync(d_inst, inst.data(), sizeof(DInst) * inst.size(),
                          cudaMemcpyHostToDevice, st));
    unsigned long long ext0[7] = {~0ull, ~0ull, ~0ull, 0, 0, 0, 0};
    ISTEP(cudaMemcpyAsync(ext, ext0, sizeof ext0, cudaMemcpyHostToDevice, st));
    const int32_t bad0 = INT32_MAX;
    ISTEP(cudaMemcpyAsync(bad, &bad0, 4, cudaMemcpyHostToDevice, st));
    if (n_pos > 0) k_decode_idx<<<grid(n_pos, B), B, 0, st>>>(d_raw, d_prims, np, n_pos, gidx, bad);
    if (n_vtx > 0) k_decode_vtx<<<grid(n_vtx, B), B, 0, st>>>(d_raw, d_prims, np, n_vtx, pos, nrm);
    ISTEP(cudaGetLastError());
    int32_t bad_h = INT32_MAX;
    ISTEP(cudaMemcpyAsync(&bad_h, bad, 4, cudaMemcpyDeviceToHost, st));
    ISTEP(cudaStreamSynchronize(st));
    if (bad_h != INT32_MAX) {
      rc = lt_fail(LT_ERR_INVALID, "primitive %d: index out of range", bad_h);
      break;
    }
    if (any_smooth) {
      uint32_t *key = reinterpret_cast<uint32_t *>(take(4 * (size_t)n_pos));
      uint32_t *val = reinterpret_cast<uint32_t *>(take(4 * (size_t)n_pos));
      uint32_t *key2 = reinterpret_cast<uint32_t *>(take(4 * (size_t)n_pos));
      uint32_t *val2 = reinterpret_cast<uint32_t *>(take(4 * (size_t)n_pos));
      int32_t *seg_s = reinterpret_cast<int32_t *>(take(4 * (size_t)n_vtx));
      int32_t *seg_e = reinterpret_cast<int32_t *>(take(4 * (size_t)n_vtx));
      void *sort_buf = take(sort_tmp);
      k_contrib<<<grid(n_tris, B), B, 0, st>>>(d_prims, np, gidx, n_tris, sentinel, key, val);
      ISTEP(cub::DeviceRadixSort::SortPairs(sort_buf, sort_tmp, key, key2, val, val2, (int)n_pos,
                                            0, end_bit, st));
      ISTEP(cudaMemsetAsync(seg_s, 0, 4 * (size_t)n_vtx, st));
      ISTEP(cudaMemsetAsync(seg_e, 0, 4 * (size_t)n_vtx, st));
      k_segments<<<grid(n_pos, B), B, 0, st>>>(key2, n_pos, sentinel, seg_s, seg_e);
      k_smooth<<<grid(n_vtx, B), B, 0, st>>>(d_prims, np, pos, gidx, val2, seg_s, seg_e, n_vtx,
                                             nrm);
      ISTEP(cudaGetLastError());
    }
    k_extent<<<grid(n_out, B), B, 0, st>>>(d_inst, ni, d_prims, pos, gidx, n_out, ext);
    k_keep<<<grid(n_out, B), B, 0, st>>>(d_inst, ni, d_prims, pos, gidx, n_out, ext, keep);
    ISTEP(cudaGetLastError());
    ISTEP(cub::DeviceScan::ExclusiveSum(scan_buf, scan_tmp, keep, slot, (int)n_out, st));
    k_emit<<<grid(n_out, B), B, 0, st>>>(d_inst, ni, d_prims, pos, nrm, gidx, n_out, keep, slot,
                                         out->v[0], out->v[1], out->v[2], out->v[3], out->v[4],
                                         out->v[5], out->mat);
    ISTEP(cudaGetLastError());
    int32_t last[2];
    ISTEP(cudaMemcpyAsync(&last[0], slot + n_out - 1, 4, cudaMemcpyDeviceToHost, st));
    ISTEP(cudaMemcpyAsync(&last[1], keep + n_out - 1, 4, cudaMemcpyDeviceToHost, st));
    ISTEP(cudaStreamSynchronize(st));
#undef ISTEP
    out->n_kept = (int64_t)last[0] + last[1];
    out->n_dropped = n_out - out->n_kept;
    if (out->n_kept == 0) rc = lt_fail(LT_ERR_INVALID, "empty scene");
  } while (0);
  if (rc != LT_OK) lt_ingest_free(out, st);
  return rc;
}
