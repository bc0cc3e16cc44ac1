// lt_api.cu -- the C-ABI (include/luxb200.h): scene residency, the render
// pass orchestration (the wavefront loop), ray queries and host-buffer
// drop-ins with the reference's dtypes.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "lt_internal.h"
#include "lt_kernels.h"
#include "lt_staged.h"

using namespace lt;

// ------------------------------------------------------------------ errors

static thread_local std::string g_last_error;

int lt_fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return lt_fail(e_ == cudaErrorMemoryAllocation ? LT_ERR_NOMEM : LT_ERR_CUDA, \
                     "%s failed: %s", #call, cudaGetErrorString(e_));              \
  } while (0)

#define RET(expr)            \
  do {                       \
    int r_ = (expr);         \
    if (r_ != LT_OK) return r_; \
  } while (0)

namespace {

// Paths per wavefront batch.  Large batches amortize the drain tail of every
// persistent trace launch (the last, longest rays of a bounce run on a few
// lanes while the rest of the GPU idles): 4M -> 64M paths took the C4 step
// from 452 to 277 ms (profiles/r01_batch_sweep.jsonl).  128 B of queues and
// path state per path: 64M paths = 8 GB, bounded by a quarter of free HBM.
#ifndef LT_MAX_BATCH_LOG2
#define LT_MAX_BATCH_LOG2 28
#endif
constexpr int64_t kMaxBatchPaths = int64_t(1) << LT_MAX_BATCH_LOG2;
// Passes of at most this many paths run as one fused launch per batch
// (k_path_small) instead of the wavefront: 2x faster at 1-2 M paths (a
// 1080p 1-spp progressive update: 2.21 -> 1.08 ms), even at ~8 M, 1.5x
// slower at full frames (profiles/r02_fused_small.jsonl, _scale.jsonl).
constexpr int64_t kFusedMaxPaths = int64_t(1) << 22;

// Device buffer.  With `ast` set the memory comes stream-ordered from the
// device's default mempool (cudaMallocAsync / cudaFreeAsync on `ast`), so a
// scene's lifetime never costs a device-wide cudaFree synchronization (which
// measured up to 1.5 s per scene destroy on the B200 box).
struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  cudaStream_t ast = nullptr;
  bool stream_ordered = false;
  int ensure(size_t want) {
    if (want <= bytes) return LT_OK;
    release();
    if (stream_ordered) {
      CK(cudaMallocAsync(&p, want, ast));
      // usable from any stream once the allocation has executed (growth is rare)
      CK(cudaStreamSynchronize(ast));
    } else {
      CK(cudaMalloc(&p, want));
    }
    bytes = want;
    return LT_OK;
  }
  void release() {
    if (p) {
      if (stream_ordered) cudaFreeAsync(p, ast);
      else cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T *as() const {
    return static_cast<T *>(p);
  }
};

// Stream-ordered temporary (cudaMallocAsync / cudaFreeAsync): scene upload
// staging without the device-wide synchronization of cudaFree.
struct TmpBuf {
  void *p = nullptr;
  cudaStream_t st = nullptr;
  bool view = false;  // points into another TmpBuf (not freed here)
  int alloc(size_t want, cudaStream_t s) {
    st = s;
    CK(cudaMallocAsync(&p, std::max<size_t>(want, 16), s));
    return LT_OK;
  }
  void set_view(void *q) {
    p = q;
    view = true;
  }
  ~TmpBuf() {
    if (p && !view) cudaFreeAsync(p, st);
  }
  template <class T>
  T *as() const {
    return static_cast<T *>(p);
  }
};

struct HostBuf {
  void *p = nullptr;
  size_t bytes = 0;
  int ensure(size_t want) {
    if (want <= bytes) return LT_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    CK(cudaMallocHost(&p, want));
    bytes = want;
    return LT_OK;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T *as() const {
    return static_cast<T *>(p);
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

// The wavefront queues and path state (up to 8 GB at the default batch) are
// cached per device and shared by every scene on it, so creating a scene per
// render call (the reference's render_progressive does) never re-allocates
// them.  Users serialize on `mu` while enqueueing and on the `last_use` event
// on the device: a pass on another stream waits for the previous pass.
// A render pass runs kLanes independent batch streams ("lanes") over
// disjoint pixel ranges, so the drain tail of one lane's bounce launches
// overlaps the other lane's work; each lane owns its queues.
constexpr int kLanes = 4;          // upper bound; LT_LANES picks 1..kLanes (default 2)
constexpr int kDefaultLanes = 2;
// pinned staging ring for pageable scene arrays: kRingWorkers host threads,
// two kRingSlot slots each
#ifndef LT_RING_WORKERS
#define LT_RING_WORKERS 6
#endif
#ifndef LT_BVH_WORKERS
#define LT_BVH_WORKERS 2
#endif
constexpr int kRingWorkers = LT_RING_WORKERS;
constexpr int kBvhWorkers = LT_BVH_WORKERS;  // of them staging the BVH arrays
constexpr int kRingSlots = 2 * kRingWorkers;
constexpr size_t kRingSlot = size_t(4) << 20;
// resident buffers of destroyed scenes kept for reuse
constexpr size_t kCacheBytes = size_t(2) << 30;

struct Lane {
  int64_t cap = 0;
  int32_t depth_cap = 0;
  DevBuf q_o[2], q_d[2], hits, S, inc, counters;
  DevBuf rng;  // per-batch PCG tables (launch_rng_tables)
  // LT_FLAG_SORT_MATERIALS: per-entry class, the class-grouped slot order,
  // class totals + cursors
  DevBuf cls, perm, cls_ctr;
};

struct Workspace {
  std::mutex mu;
  Lane lane[kLanes];
  cudaEvent_t last_use = nullptr;
  // the lanes' streams and the fork / join events, created on first use and
  // shared by every scene on the device (passes are serialized by `mu`)
  cudaStream_t lane_st[kLanes] = {};
  cudaEvent_t fork_ev = nullptr, join_ev[kLanes] = {};
  // side stream for scene triangle uploads (overlaps the BVH layout)
  cudaStream_t upload_st = nullptr;
  std::mutex upload_mu;
  // scene streams, reused across scenes (stream creation + destruction cost
  // ~0.2 ms per scene, most of a tiny scene's set-up); a returned stream may
  // still carry its last scene's stream-ordered frees, which simply run
  // before the next scene's work
  std::vector<cudaStream_t> free_streams;
  std::mutex stream_mu;
  bool pool_configured = false;
  // pinned staging for small scenes: all arrays in one host buffer and one
  // copy (stage_ev: the last copy out of it; guarded by upload_mu)
  HostBuf stage;
  cudaEvent_t stage_ev = nullptr;
  // scene creation is serialized per device (create_mu): the float64 / int32
  // upload temporaries live in one grow-only device scratch buffer (no
  // stream-ordered pool growth per scene: a pool that had to map new memory
  // for a 150 MB scene stalled creation by up to ~0.5 s on the B200 box), and
  // pageable caller arrays are staged through a pinned ring (ring_ev[k]: the
  // last copy out of slot k)
  std::mutex create_mu;
  DevBuf scratch;
  HostBuf ring;
  cudaEvent_t ring_ev[kRingSlots] = {};
  // resident buffers of destroyed scenes, reused by the next scene of a
  // similar size (ev: the destroyed scene's last use); bounded by kCacheBytes
  struct Cached {
    void *p;
    size_t bytes;
    cudaEvent_t ev;
  };
  std::vector<Cached> cache;
  std::mutex cache_mu;
  cudaEvent_t scratch_ev = nullptr;  // the last read of `scratch`
};

// ---- host -> device copies for scene creation

struct CopyItem {
  void *dst;
  const void *src;
  size_t bytes;
};

// Page-locked host memory (cudaHostAlloc'd or registered): the copy engine
// reads it directly.
static bool host_pinned(const void *p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Host -> device copies of `items` on `st`.  Page-locked sources go straight
// to the copy engine; pageable ones (plain numpy arrays, as luxtrace callers
// pass them) are cut into kRingSlot chunks that kRingWorkers host threads
// copy into the pinned ring, two slots per worker, each slot's copy-out
// issued as soon as it is filled -- the host memcpy of one chunk overlaps
// the DMA of the previous ones (~45 GB/s against 11 GB/s for the driver's
// own pageable path, tools/h2d_probe.py).  Returns after the last copy is
// enqueued.
static int staged_h2d(Workspace &W, int device, const std::vector<CopyItem> &items,
                      cudaStream_t st, int worker0 = 0, int max_workers = kRingWorkers) {
  struct Chunk {
    char *dst;
    const char *src;
    size_t bytes;
  };
  std::vector<Chunk> chunks;
  for (const CopyItem &it : items) {
    if (!it.bytes) continue;
    if (host_pinned(it.src)) {
      CK(cudaMemcpyAsync(it.dst, it.src, it.bytes, cudaMemcpyHostToDevice, st));
      continue;
    }
    for (size_t off = 0; off < it.bytes; off += kRingSlot)
      chunks.push_back(Chunk{static_cast<char *>(it.dst) + off,
                             static_cast<const char *>(it.src) + off,
                             std::min(kRingSlot, it.bytes - off)});
  }
  if (chunks.empty()) return LT_OK;
  const int n_workers = (int)std::min<size_t>(max_workers, chunks.size());
  std::vector<int> rc(n_workers, LT_OK);
  std::vector<std::string> msg(n_workers);
  auto work = [&](int w) {
    cudaSetDevice(device);
    int i = 0;
    for (size_t c = w; c < chunks.size(); c += n_workers, ++i) {
      const int slot = 2 * (worker0 + w) + (i & 1);
      char *buf = W.ring.as<char>() + kRingSlot * slot;
      cudaError_t e = cudaEventSynchronize(W.ring_ev[slot]);  // slot drained
      if (e == cudaSuccess) {
        std::memcpy(buf, chunks[c].src, chunks[c].bytes);
        e = cudaMemcpyAsync(chunks[c].dst, buf, chunks[c].bytes, cudaMemcpyHostToDevice, st);
      }
      if (e == cudaSuccess) e = cudaEventRecord(W.ring_ev[slot], st);
      if (e != cudaSuccess) {
        rc[w] = lt_fail(LT_ERR_CUDA, "staged upload failed: %s", cudaGetErrorString(e));
        msg[w] = g_last_error;
        return;
      }
    }
  };
  std::vector<std::thread> th;
  for (int w = 1; w < n_workers; ++w) th.emplace_back(work, w);
  work(0);
  for (auto &t : th) t.join();
  for (int w = 0; w < n_workers; ++w)
    if (rc[w] != LT_OK) {
      g_last_error = msg[w];
      return rc[w];
    }
  return LT_OK;
}

static int ensure_ring(Workspace &W) {
  RET(W.ring.ensure(kRingSlot * kRingSlots));
  for (int k = 0; k < kRingSlots; ++k)
    if (!W.ring_ev[k]) CK(cudaEventCreateWithFlags(&W.ring_ev[k], cudaEventDisableTiming));
  return LT_OK;
}

// A resident scene buffer: a cached block of a destroyed scene when one fits
// (ordered after that scene's last use on `st`), else a new allocation.
static int take_cached(Workspace &W, DevBuf &b, size_t want, cudaStream_t st) {
  if (b.bytes >= want) return LT_OK;
  {
    std::lock_guard<std::mutex> lk(W.cache_mu);
    int best = -1;
    for (int i = 0; i < (int)W.cache.size(); ++i) {
      const size_t sz = W.cache[i].bytes;
      if (sz >= want && sz <= want + want / 2 + (size_t(16) << 20) &&
          (best < 0 || sz < W.cache[best].bytes))
        best = i;
    }
    if (best >= 0) {
      b.release();
      Workspace::Cached c = W.cache[best];
      W.cache.erase(W.cache.begin() + best);
      CK(cudaStreamWaitEvent(st, c.ev, 0));
      cudaEventDestroy(c.ev);
      b.p = c.p;
      b.bytes = c.bytes;
      return LT_OK;
    }
  }
  return b.ensure(want);
}

// Park a destroyed scene's stream-ordered buffer for reuse (after its last
// use on `st`); the oldest blocks are freed beyond kCacheBytes.
static void park_cached(Workspace &W, DevBuf &b, cudaStream_t st) {
  if (!b.p) return;
  if (!b.stream_ordered) {
    b.release();
    return;
  }
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(ev, st) != cudaSuccess) {
    if (ev) cudaEventDestroy(ev);
    b.release();
    return;
  }
  std::lock_guard<std::mutex> lk(W.cache_mu);
  W.cache.push_back(Workspace::Cached{b.p, b.bytes, ev});
  b.p = nullptr;
  b.bytes = 0;
  size_t total = 0;
  for (const auto &c : W.cache) total += c.bytes;
  while (total > kCacheBytes && !W.cache.empty()) {
    Workspace::Cached c = W.cache.front();
    W.cache.erase(W.cache.begin());
    cudaStreamWaitEvent(st, c.ev, 0);
    cudaEventDestroy(c.ev);
    cudaFreeAsync(c.p, st);
    total -= c.bytes;
  }
}

static Workspace *workspace_for(int device) {
  static std::mutex g_mu;
  static std::vector<Workspace *> g_ws;
  std::lock_guard<std::mutex> lk(g_mu);
  if ((int)g_ws.size() <= device) g_ws.resize(device + 1, nullptr);
  if (!g_ws[device]) g_ws[device] = new Workspace();  // process lifetime
  return g_ws[device];
}

// LT_VERBOSE=1: host-side phase timings on stderr (scene create / destroy).
struct PhaseTimer {
  bool on;
  std::chrono::steady_clock::time_point t;
  PhaseTimer() : on(std::getenv("LT_VERBOSE") != nullptr), t(std::chrono::steady_clock::now()) {}
  void mark(const char *what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[luxb200] %-28s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Enqueue-side exclusive use of a device workspace on stream `st`.
struct WorkspaceLease {
  Workspace *ws;
  cudaStream_t st;
  std::unique_lock<std::mutex> lk;
  WorkspaceLease(Workspace *w, cudaStream_t s) : ws(w), st(s), lk(w->mu) {
    if (!ws->last_use) cudaEventCreateWithFlags(&ws->last_use, cudaEventDisableTiming);
    else cudaStreamWaitEvent(st, ws->last_use, 0);
  }
  ~WorkspaceLease() { cudaEventRecord(ws->last_use, st); }
};

struct lt_scene {
  // serializes the host calls that use the scene's scratch buffers, stats
  // and pixel-list cache (render passes, ray queries) across host threads;
  // taken before the device's workspace lease, never after it
  mutable std::recursive_mutex mu;
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  SceneView view{};
  int64_t n_tris = 0, n_nodes = 0, n_internal = 0, n_bfs = 0;
  int64_t device_bytes = 0;
  // nodes and leaf-ordered triangles share one allocation so a single L2
  // access-policy window keeps the whole traversal set persisting
  DevBuf geo, shade, mats, env, nodes2;
  size_t nodes_bytes = 0, geo_bytes = 0, shade_off = 0;
  int64_t n_wide = 0;
  bool use_window = false;
  cudaAccessPolicyWindow window{}, shade_window{};
  bool use_shade_window = false;
  size_t persist_bytes = 0;
  // wavefront workspace: shared per device (see Workspace)
  struct Workspace *ws = nullptr;
  DevBuf ray_ctr;
  // sharding pixel list cache
  DevBuf pix_list;
  int64_t pix_key[5] = {-1, -1, -1, -1, -1};
  int64_t pix_count = 0;
  // scratch for ray queries / host drop-ins
  DevBuf s_a, s_b, s_c, s_d, s_e, s_f;
  HostBuf h_stage;
  // launch configuration
  int trace_grid[2] = {0, 0};  // [no smem, smem]
  int shade_grid = 0;
  int64_t default_batch = int64_t(1) << 22;
  int n_lanes = kLanes;
  bool octant_sort = false;
  // stats of the last pass
  lt_render_stats stats{};
  std::vector<cudaEvent_t> ev_pool;
  int ev_used = 0;
};

// ------------------------------------------------------------------ library

extern "C" int lt_abi_version(void) { return LT_ABI_VERSION; }

extern "C" const char *lt_last_error(void) { return g_last_error.c_str(); }

extern "C" int lt_device_count(int32_t *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return lt_fail(LT_ERR_CUDA, "cudaGetDeviceCount failed: %s", cudaGetErrorString(e));
  }
  *count = n;
  return LT_OK;
}

extern "C" int lt_build_bvh(const double *v0, const double *v1, const double *v2, int64_t n,
                            int32_t leaf_size, int32_t bins, double *bounds_min,
                            double *bounds_max, int32_t *left_child, int32_t *right_child,
                            int32_t *first_triangle, int32_t *triangle_count,
                            int32_t *triangle_order, int64_t *n_nodes, int64_t *leaf_count,
                            int64_t *max_depth) {
  if (!v0 || !v1 || !v2 || !bounds_min || !bounds_max || !left_child || !right_child ||
      !first_triangle || !triangle_count || !triangle_order || !n_nodes || !leaf_count ||
      !max_depth)
    return lt_fail(LT_ERR_INVALID, "lt_build_bvh: null pointer");
  return lt_build_bvh_impl(v0, v1, v2, n, leaf_size, bins, bounds_min, bounds_max, left_child,
                           right_child, first_triangle, triangle_count, triangle_order, n_nodes,
                           leaf_count, max_depth);
}

// ------------------------------------------------------------------ scene

// f(i) for i in [0, n) on up to 16 host threads.
template <class F>
static void parallel_for(int64_t n, F f) {
  if (n <= 0) return;
  const int64_t hw = std::max<int64_t>(1, (int64_t)std::thread::hardware_concurrency());
  const int64_t nt = std::min<int64_t>({n, hw, 16});
  if (nt <= 1 || n < 4) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int64_t> next{0};  // dynamic: subtree sizes vary widely
  std::vector<std::thread> th;
  th.reserve(nt);
  for (int64_t t = 0; t < nt; ++t)
    th.emplace_back([&] {
      for (int64_t i = next++; i < n; i = next++) f(i);
    });
  for (auto &x : th) x.join();
}

// materials + environment of a description (all creation paths)
static int validate_shading(const lt_scene_desc *d) {
  if (d->n_materials < 1 || !d->base_weight || !d->base_color || !d->base_metalness ||
      !d->specular_weight || !d->specular_color || !d->specular_roughness ||
      !d->specular_ior || !d->emission_luminance || !d->emission_color)
    return lt_fail(LT_ERR_INVALID, "material arrays must be non-null");
  if (d->env_kind < LT_ENV_UNIFORM || d->env_kind > LT_ENV_LATLONG)
    return lt_fail(LT_ERR_INVALID, "unknown environment kind %d", d->env_kind);
  if (d->env_kind == LT_ENV_LATLONG &&
      (!d->env_texels || d->env_width < 1 || d->env_height < 1))
    return lt_fail(LT_ERR_INVALID, "lat-long environment needs texels and a size");
  return LT_OK;
}

static int validate_desc(const lt_scene_desc *d) {
  if (!d) return lt_fail(LT_ERR_INVALID, "null scene description");
  if (d->n_triangles < 1) return lt_fail(LT_ERR_INVALID, "empty scene");
  if (d->n_triangles >= (int64_t(1) << 31) - 1)
    return lt_fail(LT_ERR_INVALID, "too many triangles (%lld)", (long long)d->n_triangles);
  if (!d->v0 || !d->v1 || !d->v2 || !d->n0 || !d->n1 || !d->n2 || !d->material_index)
    return lt_fail(LT_ERR_INVALID, "triangle arrays must be non-null");
  // n_nodes == 0 with no BVH arrays: the scene builds the reference's tree on
  // the device (lt_scene_desc in luxb200.h)
  const bool build_here = d->n_nodes == 0 && !d->bounds_min && !d->bounds_max &&
                          !d->left_child && !d->right_child && !d->first_triangle &&
                          !d->triangle_count && !d->triangle_order;
  if (!build_here && (d->n_nodes < 1 || !d->bounds_min || !d->bounds_max || !d->left_child ||
                      !d->right_child || !d->first_triangle || !d->triangle_count ||
                      !d->triangle_order))
    return lt_fail(LT_ERR_INVALID, "bvh arrays must be non-null");
  return validate_shading(d);
}

// The O(n) index checks of a description (material indices, triangle
// order, child / leaf ranges): scene creation runs them on host threads
// while the uploads' DMA is in flight, before any kernel reads an index.
static int validate_indices(const lt_scene_desc *d) {
  const bool build_here = d->n_nodes == 0;
  const int64_t n = d->n_triangles, nn = d->n_nodes;
  // chunked scans on host threads; the reported failure is the first index,
  // as a sequential scan would report it
  auto tri_bad = [&](int64_t i) {
    const int32_t m = d->material_index[i];
    if (m < 0 || m >= d->n_materials) return true;
    if (build_here) return false;
    const int32_t o = d->triangle_order[i];
    return o < 0 || o >= n;
  };
  auto node_bad = [&](int64_t i) {
    if (d->triangle_count[i] > 0) {
      const int64_t f = d->first_triangle[i], c = d->triangle_count[i];
      return f < 0 || f + c > n;
    }
    const int32_t l = d->left_child[i], r = d->right_child[i];
    return l <= i || r <= i || l >= nn || r >= nn;
  };
  auto first_bad = [&](int64_t count, auto bad) {
    // ~16 K items per chunk: tiny scenes scan inline (no thread start-up)
    const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(64, count >> 14));
    std::vector<int64_t> hit(chunks, -1);
    parallel_for(chunks, [&](int64_t c) {
      for (int64_t i = count * c / chunks; i < count * (c + 1) / chunks; ++i)
        if (bad(i)) {
          hit[c] = i;
          return;
        }
    });
    for (int64_t h : hit)
      if (h >= 0) return h;
    return (int64_t)-1;
  };
  const int64_t bt = first_bad(n, tri_bad);
  if (bt >= 0) {
    const int32_t m = d->material_index[bt];
    if (m < 0 || m >= d->n_materials)
      return lt_fail(LT_ERR_INVALID, "triangle %lld: material index %d out of range [0, %d)",
                     (long long)bt, m, d->n_materials);
    // (only reachable with a host BVH: build_here has no triangle_order)
    return lt_fail(LT_ERR_INVALID, "triangle_order[%lld] = %d out of range", (long long)bt,
                   d->triangle_order[bt]);
  }
  const int64_t bn = build_here ? -1 : first_bad(nn, node_bad);
  if (bn >= 0) {
    if (d->triangle_count[bn] > 0) {
      const int64_t f = d->first_triangle[bn], c = d->triangle_count[bn];
      return lt_fail(LT_ERR_INVALID, "node %lld: leaf range [%lld, %lld) out of bounds",
                     (long long)bn, (long long)f, (long long)(f + c));
    }
    return lt_fail(LT_ERR_INVALID, "node %lld: invalid children (%d, %d)", (long long)bn,
                   d->left_child[bn], d->right_child[bn]);
  }
  return LT_OK;
}

// float64 -> float32 rounded toward -inf / +inf (host side of the outward
// rounding the flatten kernel does with __double2float_rd/_ru)
static float f32_down(double x) {
  float f = (float)x;
  if ((double)f > x) f = std::nextafterf(f, -INFINITY);
  return f;
}
static float f32_up(double x) {
  float f = (float)x;
  if ((double)f < x) f = std::nextafterf(f, INFINITY);
  return f;
}

static double alpha_of(double r) {
  double a = r * r;
  return a < 1e-4 ? 1e-4 : a;
}
static double f0_from_ior(double ior) {
  double r = (ior - 1.0) / (ior + 1.0);
  return r * r;
}

static void build_material(const lt_scene_desc *d, int i, GpuMaterial &g) {
  std::memset(&g, 0, sizeof(g));
  const double bw = d->base_weight[i], m = d->base_metalness[i], sw = d->specular_weight[i];
  const double alpha = alpha_of(d->specular_roughness[i]);
  const double f0d = f0_from_ior(d->specular_ior[i]);
  const double avg = sw * (f0d + (1.0 - f0d) / 21.0);
  g.bw = (float)bw;
  for (int k = 0; k < 3; ++k) {
    g.bc[k] = (float)d->base_color[3 * i + k];
    g.sc[k] = (float)d->specular_color[3 * i + k];
    g.ec[k] = (float)d->emission_color[3 * i + k];
  }
  g.m = (float)m;
  g.sw = (float)sw;
  g.alpha = (float)alpha;
  g.a2 = (float)(alpha * alpha);
  g.f0d = (float)f0d;
  g.fdavg = (float)avg;
  g.diff = (float)(bw * (1.0 / 3.141592653589793) * (1.0 - avg));
  g.el = (float)d->emission_luminance[i];
  g.ior = (float)d->specular_ior[i];
  uint32_t flags = 0;
  if (m <= 0.0 && sw <= 0.0) flags |= MAT_DIFFUSE_ONLY;
  if (d->emission_luminance[i] > 0.0) flags |= MAT_EMISSIVE;
  const double cw = d->coat_weight ? d->coat_weight[i] : 0.0;
  if (cw > 0.0) {
    flags |= MAT_COAT;
    const double ca = alpha_of(d->coat_roughness ? d->coat_roughness[i] : 0.0);
    const double f0c = f0_from_ior(d->coat_ior ? d->coat_ior[i] : 1.5);
    g.cw = (float)cw;
    g.calpha = (float)ca;
    g.ca2 = (float)(ca * ca);
    g.f0c = (float)f0c;
  }
  for (int k = 0; k < 3; ++k) {
    g.cc[k] = d->coat_color ? (float)d->coat_color[3 * i + k] : 1.f;
    g.tc[k] = d->transmission_color ? (float)d->transmission_color[3 * i + k] : 1.f;
  }
  const double tw = d->transmission_weight ? d->transmission_weight[i] : 0.0;
  if (tw > 0.0 && m < 1.0) {
    flags |= MAT_GLASS;
    g.tw = (float)tw;
  }
  g.flags = flags;
}

template <class T>
static int upload(DevBuf &b, const T *src, size_t count, cudaStream_t st) {
  RET(b.ensure(std::max<size_t>(count * sizeof(T), 16)));
  if (count) CK(cudaMemcpyAsync(b.p, src, count * sizeof(T), cudaMemcpyHostToDevice, st));
  return LT_OK;
}
template <class T>
static int upload(TmpBuf &b, const T *src, size_t count, cudaStream_t st) {
  RET(b.alloc(count * sizeof(T), st));
  if (count) CK(cudaMemcpyAsync(b.p, src, count * sizeof(T), cudaMemcpyHostToDevice, st));
  return LT_OK;
}

static void destroy_scene(lt_scene *s) {
  if (!s) return;
  DeviceGuard g(s->device);
  PhaseTimer pt;
  // every render pass records the workspace event on its stream when it
  // ends: frees on the scene stream wait for it (no use-after-free when the
  // caller destroys a scene while its last pass is still in flight)
  if (s->stream && s->ws) {
    std::lock_guard<std::mutex> lk(s->ws->mu);
    if (s->ws->last_use) cudaStreamWaitEvent(s->stream, s->ws->last_use, 0);
  }
  pt.mark("destroy: order after last pass");
  if (s->stream && s->ws) {
    park_cached(*s->ws, s->geo, s->stream);
    park_cached(*s->ws, s->nodes2, s->stream);
  }
  for (DevBuf *b : {&s->geo, &s->nodes2, &s->shade, &s->mats, &s->env, &s->ray_ctr,
                    &s->pix_list, &s->s_a, &s->s_b, &s->s_c, &s->s_d, &s->s_e, &s->s_f})
    b->release();
  pt.mark("destroy: device frees");
  s->h_stage.release();
  for (cudaEvent_t e : s->ev_pool) cudaEventDestroy(e);
  if (s->stream) {
    if (s->ws) {
      std::lock_guard<std::mutex> lk(s->ws->stream_mu);
      s->ws->free_streams.push_back(s->stream);
    } else {
      cudaStreamDestroy(s->stream);
    }
  }
  pt.mark("destroy: host + stream");
  delete s;
}

// Launch geometry that depends only on the device (occupancy of the trace /
// shade kernels, the default batch from the free memory seen by the first
// scene), computed once per device: the occupancy and memory queries cost up
// to ~16 ms per scene otherwise.
struct LaunchCache {
  bool ok = false;
  int trace_grid = 0, shade_grid = 0;
  int64_t default_batch = 0;
};

static int configure_launches(lt_scene *s) {
  static std::mutex mu;
  static std::map<int, LaunchCache> cache;
  LaunchCache lc;
  {
    std::lock_guard<std::mutex> lk(mu);
    lc = cache[s->device];
  }
  if (!lc.ok) {
    const size_t smem = trace_smem_bytes();
    for (bool c : {false, true})
      CK(cudaFuncSetAttribute(trace_kernel_ptr(c), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
    int blocks = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, trace_kernel_ptr(false),
                                                     kTraceThreads, smem));
    lc.trace_grid = std::max(1, blocks) * s->sm_count;
    size_t free_b = 0, total_b = 0;
    lc.default_batch = kMaxBatchPaths;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      const int64_t by_mem = (int64_t)(free_b / 4 / 128);
      lc.default_batch = std::max<int64_t>(int64_t(1) << 20, std::min(kMaxBatchPaths, by_mem));
    }
    blocks = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, shade_kernel_ptr(), kShadeThreads,
                                                     0));
    lc.shade_grid = std::max(1, blocks) * s->sm_count;
    lc.ok = true;
    std::lock_guard<std::mutex> lk(mu);
    cache[s->device] = lc;
  }
  s->trace_grid[0] = lc.trace_grid;
  s->shade_grid = lc.shade_grid;
  s->default_batch = lc.default_batch;
  // L2 residency of the traversal set (nodes + leaf-ordered triangles)
  const char *pe = std::getenv("LT_L2_PERSIST");
  int max_persist = 0, max_window = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, s->device);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, s->device);
  // Off by default: the persisting carve-out did not speed up k_trace (the
  // traversal set stays L2-hot anyway) and starved the streaming kernels of
  // L2 (2071 vs 1789 M samples/s on C4, profiles/r01_l2_window_sweep.jsonl).
  s->use_window = (pe && pe[0] == '1') && max_persist > 0 && max_window > 0;
  if (s->use_window) {
    // geo = [wide nodes | triangles | shading]; trace launches keep
    // [nodes, triangles] persisting, shade launches [triangles, shading]
    const size_t tri_bytes = 16 * LT_TRI_F4 * (size_t)s->n_tris;
    const size_t trace_bytes = s->nodes_bytes + tri_bytes;
    const size_t shade_bytes = s->geo_bytes - s->nodes_bytes;
    const char *se = std::getenv("LT_L2_SHADE");
    s->use_shade_window = se && se[0] == '1';
    const size_t limit = std::min<size_t>(
        (size_t)max_persist, s->use_shade_window ? std::max(trace_bytes, shade_bytes) : trace_bytes);
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur < limit) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, limit));
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    s->persist_bytes = cur;
    auto make = [&](void *base, size_t bytes) {
      cudaAccessPolicyWindow w{};
      const size_t win = std::min<size_t>((size_t)max_window, bytes);
      w.base_ptr = base;
      w.num_bytes = win;
      w.hitRatio = win > 0 ? (float)std::min(1.0, (double)cur / (double)win) : 0.f;
      w.hitProp = cudaAccessPropertyPersisting;
      w.missProp = cudaAccessPropertyStreaming;
      return w;
    };
    s->window = make(s->geo.p, trace_bytes);
    s->shade_window = make(static_cast<char *>(s->geo.p) + s->nodes_bytes, shade_bytes);
  }
  return LT_OK;
}

// Layout of a device-built BVH without a host round trip: the internal
// binary nodes in index order (prefix sum) for the counter query, and the
// 4-wide collapse (greedy largest-area expansion) in one single-CTA launch,
// wide nodes numbered breadth first.
static int device_layout(lt_scene *s, const double *bmin, const double *bmax,
                         const int32_t *left, const int32_t *right, const int32_t *count,
                         int64_t nn, bool root_leaf, TmpBuf &t_perm, TmpBuf &t_new,
                         TmpBuf &t_wch, TmpBuf &t_wof) {
  cudaStream_t st = s->stream;
  TmpBuf flags, scan, tmp;
  RET(flags.alloc((size_t)(nn + 1) * 4, st));
  RET(scan.alloc((size_t)(nn + 1) * 4, st));
  CK(cudaMemsetAsync(flags.p, 0, (size_t)(nn + 1) * 4, st));
  launch_internal_flags(count, nn, flags.as<int32_t>(), st);
  size_t tmp_bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flags.as<int32_t>(), scan.as<int32_t>(),
                                   (int)(nn + 1), st));
  RET(tmp.alloc(std::max<size_t>(tmp_bytes, 16), st));
  CK(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, flags.as<int32_t>(), scan.as<int32_t>(),
                                   (int)(nn + 1), st));
  RET(t_perm.alloc((size_t)std::max<int64_t>(nn, 1) * 4, st));
  RET(t_new.alloc((size_t)std::max<int64_t>(nn, 1) * 4, st));
  launch_internal_scatter(flags.as<int32_t>(), scan.as<int32_t>(), nn, t_perm.as<int32_t>(),
                          t_new.as<int32_t>(), st);
  int32_t n_internal = 0;
  CK(cudaMemcpyAsync(&n_internal, scan.as<int32_t>() + nn, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  s->n_internal = n_internal;
  s->n_bfs = 0;
  s->n_wide = 0;
  RET(t_wch.alloc((size_t)std::max<int64_t>(n_internal, 1) * 16, st));
  RET(t_wof.alloc((size_t)std::max<int64_t>(nn, 1) * 4, st));
  if (root_leaf || n_internal == 0) return LT_OK;
  // breadth-first 4-wide collapse in one single-CTA launch; it also reports
  // the deepest traversal stack the tree can need
  TmpBuf fifo, nw;
  RET(fifo.alloc((size_t)n_internal * 12, st));
  RET(nw.alloc(16, st));
  int32_t res[3] = {n_internal, 0, 0};
  CK(cudaMemcpyAsync(nw.p, res, 4, cudaMemcpyHostToDevice, st));
  launch_collapse_all(bmin, bmax, left, right, count, fifo.as<int32_t>(), t_wch.as<int32_t>(),
                      t_wof.as<int32_t>(), nw.as<int32_t>(), st);
  CK(cudaMemcpyAsync(res, nw.p, 12, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  s->n_wide = res[0];
  if (res[1] >= LT_STACK || res[2] >= LT_STACK)
    return lt_fail(LT_ERR_UNSUPPORTED,
                   "BVH too deep for the traversal stack: the 4-wide tree can hold %d pending "
                   "entries and the binary tree is %d levels deep (limit %d)",
                   res[1], res[2], LT_STACK);
  return LT_OK;
}

// gltf != NULL: the triangle arrays come from lt_ingest_run on the scene's
// stream (the description's triangle / BVH fields are unused), the BVH is
// built on the device
static int scene_create_impl(const lt_scene_desc *d, int32_t device, lt_scene *s,
                             const lt_gltf_desc *gltf = nullptr, int64_t *n_kept = nullptr,
                             int64_t *n_dropped = nullptr) {
  PhaseTimer pt;
  s->device = device;
  CK(cudaSetDevice(device));
  CK(cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, device));
  s->ws = workspace_for(device);
  {
    std::lock_guard<std::mutex> lk(s->ws->stream_mu);
    if (!s->ws->free_streams.empty()) {
      s->stream = s->ws->free_streams.back();
      s->ws->free_streams.pop_back();
    }
  }
  if (!s->stream) CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  {
    const char *ls = std::getenv("LT_LANES");
    s->n_lanes = std::max(1, std::min(kLanes, ls ? std::atoi(ls) : kDefaultLanes));
  }
  {
    // keep stream-ordered scene / staging memory mapped between scenes (once
    // per device)
    std::lock_guard<std::mutex> lk(s->ws->stream_mu);
    cudaMemPool_t pool;
    if (!s->ws->pool_configured && cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;  // never trim: the pool peaks at the scene + staging + build scratch
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      s->ws->pool_configured = true;
    }
  }
  for (DevBuf *b : {&s->geo, &s->nodes2, &s->shade, &s->mats, &s->env, &s->ray_ctr,
                    &s->pix_list, &s->s_a, &s->s_b, &s->s_c, &s->s_d, &s->s_e, &s->s_f}) {
    b->stream_ordered = true;
    b->ast = s->stream;
  }
  cudaStream_t st = s->stream;
  int64_t n = d->n_triangles;
  // no host BVH (n_nodes == 0): build the reference's tree (leaf size 4, 12
  // bins, build_bvh's defaults) on the device from the uploaded vertices and
  // lay it out without a host round trip
  const bool build_here = gltf || d->n_nodes == 0;
  int64_t nn = gltf ? 0 : d->n_nodes;
  pt.mark("stream + attributes");

  // --- uploads.  Small scenes: every array through one pinned staging
  // buffer and ONE copy.  Otherwise the arrays land in the workspace's
  // device scratch (serialized by create_mu): page-locked sources by direct
  // DMA, pageable ones through the pinned ring (staged_h2d); the BVH arrays
  // first, then the triangle arrays on a host thread + the side stream
  // while the device lays the tree out.
  TmpBuf t_v[6], t_mat, t_order, t_end, t_bmin, t_bmax, t_left, t_right, t_first, t_count,
      t_perm, t_new, t_wch, t_wof, t_env;
  const double *src[6] = {d->v0, d->v1, d->v2, d->n0, d->n1, d->n2};
  struct TreeGuard {
    lt_gpu_tree t{};
    ~TreeGuard() { lt_gpu_tree_free(&t); }
  } tree;
  const double *g_bmin, *g_bmax;
  const int32_t *g_left, *g_right, *g_first, *g_count, *g_order;
  bool root_leaf;
  int32_t root_first;
  double root_lo[3], root_hi[3];
  const size_t kSmallUpload = size_t(4) << 20;
  TmpBuf t_all, t_raw;
  Workspace &W = *s->ws;
  std::unique_lock<std::mutex> create_lk(W.create_mu);
  // --- glTF ingest: the buffers' raw bytes up (through the pinned ring),
  // flatten_scene on the device; its output stands in for the uploads below
  struct IngestGuard {
    lt_ingest_out o{};
    cudaStream_t st;
    ~IngestGuard() { lt_ingest_free(&o, st); }  // stream-ordered, after the flatten reads it
  } ing{{}, st};
  if (gltf) {
    std::vector<int64_t> at(std::max<int32_t>(1, gltf->n_buffers));
    size_t raw_total = 0;
    for (int32_t b = 0; b < gltf->n_buffers; ++b) {
      at[b] = (int64_t)raw_total;
      raw_total += ((size_t)gltf->buffer_bytes[b] + 255) / 256 * 256;
    }
    RET(t_raw.alloc(raw_total, st));
    std::vector<CopyItem> raw_items;
    for (int32_t b = 0; b < gltf->n_buffers; ++b)
      if (gltf->buffer_bytes[b] > 0)
        raw_items.push_back(CopyItem{t_raw.as<char>() + at[b], gltf->buffers[b],
                                     (size_t)gltf->buffer_bytes[b]});
    RET(ensure_ring(W));
    RET(staged_h2d(W, device, raw_items, st));
    pt.mark("glTF buffers staged");
    RET(lt_ingest_run(gltf, t_raw.as<uint8_t>(), at.data(), st, &ing.o));
    pt.mark("device flatten_scene");
    n = ing.o.n_kept;
    if (n_kept) *n_kept = ing.o.n_kept;
    if (n_dropped) *n_dropped = ing.o.n_dropped;
    for (int k = 0; k < 6; ++k) t_v[k].set_view(ing.o.v[k]);
    t_mat.set_view(ing.o.mat);
  }
  s->n_tris = n;
  struct Item {
    TmpBuf *dst;
    const void *src;
    size_t bytes;
    bool tri;  // a triangle array (uploaded after the BVH arrays)
  };
  std::vector<Item> items;
  if (!gltf) {
    for (int k = 0; k < 6; ++k) items.push_back({&t_v[k], src[k], 24 * (size_t)n, true});
    items.push_back({&t_mat, d->material_index, 4 * (size_t)n, true});
  }
  // the lat-long texels travel with the triangle arrays (on the side stream
  // when there is one), not after the layout
  const int64_t env_np = d->env_kind == LT_ENV_LATLONG ? (int64_t)d->env_width * d->env_height : 0;
  if (env_np) items.push_back({&t_env, d->env_texels, sizeof(float) * 3 * (size_t)env_np, true});
  if (!build_here) {
    items.push_back({&t_order, d->triangle_order, 4 * (size_t)n, false});
    items.push_back({&t_bmin, d->bounds_min, 24 * (size_t)nn, false});
    items.push_back({&t_bmax, d->bounds_max, 24 * (size_t)nn, false});
    items.push_back({&t_left, d->left_child, 4 * (size_t)nn, false});
    items.push_back({&t_right, d->right_child, 4 * (size_t)nn, false});
    items.push_back({&t_first, d->first_triangle, 4 * (size_t)nn, false});
    items.push_back({&t_count, d->triangle_count, 4 * (size_t)nn, false});
  }
  std::vector<size_t> off(items.size());
  size_t total = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    off[i] = total;
    total += (items[i].bytes + 255) / 256 * 256;
  }
  const bool small_upload = total <= kSmallUpload;
  char *base = nullptr;
  if (total == 0) {
    // (glTF ingest: nothing to upload)
  } else if (small_upload) {
    RET(t_all.alloc(total, st));
    std::lock_guard<std::mutex> lk(W.upload_mu);
    if (W.stage_ev)
      CK(cudaEventSynchronize(W.stage_ev));  // the previous small scene's copy
    else
      CK(cudaEventCreateWithFlags(&W.stage_ev, cudaEventDisableTiming));
    RET(W.stage.ensure(kSmallUpload));
    for (size_t i = 0; i < items.size(); ++i)
      std::memcpy(static_cast<char *>(W.stage.p) + off[i], items[i].src, items[i].bytes);
    CK(cudaMemcpyAsync(t_all.p, W.stage.p, total, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(W.stage_ev, st));
    base = static_cast<char *>(t_all.p);
  } else {
    // the scratch is reused by every creation on the device: order this
    // one's copies after the previous creation's last read of it (growth is
    // a plain, rare allocation)
    if (W.scratch_ev) CK(cudaEventSynchronize(W.scratch_ev));
    else CK(cudaEventCreateWithFlags(&W.scratch_ev, cudaEventDisableTiming));
    RET(W.scratch.ensure(total));
    base = W.scratch.as<char>();
  }
  struct ScratchGuard {
    Workspace &W;
    cudaStream_t st;
    bool on;
    ~ScratchGuard() {
      if (!on) return;
      if (W.upload_st) {  // side-stream copies (joined before this runs)
        cudaEventRecord(W.scratch_ev, W.upload_st);
        cudaStreamWaitEvent(st, W.scratch_ev, 0);
      }
      cudaEventRecord(W.scratch_ev, st);
    }
  } scratch_guard{W, st, !small_upload};
  for (size_t i = 0; i < items.size(); ++i) items[i].dst->set_view(base + off[i]);
  auto copies = [&](bool tri) {
    std::vector<CopyItem> c;
    for (const Item &it : items)
      if (it.tri == tri) c.push_back(CopyItem{it.dst->p, it.src, it.bytes});
    return c;
  };
  // triangle arrays in flight on a host thread (large host-BVH scenes);
  // every exit path joins it before its captures go out of scope
  cudaEvent_t tri_done = nullptr;
  struct EventGuard {
    cudaEvent_t &e;
    ~EventGuard() {
      if (e) cudaEventDestroy(e);  // released once the recorded work completes
    }
  } tri_done_guard{tri_done};
  int tri_rc = LT_OK;
  std::string tri_msg;
  std::thread tri_thread;
  struct JoinGuard {
    std::thread &t;
    ~JoinGuard() {
      if (t.joinable()) t.join();
    }
  } tri_join_guard{tri_thread};
  auto join_triangles = [&]() -> int {
    if (tri_thread.joinable()) tri_thread.join();
    if (tri_rc != LT_OK) {
      g_last_error = tri_msg;
      return tri_rc;
    }
    return LT_OK;
  };
  if (build_here) {
    if (!small_upload) {
      RET(ensure_ring(W));
      RET(staged_h2d(W, device, copies(true), st));  // the build reads vertices
    }
    RET(lt_gpu_tree_build(t_v[0].as<double>(), t_v[1].as<double>(), t_v[2].as<double>(), n, 4,
                          12, st, &tree.t));
    nn = tree.t.n_nodes;
    g_bmin = tree.t.bmin;
    g_bmax = tree.t.bmax;
    g_left = tree.t.left;
    g_right = tree.t.right;
    g_first = tree.t.first;
    g_count = tree.t.count;
    g_order = tree.t.order;
    int32_t rc0[2];
    CK(cudaMemcpyAsync(&rc0[0], g_count, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&rc0[1], g_first, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(root_lo, g_bmin, 24, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(root_hi, g_bmax, 24, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    root_leaf = rc0[0] > 0;
    root_first = rc0[1];
    pt.mark("device BVH build");
  } else {
    if (!small_upload) {
      // two concurrent staging jobs on disjoint halves of the ring: the
      // triangle arrays (the bulk) on the side stream from a host thread,
      // the BVH arrays on the scene stream from this one (the device
      // layout needs them first)
      {
        std::lock_guard<std::mutex> lk(W.upload_mu);
        if (!W.upload_st) CK(cudaStreamCreateWithFlags(&W.upload_st, cudaStreamNonBlocking));
      }
      RET(ensure_ring(W));
      CK(cudaEventCreateWithFlags(&tri_done, cudaEventDisableTiming));
      tri_thread = std::thread([&, tri_items = copies(true)]() {
        tri_rc = staged_h2d(W, device, tri_items, W.upload_st, kBvhWorkers,
                            kRingWorkers - kBvhWorkers);
        if (tri_rc == LT_OK) {
          const cudaError_t e = cudaEventRecord(tri_done, W.upload_st);
          if (e != cudaSuccess)
            tri_rc = lt_fail(LT_ERR_CUDA, "cudaEventRecord failed: %s", cudaGetErrorString(e));
        }
        if (tri_rc != LT_OK) tri_msg = g_last_error;
      });
      RET(staged_h2d(W, device, copies(false), st, 0, kBvhWorkers));
      pt.mark("BVH arrays staged");
    }
    g_bmin = t_bmin.as<double>();
    g_bmax = t_bmax.as<double>();
    g_left = t_left.as<int32_t>();
    g_right = t_right.as<int32_t>();
    g_first = t_first.as<int32_t>();
    g_count = t_count.as<int32_t>();
    g_order = t_order.as<int32_t>();
    root_leaf = d->triangle_count[0] > 0;
    root_first = d->first_triangle[0];
    for (int a = 0; a < 3; ++a) {
      root_lo[a] = d->bounds_min[a];
      root_hi[a] = d->bounds_max[a];
    }
  }
  // index checks on host threads while the DMA runs; nothing on the device
  // has read an index yet (the device build reads only vertices)
  if (int rc = gltf ? LT_OK : validate_indices(d)) {
    join_triangles();
    cudaStreamSynchronize(st);
    if (W.upload_st) cudaStreamSynchronize(W.upload_st);
    return rc;
  }
  pt.mark("validate indices (overlaps DMA)");
  s->n_nodes = nn;
  // leaf-end flags of the leaf-ordered triangle stream, on the device
  RET(t_end.alloc(std::max<int64_t>(n, 16), st));
  CK(cudaMemsetAsync(t_end.p, 0, (size_t)n, st));
  launch_leaf_end(g_first, g_count, nn, t_end.as<uint8_t>(), st);
  pt.mark("uploads enqueue");

  // --- layout on the device for both paths: the internal binary nodes in
  // index order (prefix sum) for the counter query, and the 4-wide collapse
  // (greedy largest-area expansion, one single-CTA launch; the host-side
  // version took ~4.6 ms of host time at 1 M triangles, the level-by-level
  // launches ~2 ms of per-level synchronizations)
  {
    const int rc = device_layout(s, g_bmin, g_bmax, g_left, g_right, g_count, nn, root_leaf,
                                 t_perm, t_new, t_wch, t_wof);
    if (rc != LT_OK) {
      join_triangles();
      if (W.upload_st) cudaStreamSynchronize(W.upload_st);
      return rc;
    }
  }
  pt.mark("device layout");
  RET(join_triangles());
  if (tri_done) CK(cudaStreamWaitEvent(st, tri_done, 0));  // the triangle uploads
  pt.mark("triangle arrays staged");
  // --- flatten on the device
  int rc = LT_OK;
  do {
    s->nodes_bytes = (size_t)std::max<int64_t>(1, s->n_wide) * 16 * LT_NODE_F4;
    // shading records start on a 128 B boundary so each 64 B record is
    // half of one cache line
    s->shade_off = (s->nodes_bytes + 16 * LT_TRI_F4 * (size_t)n + 127) / 128 * 128;
    s->geo_bytes = s->shade_off + 64 * (size_t)n;
    if ((rc = take_cached(W, s->geo, s->geo_bytes, st))) break;
    pt.mark("geo alloc");
    if ((rc = take_cached(W, s->nodes2, (size_t)std::max<int64_t>(1, s->n_internal) * 64, st)))
      break;
    pt.mark("nodes2 alloc");
    float4 *g_wide = s->geo.as<float4>();
    float4 *g_tris = g_wide + s->nodes_bytes / 16;
    float4 *g_shade = g_wide + s->shade_off / 16;
    float4 *g_nodes = s->nodes2.as<float4>();
    launch_flatten_tris(t_v[0].as<double>(), t_v[1].as<double>(), t_v[2].as<double>(),
                        t_v[3].as<double>(), t_v[4].as<double>(), t_v[5].as<double>(),
                        t_mat.as<int32_t>(), g_order, t_end.as<uint8_t>(), n, g_tris, g_shade,
                        st);
    if (s->n_internal > 0) {
      launch_flatten_nodes(g_bmin, g_bmax, g_left, g_right, g_first, g_count,
                           t_perm.as<int32_t>(), t_new.as<int32_t>(), s->n_internal, g_nodes,
                           st);
      launch_flatten_wide(g_bmin, g_bmax, g_first, g_count, t_wch.as<int32_t>(),
                          t_wof.as<int32_t>(), s->n_wide, g_wide, st);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      rc = lt_fail(LT_ERR_CUDA, "flatten launch failed: %s", cudaGetErrorString(e));
      break;
    }
    pt.mark("uploads + flatten enqueue");
    // materials
    std::vector<GpuMaterial> mats(d->n_materials);
    for (int i = 0; i < d->n_materials; ++i) build_material(d, i, mats[i]);
    if ((rc = upload(s->mats, mats.data(), mats.size(), st))) break;
    // environment
    if (env_np) {
      // float3 texels as given (uploaded with the triangle arrays), widened
      // to float4 records on the device
      if ((rc = s->env.ensure((size_t)env_np * 16))) break;
      launch_expand_rgb(t_env.as<float>(), env_np, s->env.as<float4>(), st);
    }
    pt.mark("materials + env");
    e = cudaStreamSynchronize(st);
    pt.mark("device flatten (sync)");
    if (e != cudaSuccess) {
      rc = lt_fail(LT_ERR_CUDA, "scene upload failed: %s", cudaGetErrorString(e));
      break;
    }
  } while (0);
  RET(rc);  // the TmpBuf staging is released stream-ordered when it leaves scope

  SceneView &v = s->view;
  v.wnodes = s->geo.as<float4>();
  v.wroot_link = root_leaf ? ~root_first : 0;
  v.nodes = s->nodes2.as<float4>();
  v.tris = s->geo.as<float4>() + s->nodes_bytes / 16;
  v.shade = s->geo.as<float4>() + s->shade_off / 16;
  v.mats = s->mats.as<GpuMaterial>();
  v.env_map = s->env.as<float4>();
  v.root_link = root_leaf ? ~root_first : 0;
  for (int a = 0; a < 3; ++a) {
    v.root_lo[a] = f32_down(root_lo[a]);
    v.root_hi[a] = f32_up(root_hi[a]);
  }
  v.n_wide = (int32_t)s->n_wide;
  v.n_tris = (int32_t)n;
  v.n_mats = d->n_materials;
  v.env_kind = d->env_kind;
  v.env_w = d->env_width;
  v.env_h = d->env_height;
  v.env_scale = (float)(d->env_kind == LT_ENV_LATLONG ? d->env_scale : 1.0);
  for (int k = 0; k < 3; ++k) {
    v.env_a[k] = (float)d->env_a[k];
    v.env_b[k] = (float)d->env_b[k];
  }
  s->device_bytes = (int64_t)(s->geo.bytes + s->nodes2.bytes + s->shade.bytes + s->mats.bytes +
                              s->env.bytes);
  pt.mark("free temporaries + view");
  RET(configure_launches(s));
  pt.mark("configure launches");
  // continuation rays appended grouped by direction octant (+3 % on C4,
  // profiles/r01_octant_sweep.jsonl); LT_OCTANT_SORT=0 disables
  const char *os_env = std::getenv("LT_OCTANT_SORT");
  s->octant_sort = os_env ? os_env[0] == '1' : true;
  const char *rf = std::getenv("LT_REFILL");
  v.refill_min = std::max(1, std::min(32, rf ? std::atoi(rf) : 16));
  const char *lm = std::getenv("LT_LEAF_MIN");
  v.leaf_min = std::max(1, std::min(33, lm ? std::atoi(lm) : 8));
  return LT_OK;
}

extern "C" int lt_scene_create(const lt_scene_desc *desc, int32_t device, lt_scene **out) {
  if (!out) return lt_fail(LT_ERR_INVALID, "null output handle");
  *out = nullptr;
  {
    PhaseTimer pv;
    RET(validate_desc(desc));
    pv.mark("validate");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return lt_fail(LT_ERR_CUDA, "no CUDA device available");
  if (device < 0 || device >= ndev)
    return lt_fail(LT_ERR_INVALID, "device %d out of range [0, %d)", device, ndev);
  DeviceGuard g(device);
  lt_scene *s = new lt_scene();
  int rc = scene_create_impl(desc, device, s);
  if (rc != LT_OK) {
    std::string msg = g_last_error;
    destroy_scene(s);
    g_last_error = msg;
    return rc;
  }
  *out = s;
  return LT_OK;
}

static int check_device(int32_t device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return lt_fail(LT_ERR_CUDA, "no CUDA device available");
  if (device < 0 || device >= ndev)
    return lt_fail(LT_ERR_INVALID, "device %d out of range [0, %d)", device, ndev);
  return LT_OK;
}

extern "C" int lt_scene_create_gltf(const lt_gltf_desc *gltf, const lt_scene_desc *desc,
                                    int32_t device, lt_scene **out, int64_t *n_kept,
                                    int64_t *n_dropped) {
  if (!out) return lt_fail(LT_ERR_INVALID, "null output handle");
  *out = nullptr;
  if (!desc) return lt_fail(LT_ERR_INVALID, "null scene description");
  if (desc->n_triangles != 0 || desc->n_nodes != 0 || desc->v0 || desc->material_index ||
      desc->bounds_min || desc->triangle_order)
    return lt_fail(LT_ERR_INVALID, "lt_scene_create_gltf: triangle and BVH fields must be empty");
  RET(validate_shading(desc));
  int64_t n_tris = 0;
  RET(lt_ingest_check(gltf, desc->n_materials, &n_tris));
  if (n_tris == 0) return lt_fail(LT_ERR_INVALID, "empty scene");
  RET(check_device(device));
  DeviceGuard g(device);
  lt_scene *s = new lt_scene();
  int rc = scene_create_impl(desc, device, s, gltf, n_kept, n_dropped);
  if (rc != LT_OK) {
    std::string msg = g_last_error;
    destroy_scene(s);
    g_last_error = msg;
    return rc;
  }
  *out = s;
  return LT_OK;
}

extern "C" int lt_gltf_flatten(const lt_gltf_desc *gltf, int32_t device, int64_t cap, double *v0,
                               double *v1, double *v2, double *n0, double *n1, double *n2,
                               int32_t *material_index, int64_t *n_kept, int64_t *n_dropped) {
  int64_t n_tris = 0;
  RET(lt_ingest_check(gltf, 0, &n_tris));
  if (n_tris == 0) return lt_fail(LT_ERR_INVALID, "empty scene");
  if (cap < n_tris) return lt_fail(LT_ERR_INVALID, "capacity %lld < %lld triangles",
                                   (long long)cap, (long long)n_tris);
  if (!v0 || !v1 || !v2 || !n0 || !n1 || !n2 || !material_index || !n_kept || !n_dropped)
    return lt_fail(LT_ERR_INVALID, "output arrays must be non-null");
  RET(check_device(device));
  DeviceGuard g(device);
  // one upload, kernels and download on the query stream, serialized by its
  // scratch (lt_staged.h) for the raw bytes
  lt_staged::Staged S;
  std::vector<int> ids(std::max<int32_t>(1, gltf->n_buffers));
  for (int32_t b = 0; b < gltf->n_buffers; ++b)
    ids[b] = S.add(gltf->buffers[b], nullptr, (size_t)gltf->buffer_bytes[b]);
  RET(S.begin());
  std::vector<int64_t> at(ids.size(), 0);
  const char *base = S.dev<char>(0);
  for (int32_t b = 0; b < gltf->n_buffers; ++b) at[b] = S.dev<char>(ids[b]) - base;
  struct Guard {
    lt_ingest_out o{};
    cudaStream_t st;
    ~Guard() { lt_ingest_free(&o, st); }
  } ing{{}, S.stream()};
  RET(lt_ingest_run(gltf, reinterpret_cast<const uint8_t *>(base), at.data(), S.stream(), &ing.o));
  const int64_t k = ing.o.n_kept;
  double *dst[6] = {v0, v1, v2, n0, n1, n2};
  for (int a = 0; a < 6; ++a)
    CK(cudaMemcpyAsync(dst[a], ing.o.v[a], 24 * (size_t)k, cudaMemcpyDeviceToHost, S.stream()));
  CK(cudaMemcpyAsync(material_index, ing.o.mat, 4 * (size_t)k, cudaMemcpyDeviceToHost,
                     S.stream()));
  CK(cudaStreamSynchronize(S.stream()));
  *n_kept = k;
  *n_dropped = ing.o.n_dropped;
  return LT_OK;
}

extern "C" int lt_scene_destroy(lt_scene *scene) {
  destroy_scene(scene);
  return LT_OK;
}

extern "C" int lt_scene_info_get(const lt_scene *s, lt_scene_info *info) {
  if (!s || !info) return lt_fail(LT_ERR_INVALID, "null argument");
  info->device = s->device;
  info->n_triangles = s->n_tris;
  info->n_nodes = s->n_nodes;
  info->n_internal = s->n_internal;
  info->device_bytes = s->device_bytes;
  info->sm_count = s->sm_count;
  info->n_wide = s->n_wide;
  info->l2_persist_bytes = s->use_window ? (int64_t)s->persist_bytes : 0;
  info->l2_window_bytes = s->use_window ? (int64_t)s->window.num_bytes : 0;
  info->default_batch_paths = s->default_batch;
  return LT_OK;
}

// ------------------------------------------------------------------ workspace

static int ensure_lane(lt_scene *s, Lane &ln, int64_t cap, int32_t max_depth) {
  if (cap > ln.cap) {
    for (int k = 0; k < 2; ++k) {
      RET(ln.q_o[k].ensure(16 * cap));
      RET(ln.q_d[k].ensure(16 * cap));
    }
    RET(ln.hits.ensure(16 * cap));
    RET(ln.S.ensure(32 * cap));
    RET(ln.cls.ensure(cap));
    RET(ln.perm.ensure(4 * cap));
    RET(ln.cls_ctr.ensure(sizeof(int32_t) * 2 * kShadeClasses));
    ln.cap = cap;
  }
  if (max_depth > ln.depth_cap) {
    RET(ln.counters.ensure(sizeof(int32_t) * (2 * (size_t)max_depth + 2)));
    ln.depth_cap = max_depth;
  }
  RET(s->ray_ctr.ensure(6 * sizeof(unsigned long long)));
  return LT_OK;
}

static PathArrays path_arrays(Lane &ln, bool explicit_inc = false) {
  return PathArrays{ln.S.as<float4>(), explicit_inc ? ln.inc.as<uint64_t>() : nullptr};
}

static int record_event(lt_scene *s, cudaStream_t st) {
  if (s->ev_used == (int)s->ev_pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    s->ev_pool.push_back(e);
  }
  CK(cudaEventRecord(s->ev_pool[s->ev_used++], st));
  return LT_OK;
}

// The bounce loop of _trace (integrator.py:160-226) over the whole queue:
// trace -> shade per segment.  With `primary` the depth-0 launches generate
// the camera rays themselves (render batches); otherwise queue 0 must hold
// the primary rays and counters[0] their number (explicit rays).
static int run_bounces(lt_scene *s, Lane &lane, int32_t max_depth, int32_t rr_start, float t_min,
                       uint32_t flags, cudaStream_t st, const RaygenArgs *primary,
                       int64_t max_rays, bool explicit_paths = false) {
  SceneView sc = s->view;
  // a batch never holds more than max_rays rays: small batches (tiny frames)
  // launch only the CTAs that can find work
  const int trace_grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(s->trace_grid[0],
                                                  (max_rays + kTraceThreads - 1) / kTraceThreads));
  const int shade_grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(s->shade_grid,
                                                  (max_rays + kShadeThreads - 1) / kShadeThreads));
  Lane *ws = &lane;
  int32_t *ctr = ws->counters.as<int32_t>();
  int32_t *fetch = ctr + max_depth + 1;
  const PathArrays pa = path_arrays(lane, explicit_paths);
  int cur = 0;
  for (int32_t depth = 0; depth < max_depth; ++depth) {
    if (flags & LT_FLAG_PROFILE) RET(record_event(s, st));
    // (in-kernel ray generation for trace measured slower than reading the
    // 32 B ray record: the float64 camera math serializes the refill path)
    // a render batch's primary rays carry no origin record (the camera)
    const bool prim_rays = depth == 0 && primary;
    const float4 cam_o = primary ? make_float4((float)primary->cam[0], (float)primary->cam[1],
                                               (float)primary->cam[2], 0.f)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    CK(launch_trace(sc, (flags & LT_FLAG_COUNT) != 0, trace_grid,
                    s->use_window ? &s->window : nullptr,
                    prim_rays ? nullptr : ws->q_o[cur].as<float4>(), ws->q_d[cur].as<float4>(),
                    ctr + depth, fetch + depth, ws->hits.as<float4>(),
                    s->ray_ctr.as<unsigned long long>(), cam_o, st));
    if (flags & LT_FLAG_PROFILE) RET(record_event(s, st));
    const int32_t *perm = nullptr;
    if (flags & LT_FLAG_SORT_MATERIALS) {
      CK(cudaMemsetAsync(ws->cls_ctr.p, 0, sizeof(int32_t) * 2 * kShadeClasses, st));
      launch_material_sort(sc, ws->hits.as<float4>(), ctr + depth, depth != max_depth - 1,
                           shade_grid, ws->cls.as<uint8_t>(), ws->cls_ctr.as<int32_t>(),
                           ws->perm.as<int32_t>(), st);
      perm = ws->perm.as<int32_t>();
      s->stats.kernel_launches += 2;
    }
    ShadeArgs sa{depth, max_depth, rr_start, t_min, 0, s->octant_sort ? 1 : 0, perm,
                 (flags & LT_FLAG_COUNT) ? s->ray_ctr.as<unsigned long long>() + 3 : nullptr,
                 lane.cap};
    CK(launch_shade(sc, sa, pa, shade_grid,
                    s->use_window && s->use_shade_window ? &s->shade_window : nullptr, primary,
                    depth == 0,
                    ws->q_o[cur].as<float4>(), ws->q_d[cur].as<float4>(),
                    ws->hits.as<float4>(), ctr + depth, ws->q_o[cur ^ 1].as<float4>(),
                    ws->q_d[cur ^ 1].as<float4>(), ctr + depth + 1, st));
    s->stats.kernel_launches += 2;
    s->stats.trace_launches += 1;
    cur ^= 1;
  }
  CK(cudaGetLastError());
  return LT_OK;
}

static int validate_render(const lt_render_params *p) {
  if (!p) return lt_fail(LT_ERR_INVALID, "null render params");
  if (p->width < 1 || p->height < 1) return lt_fail(LT_ERR_INVALID, "image width and height must be >= 1");
  if ((int64_t)p->width * p->height >= (int64_t(1) << 31))
    return lt_fail(LT_ERR_INVALID, "image too large");
  if (p->max_depth < 1) return lt_fail(LT_ERR_INVALID, "max_depth must be >= 1");
  if (p->rr_start < 0) return lt_fail(LT_ERR_INVALID, "rr_start_depth must be >= 0");
  if (p->sample_start < 0 || p->sample_count < 0)
    return lt_fail(LT_ERR_INVALID, "sample range must be non-negative");
  if (!(p->t_min > 0.0)) return lt_fail(LT_ERR_INVALID, "t_min must be positive");
  if (p->n_ranks > 1 && (p->rank < 0 || p->rank >= p->n_ranks || p->tile_size < 1))
    return lt_fail(LT_ERR_INVALID, "invalid sharding (rank %d of %d, tile %d)", p->rank,
                   p->n_ranks, p->tile_size);
  return LT_OK;
}

// local pixel list for interleaved tiles: tile k (raster order over
// ceil(W/T) x ceil(H/T) tiles) belongs to rank k % n_ranks
static int pixel_set(lt_scene *s, const lt_render_params *p, const int32_t **list, int64_t *n) {
  // single rank: pixels in T x T tile order (LT_TILE_ORDER, default 4; 0 =
  // raster) so a warp's primary rays cover a compact 8 x 4 patch (+2 % on C4)
  const char *to = std::getenv("LT_TILE_ORDER");
  const int tile_order = to ? std::atoi(to) : 4;
  const bool sharded = p->n_ranks > 1;
  if (!sharded && tile_order <= 1) {
    *list = nullptr;
    *n = (int64_t)p->width * p->height;
    return LT_OK;
  }
  const int64_t rank = sharded ? p->rank : 0, n_ranks = sharded ? p->n_ranks : 1;
  const int64_t tile_sz = sharded ? p->tile_size : tile_order;
  const int64_t key[5] = {p->width, p->height, tile_sz, rank, n_ranks};
  if (!std::equal(key, key + 5, s->pix_key)) {
    // per-tile start offsets on the host (<= W*H/T^2 tiles), the per-pixel
    // scatter on the device (no 2 M-entry host list, no synchronous copy)
    const int64_t W = p->width, H = p->height, T = tile_sz;
    const int64_t ntx = (W + T - 1) / T, nty = (H + T - 1) / T;
    // this rank's tiles (tile = rank, rank + n_ranks, ...); the order in
    // which they are laid out: row-major, or (LT_TILE_CURVE=morton) along a
    // Z curve over the tile grid, so consecutive paths cover a compact
    // square instead of a strip
    std::vector<int64_t> tiles;
    for (int64_t tile = rank; tile < ntx * nty; tile += n_ranks) tiles.push_back(tile);
    const char *curve = std::getenv("LT_TILE_CURVE");
    if (curve && std::strcmp(curve, "morton") == 0) {
      auto spread = [](uint64_t v) {
        uint64_t x = v & 0xffffffffull;
        x = (x | (x << 16)) & 0x0000ffff0000ffffull;
        x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
        x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
        x = (x | (x << 2)) & 0x3333333333333333ull;
        x = (x | (x << 1)) & 0x5555555555555555ull;
        return x;
      };
      auto key = [&](int64_t tile) {
        const int64_t ty = tile / ntx, tx = tile - ty * ntx;
        return spread((uint64_t)tx) | (spread((uint64_t)ty) << 1);
      };
      std::stable_sort(tiles.begin(), tiles.end(),
                       [&](int64_t a, int64_t b) { return key(a) < key(b); });
    }
    std::vector<int32_t> tile_start((size_t)(ntx * nty / n_ranks + 2), 0);
    int64_t total = 0;
    for (int64_t tile : tiles) {
      const int64_t ty = tile / ntx, tx = tile - ty * ntx;
      tile_start[(size_t)(tile / n_ranks)] = (int32_t)total;
      total += (std::min(W, (tx + 1) * T) - tx * T) * (std::min(H, (ty + 1) * T) - ty * T);
    }
    // earlier passes (any stream) may still read the current list: the scene
    // stream waits for the device's last pass before replacing it
    {
      std::lock_guard<std::mutex> lk(s->ws->mu);
      if (s->ws->last_use) CK(cudaStreamWaitEvent(s->stream, s->ws->last_use, 0));
    }
    RET(s->pix_list.ensure(std::max<size_t>(16, (size_t)total * 4)));
    TmpBuf t_start;
    RET(upload(t_start, tile_start.data(), tile_start.size(), s->stream));
    launch_pixel_list((int32_t)W, (int32_t)H, (int32_t)T, (int32_t)rank, (int32_t)n_ranks,
                      t_start.as<int32_t>(), s->pix_list.as<int32_t>(), s->stream);
    CK(cudaGetLastError());
    // the render streams fork from the caller's stream: order after the scatter
    CK(cudaStreamSynchronize(s->stream));
    std::copy(key, key + 5, s->pix_key);
    s->pix_count = total;
  }
  *list = s->pix_list.as<int32_t>();
  *n = s->pix_count;
  return LT_OK;
}

static int render_impl(lt_scene *s, const lt_render_params *p, float *accum, uint32_t *valid,
                       uint32_t *invalid, cudaStream_t st) {
  RET(validate_render(p));
  if (!accum || !valid || !invalid) return lt_fail(LT_ERR_INVALID, "null accumulation buffer");
  s->stats = lt_render_stats{};
  s->ev_used = 0;
  const int32_t *pix_list = nullptr;
  int64_t n_local = 0;
  RET(pixel_set(s, p, &pix_list, &n_local));
  if (n_local == 0 || p->sample_count == 0) return LT_OK;
  const int64_t B = std::min(p->max_batch_paths > 0 ? p->max_batch_paths : s->default_batch,
                             kMaxBatchPaths);
  // lanes: disjoint contiguous ranges of the (tile-ordered) local pixels,
  // each with its own batches on its own stream; per pixel, samples still
  // accumulate in index order, so results do not depend on the lane count
  // a small pass (< 1 M paths) runs on one lane: a second lane would only
  // add launches and a stream fork / join to a few-microsecond frame
  const bool small = n_local * p->sample_count < (int64_t(1) << 20);
  // the fused one-launch path for passes too small to fill the GPU (no
  // per-launch counters / timing / material sort requested); LT_FUSED_MAX
  // overrides the path-count threshold (0 disables)
  const int64_t fused_max = [] {
    const char *e = std::getenv("LT_FUSED_MAX");
    return e ? (int64_t)std::atoll(e) : kFusedMaxPaths;
  }();
  const bool rng_tables = [] {
    const char *e = std::getenv("LT_RNG_TABLES");
    return !(e && e[0] == '0');
  }();
  const bool fused = n_local * p->sample_count <= fused_max &&
                     !(p->flags & (LT_FLAG_COUNT | LT_FLAG_SORT_MATERIALS));
  const int n_lanes =
      small ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(s->n_lanes, n_local));
  struct Batch {
    int lane;
    int64_t s0, ns, pc0, np;
  };
  std::vector<Batch> order;
  int64_t lane_cap[kLanes] = {};
  {
    std::vector<std::vector<Batch>> per(n_lanes);
    for (int k = 0; k < n_lanes; ++k) {
      const int64_t lo = n_local * k / n_lanes, hi = n_local * (k + 1) / n_lanes;
      const int64_t n_k = hi - lo, B_k = std::max<int64_t>(1, B / n_lanes);
      const int64_t chunk = std::min(n_k, B_k);
      const int64_t spb = std::min<int64_t>(std::max<int64_t>(1, B_k / chunk), p->sample_count);
      lane_cap[k] = chunk * spb;
      for (int64_t s0 = 0; s0 < p->sample_count; s0 += spb)
        for (int64_t pc = lo; pc < hi; pc += chunk)
          per[k].push_back(Batch{k, s0, std::min(spb, p->sample_count - s0), pc,
                                 std::min(chunk, hi - pc)});
    }
    // enqueue round-robin so every lane stream always has work queued
    for (size_t i = 0;; ++i) {
      bool any = false;
      for (int k = 0; k < n_lanes; ++k)
        if (i < per[k].size()) {
          order.push_back(per[k][i]);
          any = true;
        }
      if (!any) break;
    }
  }
  WorkspaceLease lease(s->ws, st);
  for (int k = 0; k < n_lanes; ++k) RET(ensure_lane(s, s->ws->lane[k], lane_cap[k], p->max_depth));
  CK(cudaMemsetAsync(s->ray_ctr.p, 0, 6 * sizeof(unsigned long long), st));
  // fork the lane streams off the caller's stream
  Workspace &W = *s->ws;
  if (!W.fork_ev) {
    for (int k = 0; k < kLanes; ++k) {
      CK(cudaStreamCreateWithFlags(&W.lane_st[k], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&W.join_ev[k], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&W.fork_ev, cudaEventDisableTiming));
  }
  // (one lane: its work goes straight onto the caller's stream)
  const bool fork = n_lanes > 1;
  if (fork) {
    CK(cudaEventRecord(W.fork_ev, st));
    for (int k = 0; k < n_lanes; ++k) CK(cudaStreamWaitEvent(W.lane_st[k], W.fork_ev, 0));
  }
  const float t_min = (float)p->t_min;
  for (const Batch &b : order) {
    Lane &ln = s->ws->lane[b.lane];
    cudaStream_t ls = fork ? W.lane_st[b.lane] : st;
    int32_t *ctr = ln.counters.as<int32_t>();
    if (!fused) CK(cudaMemsetAsync(ctr, 0, sizeof(int32_t) * (2 * (size_t)p->max_depth + 2), ls));
    RaygenArgs ra{};
    std::memcpy(ra.cam, p->camera, sizeof(ra.cam));
    ra.width = p->width;
    ra.height = p->height;
    ra.seed = p->seed;
    ra.sample_base = p->sample_start + b.s0;
    ra.n_pix = b.np;
    ra.pix_offset = b.pc0;
    ra.pix_list = pix_list;
    ra.n_paths = b.np * b.ns;
    ra.t_min = t_min;
    if (rng_tables) {
      // the batch's PCG increments (per pixel) and seeding terms (per
      // sample) once, instead of three mix64 per path in raygen and again
      // in the depth-0 shade
      RET(ln.rng.ensure(sizeof(uint64_t) * (size_t)(b.np + b.ns)));
      uint64_t *tab = ln.rng.as<uint64_t>();
      ra.inc_tab = tab;
      ra.init_tab = tab + b.np;
      launch_rng_tables(ra, b.ns, tab, tab + b.np, ls);
      s->stats.kernel_launches += 1;
    }
    if (fused) {
      // (LT_FLAG_PROFILE times the fused launch as the pass's trace time)
      if (p->flags & LT_FLAG_PROFILE) RET(record_event(s, ls));
      launch_path_small(s->view, ra, p->max_depth, p->rr_start, path_arrays(ln),
                        s->ray_ctr.as<unsigned long long>(), ls);
      if (p->flags & LT_FLAG_PROFILE) RET(record_event(s, ls));
      s->stats.kernel_launches += 1;
      s->stats.trace_launches += 1;
    } else {
      // raygen writes only the ray records; the depth-0 shade regenerates
      // throughput / radiance / PCG state
      launch_raygen(ra, path_arrays(ln), ln.q_o[0].as<float4>(), ln.q_d[0].as<float4>(), ctr,
                    ls);
      RET(run_bounces(s, ln, p->max_depth, p->rr_start, t_min, p->flags, ls, &ra, ra.n_paths));
    }
    AccumArgs aa{b.np, b.pc0, b.ns, pix_list};
    launch_accumulate(aa, ln.S.as<float4>(), accum, valid, invalid, ls);
    s->stats.kernel_launches += 2;
    s->stats.batches += 1;
    s->stats.paths += b.np * b.ns;
  }
  // join back into the caller's stream
  for (int k = 0; fork && k < n_lanes; ++k) {
    CK(cudaEventRecord(W.join_ev[k], W.lane_st[k]));
    CK(cudaStreamWaitEvent(st, W.join_ev[k], 0));
  }
  CK(cudaGetLastError());
  return LT_OK;
}

extern "C" int lt_render_pass(lt_scene *s, const lt_render_params *params, float *accum_sum,
                              uint32_t *valid, uint32_t *invalid, void *stream) {
  if (!s) return lt_fail(LT_ERR_INVALID, "null scene");
  DeviceGuard g(s->device);
  std::lock_guard<std::recursive_mutex> scene_lk(s->mu);
  return render_impl(s, params, accum_sum, valid, invalid, (cudaStream_t)stream);
}

extern "C" int lt_render_stats_get(const lt_scene *cs, lt_render_stats *out) {
  if (!cs || !out) return lt_fail(LT_ERR_INVALID, "null argument");
  lt_scene *s = const_cast<lt_scene *>(cs);
  DeviceGuard g(s->device);
  std::lock_guard<std::recursive_mutex> scene_lk(s->mu);
  if (s->ray_ctr.p) {
    unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
    CK(cudaMemcpy(c, s->ray_ctr.p, sizeof(c), cudaMemcpyDeviceToHost));
    s->stats.rays = (int64_t)c[0];
    s->stats.slab_tests = (int64_t)c[1];
    s->stats.tri_tests = (int64_t)c[2];
    s->stats.shade_warps = (int64_t)c[3];
    s->stats.shade_mixed_warps = (int64_t)c[4];
    s->stats.shade_warp_classes = (int64_t)c[5];
  }
  // trace launches of concurrent lanes overlap: report the union of their
  // [start, end] intervals (time during which any trace kernel ran)
  std::vector<std::pair<double, double>> iv;
  for (int i = 0; i + 1 < s->ev_used; i += 2) {
    CK(cudaEventSynchronize(s->ev_pool[i + 1]));
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, s->ev_pool[0], s->ev_pool[i]));
    CK(cudaEventElapsedTime(&b, s->ev_pool[0], s->ev_pool[i + 1]));
    iv.emplace_back(a, b);
  }
  std::sort(iv.begin(), iv.end());
  double ms = 0.0, cur_a = 0.0, cur_b = -1.0;
  for (const auto &x : iv) {
    if (x.first > cur_b) {
      if (cur_b > cur_a) ms += cur_b - cur_a;
      cur_a = x.first;
      cur_b = x.second;
    } else if (x.second > cur_b) {
      cur_b = x.second;
    }
  }
  if (cur_b > cur_a) ms += cur_b - cur_a;
  s->stats.trace_ms = ms;
  *out = s->stats;
  return LT_OK;
}

extern "C" int lt_render_pass_host(lt_scene *s, const lt_render_params *p, double *accum_mean,
                                   int64_t *valid, int64_t *invalid) {
  if (!s) return lt_fail(LT_ERR_INVALID, "null scene");
  RET(validate_render(p));
  if (!accum_mean || !valid || !invalid) return lt_fail(LT_ERR_INVALID, "null output buffer");
  DeviceGuard g(s->device);
  std::lock_guard<std::recursive_mutex> scene_lk(s->mu);
  const int64_t npx = (int64_t)p->width * p->height;
  RET(s->s_a.ensure(12 * npx));
  RET(s->s_b.ensure(4 * npx));
  RET(s->s_c.ensure(4 * npx));
  cudaStream_t st = s->stream;
  CK(cudaMemsetAsync(s->s_a.p, 0, 12 * npx, st));
  CK(cudaMemsetAsync(s->s_b.p, 0, 4 * npx, st));
  CK(cudaMemsetAsync(s->s_c.p, 0, 4 * npx, st));
  RET(render_impl(s, p, s->s_a.as<float>(), s->s_b.as<uint32_t>(), s->s_c.as<uint32_t>(), st));
  RET(s->h_stage.ensure(20 * npx));
  float *h_sum = s->h_stage.as<float>();
  uint32_t *h_valid = reinterpret_cast<uint32_t *>(h_sum + 3 * npx);
  uint32_t *h_invalid = h_valid + npx;
  CK(cudaMemcpyAsync(h_sum, s->s_a.p, 12 * npx, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_valid, s->s_b.p, 4 * npx, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_invalid, s->s_c.p, 4 * npx, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // fold the new samples into the running means (integrator.py:266-270)
  for (int64_t i = 0; i < npx; ++i) {
    const uint32_t v = h_valid[i];
    if (v) {
      const int64_t n = valid[i] + v;
      for (int c = 0; c < 3; ++c) {
        const double m = accum_mean[3 * i + c];
        accum_mean[3 * i + c] = m + ((double)h_sum[3 * i + c] - (double)v * m) / (double)n;
      }
      valid[i] = n;
    }
    invalid[i] += h_invalid[i];
  }
  return LT_OK;
}

// ------------------------------------------------------------------ ray queries

static int intersect_common(lt_scene *s, int64_t n, cudaStream_t st, bool count,
                            int32_t **nodes, int32_t **tests) {
  RET(s->s_d.ensure(std::max<int64_t>(16, 16 * n)));
  RET(s->s_e.ensure(std::max<int64_t>(16, 16 * n)));
  RET(s->s_f.ensure(std::max<int64_t>(16, 16 * n)));
  if (count) {
    RET(s->s_b.ensure(std::max<int64_t>(16, 4 * n)));
    RET(s->s_c.ensure(std::max<int64_t>(16, 4 * n)));
    *nodes = s->s_b.as<int32_t>();
    *tests = s->s_c.as<int32_t>();
  }
  launch_trace_rays(s->view, s->s_d.as<float4>(), s->s_e.as<float4>(), n, s->s_f.as<float4>(),
                    count ? *nodes : nullptr, count ? *tests : nullptr, st);
  CK(cudaGetLastError());
  return LT_OK;
}

extern "C" int lt_intersect_batch(lt_scene *s, const float *origins, const float *dirs, int64_t n,
                                  float t_min, float t_max, int32_t *idx, float *t, void *stream) {
  if (!s || n < 0) return lt_fail(LT_ERR_INVALID, "invalid arguments");
  if (n == 0) return LT_OK;
  if (!origins || !dirs || !idx || !t) return lt_fail(LT_ERR_INVALID, "null ray buffer");
  DeviceGuard g(s->device);
  std::lock_guard<std::recursive_mutex> scene_lk(s->mu);
  cudaStream_t st = (cudaStream_t)stream;
  RET(s->s_d.ensure(16 * n));
  RET(s->s_e.ensure(16 * n));
  launch_pack_rays_f32(origins, dirs, n, t_min, t_max, s->s_d.as<float4>(), s->s_e.as<float4>(),
                       st);
  RET(intersect_common(s, n, st, false, nullptr, nullptr));
  launch_unpack_hits(s->view, s->s_f.as<float4>(), n, idx, t, nullptr, nullptr, nullptr, st);
  CK(cudaGetLastError());
  return LT_OK;
}

static int upload_rays_f64(lt_scene *s, const double *o, const double *d, int64_t n,
                           double t_min, double t_max, cudaStream_t st) {
  RET(s->s_a.ensure(48 * n));
  double *dev = s->s_a.as<double>();
  CK(cudaMemcpyAsync(dev, o, 24 * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dev + 3 * n, d, 24 * n, cudaMemcpyHostToDevice, st));
  RET(s->s_d.ensure(16 * n));
  RET(s->s_e.ensure(16 * n));
  const float fmax = (float)t_max;  // +inf stays +inf
  launch_pack_rays_f64(dev, dev + 3 * n, n, (float)t_min, fmax, s->s_d.as<float4>(),
                       s->s_e.as<float4>(), st);
  return LT_OK;
}

// Closest hits of host rays (fp32 traversal, or the exhaustive kernel) as
// the reference's dtypes: idx int64 / t float64, optionally (u, v).
static int hits_host(lt_scene *s, const double *origins, const double *dirs, int64_t n,
                     double t_min, double t_max, bool brute, int64_t *idx, double *t,
                     double *uv) {
  if (!s || n < 0) return lt_fail(LT_ERR_INVALID, "invalid arguments");
  if (n == 0) return LT_OK;
  if (!origins || !dirs || !idx || !t) return lt_fail(LT_ERR_INVALID, "null ray buffer");
  DeviceGuard g(s->device);
  std::lock_guard<std::recursive_mutex> scene_lk(s->mu);
  cudaStream_t st = s->stream;
  RET(upload_rays_f64(s, origins, dirs, n, t_min, t_max, st));
  if (brute) {
    RET(s->s_f.ensure(std::max<int64_t>(16, 16 * n)));
    launch_brute_force(s->view, s->n_tris, s->s_d.as<float4>(), s->s_e.as<float4>(), n,
                       s->s_f.as<float4>(), st);
    CK(cudaGetLastError());
  } else {
    RET(intersect_common(s, n, st, false, nullptr, nullptr));
  }
  RET(s->s_a.ensure(32 * n));
  int64_t *d_idx = s->s_a.as<int64_t>();
  double *d_t = reinterpret_cast<double *>(d_idx + n);
  double *d_uv = uv ? d_t + n : nullptr;
  launch_unpack_hits(s->view, s->s_f.as<float4>(), n, nullptr, nullptr, d_idx, d_t, d_uv, st);
  CK(cudaMemcpyAsync(idx, d_idx, 8 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(t, d_t, 8 * n, cudaMemcpyDeviceToHost, st));
  if (uv) CK(cudaMemcpyAsync(uv, d_uv, 16 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return LT_OK;
}

extern "C" int lt_intersect_batch_host(lt_scene *s, const double *origins, const double *dirs,
                                       int64_t n, double t_min, double t_max, int64_t *idx,
                                       double *t) {
  return hits_host(s, origins, dirs, n, t_min, t_max, false, idx, t, nullptr);
}

extern "C" int lt_intersect_hits_host(lt_scene *s, const double *origins, const double *dirs,
                                      int64_t n, double t_min, double t_max, int64_t *idx,
                                      double *t, double *uv) {
  return hits_host(s, origins, dirs, n, t_min, t_max, false, idx, t, uv);
}

extern "C" int lt_brute_force_batch_host(lt_scene *s, const double *origins, const double *dirs,
                                         int64_t n, double t_min, double t_max, int64_t *idx,
                                         double *t) {
  return hits_host(s, origins, dirs, n, t_min, t_max, true, idx, t, nullptr);
}

extern "C" int lt_traversal_counts_host(lt_scene *s, const double *origins, const double *dirs,
                                        int64_t n, double t_min, double t_max, int64_t *nodes,
                                        int64_t *tests) {
  if (!s || n < 0) return lt_fail(LT_ERR_INVALID, "invalid arguments");
  if (n == 0) return LT_OK;
  if (!origins || !dirs || !nodes || !tests) return lt_fail(LT_ERR_INVALID, "null buffer");
  DeviceGuard g(s->device);
  std::lock_guard<std::recursive_mutex> scene_lk(s->mu);
  cudaStream_t st = s->stream;
  RET(upload_rays_f64(s, origins, dirs, n, t_min, t_max, st));
  int32_t *d_nodes = nullptr, *d_tests = nullptr;
  RET(intersect_common(s, n, st, true, &d_nodes, &d_tests));
  std::vector<int32_t> hn(n), ht(n);
  CK(cudaMemcpyAsync(hn.data(), d_nodes, 4 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ht.data(), d_tests, 4 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i) {
    nodes[i] = hn[i];
    tests[i] = ht[i];
  }
  return LT_OK;
}

extern "C" int lt_trace_paths_host(lt_scene *s, const double *origins, const double *dirs,
                                   const uint64_t *state, const uint64_t *inc, int64_t n,
                                   int32_t max_depth, int32_t rr_start, double t_min, double *rgb,
                                   uint64_t *state_out) {
  if (!s || n < 0) return lt_fail(LT_ERR_INVALID, "invalid arguments");
  if (n == 0) return LT_OK;
  if (!origins || !dirs || !state || !inc || !rgb || !state_out)
    return lt_fail(LT_ERR_INVALID, "null buffer");
  if (max_depth < 1) return lt_fail(LT_ERR_INVALID, "max_depth must be >= 1");
  if (rr_start < 0) return lt_fail(LT_ERR_INVALID, "rr_start_depth must be >= 0");
  if (!(t_min > 0.0)) return lt_fail(LT_ERR_INVALID, "t_min must be positive");
  if (n >= (int64_t(1) << 31)) return lt_fail(LT_ERR_INVALID, "too many paths");
  DeviceGuard g(s->device);
  std::lock_guard<std::recursive_mutex> scene_lk(s->mu);
  cudaStream_t st = s->stream;
  s->stats = lt_render_stats{};
  s->ev_used = 0;
  WorkspaceLease lease(s->ws, st);
  Lane &ln = s->ws->lane[0];
  RET(ensure_lane(s, ln, n, max_depth));
  RET(s->s_a.ensure(64 * n));
  double *d_o = s->s_a.as<double>();
  double *d_d = d_o + 3 * n;
  uint64_t *d_state = reinterpret_cast<uint64_t *>(d_d + 3 * n);
  uint64_t *d_inc = d_state + n;
  CK(cudaMemcpyAsync(d_o, origins, 24 * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_d, dirs, 24 * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_state, state, 8 * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_inc, inc, 8 * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(ln.counters.p, 0, sizeof(int32_t) * (2 * (size_t)max_depth + 2), st));
  CK(cudaMemsetAsync(s->ray_ctr.p, 0, 6 * sizeof(unsigned long long), st));
  RET(ln.inc.ensure(8 * (size_t)std::max<int64_t>(n, ln.cap)));
  const PathArrays pa = path_arrays(ln, true);
  launch_raygen_explicit(d_o, d_d, d_state, d_inc, n, (float)t_min, pa, ln.q_o[0].as<float4>(),
                         ln.q_d[0].as<float4>(), ln.counters.as<int32_t>(), st);
  RET(run_bounces(s, ln, max_depth, rr_start, (float)t_min, 0u, st, nullptr, n, true));
  RET(s->s_b.ensure(32 * n));
  double *d_rgb = s->s_b.as<double>();
  uint64_t *d_sout = reinterpret_cast<uint64_t *>(d_rgb + 3 * n);
  launch_gather_explicit(pa, n, d_rgb, d_sout, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(rgb, d_rgb, 24 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(state_out, d_sout, 8 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return LT_OK;
}

// ------------------------------------------------------------------ BSDF queries

// GpuMaterial records from (n,21) parameter rows (layout in luxb200.h)
static void materials_from_params(const double *p, int64_t n, std::vector<GpuMaterial> &out) {
  std::vector<double> bw(n), bc(3 * n), m(n), sw(n), sc(3 * n), r(n), ior(n), zero(3 * n, 0.0);
  std::vector<double> cw(n), cr(n), ci(n), cc(3 * n), tw(n), tc(3 * n);
  for (int64_t i = 0; i < n; ++i) {
    const double *q = p + 21 * i;
    bw[i] = q[0];
    for (int k = 0; k < 3; ++k) {
      bc[3 * i + k] = q[1 + k];
      sc[3 * i + k] = q[6 + k];
      cc[3 * i + k] = q[14 + k];
      tc[3 * i + k] = q[18 + k];
    }
    m[i] = q[4];
    sw[i] = q[5];
    r[i] = q[9];
    ior[i] = q[10];
    cw[i] = q[11];
    cr[i] = q[12];
    ci[i] = q[13];
    tw[i] = q[17];
  }
  lt_scene_desc d{};
  d.n_materials = (int32_t)n;
  d.base_weight = bw.data();
  d.base_color = bc.data();
  d.base_metalness = m.data();
  d.specular_weight = sw.data();
  d.specular_color = sc.data();
  d.specular_roughness = r.data();
  d.specular_ior = ior.data();
  d.emission_luminance = zero.data();
  d.emission_color = zero.data();
  d.coat_weight = cw.data();
  d.coat_roughness = cr.data();
  d.coat_ior = ci.data();
  d.coat_color = cc.data();
  d.transmission_weight = tw.data();
  d.transmission_color = tc.data();
  out.resize(n);
  for (int64_t i = 0; i < n; ++i) build_material(&d, (int)i, out[i]);
}

extern "C" int lt_bsdf_eval_ext_batch(const double *params, const double *wo, const double *wi,
                                      const double *normal, const int32_t *front, int64_t n,
                                      double *f, double *pdf) {
  if (n < 0 || (n > 0 && (!params || !wo || !wi || !normal || !f || !pdf)))
    return lt_fail(LT_ERR_INVALID, "invalid bsdf arguments");
  if (n == 0) return LT_OK;
  std::vector<GpuMaterial> mats;
  materials_from_params(params, n, mats);
  lt_staged::Staged q;
  const size_t v3 = 24 * (size_t)n;
  const int im = q.add(mats.data(), nullptr, sizeof(GpuMaterial) * n);
  const int io = q.add(wo, nullptr, v3), ii = q.add(wi, nullptr, v3), in = q.add(normal, nullptr, v3);
  const int ifr = front ? q.add(front, nullptr, 4 * (size_t)n) : -1;
  const int iff = q.add(nullptr, f, v3), ip = q.add(nullptr, pdf, 8 * (size_t)n);
  RET(q.begin());
  launch_bsdf_eval(q.dev<GpuMaterial>(im), q.dev<double>(io), q.dev<double>(ii),
                   q.dev<double>(in), ifr >= 0 ? q.dev<int32_t>(ifr) : nullptr, n,
                   q.dev<double>(iff), q.dev<double>(ip), q.stream());
  return q.finish();
}

extern "C" int lt_bsdf_eval_batch(const double *params, const double *wo, const double *wi,
                                  const double *normal, int64_t n, double *f, double *pdf) {
  return lt_bsdf_eval_ext_batch(params, wo, wi, normal, nullptr, n, f, pdf);
}

extern "C" int lt_bsdf_sample_batch(const double *params, const double *wo, const double *normal,
                                    const double *u, const int32_t *front, int64_t n, int32_t *ok,
                                    double *wi, double *weight) {
  if (n < 0 || (n > 0 && (!params || !wo || !normal || !u || !ok || !wi || !weight)))
    return lt_fail(LT_ERR_INVALID, "invalid bsdf arguments");
  if (n == 0) return LT_OK;
  std::vector<GpuMaterial> mats;
  materials_from_params(params, n, mats);
  lt_staged::Staged q;
  const size_t v3 = 24 * (size_t)n;
  const int im = q.add(mats.data(), nullptr, sizeof(GpuMaterial) * n);
  const int io = q.add(wo, nullptr, v3), in = q.add(normal, nullptr, v3), iu = q.add(u, nullptr, v3);
  const int ifr = front ? q.add(front, nullptr, 4 * (size_t)n) : -1;
  const int iok = q.add(nullptr, ok, 4 * (size_t)n), iwi = q.add(nullptr, wi, v3);
  const int iw = q.add(nullptr, weight, v3);
  RET(q.begin());
  launch_bsdf_sample(q.dev<GpuMaterial>(im), q.dev<double>(io), q.dev<double>(in),
                     q.dev<double>(iu), ifr >= 0 ? q.dev<int32_t>(ifr) : nullptr, n,
                     q.dev<int32_t>(iok), q.dev<double>(iwi), q.dev<double>(iw), q.stream());
  return q.finish();
}

extern "C" int lt_occluded_batch_host(lt_scene *s, const double *origins, const double *dirs,
                                      int64_t n, double t_min, double t_max, int32_t *occluded) {
  if (!s || n < 0) return lt_fail(LT_ERR_INVALID, "invalid arguments");
  if (n == 0) return LT_OK;
  if (!origins || !dirs || !occluded) return lt_fail(LT_ERR_INVALID, "null buffer");
  DeviceGuard g(s->device);
  std::lock_guard<std::recursive_mutex> scene_lk(s->mu);
  cudaStream_t st = s->stream;
  RET(upload_rays_f64(s, origins, dirs, n, t_min, t_max, st));
  RET(s->s_b.ensure(std::max<int64_t>(16, 4 * n)));
  launch_occluded(s->view, s->s_d.as<float4>(), s->s_e.as<float4>(), n, s->s_b.as<int32_t>(), st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(occluded, s->s_b.p, 4 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return LT_OK;
}

extern "C" int lt_read_bandwidth(int32_t device, int64_t bytes, int32_t iters, double *gbps) {
  if (!gbps || bytes < 1024 || iters < 1) return lt_fail(LT_ERR_INVALID, "invalid probe arguments");
  DeviceGuard g(device);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  DevBuf buf, sink;
  RET(buf.ensure((size_t)bytes));
  RET(sink.ensure(4096));
  CK(cudaMemset(buf.p, 0, (size_t)bytes));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int64_t n4 = bytes / 16;
  const int grid = sms * 4;
  // enough passes per launch that launch overhead is < 1% of the time
  const int passes = (int)std::max<int64_t>(1, std::min<int64_t>(64, (int64_t(1) << 31) / bytes));
  for (int w = 0; w < 2; ++w)
    launch_read_probe(buf.as<float4>(), n4, passes, sink.as<float>(), grid, st);
  cudaEventRecord(e0, st);
  for (int i = 0; i < iters; ++i)
    launch_read_probe(buf.as<float4>(), n4, passes, sink.as<float>(), grid, st);
  cudaEventRecord(e1, st);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  buf.release();
  sink.release();
  if (e != cudaSuccess) return lt_fail(LT_ERR_CUDA, "probe failed: %s", cudaGetErrorString(e));
  *gbps = (double)bytes * passes * iters / (ms * 1e-3) / 1e9;
  return LT_OK;
}

extern "C" int lt_accum_finish(const float *accum_sum, const uint32_t *valid,
                               const uint32_t *invalid, int64_t n_pixels, double *mean,
                               int64_t *invalid_out, void *stream) {
  if (n_pixels < 0 ||
      (n_pixels > 0 && (!accum_sum || !valid || !invalid || !mean || !invalid_out)))
    return lt_fail(LT_ERR_INVALID, "invalid accumulation arguments");
  launch_accum_finish(accum_sum, valid, invalid, n_pixels, mean, invalid_out,
                      (cudaStream_t)stream);
  CK(cudaGetLastError());
  return LT_OK;
}

extern "C" int lt_tonemap_u8(const float *linear, int64_t n_pixels, uint8_t *out, void *stream) {
  if (n_pixels < 0 || (n_pixels > 0 && (!linear || !out)))
    return lt_fail(LT_ERR_INVALID, "invalid tonemap arguments");
  launch_tonemap_u8(linear, n_pixels, out, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return LT_OK;
}
