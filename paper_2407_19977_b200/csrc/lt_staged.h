// lt_staged.h -- host-buffer staging for the synchronous query entry points
// (lt_query64.cu, the BSDF batches of lt_api.cu): every call's arrays go
// through one per-device scratch buffer (grow-only, serialized by a mutex)
// on a per-device non-blocking stream, so a query never waits for -- or
// blocks -- render work on other streams and never allocates per call.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "lt_internal.h"

namespace lt_staged {

struct Scratch {
  std::mutex mu;
  void *p = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;
};

inline Scratch &scratch_for(int dev) {
  static std::mutex g_mu;
  static std::vector<Scratch *> g;
  std::lock_guard<std::mutex> lk(g_mu);
  if ((int)g.size() <= dev) g.resize(dev + 1, nullptr);
  if (!g[dev]) g[dev] = new Scratch();  // process lifetime
  return *g[dev];
}

// One staged call: `add` registers an input (copied in) and / or output
// (copied back) array and returns its index; begin() uploads, dev<T>(i) is
// the device pointer, finish() downloads and synchronizes.
struct Staged {
  struct Arr {
    const void *in;
    void *out;
    size_t bytes, off;
  };
  std::vector<Arr> arrs;
  size_t total = 0;
  Scratch *sc = nullptr;
  std::unique_lock<std::mutex> lk;
  int add(const void *in, void *out, size_t bytes) {
    arrs.push_back(Arr{in, out, bytes, total});
    total += (bytes + 255) / 256 * 256;
    return (int)arrs.size() - 1;
  }
  int begin() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return lt_fail(LT_ERR_CUDA, "no CUDA device");
    sc = &scratch_for(dev);
    lk = std::unique_lock<std::mutex>(sc->mu);
    if (!sc->st) {
      const cudaError_t e = cudaStreamCreateWithFlags(&sc->st, cudaStreamNonBlocking);
      if (e != cudaSuccess) return lt_fail(LT_ERR_CUDA, "query stream: %s", cudaGetErrorString(e));
    }
    if (sc->bytes < total) {
      if (sc->p) cudaFree(sc->p);
      sc->p = nullptr;
      sc->bytes = 0;
      const size_t want = std::max<size_t>(total, size_t(1) << 20);
      const cudaError_t e = cudaMalloc(&sc->p, want);
      if (e != cudaSuccess)
        return lt_fail(LT_ERR_NOMEM, "query scratch: %s", cudaGetErrorString(e));
      sc->bytes = want;
    }
    for (const Arr &a : arrs)
      if (a.in && a.bytes) {
        const cudaError_t e =
            cudaMemcpyAsync(ptr(a), a.in, a.bytes, cudaMemcpyHostToDevice, sc->st);
        if (e != cudaSuccess) return lt_fail(LT_ERR_CUDA, "query upload: %s", cudaGetErrorString(e));
      }
    return LT_OK;
  }
  char *ptr(const Arr &a) const { return static_cast<char *>(sc->p) + a.off; }
  cudaStream_t stream() const { return sc->st; }
  template <class T>
  T *dev(int i) const {
    return reinterpret_cast<T *>(ptr(arrs[i]));
  }
  int finish() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return lt_fail(LT_ERR_CUDA, "query kernel: %s", cudaGetErrorString(e));
    for (const Arr &a : arrs)
      if (a.out && a.bytes) {
        e = cudaMemcpyAsync(a.out, ptr(a), a.bytes, cudaMemcpyDeviceToHost, sc->st);
        if (e != cudaSuccess) return lt_fail(LT_ERR_CUDA, "query download: %s", cudaGetErrorString(e));
      }
    e = cudaStreamSynchronize(sc->st);
    if (e != cudaSuccess) return lt_fail(LT_ERR_CUDA, "query: %s", cudaGetErrorString(e));
    return LT_OK;
  }
};

}  // namespace lt_staged

#define Q_RET(expr)             \
  do {                          \
    const int r_ = (expr);      \
    if (r_ != LT_OK) return r_; \
  } while (0)
