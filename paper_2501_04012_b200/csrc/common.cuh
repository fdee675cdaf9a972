// common.cuh — shared host/device plumbing for the FlexCache B200 library:
// error mapping (reference exception types -> lc_status), the per-GPU
// context, stream-ordered scratch buffers and host<->device staging for the
// C-ABI's "host or device pointer" arguments.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "flexcache_b200.h"

namespace fc {

// One exception type carrying the lc_status; thrown inside the library and
// converted at the C boundary (LC_API_BEGIN/END).
struct Error : std::runtime_error {
  lc_status code;
  Error(lc_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(lc_status c, const std::string& m) { throw Error(c, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line, cudaGetErrorString(e));
    throw Error(e == cudaErrorMemoryAllocation ? LC_ERR_OOM : LC_ERR_CUDA, buf);
  }
}
#define FC_CUDA(x) ::fc::cuda_check((x), #x, __FILE__, __LINE__)
#define FC_LAUNCH_CHECK() ::fc::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

void set_last_error(const std::string& m);
void set_last_oversize(uint64_t needed, uint64_t limit);
// SnapshotError(what, offset) (errors.hpp:30-35): message "<what> at byte <offset>"
[[noreturn]] void raise_snap(const std::string& what, uint64_t offset);

#define LC_API_BEGIN try {
#define LC_API_END                                   \
  }                                                  \
  catch (const ::fc::Error& e) {                     \
    ::fc::set_last_error(e.what());                  \
    return e.code;                                   \
  }                                                  \
  catch (const std::bad_alloc& e) {                  \
    ::fc::set_last_error("host allocation failed");  \
    return LC_ERR_OOM;                               \
  }                                                  \
  catch (const std::exception& e) {                  \
    ::fc::set_last_error(e.what());                  \
    return LC_ERR_INTERNAL;                          \
  }                                                  \
  return LC_OK;

#define FC_REQUIRE(cond, msg) \
  do {                        \
    if (!(cond)) ::fc::raise(LC_ERR_INVALID_ARGUMENT, (msg)); \
  } while (0)

}  // namespace fc

namespace fc {
struct Comm;  // shard.cu: NCCL communicator or host all-gather callback
void comm_free(Comm* c);
}  // namespace fc

struct lc_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::atomic<uint64_t> launches{0};
  // codec instrumentation (lc_codec_stats)
  std::atomic<uint64_t> inter_items{0}, inter_exact_items{0};
  // per-kernel CUDA-event timing (lc_ctx_profile / lc_ctx_kernel_time)
  bool profile = false;
  std::mutex prof_mu;
  std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> prof;
  // child contexts (own stream, same device) for work a call splits across
  // streams; launches and kernel timings are accounted on the root
  lc_ctx* root = nullptr;
  std::mutex aux_mu;
  std::vector<lc_ctx*> aux;
  lc_ctx* top() { return root ? root : this; }
  // entry-sharded multi-GPU (lc_ctx_comm_init / lc_ctx_comm_host)
  fc::Comm* comm = nullptr;
};

namespace fc {
// Records a CUDA event pair around the launches in its scope (on the
// context stream) when profiling is enabled.
struct KTimer {
  lc_ctx* ctx;
  const char* name;
  cudaEvent_t a = nullptr, b = nullptr;
  KTimer(lc_ctx* c, const char* n) : ctx(c), name(n) {
    if (!ctx->top()->profile) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, ctx->stream);
  }
  void stop() {
    if (!a) return;
    cudaEventRecord(b, ctx->stream);
    lc_ctx* t = ctx->top();
    std::lock_guard<std::mutex> g(t->prof_mu);
    t->prof[name].emplace_back(a, b);
    a = nullptr;
  }
  void cancel() {  // drop the interval (the caller times a narrower one)
    if (!a) return;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    a = b = nullptr;
  }
  ~KTimer() { stop(); }
};
}  // namespace fc

namespace fc {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) FC_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// For destructors: switches device like DeviceGuard but never throws (a
// destructor that throws terminates the process, e.g. during CUDA teardown).
struct QuietDeviceGuard {
  int prev = -1;
  explicit QuietDeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev && cudaSetDevice(dev) != cudaSuccess) cudaGetLastError();
  }
  ~QuietDeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
    cudaGetLastError();
  }
};

inline void count_launch(lc_ctx* ctx, uint64_t n = 1) { ctx->top()->launches.fetch_add(n, std::memory_order_relaxed); }
// i-th child context of ctx (created on first use; destroyed with ctx)
lc_ctx* aux_ctx(lc_ctx* ctx, int i);

// Stream-ordered device buffer (cudaMallocAsync / cudaFreeAsync).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t st) : bytes(n), s(st) {
    if (n) FC_CUDA(cudaMallocAsync(&p, n, st));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; bytes = o.bytes; s = o.s;
      o.p = nullptr; o.bytes = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

inline bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Read-only argument that may live on host or device.
template <class T>
struct InArg {
  const T* dev = nullptr;
  DevBuf tmp;
  InArg(lc_ctx* ctx, const T* p, size_t count) {
    if (!p || count == 0) return;
    if (is_device_ptr(p)) {
      dev = p;
    } else {
      tmp = DevBuf(count * sizeof(T), ctx->stream);
      FC_CUDA(cudaMemcpyAsync(tmp.p, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
      dev = tmp.as<T>();
    }
  }
};

void* pinned_acquire(size_t bytes);
void pinned_release(void* p);

// Output argument that may live on host or device; finish() copies back.
// stage = true: a pageable host destination is reached through a pooled
// pinned buffer (an async DMA instead of the driver's staged pageable copy);
// the caller calls deliver() after its stream sync.
template <class T>
struct OutArg {
  T* user = nullptr;
  T* dev = nullptr;
  size_t count = 0;
  bool host = false;
  T* pin = nullptr;
  DevBuf tmp;
  OutArg(lc_ctx* ctx, T* p, size_t n, bool stage = false) : user(p), count(n) {
    if (!p || n == 0) return;
    if (is_device_ptr(p)) {
      dev = p;
    } else {
      host = true;
      tmp = DevBuf(n * sizeof(T), ctx->stream);
      dev = tmp.as<T>();
      if (stage) pin = static_cast<T*>(pinned_acquire(n * sizeof(T)));
    }
  }
  OutArg(const OutArg&) = delete;
  OutArg& operator=(const OutArg&) = delete;
  ~OutArg() {
    if (pin) pinned_release(pin);
  }
  void finish(lc_ctx* ctx) {
    if (host && count)
      FC_CUDA(cudaMemcpyAsync(pin ? pin : user, dev, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  }
  void deliver() {  // after the stream sync
    if (pin) memcpy(user, pin, count * sizeof(T));
  }
};

inline unsigned grid_for(int64_t n, int block, int64_t cap = 1 << 30) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

inline void sync(lc_ctx* ctx) { FC_CUDA(cudaStreamSynchronize(ctx->stream)); }

}  // namespace fc

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
namespace fc {

// (score desc, id asc) ordering used by every top-k in the library: the
// generalisation of query_top1's strict '>' over ascending ids
// (vindex.cpp:58-72).
__host__ __device__ __forceinline__ bool better(double s1, uint64_t i1, double s2, uint64_t i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}

__device__ __forceinline__ double warp_shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

}  // namespace fc

namespace fc {
// Page-locked host staging with a process-wide cache of blocks: D2H / H2D of
// the compress orchestration's small arrays (maps, norms, per-key results,
// copy jobs, recipes) run at PCIe/NVLink-C2C speed instead of through the
// driver's pageable bounce buffers, without a cudaHostAlloc per call.
void* pinned_acquire(size_t bytes);
void pinned_release(void* p);
template <class T>
struct PinnedBuf {
  T* p = nullptr;
  size_t n = 0;
  PinnedBuf() = default;
  explicit PinnedBuf(size_t count) : n(count) {
    if (count) p = static_cast<T*>(pinned_acquire(count * sizeof(T)));
  }
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  PinnedBuf(PinnedBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  PinnedBuf& operator=(PinnedBuf&& o) noexcept {
    if (this != &o) {
      if (p) pinned_release(p);
      p = o.p; n = o.n;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~PinnedBuf() {
    if (p) pinned_release(p);
  }
  T* data() { return p; }
  const T* data() const { return p; }
  size_t size() const { return n; }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
  bool empty() const { return n == 0; }
};
}  // namespace fc
