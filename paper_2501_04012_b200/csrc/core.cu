// core.cu — context, error plumbing and the scalar primitives of
// core.cpp (embedding normalisation, cosine similarity), the engine's
// decide/similarity_to_step rule and the shard merge.
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>

#include "common.cuh"
#include "decide.cuh"

namespace fc {

// POD storage: no TLS destructor, so a C-ABI call made while the process is
// exiting (e.g. a static owner destroying its context) can still record its error
static thread_local char g_err[1024];
static thread_local uint64_t g_over_needed = 0, g_over_limit = 0, g_snap_off = 0;

// ---- pinned host staging cache ----
namespace {
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;   // size -> block
std::map<void*, size_t> g_pin_size;        // block -> size
}  // namespace

void* pinned_acquire(size_t bytes) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  auto it = g_pin_free.lower_bound(bytes);
  if (it != g_pin_free.end() && it->first <= 4 * bytes + (1 << 20)) {
    void* p = it->second;
    g_pin_free.erase(it);
    return p;
  }
  size_t sz = 1 << 16;
  while (sz < bytes) sz <<= 1;
  void* p = nullptr;
  FC_CUDA(cudaHostAlloc(&p, sz, cudaHostAllocPortable));
  g_pin_size[p] = sz;
  return p;
}

void pinned_release(void* p) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.emplace(g_pin_size.at(p), p);
}

void set_last_error(const std::string& m) {
  const size_t n = std::min(m.size(), sizeof(g_err) - 1);
  memcpy(g_err, m.data(), n);
  g_err[n] = 0;
}
void raise_snap(const std::string& what, uint64_t offset) {
  g_snap_off = offset;
  raise(LC_ERR_SNAPSHOT, what + " at byte " + std::to_string(offset));
}

void set_last_oversize(uint64_t needed, uint64_t limit) {
  g_over_needed = needed;
  g_over_limit = limit;
}

// Embedding ctor, core.cpp:50-59: sq = sum (double)v*v in element order;
// inv = 1/sqrt(sq); out = (float)(v*inv). One thread per row keeps the
// reduction sequential (bit-exact); rows are independent.
__global__ void k_normalize(const float* __restrict__ v, int64_t n, int dim, float* __restrict__ out,
                            int* __restrict__ bad) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float* x = v + r * dim;
  double sq = 0.0;
  bool finite = true;
  for (int i = 0; i < dim; ++i) {
    const double t = x[i];
    finite &= isfinite(x[i]);
    sq = fma(t, t, sq);  // t*t is exact in fp64, so fma == mul+add
  }
  if (!finite || sq == 0.0) {
    atomicExch(bad, 1);
    return;
  }
  const double inv = 1.0 / sqrt(sq);
  float* o = out + r * dim;
  for (int i = 0; i < dim; ++i) o[i] = (float)((double)x[i] * inv);
}

// cosine_similarity, core.cpp:101-114 (three sequential fp64 chains).
__global__ void k_cosine(const float* __restrict__ a, const float* __restrict__ b, int64_t n, int64_t len,
                         double* __restrict__ out, int* __restrict__ bad) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float* x = a + r * len;
  const float* y = b + r * len;
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (int64_t i = 0; i < len; ++i) {
    const double p = x[i], q = y[i];
    dot = fma(p, q, dot);
    na = fma(p, p, na);
    nb = fma(q, q, nb);
  }
  if (na == 0.0 || nb == 0.0) {
    atomicExch(bad, 1);
    out[r] = 0.0;
    return;
  }
  out[r] = dot / (sqrt(na) * sqrt(nb));
}

__global__ void k_decide(const uint64_t* wi, const double* ws, const uint64_t* oi, const double* os,
                         const uint64_t* bi, const double* bs, const int32_t* wc, int64_t n, double thr,
                         double e0, double e1, double e2, double e3, lc_decision* out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double e[4] = {e0, e1, e2, e3};
  lc_decision d;
  d.whole_id = wi[r];
  d.object_id = oi[r];
  d.background_id = bi[r];
  decide_one(ws[r], os[r], bs[r], wc ? wc[r] > 0 : true, thr, e, &d);
  out[r] = d;
}

// Global top-k of the union of G per-shard exact top-k lists (a23): each
// shard list is already ordered, the union order is (score desc, id asc),
// which is partition-independent, so the merge is exact.
__global__ void k_topk_merge(const uint64_t* __restrict__ ids, const double* __restrict__ sc,
                             const int32_t* __restrict__ cnt, int G, int64_t n, int k,
                             uint64_t* __restrict__ oid, double* __restrict__ osc, int32_t* __restrict__ ocnt) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  int pos[16];
  for (int g = 0; g < G; ++g) pos[g] = 0;
  int outn = 0;
  while (outn < k) {
    int bg = -1;
    double bs = 0.0;
    uint64_t bid = 0;
    for (int g = 0; g < G; ++g) {
      const int64_t base = ((int64_t)g * n + q);
      if (pos[g] >= cnt[base]) continue;
      const double s = sc[base * k + pos[g]];
      const uint64_t id = ids[base * k + pos[g]];
      if (bg < 0 || better(s, id, bs, bid)) {
        bg = g;
        bs = s;
        bid = id;
      }
    }
    if (bg < 0) break;
    oid[q * k + outn] = bid;
    osc[q * k + outn] = bs;
    ++outn;
    ++pos[bg];
  }
  for (int j = outn; j < k; ++j) {
    oid[q * k + j] = 0;
    osc[q * k + j] = 0.0;
  }
  ocnt[q] = outn;
}

// lrbu_priority / lcbfu_priority (store.cpp:32-42); FIFO/LRU keys are the
// store's min_priority_step keys (store.cpp:125-126).
__device__ __forceinline__ double policy_key(int policy, uint64_t f, int step, uint64_t last, uint64_t seq,
                                             uint64_t cap, uint64_t now, int* bad) {
  switch (policy) {
    case LC_POLICY_FIFO: return (double)seq;
    case LC_POLICY_LRU: return (double)last;
    case LC_POLICY_LCBFU: return __dmul_rn((double)(f + 1), (double)step);
    default: {
      if (now < last || cap == 0) {
        *bad = 1;
        return 0.0;
      }
      const uint64_t dd = now - last;
      const double duration = (double)(dd > 1 ? dd : 1);
      return __ddiv_rn(__dmul_rn((double)(f + 1), (double)step), __dmul_rn((double)cap, duration));
    }
  }
}

__global__ void k_priority(int policy, const lc_step_entry* __restrict__ e, int64_t n, uint64_t now,
                           double* __restrict__ out, int* __restrict__ bad) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int b = 0;
  out[r] = policy_key(policy, e[r].f, e[r].step, e[r].last_access, e[r].inserted_seq, e[r].capacity, now, &b);
  if (b) atomicExch(bad, 1);
}

lc_ctx* aux_ctx(lc_ctx* ctx, int i) {
  lc_ctx* t = ctx->top();
  std::lock_guard<std::mutex> lk(t->aux_mu);
  while ((int)t->aux.size() <= i) {
    auto* c = new lc_ctx();
    c->device = t->device;
    c->sm_count = t->sm_count;
    c->root = t;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      raise(LC_ERR_CUDA, "aux stream creation failed");
    }
    c->own_stream = true;
    t->aux.push_back(c);
  }
  return t->aux[i];
}

}  // namespace fc

using namespace fc;

extern "C" {

const char* lc_last_error(void) { return g_err; }
void lc_last_oversize(uint64_t* needed, uint64_t* limit) {
  if (needed) *needed = g_over_needed;
  if (limit) *limit = g_over_limit;
}
uint64_t lc_last_snapshot_offset(void) { return g_snap_off; }
const char* lc_version(void) { return "flexcache-b200 0.1 (sm_100a)"; }


lc_status lc_ctx_create(int device, lc_ctx** out) {
  LC_API_BEGIN
  FC_REQUIRE(out != nullptr, "lc_ctx_create: null out");
  int n = 0;
  FC_CUDA(cudaGetDeviceCount(&n));
  FC_REQUIRE(device >= 0 && device < n, "lc_ctx_create: bad device ordinal");
  cudaDeviceProp prop{};
  FC_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) raise(LC_ERR_CUDA, "lc_ctx_create: this build targets sm_100a (B200); device is sm_" +
                                               std::to_string(prop.major) + std::to_string(prop.minor));
  DeviceGuard g(device);
  auto* c = new lc_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  FC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = true;
  // stream-ordered scratch and entry storage come from the device's default
  // pool; keep freed blocks cached instead of unmapping them at every sync
  // (re-mapping ~1 GB of entries per compress batch cost ~10 ms of host time)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  *out = c;
  LC_API_END
}

lc_status lc_ctx_destroy(lc_ctx* ctx) {
  LC_API_BEGIN
  if (!ctx) return LC_OK;
  DeviceGuard g(ctx->device);
  for (lc_ctx* c : ctx->aux) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
    delete c;
  }
  cudaStreamSynchronize(ctx->stream);
  comm_free(ctx->comm);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  LC_API_END
}

lc_status lc_ctx_set_stream(lc_ctx* ctx, void* s) {
  LC_API_BEGIN
  DeviceGuard g(ctx->device);
  FC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  if (s) {
    ctx->stream = static_cast<cudaStream_t>(s);
    ctx->own_stream = false;
  } else {
    FC_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  LC_API_END
}

void* lc_ctx_stream(lc_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

lc_status lc_ctx_synchronize(lc_ctx* ctx) {
  LC_API_BEGIN
  DeviceGuard g(ctx->device);
  sync(ctx);
  LC_API_END
}

uint64_t lc_ctx_launches(lc_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

lc_status lc_ctx_profile(lc_ctx* ctx, int enable) {
  LC_API_BEGIN
  ctx->profile = enable != 0;
  LC_API_END
}

lc_status lc_ctx_kernel_time(lc_ctx* ctx, const char* name, uint64_t* launches, double* total_ms, int reset) {
  LC_API_BEGIN
  DeviceGuard g(ctx->device);
  sync(ctx);
  std::lock_guard<std::mutex> lk(ctx->prof_mu);
  uint64_t n = 0;
  double ms = 0.0;
  auto it = ctx->prof.find(name ? name : "");
  if (it != ctx->prof.end()) {
    for (auto& pr : it->second) {
      float t = 0.f;
      FC_CUDA(cudaEventElapsedTime(&t, pr.first, pr.second));
      ms += t;
      ++n;
    }
    if (reset) {
      for (auto& pr : it->second) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
      }
      ctx->prof.erase(it);
    }
  }
  if (launches) *launches = n;
  if (total_ms) *total_ms = ms;
  LC_API_END
}

lc_status lc_embedding_normalize(lc_ctx* ctx, const float* v, int64_t n, int dim, float* out) {
  LC_API_BEGIN
  FC_REQUIRE(dim > 0, "Embedding: empty vector");
  if (n <= 0) return LC_OK;
  DeviceGuard g(ctx->device);
  InArg<float> in(ctx, v, (size_t)n * dim);
  OutArg<float> o(ctx, out, (size_t)n * dim);
  DevBuf bad(sizeof(int), ctx->stream);
  FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
  k_normalize<<<grid_for(n, 128), 128, 0, ctx->stream>>>(in.dev, n, dim, o.dev, bad.as<int>());
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  o.finish(ctx);
  int hb = 0;
  FC_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  if (hb) raise(LC_ERR_INVALID_ARGUMENT, "Embedding: zero norm or non-finite element");
  LC_API_END
}

lc_status lc_cosine_batch(lc_ctx* ctx, const float* a, const float* b, int64_t n, int64_t len, double* out) {
  LC_API_BEGIN
  FC_REQUIRE(len > 0, "cosine_similarity: empty vectors");
  if (n <= 0) return LC_OK;
  DeviceGuard g(ctx->device);
  InArg<float> ia(ctx, a, (size_t)n * len), ib(ctx, b, (size_t)n * len);
  OutArg<double> o(ctx, out, (size_t)n);
  DevBuf bad(sizeof(int), ctx->stream);
  FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
  k_cosine<<<grid_for(n, 128), 128, 0, ctx->stream>>>(ia.dev, ib.dev, n, len, o.dev, bad.as<int>());
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  o.finish(ctx);
  int hb = 0;
  FC_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  if (hb) raise(LC_ERR_INVALID_ARGUMENT, "cosine_similarity: zero-norm operand");
  LC_API_END
}

lc_status lc_topk_merge(lc_ctx* ctx, const uint64_t* ids, const double* scores, const int32_t* counts, int G,
                        int64_t n, int k, uint64_t* out_ids, double* out_scores, int32_t* out_counts) {
  LC_API_BEGIN
  FC_REQUIRE(G >= 1 && G <= 16, "lc_topk_merge: 1 <= G <= 16");
  FC_REQUIRE(k >= 1, "lc_topk_merge: k >= 1");
  if (n <= 0) return LC_OK;
  DeviceGuard g(ctx->device);
  InArg<uint64_t> ii(ctx, ids, (size_t)G * n * k);
  InArg<double> is(ctx, scores, (size_t)G * n * k);
  InArg<int32_t> ic(ctx, counts, (size_t)G * n);
  OutArg<uint64_t> oi(ctx, out_ids, (size_t)n * k);
  OutArg<double> os(ctx, out_scores, (size_t)n * k);
  OutArg<int32_t> oc(ctx, out_counts, (size_t)n);
  k_topk_merge<<<grid_for(n, 128), 128, 0, ctx->stream>>>(ii.dev, is.dev, ic.dev, G, n, k, oi.dev, os.dev, oc.dev);
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  oi.finish(ctx);
  os.finish(ctx);
  oc.finish(ctx);
  sync(ctx);
  LC_API_END
}

lc_status lc_decide_batch(lc_ctx* ctx, const uint64_t* w_ids, const double* w_scores, const uint64_t* o_ids,
                          const double* o_scores, const uint64_t* b_ids, const double* b_scores, int64_t n,
                          double thr, const double* edges4, lc_decision* out) {
  LC_API_BEGIN
  if (n <= 0) return LC_OK;
  DeviceGuard g(ctx->device);
  const double def[4] = {0.72, 0.79, 0.86, 0.93};
  const double* e = edges4 ? edges4 : def;
  InArg<uint64_t> wi(ctx, w_ids, n), oi(ctx, o_ids, n), bi(ctx, b_ids, n);
  InArg<double> ws(ctx, w_scores, n), os(ctx, o_scores, n), bs(ctx, b_scores, n);
  OutArg<lc_decision> o(ctx, out, n);
  k_decide<<<grid_for(n, 128), 128, 0, ctx->stream>>>(wi.dev, ws.dev, oi.dev, os.dev, bi.dev, bs.dev, nullptr, n,
                                                      thr, e[0], e[1], e[2], e[3], o.dev);
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  o.finish(ctx);
  sync(ctx);
  LC_API_END
}

lc_status lc_priority_batch(lc_ctx* ctx, int policy, const lc_step_entry* e, int64_t n, uint64_t now, double* out) {
  LC_API_BEGIN
  FC_REQUIRE(policy >= 0 && policy <= 3, "invalid policy value");
  if (n <= 0) return LC_OK;
  DeviceGuard g(ctx->device);
  InArg<lc_step_entry> ie(ctx, e, n);
  OutArg<double> o(ctx, out, n);
  DevBuf bad(sizeof(int), ctx->stream);
  FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
  k_priority<<<grid_for(n, 128), 128, 0, ctx->stream>>>(policy, ie.dev, n, now, o.dev, bad.as<int>());
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  o.finish(ctx);
  int hb = 0;
  FC_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  if (hb) raise(LC_ERR_INVALID_ARGUMENT, "lrbu_priority: now precedes last access or zero capacity");
  LC_API_END
}

}  // extern "C"
