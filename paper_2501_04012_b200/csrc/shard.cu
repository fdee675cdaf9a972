// shard.cu — entry-sharded multi-GPU cache behind the C-ABI.
//
// One process (or thread) per GPU; prompt p is owned by rank p mod G, which
// holds its three index rows, its compressed entry and its live steps. The
// context carries the communicator:
//   * NCCL (lc_ctx_comm_init, ncclCommInitRank over NVLink/NVSwitch; NCCL is
//     dlopen'ed on first use so the library loads without it), or
//   * a host all-gather callback (lc_ctx_comm_host) for callers that bring
//     their own transport (MPI, a torch.distributed gloo group in the tests).
//
// Lookup (lc_sharded_query_topk / lc_sharded_lookup_decide): every rank runs
// the exact local top-k of the same query batch (tensor-core shortlist +
// certified fp64 rescore, index.cu), ONE grouped all-gather moves the
// [G][n][k] (id, score) lists and counts, and k_topk_merge takes the top-k of
// their union by (score desc, id asc) — a total order independent of the
// partition, so the result equals the unsharded query_top1 / top-k
// (vindex.cpp:58-72) bit for bit.
//
// Store (lc_sharded_store_*): one global capacity budget (store.cpp:53-91).
// A step's policy key depends only on its own prompt's records, which all live
// on the owner, so each shard's victim sequence at a fixed `now` is
// independent of the other shards' evictions, and the global sequence of
// repeated evict_one (store.cpp:80, 113-157) is the (key, seq) merge of the
// per-shard sequences. Each eviction burst therefore costs one all-gather of
// every shard's next m victims (lc_store_peek_many: key, StepEntry, used()
// after) per round instead of one collective per eviction; every rank runs the
// same merge and evicts its own consumed prefix. The global sequence counter
// (store.hpp:113 next_seq_) is replayed identically on every rank.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "lookup.cuh"

namespace fc {
__global__ void k_topk_merge(const uint64_t* __restrict__ ids, const double* __restrict__ sc,
                             const int32_t* __restrict__ cnt, int G, int64_t n, int k, uint64_t* __restrict__ oid,
                             double* __restrict__ osc, int32_t* __restrict__ ocnt);
lc_ctx* index_ctx(lc_index* ix);
int index_dim(lc_index* ix);
void index_topk_dev(lc_index* ix, int kind, const float* Qdev, int nq, int k, uint64_t* oid, double* osc,
                    int32_t* ocnt, const BoundExchange* xchg);
}  // namespace fc

using namespace fc;

namespace {

// ---- NCCL, resolved at run time -------------------------------------------
// (types restated from nccl.h; the ABI of these entry points is stable)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclSuccess = 0, ncclUint8 = 1 };

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the copy already mapped into the process (e.g. torch's) wins
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    auto sym = [&](auto& f, const char* s) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(api.h, s)); };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommCount, "ncclCommCount");
    sym(api.AllGather, "ncclAllGather");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
  });
  if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.AllGather)
    raise(LC_ERR_NCCL, "NCCL (libnccl.so.2) is not available in this process");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    raise(LC_ERR_NCCL, std::string(what) + " failed: " + m);
  }
}

}  // namespace

namespace fc {

struct Comm {
  int nranks = 1, rank = 0;
  ncclComm_t nccl = nullptr;
  lc_allgather_fn fn = nullptr;
  void* user = nullptr;
  uint64_t collectives = 0;

  struct Part {
    const void* send;
    void* recv;  // [nranks][bytes]
    size_t bytes;
  };

  // Grouped all-gather of device buffers (stream-ordered on ctx->stream).
  void allgather_dev(lc_ctx* ctx, const std::vector<Part>& parts) {
    ++collectives;
    if (nccl) {
      Nccl& api = ::nccl();
      nccl_check(api.GroupStart(), "ncclGroupStart");
      for (const Part& p : parts) nccl_check(api.AllGather(p.send, p.recv, p.bytes, ncclUint8, nccl, ctx->stream), "ncclAllGather");
      nccl_check(api.GroupEnd(), "ncclGroupEnd");
      return;
    }
    // host transport: pack, one callback, unpack
    size_t tot = 0;
    for (const Part& p : parts) tot += p.bytes;
    std::vector<uint8_t> send(tot), recv(tot * nranks);
    size_t off = 0;
    for (const Part& p : parts) {
      FC_CUDA(cudaMemcpyAsync(send.data() + off, p.send, p.bytes, cudaMemcpyDeviceToHost, ctx->stream));
      off += p.bytes;
    }
    sync(ctx);
    if (fn(user, send.data(), recv.data(), tot) != 0) raise(LC_ERR_NCCL, "host all-gather callback failed");
    off = 0;
    for (const Part& p : parts) {
      for (int r = 0; r < nranks; ++r)
        FC_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(p.recv) + (size_t)r * p.bytes, recv.data() + (size_t)r * tot + off,
                                p.bytes, cudaMemcpyHostToDevice, ctx->stream));
      off += p.bytes;
    }
    sync(ctx);  // the host staging dies with this scope
  }

  // All-gather of a small host record (control plane of the sharded store).
  std::vector<uint8_t> allgather_host(lc_ctx* ctx, const void* rec, size_t bytes) {
    std::vector<uint8_t> out(bytes * nranks);
    if (nccl) {
      ++collectives;
      DevBuf d(bytes * (nranks + 1), ctx->stream);
      FC_CUDA(cudaMemcpyAsync(d.p, rec, bytes, cudaMemcpyHostToDevice, ctx->stream));
      nccl_check(::nccl().AllGather(d.p, d.as<uint8_t>() + bytes, bytes, ncclUint8, nccl, ctx->stream), "ncclAllGather");
      FC_CUDA(cudaMemcpyAsync(out.data(), d.as<uint8_t>() + bytes, bytes * nranks, cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      return out;
    }
    ++collectives;
    if (fn(user, rec, out.data(), bytes) != 0) raise(LC_ERR_NCCL, "host all-gather callback failed");
    return out;
  }
};

void comm_free(Comm* c) {
  if (!c) return;
  if (c->nccl) ::nccl().CommDestroy(c->nccl);
  delete c;
}

}  // namespace fc

namespace {

Comm& need_comm(lc_ctx* ctx) {
  if (!ctx->comm) raise(LC_ERR_INVALID_ARGUMENT, "sharded call on a context without a communicator (lc_ctx_comm_init)");
  return *ctx->comm;
}

// Exact local top-k of one table into device buffers, all-gathered and merged.
struct ShardLists {
  DevBuf ids, sc, cnt, gids, gsc, gcnt;
};

__global__ void k_bound_max(const float* __restrict__ all, int G, int n, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float m = all[i];
  for (int g = 1; g < G; ++g) m = fmaxf(m, all[(size_t)g * n + i]);
  out[i] = m;
}

// Rank-local lists for the merge. With G > 1 the int8 tier runs two-phase:
// after its candidate pass each rank's per-query lower bound of its k-th score
// is all-gathered and max-reduced, a lower bound of the GLOBAL k-th score, so
// each rank rescores only the candidates that can reach the merged top-k
// (~1/G of them) instead of its whole local top-k.
void local_lists(lc_ctx* ctx, Comm& cm, lc_index* ix, int kind, const float* qdev, int64_t n, int k, ShardLists& L) {
  const cudaStream_t st = ctx->stream;
  const int G = cm.nranks;
  L.ids = DevBuf((size_t)n * k * 8, st);
  L.sc = DevBuf((size_t)n * k * 8, st);
  L.cnt = DevBuf((size_t)n * 4, st);
  L.gids = DevBuf((size_t)G * n * k * 8, st);
  L.gsc = DevBuf((size_t)G * n * k * 8, st);
  L.gcnt = DevBuf((size_t)G * n * 4, st);
  static const bool two_phase = !(getenv("FC_SHARD_TWO_PHASE") && atoi(getenv("FC_SHARD_TWO_PHASE")) == 0);
  BoundExchange ex = [&](float* b, int nb) {
    DevBuf all((size_t)G * nb * sizeof(float), st);
    std::vector<Comm::Part> parts{{b, all.p, (size_t)nb * sizeof(float)}};
    cm.allgather_dev(ctx, parts);
    k_bound_max<<<grid_for(nb, 256), 256, 0, st>>>(all.as<float>(), G, nb, b);
    FC_LAUNCH_CHECK();
    count_launch(ctx);
  };
  index_topk_dev(ix, kind, qdev, (int)n, k, L.ids.as<uint64_t>(), L.sc.as<double>(), L.cnt.as<int32_t>(),
                 (G > 1 && two_phase) ? &ex : nullptr);
}

void add_parts(std::vector<Comm::Part>& parts, ShardLists& L, int64_t n, int k) {
  parts.push_back({L.ids.p, L.gids.p, (size_t)n * k * 8});
  parts.push_back({L.sc.p, L.gsc.p, (size_t)n * k * 8});
  parts.push_back({L.cnt.p, L.gcnt.p, (size_t)n * 4});
}

void merge(lc_ctx* ctx, ShardLists& L, int G, int64_t n, int k, uint64_t* oid, double* osc, int32_t* ocnt) {
  k_topk_merge<<<grid_for(n, 128), 128, 0, ctx->stream>>>(L.gids.as<uint64_t>(), L.gsc.as<double>(), L.gcnt.as<int32_t>(),
                                                          G, n, k, oid, osc, ocnt);
  FC_LAUNCH_CHECK();
  count_launch(ctx);
}

}  // namespace

// ---------------------------------------------------------------------------
// sharded store
// ---------------------------------------------------------------------------
struct lc_sharded_store {
  lc_ctx* ctx = nullptr;
  lc_store* local = nullptr;
  uint64_t capacity = 0;
  uint64_t seq = 0;  // global next_seq_ (store.hpp:113), identical on every rank
  int batch = 64;    // victims per shard per all-gather round
  uint64_t rounds = 0, evictions = 0;
};

namespace {

void ok(lc_status s) {
  if (s != LC_OK) raise(s, lc_last_error());
}

// One shard's next victims as exchanged in a round.
struct PeekHdr {
  int32_t n, more;
  uint64_t used;
};
struct PeekRec {
  lc_step_entry e;
  double key;
  uint64_t used_after;
};

// Evict globally at `now` until used + extra <= capacity (want < 0) or
// exactly `want` steps; every rank returns the same victim list.
std::vector<lc_step_entry> global_evict(lc_sharded_store* ss, uint64_t now, uint64_t extra, int want) {
  Comm& cm = need_comm(ss->ctx);
  const int G = cm.nranks, m = ss->batch;
  std::vector<lc_step_entry> out;
  const size_t rec_bytes = sizeof(PeekHdr) + (size_t)m * sizeof(PeekRec);
  std::vector<uint8_t> mine(rec_bytes);
  uint64_t total = 0;
  if (want < 0) {  // the common case of no eviction costs one 8-byte all-gather
    const uint64_t u = lc_store_used(ss->local);
    std::vector<uint8_t> all = cm.allgather_host(ss->ctx, &u, sizeof u);
    for (int r = 0; r < G; ++r) {
      uint64_t x;
      memcpy(&x, all.data() + (size_t)r * 8, 8);
      total += x;
    }
    if (total + extra <= ss->capacity) return out;
  }
  for (;;) {
    PeekHdr h{0, 0, lc_store_used(ss->local)};
    auto* recs = reinterpret_cast<PeekRec*>(mine.data() + sizeof(PeekHdr));
    std::vector<lc_step_entry> e(m);
    std::vector<double> key(m);
    std::vector<uint64_t> ua(m);
    if (lc_store_step_count(ss->local) > 0) {
      int n = 0, more = 0;
      ok(lc_store_peek_many(ss->local, now, m, e.data(), key.data(), ua.data(), &n, &more));
      h.n = n;
      h.more = more;
      for (int i = 0; i < n; ++i) recs[i] = PeekRec{e[i], key[i], ua[i]};
    }
    memcpy(mine.data(), &h, sizeof h);
    std::vector<uint8_t> all = cm.allgather_host(ss->ctx, mine.data(), rec_bytes);
    ++ss->rounds;
    std::vector<PeekHdr> H(G);
    std::vector<const PeekRec*> R(G);
    total = 0;
    for (int r = 0; r < G; ++r) {
      memcpy(&H[r], all.data() + (size_t)r * rec_bytes, sizeof(PeekHdr));
      R[r] = reinterpret_cast<const PeekRec*>(all.data() + (size_t)r * rec_bytes + sizeof(PeekHdr));
      total += H[r].used;
    }
    auto done = [&] { return want >= 0 ? (int)out.size() >= want : total + extra <= ss->capacity; };
    if (done()) break;
    std::vector<int> ptr(G, 0);
    std::vector<uint64_t> used_r(G);
    for (int r = 0; r < G; ++r) used_r[r] = H[r].used;
    bool blocked = false, progressed = false;
    while (!done()) {
      int best = -1;
      for (int r = 0; r < G; ++r) {
        if (ptr[r] >= H[r].n) {
          if (H[r].more) blocked = true;  // this shard's next victim is unknown until it re-scores
          continue;
        }
        const PeekRec& c = R[r][ptr[r]];
        if (best < 0) {
          best = r;
          continue;
        }
        const PeekRec& b = R[best][ptr[best]];
        if (c.key < b.key || (c.key == b.key && c.e.inserted_seq < b.e.inserted_seq)) best = r;
      }
      if (blocked) break;
      if (best < 0) raise(LC_ERR_LOGIC, "evict_one: store is empty");
      const PeekRec& v = R[best][ptr[best]];
      total -= used_r[best] - v.used_after;
      used_r[best] = v.used_after;
      out.push_back(v.e);
      ++ptr[best];
      progressed = true;
    }
    // every rank applies its own consumed prefix (identical to the peek)
    for (int i = 0; i < ptr[cm.rank]; ++i) {
      lc_step_entry got{};
      ok(lc_store_evict_one(ss->local, now, &got));
      const PeekRec& p = R[cm.rank][i];
      if (memcmp(&got, &p.e, sizeof got) != 0) raise(LC_ERR_INTERNAL, "sharded eviction: local victim differs from its peek");
    }
    ss->evictions += ptr[cm.rank];
    if (done()) break;
    if (!blocked && !progressed) raise(LC_ERR_LOGIC, "evict_one: store is empty");
  }
  return out;
}

}  // namespace

extern "C" {

lc_status lc_comm_unique_id(uint8_t* id128) {
  LC_API_BEGIN
  FC_REQUIRE(id128, "null argument");
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(id128, &id, sizeof id);
  LC_API_END
}

lc_status lc_ctx_comm_init(lc_ctx* ctx, int nranks, int rank, const uint8_t* id128) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && id128, "null argument");
  FC_REQUIRE(nranks >= 1 && nranks <= 16 && rank >= 0 && rank < nranks, "lc_ctx_comm_init: bad nranks/rank");
  FC_REQUIRE(!ctx->comm, "lc_ctx_comm_init: context already has a communicator");
  DeviceGuard g(ctx->device);
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  auto* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclResult_t r = nccl().CommInitRank(&c->nccl, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    nccl_check(r, "ncclCommInitRank");
  }
  ctx->comm = c;
  LC_API_END
}

lc_status lc_ctx_comm_host(lc_ctx* ctx, int nranks, int rank, lc_allgather_fn fn, void* user) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && fn, "null argument");
  FC_REQUIRE(nranks >= 1 && nranks <= 16 && rank >= 0 && rank < nranks, "lc_ctx_comm_host: bad nranks/rank");
  FC_REQUIRE(!ctx->comm, "lc_ctx_comm_host: context already has a communicator");
  auto* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  c->fn = fn;
  c->user = user;
  ctx->comm = c;
  LC_API_END
}

lc_status lc_ctx_comm_info(lc_ctx* ctx, int* nranks, int* rank, int* backend, uint64_t* collectives) {
  LC_API_BEGIN
  FC_REQUIRE(ctx, "null argument");
  const Comm* c = ctx->comm;
  int nr = c ? c->nranks : 1;
  if (c && c->nccl && nccl().CommCount) nccl_check(nccl().CommCount(c->nccl, &nr), "ncclCommCount");
  if (nranks) *nranks = nr;
  if (rank) *rank = c ? c->rank : 0;
  if (backend) *backend = !c ? 0 : c->nccl ? 1 : 2;
  if (collectives) *collectives = c ? c->collectives : 0;
  LC_API_END
}

uint64_t lc_shard_owner(uint64_t prompt, int nranks) { return nranks > 0 ? prompt % (uint64_t)nranks : 0; }

lc_status lc_sharded_query_topk(lc_index* ix, int kind, const float* q, int64_t n, int dim, int k, uint64_t* out_ids,
                                double* out_scores, int32_t* out_counts) {
  LC_API_BEGIN
  FC_REQUIRE(ix, "null index");
  FC_REQUIRE(kind >= 0 && kind <= 2, "bad embedding kind");
  FC_REQUIRE(k >= 1 && k <= 64, "k must be in [1, 64]");
  FC_REQUIRE(n >= 0 && n < (1ll << 31), "bad query count");
  lc_ctx* ctx = index_ctx(ix);
  Comm& cm = need_comm(ctx);
  DeviceGuard g(ctx->device);
  if (n == 0) return LC_OK;
  const int d0 = index_dim(ix);
  FC_REQUIRE(dim > 0 && (d0 == 0 || d0 == dim), "SimilarityIndex: query dimension mismatch");
  InArg<float> qa(ctx, q, (size_t)n * dim);
  OutArg<uint64_t> oi(ctx, out_ids, (size_t)n * k);
  OutArg<double> os(ctx, out_scores, (size_t)n * k);
  OutArg<int32_t> oc(ctx, out_counts, (size_t)n);
  ShardLists L;
  local_lists(ctx, cm, ix, kind, qa.dev, n, k, L);
  std::vector<Comm::Part> parts;
  add_parts(parts, L, n, k);
  cm.allgather_dev(ctx, parts);
  merge(ctx, L, cm.nranks, n, k, oi.dev, os.dev, oc.dev);
  oi.finish(ctx);
  os.finish(ctx);
  oc.finish(ctx);
  sync(ctx);
  LC_API_END
}

lc_status lc_sharded_lookup_decide(lc_index* ix, const float* qw, const float* qo, const float* qb, int64_t n, int dim,
                                   double thr, const double* edges4, lc_decision* out) {
  LC_API_BEGIN
  FC_REQUIRE(ix && qw && qo && qb && out, "null argument");
  FC_REQUIRE(n >= 0 && n < (1ll << 31), "bad query count");
  lc_ctx* ctx = index_ctx(ix);
  Comm& cm = need_comm(ctx);
  DeviceGuard g(ctx->device);
  if (n == 0) return LC_OK;
  const int d0 = index_dim(ix);
  FC_REQUIRE(dim > 0 && (d0 == 0 || d0 == dim), "SimilarityIndex: query dimension mismatch");
  const double def[4] = {0.72, 0.79, 0.86, 0.93};
  const double* e = edges4 ? edges4 : def;
  const float* qs[3] = {qw, qo, qb};
  ShardLists L[3];
  std::vector<Comm::Part> parts;
  for (int t = 0; t < 3; ++t) {
    InArg<float> qa(ctx, qs[t], (size_t)n * dim);
    local_lists(ctx, cm, ix, t, qa.dev, n, 1, L[t]);
    add_parts(parts, L[t], n, 1);
  }
  cm.allgather_dev(ctx, parts);
  DevBuf ids(3 * (size_t)n * 8, ctx->stream), sc(3 * (size_t)n * 8, ctx->stream), cnt(3 * (size_t)n * 4, ctx->stream);
  for (int t = 0; t < 3; ++t)
    merge(ctx, L[t], cm.nranks, n, 1, ids.as<uint64_t>() + t * n, sc.as<double>() + t * n, cnt.as<int32_t>() + t * n);
  OutArg<lc_decision> o(ctx, out, (size_t)n);
  k_decide<<<grid_for(n, 128), 128, 0, ctx->stream>>>(ids.as<uint64_t>(), sc.as<double>(), ids.as<uint64_t>() + n,
                                                      sc.as<double>() + n, ids.as<uint64_t>() + 2 * n,
                                                      sc.as<double>() + 2 * n, cnt.as<int32_t>(), n, thr, e[0], e[1],
                                                      e[2], e[3], o.dev);
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  o.finish(ctx);
  sync(ctx);
  LC_API_END
}

lc_status lc_sharded_store_create(lc_ctx* ctx, uint64_t capacity, int policy, int batch, lc_sharded_store** out) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && out, "null argument");
  need_comm(ctx);
  FC_REQUIRE(batch >= 0 && batch <= 4096, "lc_sharded_store_create: batch in [0, 4096]");
  auto* ss = new lc_sharded_store();
  ss->ctx = ctx;
  ss->capacity = capacity;
  if (batch) ss->batch = batch;
  lc_status st = lc_store_create(ctx, UINT64_MAX, policy, &ss->local);  // the budget is global, not per shard
  if (st != LC_OK) {
    delete ss;
    raise(st, lc_last_error());
  }
  *out = ss;
  LC_API_END
}

lc_status lc_sharded_store_destroy(lc_sharded_store* ss) {
  LC_API_BEGIN
  if (!ss) return LC_OK;
  lc_store_destroy(ss->local);
  delete ss;
  LC_API_END
}

lc_store* lc_sharded_store_local(lc_sharded_store* ss) { return ss ? ss->local : nullptr; }

lc_status lc_sharded_store_insert(lc_sharded_store* ss, uint64_t prompt, lc_entry* entry, const int32_t* steps,
                                  int n_steps, uint64_t now, lc_step_entry* evicted, int cap, int* n_evicted) {
  LC_API_BEGIN
  FC_REQUIRE(ss, "null store");
  Comm& cm = need_comm(ss->ctx);
  DeviceGuard g(ss->ctx->device);
  if (n_evicted) *n_evicted = 0;
  const int own = (int)lc_shard_owner(prompt, cm.nranks);
  // (1) the owner validates (store.cpp:53-76); every rank learns the outcome
  struct Val {
    int32_t status, n_sel;
    uint64_t standalone;
  } v{0, 0, 0};
  std::string msg;
  if (cm.rank == own) {
    if (!entry) {
      v.status = LC_ERR_INVALID_ARGUMENT;
      msg = "lc_sharded_store_insert: the owner rank must pass the entry";
    } else {
      lc_status st = lc_store_check_insert(ss->local, prompt, entry, steps, n_steps, &v.standalone);
      if (st != LC_OK) {
        v.status = st;
        msg = lc_last_error();
      } else {
        std::vector<int32_t> u(steps, steps + n_steps);
        std::sort(u.begin(), u.end());
        v.n_sel = (int32_t)(std::unique(u.begin(), u.end()) - u.begin());
        if (v.standalone > ss->capacity) v.status = LC_ERR_OVERSIZED_ENTRY;
      }
    }
  }
  std::vector<uint8_t> all = cm.allgather_host(ss->ctx, &v, sizeof v);
  memcpy(&v, all.data() + (size_t)own * sizeof v, sizeof v);
  if (v.status == LC_ERR_OVERSIZED_ENTRY) {
    set_last_oversize(v.standalone, ss->capacity);
    raise(LC_ERR_OVERSIZED_ENTRY, "entry of " + std::to_string(v.standalone) + " bytes exceeds capacity limit of " +
                                      std::to_string(ss->capacity) + " bytes");
  }
  if (v.status != LC_OK)
    raise((lc_status)v.status, msg.empty() ? "insert_steps: rejected by owner rank " + std::to_string(own) : msg);
  // (2) global evictions (store.cpp:80), batched per round
  std::vector<lc_step_entry> ev = global_evict(ss, now, v.standalone, -1);
  for (size_t i = 0; i < ev.size() && evicted && (int)i < cap; ++i) evicted[i] = ev[i];
  if (n_evicted) *n_evicted = (int)ev.size();
  // (3) the owner inserts with the global sequence numbers
  if (cm.rank == own) {
    ok(lc_store_set_next_seq(ss->local, ss->seq));
    int ne = 0;
    ok(lc_store_insert(ss->local, prompt, entry, steps, n_steps, now, nullptr, 0, &ne));
    if (ne) raise(LC_ERR_INTERNAL, "sharded insert: unexpected local eviction");
  }
  ss->seq += (uint64_t)v.n_sel;
  LC_API_END
}

lc_status lc_sharded_store_evict_one(lc_sharded_store* ss, uint64_t now, lc_step_entry* out) {
  LC_API_BEGIN
  FC_REQUIRE(ss, "null store");
  DeviceGuard g(ss->ctx->device);
  std::vector<lc_step_entry> ev = global_evict(ss, now, 0, 1);
  if (out) *out = ev.at(0);
  LC_API_END
}

lc_status lc_sharded_store_get_step(lc_sharded_store* ss, uint64_t prompt, int desired, uint64_t now, int32_t* actual,
                                    float* out_dev) {
  LC_API_BEGIN
  FC_REQUIRE(ss && actual, "null argument");
  Comm& cm = need_comm(ss->ctx);
  DeviceGuard g(ss->ctx->device);
  const int own = (int)lc_shard_owner(prompt, cm.nranks);
  int32_t a[2] = {0, 0};  // actual, status
  std::string msg;
  if (cm.rank == own) {
    lc_status st = lc_store_get_step(ss->local, prompt, desired, now, &a[0], out_dev);
    a[1] = st;
    if (st != LC_OK) msg = lc_last_error();
  }
  std::vector<uint8_t> all = cm.allgather_host(ss->ctx, a, sizeof a);
  memcpy(a, all.data() + (size_t)own * sizeof a, sizeof a);
  if (a[1] != LC_OK) raise((lc_status)a[1], msg.empty() ? "get_step: rejected by owner rank " + std::to_string(own) : msg);
  *actual = a[0];
  LC_API_END
}

lc_status lc_sharded_store_used(lc_sharded_store* ss, uint64_t* out) {
  LC_API_BEGIN
  FC_REQUIRE(ss && out, "null argument");
  Comm& cm = need_comm(ss->ctx);
  const uint64_t u = lc_store_used(ss->local);
  std::vector<uint8_t> all = cm.allgather_host(ss->ctx, &u, sizeof u);
  uint64_t t = 0;
  for (int r = 0; r < cm.nranks; ++r) {
    uint64_t x;
    memcpy(&x, all.data() + (size_t)r * 8, 8);
    t += x;
  }
  *out = t;
  LC_API_END
}

lc_status lc_sharded_store_stats(lc_sharded_store* ss, uint64_t* rounds, uint64_t* local_evictions, uint64_t* next_seq) {
  LC_API_BEGIN
  FC_REQUIRE(ss, "null store");
  if (rounds) *rounds = ss->rounds;
  if (local_evictions) *local_evictions = ss->evictions;
  if (next_seq) *next_seq = ss->seq;
  LC_API_END
}

}  // extern "C"
