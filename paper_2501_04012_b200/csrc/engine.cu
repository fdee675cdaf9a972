// engine.cu — the request pipeline of SPEC.md:453-562 (Fig. 5 of the paper):
// lookup -> decide -> step selection -> get_step / decompress+stitch ->
// simulated generation -> update_after_generation, plus the latency and cost
// models. The reference declares this module but ships no code for it
// (SURVEY §8(c)), so its rules come from the SPEC text and its examples.
//
// The engine is a client of the library's own C-ABI (index, store, codec).
// Requests are processed in order and every result equals serial
// execution; a batch of n requests shares ONE exact top-K lookup per table on
// the tensor-core path (K = 8). Request j then fixes that list up on the
// host: rows removed since the batch lookup are skipped, rows inserted since
// are scored exactly (sequential fp64, vindex.cpp:67 order) and merged by
// (score desc, id asc); only if all K listed rows are gone does j re-query
// the device index. The top-1 per table therefore equals query_top1 on the
// index state request j sees.
#include <algorithm>
#include <array>
#include <memory>
#include <cmath>
#include <cstring>
#include <map>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include <chrono>

#include "common.cuh"
#include "decide.cuh"

namespace fc {
namespace {

constexpr int KTOP = 8;
constexpr int kCached[5] = {5, 10, 15, 20, 25};

void ok(lc_status st) {
  if (st != LC_OK) raise(st, lc_last_error() ? lc_last_error() : "engine: library call failed");
}

std::vector<float> to_host(const float* p, size_t n) {
  std::vector<float> h(n);
  if (n == 0) return h;
  if (is_device_ptr(p)) FC_CUDA(cudaMemcpy(h.data(), p, n * sizeof(float), cudaMemcpyDeviceToHost));
  else memcpy(h.data(), p, n * sizeof(float));
  return h;
}

// Exact dots among the batch's own queries, per table: D[t][j][i] =
// sum_d (double)q_j[d] * (double)q_i[d] in d order (vindex.cpp:67; the
// product of two floats is exact in fp64, so fma == the reference's mul+add)
// for i < j. Rows inserted during the batch are earlier requests' query rows,
// so the per-request fix-up reads these instead of scoring on the host.
// Block = 16 x 16 (j, i) pairs, the two 16-row query slices staged in smem
// 64 dims at a time; blocks above the diagonal exit.
constexpr int BD_T = 16, BD_K = 64;
__global__ void __launch_bounds__(BD_T * BD_T) k_batch_dots(const float* __restrict__ q0, const float* __restrict__ q1,
                                                          const float* __restrict__ q2, int n, int d,
                                                          double* __restrict__ D) {
  const int t = blockIdx.z;
  const float* q = t == 0 ? q0 : t == 1 ? q1 : q2;
  const int j0 = blockIdx.y * BD_T, i0 = blockIdx.x * BD_T;
  if (i0 > j0 + BD_T - 1) return;  // every pair of the block has i > j
  __shared__ float sj[BD_T][BD_K + 1], si[BD_T][BD_K + 1];
  const int tj = threadIdx.x / BD_T, ti = threadIdx.x % BD_T;
  const int j = j0 + tj, i = i0 + ti;
  double acc = 0.0;
  for (int k0 = 0; k0 < d; k0 += BD_K) {
    const int kn = min(BD_K, d - k0);
    for (int x = threadIdx.x; x < BD_T * BD_K; x += BD_T * BD_T) {
      const int r = x / BD_K, c = x % BD_K;
      sj[r][c] = (j0 + r < n && c < kn) ? q[(size_t)(j0 + r) * d + k0 + c] : 0.f;
      si[r][c] = (i0 + r < n && c < kn) ? q[(size_t)(i0 + r) * d + k0 + c] : 0.f;
    }
    __syncthreads();
    for (int c = 0; c < kn; ++c) acc = fma((double)sj[tj][c], (double)si[ti][c], acc);
    __syncthreads();
  }
  if (j < n && i < j) D[((size_t)t * n + j) * n + i] = acc;
}

// FC_TRACE=1: accumulated host time per engine phase, printed per call
struct PhaseClock {
  bool on = getenv("FC_TRACE") && atoi(getenv("FC_TRACE")) == 1;
  double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void lap(int k) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    t[k] += std::chrono::duration<double, std::milli>(n - t0).count();
    t0 = n;
  }
  ~PhaseClock() {
    if (on)
      fprintf(stderr, "[engine] lookup %.3f fixup %.3f serve %.3f defer %.3f flush-compress %.3f flush-insert %.3f "
              "serial-update %.3f index-insert %.3f ms\n", t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
  }
};

}  // namespace
}  // namespace fc

using namespace fc;

struct lc_engine {
  lc_ctx* ctx = nullptr;
  lc_engine_config cfg{};
  lc_index* ix = nullptr;
  lc_store* st = nullptr;
  lc_engine_metrics m{};
  // device staging for the deferred compressions' inputs, kept across calls:
  // a fresh ~100 MB stream-ordered allocation per flush fragmented the pool
  // against the store's entries and cost 5-190 ms of pool growth per call
  void* stage = nullptr;
  size_t stage_bytes = 0;
  void* stage_for(size_t bytes) {
    if (bytes > stage_bytes) {
      if (stage) {
        FC_CUDA(cudaStreamSynchronize(ctx->stream));
        cudaFree(stage);
        stage = nullptr;
        stage_bytes = 0;
      }
      const size_t want = std::max(bytes, bytes + bytes / 2);
      FC_CUDA(cudaMalloc(&stage, want));
      stage_bytes = want;
    }
    return stage;
  }
  ~lc_engine() {
    if (st) lc_store_destroy(st);
    if (ix) lc_index_destroy(ix);
    if (stage) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(stage);
    }
  }
};

namespace {

// Live steps of `prompt` (ascending), via the store's cached_steps.
std::vector<int> live_steps(lc_store* st, uint64_t prompt) {
  int32_t s[8];
  int n = 0;
  ok(lc_store_cached_steps(st, prompt, s, &n));
  return std::vector<int>(s, s + n);
}

// largest live step <= desired (get_step's hole rule, store.cpp:97-103), 0 if none
int avail(const std::vector<int>& live, int desired) {
  int a = 0;
  for (int s : live)
    if (s <= desired) a = s;
  return a;
}

}  // namespace

extern "C" {

void lc_engine_config_default(lc_engine_config* c) {
  if (!c) return;
  *c = lc_engine_config{};
  c->hit_threshold = 0.65;
  c->compress_threshold = 0.99;
  const double e[4] = {0.72, 0.79, 0.86, 0.93};
  memcpy(c->bin_edges, e, sizeof e);
  c->t_per_step = 4.84;
  c->t_lookup = 0.14;
  c->t_extract = 3.6;
  c->t_stitch = 0.0;
  c->total_steps = 50;
  c->policy = LC_POLICY_LRBU;
  c->capacity = ~0ull;
  c->dim = 512;
  c->F = 64, c->H = 40, c->W = 64, c->C = 4;
}

lc_status lc_engine_create(lc_ctx* ctx, const lc_engine_config* cfg, lc_engine** out) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && cfg && out, "lc_engine_create: null argument");
  FC_REQUIRE(cfg->dim > 0 && cfg->F > 0 && cfg->H > 0 && cfg->W > 0 && cfg->C > 0, "lc_engine_create: bad geometry");
  FC_REQUIRE(cfg->t_per_step >= 0 && cfg->t_lookup >= 0 && cfg->t_extract >= 0 && cfg->t_stitch >= 0,
             "LatencyModel: all times must be >= 0");
  FC_REQUIRE(cfg->total_steps >= 25, "LatencyModel: total_steps must cover the cached steps");
  auto e = std::make_unique<lc_engine>();
  e->ctx = ctx;
  e->cfg = *cfg;
  ok(lc_index_create(ctx, cfg->dim, 0, &e->ix));
  ok(lc_store_create(ctx, cfg->capacity, cfg->policy, &e->st));
  {
    // Pre-grow the device's stream-ordered pool (its release threshold keeps
    // freed memory cached, core.cu) to about what the store will hold: entry
    // arenas then carve from mapped memory instead of growing the pool inside
    // a request batch (4-30 ms per growth step measured on B200).
    DeviceGuard g(ctx->device);
    size_t free_b = 0, total_b = 0;
    FC_CUDA(cudaMemGetInfo(&free_b, &total_b));
    size_t want = cfg->capacity > 0 ? (size_t)cfg->capacity + (size_t)cfg->capacity / 4 + (1ull << 30) : (8ull << 30);
    want = std::min(want, free_b / 2);
    void* p = nullptr;
    if (want >= (64ull << 20) && cudaMallocAsync(&p, want, ctx->stream) == cudaSuccess) {
      cudaFreeAsync(p, ctx->stream);
      FC_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
      cudaGetLastError();  // reservation is best effort
    }
  }
  *out = e.release();
  LC_API_END
}

lc_status lc_engine_destroy(lc_engine* e) {
  LC_API_BEGIN
  delete e;
  LC_API_END
}

lc_index* lc_engine_index(lc_engine* e) { return e ? e->ix : nullptr; }
lc_store* lc_engine_store(lc_engine* e) { return e ? e->st : nullptr; }

lc_status lc_engine_process(lc_engine* e, const lc_request* req, int64_t n, const float* q_whole, const float* q_object,
                            const float* q_background, const float* latents, const uint8_t* obj_masks,
                            const uint8_t* bg_masks, float* served_dev, lc_outcome* out) {
  LC_API_BEGIN
  FC_REQUIRE(e && req && out && q_whole && q_object && q_background && latents && obj_masks && bg_masks,
             "lc_engine_process: null argument");
  if (n <= 0) return LC_OK;
  DeviceGuard dg(e->ctx->device);
  const lc_engine_config& c = e->cfg;
  const int d = c.dim;
  const int64_t E = (int64_t)c.H * c.W * c.C;
  const int64_t mb = ((int64_t)c.H * c.W + 7) / 8;
  if (served_dev) FC_REQUIRE(is_device_ptr(served_dev), "lc_engine_process: served_dev must be device memory");
  // queries on the host (exact fix-up dots) and as the batch lookup input
  PhaseClock pc;
  const float* qs[3] = {q_whole, q_object, q_background};
  std::vector<float> qh[3];
  for (int t = 0; t < 3; ++t) qh[t] = to_host(qs[t], (size_t)n * d);
  // ---- one exact top-K per table for the whole batch ----
  const int64_t size0 = lc_index_size(e->ix);
  std::vector<uint64_t> bid[3];
  std::vector<double> bsc[3];
  std::vector<int32_t> bcnt[3];
  for (int t = 0; t < 3; ++t) {
    bid[t].assign((size_t)n * KTOP, 0);
    bsc[t].assign((size_t)n * KTOP, 0.0);
    bcnt[t].assign((size_t)n, 0);
    if (size0 > 0)
      ok(lc_index_query_topk(e->ix, t, qh[t].data(), n, KTOP, bid[t].data(), bsc[t].data(), bcnt[t].data()));
  }
  // exact dots among the batch's queries (the rows this batch may insert)
  std::vector<double> bdots;
  if (n >= 2 && n <= 1024) {
    DevBuf dq(3 * (size_t)n * d * sizeof(float), e->ctx->stream), dD(3 * (size_t)n * n * sizeof(double), e->ctx->stream);
    const float* qd[3];
    for (int t = 0; t < 3; ++t) {
      if (is_device_ptr(qs[t])) {
        qd[t] = qs[t];
      } else {
        float* dst = dq.as<float>() + (size_t)t * n * d;
        FC_CUDA(cudaMemcpyAsync(dst, qh[t].data(), (size_t)n * d * sizeof(float), cudaMemcpyHostToDevice, e->ctx->stream));
        qd[t] = dst;
      }
    }
    const unsigned nb = (unsigned)((n + BD_T - 1) / BD_T);
    k_batch_dots<<<dim3(nb, nb, 3), BD_T * BD_T, 0, e->ctx->stream>>>(qd[0], qd[1], qd[2], (int)n, d, dD.as<double>());
    FC_LAUNCH_CHECK();
    count_launch(e->ctx);
    bdots.resize(3 * (size_t)n * n);
    FC_CUDA(cudaMemcpyAsync(bdots.data(), dD.p, dD.bytes, cudaMemcpyDeviceToHost, e->ctx->stream));
    sync(e->ctx);
  }
  pc.lap(0);
  // index changes since the batch lookup
  std::unordered_set<uint64_t> removed;                        // present at lookup time, removed since
  std::map<uint64_t, std::array<const float*, 3>> added;       // inserted since (rows in qh)
  // index inserts are batched too (lookups inside the batch score the added
  // rows exactly on the host); they reach the device index before any device
  // query (re-query) and at the end of the batch
  std::vector<uint64_t> ix_pending;
  auto index_flush = [&]() {
    if (ix_pending.empty()) return;
    const size_t m = ix_pending.size();
    std::vector<float> rows[3];
    for (int t = 0; t < 3; ++t) {
      rows[t].resize(m * d);
      for (size_t q = 0; q < m; ++q) memcpy(rows[t].data() + q * d, added.at(ix_pending[q])[t], d * sizeof(float));
    }
    ok(lc_index_insert_batch(e->ix, ix_pending.data(), rows[0].data(), rows[1].data(), rows[2].data(), (int64_t)m, d));
    ix_pending.clear();
  };
  auto index_has = [&](uint64_t p) {
    if (std::find(ix_pending.begin(), ix_pending.end(), p) != ix_pending.end()) return true;
    int32_t inx = 0;
    ok(lc_index_contains(e->ix, p, &inx));
    return inx != 0;
  };
  auto index_add = [&](uint64_t p, const float* w, const float* ob, const float* bg) {
    ix_pending.push_back(p);
    added[p] = {w, ob, bg};
  };
  auto index_remove = [&](uint64_t p) {
    auto it = std::find(ix_pending.begin(), ix_pending.end(), p);
    if (it != ix_pending.end()) ix_pending.erase(it);  // never reached the device
    else ok(lc_index_remove(e->ix, p));
    removed.insert(p);
    added.erase(p);
  };
  // ---- deferred cache updates ----
  // An update whose insert provably evicts nothing (used + an upper bound of
  // every pending entry's compressed_size fits the capacity) does not depend
  // on anything that happens to other prompts before it is applied, so the
  // compressions of such updates are batched (one lc_compress_batch per step
  // set) and inserted in request order at the next flush: when a later
  // request needs a pending prompt's store record, when a non-deferrable
  // update comes, or at the end of the batch. The store/index states equal
  // serial execution. FC_ENGINE_SERIAL=1 disables it.
  const bool defer_ok = !(getenv("FC_ENGINE_SERIAL") && atoi(getenv("FC_ENGINE_SERIAL")) == 1);
  struct Pending {
    int64_t j;
    uint64_t prompt, now;
    int first;
    bool added_ix;              // its embeddings were registered for the index at deferral
    lc_entry* ready = nullptr;  // compressed speculatively already (owned)
  };
  std::vector<Pending> pending;
  std::unordered_set<uint64_t> pending_ids;
  uint64_t pending_bound = 0;
  // compressed_size upper bound for S steps (codec.cpp:305-338 with every
  // non-first key frame stored twice: as a base diff and as an extra)
  auto size_bound = [&](int S) {
    const uint64_t fr = 2 + 4 * (uint64_t)E, F = (uint64_t)c.F;
    return 20 + (F - 1) * fr + 2 * F * (uint64_t)mb + (uint64_t)S * (1 + 4 * (uint64_t)E + 2 * F + 4 * (F - 1) + 2 + (F - 1) * fr);
  };
  const bool lat_dev = is_device_ptr(latents), om_dev = is_device_ptr(obj_masks), bm_dev = is_device_ptr(bg_masks);
  // A deferred update that cannot be stored (its compress or insert failed)
  // must not leave its prompt in the index: a later lookup would hit a prompt
  // with no store record.
  auto unregister = [&](const Pending& pd) {
    if (!pd.added_ix) return;
    int32_t cached = 0;
    ok(lc_store_contains(e->st, pd.prompt, &cached));
    if (!cached && index_has(pd.prompt)) index_remove(pd.prompt);
  };
  // lc_compress_batch of requests jobs[i] = (j, prompt) over the step set
  // kCached[first..4], inputs staged in the engine's persistent buffer
  auto compress_group = [&](const std::vector<std::pair<int64_t, uint64_t>>& jobs, int first,
                            std::vector<lc_entry*>& ents) {
    const int S = 5 - first;
    const size_t m = jobs.size(), fe = (size_t)S * c.F * E, fm = (size_t)c.F * mb;
    const size_t lat_b = (m * fe * sizeof(float) + 255) & ~size_t(255), msk_b = (m * fm + 255) & ~size_t(255);
    auto* sbase = static_cast<uint8_t*>(e->stage_for(lat_b + 2 * msk_b));
    float* dl = reinterpret_cast<float*>(sbase);
    uint8_t* dom = sbase + lat_b;
    uint8_t* dbm = dom + msk_b;
    for (size_t q = 0; q < m; ++q) {
      const int64_t j = jobs[q].first;
      FC_CUDA(cudaMemcpyAsync(dl + q * fe, latents + ((size_t)j * 5 + first) * c.F * E, fe * sizeof(float),
                              lat_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, e->ctx->stream));
      FC_CUDA(cudaMemcpyAsync(dom + q * fm, obj_masks + (size_t)j * fm, fm,
                              om_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, e->ctx->stream));
      FC_CUDA(cudaMemcpyAsync(dbm + q * fm, bg_masks + (size_t)j * fm, fm,
                              bm_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, e->ctx->stream));
    }
    std::vector<uint64_t> pids(m);
    for (size_t q = 0; q < m; ++q) pids[q] = jobs[q].second;
    ents.assign(m, nullptr);
    std::vector<int32_t> steps(kCached + first, kCached + 5);
    ok(lc_compress_batch(e->ctx, dl, steps.data(), S, c.F, c.H, c.W, c.C, dom, dbm, c.compress_threshold, pids.data(),
                         (int64_t)m, ents.data(), nullptr));
    sync(e->ctx);  // the staging buffer is reused by the next group / call
  };
  auto flush = [&]() {
    if (pending.empty()) return;
    // one compress per step set; entries in request order
    std::map<int64_t, lc_entry*> ent_of;
    for (auto& pd : pending)
      if (pd.ready) {
        ent_of[pd.j] = pd.ready;
        pd.ready = nullptr;
      }
    try {
    for (int first = 0; first < 5; ++first) {
      std::vector<const Pending*> grp;
      for (const auto& pd : pending)
        if (pd.first == first && !ent_of.count(pd.j)) grp.push_back(&pd);
      if (grp.empty()) continue;
      std::vector<std::pair<int64_t, uint64_t>> jobs;
      for (const Pending* pd : grp) jobs.emplace_back(pd->j, pd->prompt);
      std::vector<lc_entry*> ents;
      compress_group(jobs, first, ents);
      const size_t m = grp.size();
      for (size_t q = 0; q < m; ++q) ent_of[grp[q]->j] = ents[q];
    }
    } catch (...) {
      // nothing of this flush is stored: release what was compressed and take
      // the pending prompts back out of the index
      for (auto& kv : ent_of) lc_entry_release(kv.second);
      std::vector<Pending> drop;
      drop.swap(pending);
      pending_ids.clear();
      pending_bound = 0;
      for (const auto& pd : drop) unregister(pd);
      throw;
    }
    pc.lap(4);
    std::exception_ptr err = nullptr;
    for (const auto& pd : pending) {
      lc_entry* ent = ent_of[pd.j];
      if (!err) {
        const int S = 5 - pd.first;
        std::vector<int32_t> steps(kCached + pd.first, kCached + 5);
        int nev = 0;
        lc_step_entry ev1;
        const lc_status st1 = lc_store_insert(e->st, pd.prompt, ent, steps.data(), S, pd.now, &ev1, 1, &nev);
        if (st1 != LC_OK) {
          try {
            ok(st1);
          } catch (...) {
            err = std::current_exception();
          }
        } else if (nev != 0) {
          try {
            raise(LC_ERR_INTERNAL, "engine: a deferred insert evicted (size bound violated)");
          } catch (...) {
            err = std::current_exception();
          }
        }
      }
      lc_entry_release(ent);
    }
    std::vector<Pending> done;
    done.swap(pending);
    pending_ids.clear();
    pending_bound = 0;
    if (err)
      for (const auto& pd : done) unregister(pd);  // the failed insert and every later one
    pc.lap(5);
    if (err) std::rethrow_exception(err);
  };
  // ---- speculative compression of evicting updates ----
  // An update that may evict cannot be deferred (its evictions change what
  // later requests see), and compressing it alone costs ~0.45 ms. But the
  // compressed entry depends only on the request's own latents and its step
  // set, never on the store: at the first evicting update of a batch, the
  // step set of every later request is predicted from the batch lookup and
  // the current store (decide + hole rule), and all of them are compressed in
  // one batched lc_compress_batch per step set. A request whose real step
  // set matches takes its entry (bit-identical to compressing it then); any
  // other compresses alone, as before. No state is touched by a prediction,
  // so results equal serial execution; unused entries are released.
  std::unordered_map<int64_t, std::pair<int, lc_entry*>> spec;  // j -> (first, entry)
  bool speculated = false;
  auto release_spec = [&]() {
    for (auto& kv : spec) lc_entry_release(kv.second.second);
    spec.clear();
  };
  auto take_spec = [&](int64_t j, int first) -> lc_entry* {
    auto it = spec.find(j);
    if (it == spec.end()) return nullptr;
    lc_entry* ent = it->second.first == first ? it->second.second : nullptr;
    if (!ent) lc_entry_release(it->second.second);
    spec.erase(it);
    return ent;
  };
  auto speculate = [&](int64_t from) {
    speculated = true;
    std::vector<std::pair<int64_t, uint64_t>> grp[5];
    std::unordered_set<uint64_t> seen;
    for (int64_t jj = from; jj < n; ++jj) {
      const uint64_t p = req[jj].prompt;
      if (!seen.insert(p).second) continue;  // a repeated prompt is cached by its first update
      int32_t cached = pending_ids.count(p) ? 1 : 0;
      if (!cached) ok(lc_store_contains(e->st, p, &cached));
      if (cached) continue;
      uint64_t tid[3] = {0, 0, 0};
      double tsc[3] = {0, 0, 0};
      bool have[3] = {false, false, false};
      for (int t = 0; t < 3; ++t)
        for (int k = 0; k < bcnt[t][jj]; ++k)
          if (!removed.count(bid[t][(size_t)jj * KTOP + k])) {
            have[t] = true;
            tid[t] = bid[t][(size_t)jj * KTOP + k];
            tsc[t] = bsc[t][(size_t)jj * KTOP + k];
            break;
          }
      lc_decision dc{};
      dc.whole_id = tid[0];
      dc.object_id = tid[1];
      dc.background_id = tid[2];
      decide_one(tsc[0], tsc[1], tsc[2], have[0], c.hit_threshold, c.bin_edges, &dc);
      int actual = 0;
      if (dc.kind == LC_WHOLE_HIT) {
        actual = avail(live_steps(e->st, dc.whole_id), dc.step);
      } else if (dc.kind == LC_DECOUPLED_HIT) {
        const auto lo = live_steps(e->st, dc.object_id), lb = live_steps(e->st, dc.background_id);
        int m = std::min(avail(lo, dc.step), avail(lb, dc.step));
        while (m > 0 && (avail(lo, m) != m || avail(lb, m) != m)) m = std::min(avail(lo, m), avail(lb, m));
        actual = m;
      }
      if (actual >= 25) continue;
      int first = 0;
      while (first < 5 && kCached[first] <= actual) ++first;
      grp[first].emplace_back(jj, p);
    }
    for (int first = 0; first < 5; ++first) {
      if (grp[first].empty()) continue;
      std::vector<lc_entry*> ents;
      try {
        compress_group(grp[first], first, ents);
      } catch (const Error&) {
        continue;  // e.g. a non-finite latent: that request raises when it is reached
      }
      for (size_t q = 0; q < ents.size(); ++q) spec[grp[first][q].first] = {first, ents[q]};
    }
  };
  try {
  for (int64_t j = 0; j < n; ++j) {
    const lc_request& r = req[j];
    const uint64_t now = r.arrival;
    // ---- (1) top-1 per table on the current index ----
    uint64_t tid[3] = {0, 0, 0};
    double tsc[3] = {0, 0, 0};
    bool have[3] = {false, false, false};
    for (int t = 0; t < 3; ++t) {
      const float* q = qh[t].data() + (size_t)j * d;
      const int cnt = bcnt[t][j];
      int pick = -1;
      for (int k = 0; k < cnt; ++k)
        if (!removed.count(bid[t][(size_t)j * KTOP + k])) {
          pick = k;
          break;
        }
      if (pick >= 0) {
        have[t] = true;
        tid[t] = bid[t][(size_t)j * KTOP + pick];
        tsc[t] = bsc[t][(size_t)j * KTOP + pick];
      } else if (cnt == KTOP) {
        // every listed row is gone and the table had more: the current
        // index's exact top-1 is the answer (it includes the added rows)
        uint64_t i1 = 0;
        double s1 = 0;
        int32_t c1 = 0;
        index_flush();
        ok(lc_index_query_topk(e->ix, t, q, 1, 1, &i1, &s1, &c1));
        have[t] = c1 > 0;
        tid[t] = i1;
        tsc[t] = s1;
        continue;
      }
      // exact scores of the rows added since the lookup: earlier query rows
      // of this batch come from the device dot table; anything else is
      // scored here, four independent sequential chains at a time (each in
      // vindex.cpp:67 element order)
      auto it = added.begin();
      while (it != added.end()) {
        const float* x[4];
        uint64_t id[4];
        int m = 0;
        for (; m < 4 && it != added.end(); ++it) {
          const float* row = it->second[t];
          const ptrdiff_t off = row - qh[t].data();
          if (!bdots.empty() && off >= 0 && off % d == 0 && off / d < j) {
            const double s = bdots[((size_t)t * n + j) * n + off / d];
            if (!have[t] || better(s, it->first, tsc[t], tid[t])) {
              have[t] = true;
              tid[t] = it->first;
              tsc[t] = s;
            }
            continue;
          }
          x[m] = row;
          id[m] = it->first;
          ++m;
        }
        if (m == 0) continue;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < d; ++i) {
          const double qi = (double)q[i];
          for (int u = 0; u < 4; ++u)
            if (u < m) acc[u] += qi * (double)x[u][i];
        }
        for (int u = 0; u < m; ++u)
          if (!have[t] || better(acc[u], id[u], tsc[t], tid[t])) {
            have[t] = true;
            tid[t] = id[u];
            tsc[t] = acc[u];
          }
      }
    }
    pc.lap(1);
    // ---- (2) decide + similarity_to_step ----
    lc_outcome o{};
    o.decision.whole_id = tid[0];
    o.decision.object_id = tid[1];
    o.decision.background_id = tid[2];
    decide_one(tsc[0], tsc[1], tsc[2], have[0], c.hit_threshold, c.bin_edges, &o.decision);
    // ---- (3) serve ----
    if (!pending_ids.empty() &&
        ((o.decision.kind == LC_WHOLE_HIT && pending_ids.count(o.decision.whole_id)) ||
         (o.decision.kind == LC_DECOUPLED_HIT &&
          (pending_ids.count(o.decision.object_id) || pending_ids.count(o.decision.background_id)))))
      flush();
    int actual = 0;
    float* srv = served_dev ? served_dev + (size_t)j * c.F * E : nullptr;
    if (o.decision.kind == LC_WHOLE_HIT) {
      int32_t a = 0;
      ok(lc_store_get_step(e->st, o.decision.whole_id, o.decision.step, now, &a, srv));
      actual = a;
    } else if (o.decision.kind == LC_DECOUPLED_HIT) {
      // both latents must come from the same step: the largest step both
      // sources hold at or below the desired one
      const auto lo = live_steps(e->st, o.decision.object_id), lb = live_steps(e->st, o.decision.background_id);
      int m = std::min(avail(lo, o.decision.step), avail(lb, o.decision.step));
      while (m > 0 && (avail(lo, m) != m || avail(lb, m) != m)) m = std::min(avail(lo, m), avail(lb, m));
      if (m > 0) {
        int32_t a1 = 0, a2 = 0;
        ok(lc_store_get_step(e->st, o.decision.object_id, m, now, &a1, nullptr));
        ok(lc_store_get_step(e->st, o.decision.background_id, m, now, &a2, nullptr));
        FC_REQUIRE(a1 == m && a2 == m, "engine: decoupled sources changed under the stitch");
        if (srv) {
          lc_entry *oe = nullptr, *be = nullptr;
          ok(lc_store_entry(e->st, o.decision.object_id, &oe));
          ok(lc_store_entry(e->st, o.decision.background_id, &be));
          const int32_t step = m;
          ok(lc_decompress_stitch_batch(e->ctx, &oe, &be, &step, 1, srv));
        }
        actual = m;
      }
    }
    o.actual_step = actual;
    pc.lap(2);
    // ---- (4) latency model ----
    o.latency = c.t_extract + c.t_lookup + c.t_per_step * (double)(c.total_steps - actual) +
                ((o.decision.kind == LC_DECOUPLED_HIT && actual > 0) ? c.t_stitch : 0.0);
    // ---- (5) update_after_generation ----
    if (actual < 25) {
      int32_t cached = pending_ids.count(r.prompt) ? 1 : 0;
      if (!cached) ok(lc_store_contains(e->st, r.prompt, &cached));
      int first = 0;  // first inserted step index into 5..25
      while (first < 5 && kCached[first] <= actual) ++first;
      const int S = 5 - first;
      const uint64_t bound = size_bound(S);
      if (!cached && defer_ok && lc_store_used(e->st) + pending_bound + bound <= c.capacity &&
          pending_bound + bound >= pending_bound) {
        const bool add_ix = !index_has(r.prompt);
        pending.push_back(Pending{j, r.prompt, now, first, add_ix, take_spec(j, first)});
        pending_ids.insert(r.prompt);
        pending_bound += bound;
        o.n_inserted = S;
        pc.lap(3);
        if (add_ix)
          index_add(r.prompt, qh[0].data() + (size_t)j * d, qh[1].data() + (size_t)j * d, qh[2].data() + (size_t)j * d);
        pc.lap(7);
      } else if (!cached) {
        flush();  // in-order state before an insert that may evict
        if (!speculated && defer_ok) speculate(j);
        std::vector<int32_t> steps(kCached + first, kCached + 5);
        lc_entry* ent = take_spec(j, first);
        if (!ent) {
          const float* lat = latents + ((size_t)j * 5 + first) * c.F * E;
          uint64_t sz = 0;
          ok(lc_compress_batch(e->ctx, lat, steps.data(), S, c.F, c.H, c.W, c.C, obj_masks + (size_t)j * c.F * mb,
                               bg_masks + (size_t)j * c.F * mb, c.compress_threshold, &r.prompt, 1, &ent, &sz));
        }
        std::vector<lc_step_entry> ev((size_t)lc_store_step_count(e->st) + 1);
        int nev = 0;
        lc_status s1 = lc_store_insert(e->st, r.prompt, ent, steps.data(), S, now, ev.data(), (int)ev.size(), &nev);
        lc_entry_release(ent);
        const bool skipped = s1 == LC_ERR_OVERSIZED_ENTRY && c.skip_oversized;
        if (skipped) s1 = LC_OK;
        // the eviction callback: a prompt whose last step went leaves the index
        for (int k = 0; k < std::min<int>(nev, (int)ev.size()); ++k) {
          int32_t still = 0;
          ok(lc_store_contains(e->st, ev[k].prompt, &still));
          if (!still && index_has(ev[k].prompt)) index_remove(ev[k].prompt);
        }
        ok(s1);
        o.n_inserted = skipped ? 0 : S;
        o.n_evicted = nev;
        if (!skipped && !index_has(r.prompt))
          index_add(r.prompt, qh[0].data() + (size_t)j * d, qh[1].data() + (size_t)j * d, qh[2].data() + (size_t)j * d);
      }
    }
    pc.lap(6);
    // ---- (6) metrics ----
    lc_engine_metrics& M = e->m;
    ++M.requests;
    if (o.decision.kind == LC_WHOLE_HIT) ++M.whole_hits;
    else if (o.decision.kind == LC_DECOUPLED_HIT) ++M.decoupled_hits;
    else ++M.misses;
    M.skipped_hist[actual / 5] += 1;
    M.skipped_total += (uint64_t)actual;
    M.simulated_time += o.latency;
    out[j] = o;
  }
  flush();
  index_flush();
  release_spec();
  if (served_dev) sync(e->ctx);  // decoupled hits are stitched stream-ordered (lc_decompress_stitch_batch)
  } catch (...) {
    // requests before the failing one are complete: apply their updates
    try {
      flush();
      index_flush();
    } catch (...) {
    }
    release_spec();
    for (auto& pd : pending)
      if (pd.ready) lc_entry_release(pd.ready);
    throw;
  }
  LC_API_END
}

lc_status lc_engine_metrics_get(lc_engine* e, lc_engine_metrics* out) {
  LC_API_BEGIN
  FC_REQUIRE(e && out, "lc_engine_metrics_get: null argument");
  lc_engine_metrics m = e->m;
  if (m.requests) {
    m.mean_latency = m.simulated_time / (double)m.requests;
    m.computation_savings = (double)m.skipped_total / ((double)e->cfg.total_steps * (double)m.requests);
    m.throughput_vs_nocache = (double)e->cfg.total_steps * e->cfg.t_per_step / m.mean_latency;
  }
  *out = m;
  LC_API_END
}

lc_status lc_engine_report(lc_engine* e, const lc_pricing* p, lc_cost_report* out) {
  LC_API_BEGIN
  FC_REQUIRE(e && p && out, "lc_engine_report: null argument");
  if (e->m.requests == 0) raise(LC_ERR_INVALID_ARGUMENT, "report: zero requests");
  FC_REQUIRE(p->gpu_rate >= 0 && p->storage_rate >= 0 && p->provisioned_storage >= 0,
             "PricingModel: all rates must be >= 0");
  lc_engine_metrics m;
  ok(lc_engine_metrics_get(e, &m));
  lc_cost_report r{};
  r.mean_latency = m.mean_latency;
  r.gpu_cost_per_video = p->gpu_rate * m.mean_latency / 3600.0;
  r.videos_per_month = (30.0 * 24.0 * 3600.0) / m.mean_latency;
  r.storage_cost_per_video = p->provisioned_storage * p->storage_rate / r.videos_per_month;
  r.throughput_vs_nocache = m.throughput_vs_nocache;
  *out = r;
  LC_API_END
}

}  // extern "C"
