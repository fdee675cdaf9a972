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

#include "common.cuh"
#include "decide.cuh"

namespace fc {
namespace {

constexpr int KTOP = 8;
constexpr int kCached[5] = {5, 10, 15, 20, 25};

void ok(lc_status st) {
  if (st != LC_OK) raise(st, lc_last_error() ? lc_last_error() : "engine: library call failed");
}

// vindex.cpp:58-72: sequential fp64 dot of the fp32 query with the fp32 row
double row_dot(const float* q, const float* x, int d) {
  double acc = 0.0;
  for (int i = 0; i < d; ++i) acc += (double)q[i] * (double)x[i];
  return acc;
}

std::vector<float> to_host(const float* p, size_t n) {
  std::vector<float> h(n);
  if (n == 0) return h;
  if (is_device_ptr(p)) FC_CUDA(cudaMemcpy(h.data(), p, n * sizeof(float), cudaMemcpyDeviceToHost));
  else memcpy(h.data(), p, n * sizeof(float));
  return h;
}

}  // namespace
}  // namespace fc

using namespace fc;

struct lc_engine {
  lc_ctx* ctx = nullptr;
  lc_engine_config cfg{};
  lc_index* ix = nullptr;
  lc_store* st = nullptr;
  lc_engine_metrics m{};
  ~lc_engine() {
    if (st) lc_store_destroy(st);
    if (ix) lc_index_destroy(ix);
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
  // index changes since the batch lookup
  std::unordered_set<uint64_t> removed;                        // present at lookup time, removed since
  std::map<uint64_t, std::array<const float*, 3>> added;       // inserted since (rows in qh)
  auto index_remove = [&](uint64_t p) {
    ok(lc_index_remove(e->ix, p));
    removed.insert(p);
    added.erase(p);
  };
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
        ok(lc_index_query_topk(e->ix, t, q, 1, 1, &i1, &s1, &c1));
        have[t] = c1 > 0;
        tid[t] = i1;
        tsc[t] = s1;
        continue;
      }
      for (const auto& kv : added) {
        const double s = row_dot(q, kv.second[t], d);
        if (!have[t] || better(s, kv.first, tsc[t], tid[t])) {
          have[t] = true;
          tid[t] = kv.first;
          tsc[t] = s;
        }
      }
    }
    // ---- (2) decide + similarity_to_step ----
    lc_outcome o{};
    o.decision.whole_id = tid[0];
    o.decision.object_id = tid[1];
    o.decision.background_id = tid[2];
    decide_one(tsc[0], tsc[1], tsc[2], have[0], c.hit_threshold, c.bin_edges, &o.decision);
    // ---- (3) serve ----
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
    // ---- (4) latency model ----
    o.latency = c.t_extract + c.t_lookup + c.t_per_step * (double)(c.total_steps - actual) +
                ((o.decision.kind == LC_DECOUPLED_HIT && actual > 0) ? c.t_stitch : 0.0);
    // ---- (5) update_after_generation ----
    if (actual < 25) {
      int32_t cached = 0;
      ok(lc_store_contains(e->st, r.prompt, &cached));
      if (!cached) {
        int first = 0;  // first inserted step index into 5..25
        while (first < 5 && kCached[first] <= actual) ++first;
        const int S = 5 - first;
        std::vector<int32_t> steps(kCached + first, kCached + 5);
        const float* lat = latents + ((size_t)j * 5 + first) * c.F * E;
        lc_entry* ent = nullptr;
        uint64_t sz = 0;
        ok(lc_compress_batch(e->ctx, lat, steps.data(), S, c.F, c.H, c.W, c.C, obj_masks + (size_t)j * c.F * mb,
                             bg_masks + (size_t)j * c.F * mb, c.compress_threshold, &r.prompt, 1, &ent, &sz));
        std::vector<lc_step_entry> ev((size_t)lc_store_step_count(e->st) + 1);
        int nev = 0;
        const lc_status s1 = lc_store_insert(e->st, r.prompt, ent, steps.data(), S, now, ev.data(), (int)ev.size(), &nev);
        lc_entry_release(ent);
        // the eviction callback: a prompt whose last step went leaves the index
        for (int k = 0; k < std::min<int>(nev, (int)ev.size()); ++k) {
          int32_t still = 0;
          ok(lc_store_contains(e->st, ev[k].prompt, &still));
          int32_t inx = 0;
          ok(lc_index_contains(e->ix, ev[k].prompt, &inx));
          if (!still && inx) index_remove(ev[k].prompt);
        }
        ok(s1);
        o.n_inserted = S;
        o.n_evicted = nev;
        int32_t inx = 0;
        ok(lc_index_contains(e->ix, r.prompt, &inx));
        if (!inx) {
          const float* w = qh[0].data() + (size_t)j * d;
          const float* ob = qh[1].data() + (size_t)j * d;
          const float* bg = qh[2].data() + (size_t)j * d;
          ok(lc_index_insert(e->ix, r.prompt, w, ob, bg, d));
          added[r.prompt] = {w, ob, bg};
        }
      }
    }
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
