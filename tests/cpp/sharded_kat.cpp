// sharded_kat.cpp — the entry-sharded cache through the C++ host API
// (lcache.hpp ShardedSimilarityIndex / ShardedCacheStore), the way a C++ user
// of the reference `lcache` library would shard it. Two ranks run as two
// threads of one process on the same GPU, each with its own context; the
// library's collectives go through an in-process host all-gather
// (lc_ctx_comm_host). Each rank checks the global results against an
// UNSHARDED index / store holding every prompt:
//   * top-8 ids and fp64 scores (vindex.cpp:58-72 order) and query_top1;
//   * a random insert / get_step / evict_one trace under one global capacity
//     budget: evicted StepEntry lists, actual steps, used() (store.cpp:53-176).
// Exit code 0 = all checks passed.
#include <barrier>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "lcache_b200/lcache.hpp"

using namespace lcache;

static std::atomic<int> g_fail{0}, g_pass{0};
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (cond) {                                                            \
      ++g_pass;                                                            \
    } else {                                                               \
      ++g_fail;                                                            \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)

constexpr int G = 2;

struct Hub {
  std::barrier<> bar{G};
  std::vector<std::uint8_t> slot[G];
};
struct RankUser {
  Hub* hub;
  int rank;
};

static int gather(void* user, const void* send, void* recv, std::uint64_t bytes) {
  auto* u = static_cast<RankUser*>(user);
  const auto* s = static_cast<const std::uint8_t*>(send);
  u->hub->slot[u->rank].assign(s, s + bytes);
  u->hub->bar.arrive_and_wait();
  for (int r = 0; r < G; ++r) std::memcpy(static_cast<std::uint8_t*>(recv) + (size_t)r * bytes, u->hub->slot[r].data(), bytes);
  u->hub->bar.arrive_and_wait();  // slots may be overwritten after this
  return 0;
}

static std::vector<float> unit_rows(int n, int d, std::uint64_t seed) {
  std::mt19937_64 g(seed);
  std::normal_distribution<float> nd;
  std::vector<float> v((size_t)n * d);
  for (auto& x : v) x = nd(g);
  return v;
}

static void rank_main(int rank, Hub* hub) {
  auto ctx = std::make_shared<b200::Context>(0);
  RankUser ru{hub, rank};
  b200::attach_host_transport(*ctx, G, rank, gather, &ru);

  // ---- lookup: sharded vs unsharded, same rows and queries on every rank ----
  const int n = 12000, d = 256, nq = 48;
  std::vector<float> raw = unit_rows(n, d, 7);
  std::vector<Embedding> rows;
  rows.reserve(n);
  for (int i = 0; i < n; ++i)
    rows.emplace_back(std::vector<float>(raw.begin() + (size_t)i * d, raw.begin() + (size_t)(i + 1) * d),
                      EmbeddingKind::Whole);
  rows[n - 1] = rows[3];  // exact duplicate across the shards: ties -> smaller id
  ShardedSimilarityIndex sh(d, ctx);
  SimilarityIndex full(d, ctx);
  for (int i = 0; i < n; ++i) {
    const PromptId p{(std::uint64_t)i * 3 + 1};
    sh.insert(rows[i], rows[i], rows[i], p);
    full.insert(rows[i], rows[i], rows[i], p);
  }
  b200::check(lc_index_set_lookup(sh.local().handle(), 2, 32, 0));  // tensor-core path on the shard
  b200::check(lc_index_set_lookup(full.handle(), 1, 0, 0));          // exact scan
  std::vector<float> q((size_t)nq * d);
  std::mt19937_64 g(11);
  std::normal_distribution<float> nd;
  for (int j = 0; j < nq; ++j) {
    std::vector<float> v(rows[(j * 97) % n].values().begin(), rows[(j * 97) % n].values().end());
    for (auto& x : v) x += 0.03f * nd(g);
    Embedding e(v, EmbeddingKind::Whole);
    std::memcpy(q.data() + (size_t)j * d, e.values().data(), d * sizeof(float));
  }
  std::memcpy(q.data(), rows[3].values().data(), d * sizeof(float));
  auto a = sh.query_topk(EmbeddingKind::Whole, q, 8);
  auto b = full.query_topk(EmbeddingKind::Whole, q, 8);
  bool same = a.size() == b.size();
  for (size_t j = 0; same && j < a.size(); ++j) {
    same = a[j].size() == b[j].size();
    for (size_t t = 0; same && t < a[j].size(); ++t)
      same = a[j][t].prompt.value == b[j][t].prompt.value && std::memcmp(&a[j][t].score, &b[j][t].score, 8) == 0;
  }
  CHECK(same);
  CHECK(a[0][0].prompt.value == 10 && a[0][1].prompt.value == (std::uint64_t)(n - 1) * 3 + 1);  // the tie
  auto t1 = sh.query_top1(EmbeddingKind::Object, rows[5]);
  CHECK(t1 && t1->prompt.value == 16);

  // ---- store: one global budget across the shards vs one store ----
  const int np = 24, F = 4, H = 4, W = 4, C = 2;
  const int E = H * W * C, mb = (H * W + 7) / 8;
  std::vector<std::uint64_t> seeds(np), pids(np);
  for (int i = 0; i < np; ++i) {
    seeds[i] = 500 + i;
    pids[i] = (i % 3 == 0 ? (1ull << 63) : 0) + 100 + i;  // some ids >= 2^63
  }
  std::vector<float> lat((size_t)np * 5 * F * E);
  std::vector<std::uint8_t> om((size_t)np * F * mb), bm((size_t)np * F * mb);
  b200::check(lc_synth_latents(ctx->get(), seeds.data(), np, F, H, W, C, nullptr, lat.data(), om.data(), bm.data()));
  const int32_t all_steps[5] = {5, 10, 15, 20, 25};
  std::vector<lc_entry*> eh(np, nullptr);
  std::vector<std::uint64_t> sizes(np);
  b200::check(lc_compress_batch(ctx->get(), lat.data(), all_steps, 5, F, H, W, C, om.data(), bm.data(), 0.99,
                                pids.data(), np, eh.data(), sizes.data()));
  std::vector<CompressedEntry> ents;
  for (auto* h : eh) ents.emplace_back(h, ctx);
  std::vector<std::uint64_t> srt(sizes);
  std::sort(srt.begin(), srt.end());
  const std::uint64_t cap = srt[np / 2] * 6;
  for (int policy = 0; policy < 4; ++policy) {
    ShardedCacheStore ss(cap, (Policy)policy, ctx, policy == 3 ? 2 : 0);
    CacheStore one(cap, (Policy)policy, ctx);
    std::mt19937_64 r(100 + policy);
    std::uint64_t now = 0;
    int evicted = 0;
    for (int op = 0; op < 300; ++op) {
      now += r() % 3;
      const int i = (int)(r() % np);
      const PromptId p{pids[i]};
      const int u = (int)(r() % 100);
      if (u < 45) {
        std::vector<StepId> st;
        for (int s : all_steps)
          if (r() % 2) st.emplace_back(s);
        if (st.empty()) st.emplace_back(5);
        const bool mine = (int)b200::shard_owner(p, G) == rank;
        std::string e1 = "ok", e2 = "ok";
        std::vector<StepEntry> v1, v2;
        try {
          v1 = ss.insert_steps(p, mine ? &ents[i] : nullptr, st, now);
        } catch (const OversizedEntry&) {
          e1 = "oversized";
        } catch (const std::invalid_argument&) {
          e1 = "invalid";
        }
        try {
          v2 = one.insert_steps(p, ents[i], st, now);
        } catch (const OversizedEntry&) {
          e2 = "oversized";
        } catch (const std::invalid_argument&) {
          e2 = "invalid";
        }
        CHECK(e1 == e2);
        bool eq = v1.size() == v2.size();
        for (size_t k = 0; eq && k < v1.size(); ++k)
          eq = v1[k].prompt.value == v2[k].prompt.value && v1[k].step.value() == v2[k].step.value() &&
               v1[k].f == v2[k].f && v1[k].last_access == v2[k].last_access &&
               v1[k].inserted_seq == v2[k].inserted_seq && v1[k].capacity == v2[k].capacity;
        CHECK(eq);
        if (!eq && rank == 0) {
          std::fprintf(stderr, "policy %d op %d insert %llu now %llu: sharded [", policy, op,
                       (unsigned long long)p.value, (unsigned long long)now);
          for (auto& x : v1)
            std::fprintf(stderr, " (%llu,%d,f%llu,l%llu,s%llu,c%llu)", (unsigned long long)x.prompt.value,
                         x.step.value(), (unsigned long long)x.f, (unsigned long long)x.last_access,
                         (unsigned long long)x.inserted_seq, (unsigned long long)x.capacity);
          std::fprintf(stderr, " ] single [");
          for (auto& x : v2)
            std::fprintf(stderr, " (%llu,%d,f%llu,l%llu,s%llu,c%llu)", (unsigned long long)x.prompt.value,
                         x.step.value(), (unsigned long long)x.f, (unsigned long long)x.last_access,
                         (unsigned long long)x.inserted_seq, (unsigned long long)x.capacity);
          std::fprintf(stderr, " ] used %llu / %llu\n", (unsigned long long)ss.used(), (unsigned long long)one.used());
        }
        evicted += (int)v1.size();
      } else if (u < 85) {
        const StepId want(all_steps[r() % 5]);
        const int a1 = ss.get_step(p, want, now);
        auto g2 = one.get_step(p, want, now);
        CHECK(a1 == (g2 ? g2->actual.value() : 0));
      } else {
        bool empty1 = false, empty2 = false;
        StepEntry x1, x2;
        try {
          x1 = ss.evict_one(now);
        } catch (const std::logic_error&) {
          empty1 = true;
        }
        try {
          x2 = one.evict_one(now);
        } catch (const std::logic_error&) {
          empty2 = true;
        }
        CHECK(empty1 == empty2);
        if (!empty1 && !empty2) CHECK(x1.prompt.value == x2.prompt.value && x1.inserted_seq == x2.inserted_seq);
      }
      CHECK(ss.used() == one.used());
    }
    CHECK(evicted > 0);
  }
}

int main() {
  Hub hub;
  std::vector<std::thread> th;
  for (int r = 0; r < G; ++r)
    th.emplace_back([r, &hub] {
      try {
        rank_main(r, &hub);
      } catch (const std::exception& e) {
        std::fprintf(stderr, "rank %d: %s\n", r, e.what());
        ++g_fail;
        std::exit(2);  // the other rank would wait in the all-gather forever
      }
    });
  for (auto& t : th) t.join();
  std::printf("sharded_kat: %d passed, %d failed\n", g_pass.load(), g_fail.load());
  return g_fail.load() ? 1 : 0;
}
