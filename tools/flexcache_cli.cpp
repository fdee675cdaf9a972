// flexcache — batch front-end over the B200 library (the
// reference's missing cli module): trace generation,
// simulation runs, policy benchmarks and codec round-trip reports.
//
//   flexcache gen-trace --out trace.jsonl [--requests N] [--objects 50] [--backgrounds 40]
//                       [--zipf 1.0] [--decay 0] [--dim 512] [--seed 1]
//   flexcache simulate --trace trace.jsonl [--capacity-bytes B] [--policy lrbu|lru|fifo|lcbfu|all]
//                      [--hit-threshold 0.65] [--compress-threshold 0.99] [--bins a,b,c,d]
//                      [--gpu-rate 3.67] [--storage-rate 0] [--storage-gb 0] [--frames 16]
//                      [--height 40] [--width 64] [--channels 4] [--batch 64] [--out DIR]
//   flexcache bench-policies --trace trace.jsonl --capacities 1e6,1e7,1e8 [...] [--out DIR]
//   flexcache codec [--prompts 4] [--frames 64] [--height 40] [--width 64] [--channels 4]
//                   [--redundancy r5,r10,r15,r20,r25] [--noise 0.01] [--zero-motion] [--seed 1]
//
// Exit codes: 0 success, 1 usage, 2 data/format error, 3 internal.
// Everything is deterministic under a fixed seed; outputs are byte-stable.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "flexcache_b200.h"

namespace {

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ok(lc_status s) {
  if (s == LC_OK) return;
  const std::string m = lc_last_error() ? lc_last_error() : "";
  if (s == LC_ERR_INVALID_ARGUMENT || s == LC_ERR_SNAPSHOT || s == LC_ERR_IO || s == LC_ERR_OVERSIZED_ENTRY)
    throw DataError(m);
  throw std::runtime_error(m);
}

// rng.hpp:25-31 (counter-based streams, as in csrc/simgen.cu)
uint64_t hc(uint64_t a, uint64_t b) {
  uint64_t z = a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2));
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
double unif(uint64_t s, uint64_t i) { return (double)(hc(s, i) >> 11) * 0x1.0p-53; }

struct Args {
  std::map<std::string, std::string> kv;
  std::vector<std::string> flags;
  std::string get(const std::string& k, const std::string& d) const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  double num(const std::string& k, double d) const {
    auto it = kv.find(k);
    if (it == kv.end()) return d;
    char* end = nullptr;
    const double v = strtod(it->second.c_str(), &end);
    if (!end || *end) throw Usage("--" + k + ": not a number: " + it->second);
    return v;
  }
  bool has(const std::string& f) const { return std::find(flags.begin(), flags.end(), f) != flags.end(); }
};

Args parse(int argc, char** argv, int from, const std::vector<std::string>& known_flags) {
  Args a;
  for (int i = from; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) throw Usage("unexpected argument: " + s);
    s = s.substr(2);
    if (std::find(known_flags.begin(), known_flags.end(), s) != known_flags.end()) {
      a.flags.push_back(s);
      continue;
    }
    if (i + 1 >= argc) throw Usage("--" + s + " needs a value");
    a.kv[s] = argv[++i];
  }
  return a;
}

std::vector<double> csv_nums(const std::string& s) {
  std::vector<double> v;
  std::stringstream ss(s);
  std::string t;
  while (std::getline(ss, t, ',')) v.push_back(strtod(t.c_str(), nullptr));
  return v;
}

// ---------------------------------------------------------------------------
// trace: object x background template grid, Zipf(s)
// popularity over a ranking that is reshuffled every `decay` requests.
// ---------------------------------------------------------------------------
struct Record {
  uint64_t prompt, arrival, latent_seed;
  std::vector<uint64_t> obj, bg;
};

int cmd_gen_trace(const Args& a) {
  const std::string out = a.get("out", "");
  if (out.empty()) throw Usage("gen-trace: --out is required");
  const int64_t n = (int64_t)a.num("requests", 1000);
  const int no = (int)a.num("objects", 50), nb = (int)a.num("backgrounds", 40);
  const double zs = a.num("zipf", 1.0);
  const int64_t decay = (int64_t)a.num("decay", 0);
  const int dim = (int)a.num("dim", 512);
  const uint64_t seed = (uint64_t)a.num("seed", 1);
  if (n < 1 || no < 1 || nb < 1 || dim < 1 || decay < 0) throw Usage("gen-trace: counts must be >= 1");
  if (!(zs >= 0.0)) throw Usage("gen-trace: --zipf must be >= 0");
  const int64_t nt = (int64_t)no * nb;
  std::vector<double> cdf(nt);
  double acc = 0.0;
  for (int64_t r = 0; r < nt; ++r) cdf[r] = (acc += 1.0 / std::pow((double)(r + 1), zs));
  std::vector<int64_t> rank(nt);  // popularity rank -> template
  for (int64_t t = 0; t < nt; ++t) rank[t] = t;
  auto reshuffle = [&](uint64_t epoch) {
    for (int64_t t = nt - 1; t >= 1; --t) std::swap(rank[t], rank[hc(hc(seed, 0x5eed0000 + epoch), t) % (t + 1)]);
  };
  reshuffle(0);
  FILE* f = fopen(out.c_str(), "wb");
  if (!f) throw DataError("cannot open " + out);
  fprintf(f,
          "{\"format\":\"flexcache-trace\",\"version\":1,\"n_requests\":%lld,\"n_objects\":%d,\"n_backgrounds\":%d,"
          "\"zipf_s\":%.17g,\"decay_half_life\":%lld,\"embed_dim\":%d,\"seed\":%llu}\n",
          (long long)n, no, nb, zs, (long long)decay, dim, (unsigned long long)seed);
  for (int64_t r = 0; r < n; ++r) {
    if (decay > 0 && r > 0 && r % decay == 0) reshuffle((uint64_t)(r / decay));
    const double u = unif(hc(seed, 0x7a1f), (uint64_t)r) * acc;
    const int64_t k = std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
    const int64_t tpl = rank[std::min<int64_t>(k, nt - 1)];
    const int64_t oi = tpl / nb, bi = tpl % nb;
    const uint64_t o0 = hc(hc(seed, 0x0b1), oi), b0 = hc(hc(seed, 0xb9), bi);
    fprintf(f,
            "{\"prompt\":%lld,\"arrival\":%lld,\"object\":[%llu,%llu],\"background\":[%llu,%llu],"
            "\"latent_seed\":%llu}\n",
            (long long)tpl, (long long)(r + 1), (unsigned long long)hc(o0, 1), (unsigned long long)hc(o0, 2),
            (unsigned long long)hc(b0, 1), (unsigned long long)hc(b0, 2),
            (unsigned long long)hc(seed ^ 0x1a7e47, (uint64_t)tpl));
  }
  if (fclose(f) != 0) throw DataError("write failed: " + out);
  return 0;
}

// minimal JSONL reader for the schema above (line numbers in errors)
uint64_t jnum(const std::string& line, const char* key, size_t lineno) {
  const std::string k = std::string("\"") + key + "\":";
  const size_t p = line.find(k);
  if (p == std::string::npos) throw DataError("trace line " + std::to_string(lineno) + ": missing " + key);
  return strtoull(line.c_str() + p + k.size(), nullptr, 10);
}
std::vector<uint64_t> jarr(const std::string& line, const char* key, size_t lineno) {
  const std::string k = std::string("\"") + key + "\":[";
  const size_t p = line.find(k);
  if (p == std::string::npos) throw DataError("trace line " + std::to_string(lineno) + ": missing " + key);
  std::vector<uint64_t> v;
  const char* c = line.c_str() + p + k.size();
  while (*c && *c != ']') {
    char* e = nullptr;
    v.push_back(strtoull(c, &e, 10));
    if (e == c) throw DataError("trace line " + std::to_string(lineno) + ": bad " + key);
    c = e;
    if (*c == ',') ++c;
  }
  if (v.empty() || v.size() > 8) throw DataError("trace line " + std::to_string(lineno) + ": 1..8 tokens per set");
  return v;
}

std::vector<Record> read_trace(const std::string& path, int* dim) {
  std::ifstream in(path);
  if (!in) throw DataError("cannot open trace " + path);
  std::string line;
  size_t lineno = 1;
  if (!std::getline(in, line) || line.find("\"flexcache-trace\"") == std::string::npos)
    throw DataError("trace line 1: missing flexcache-trace header");
  *dim = (int)jnum(line, "embed_dim", 1);
  std::vector<Record> out;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    Record r;
    r.prompt = jnum(line, "prompt", lineno);
    r.arrival = jnum(line, "arrival", lineno);
    r.latent_seed = jnum(line, "latent_seed", lineno);
    r.obj = jarr(line, "object", lineno);
    r.bg = jarr(line, "background", lineno);
    out.push_back(std::move(r));
  }
  return out;
}

// ---------------------------------------------------------------------------
// simulate
// ---------------------------------------------------------------------------
struct SimResult {
  lc_engine_metrics m;
  lc_cost_report cost;
  std::vector<lc_outcome> outs;
};

int policy_of(const std::string& p) {  // parse_policy (store.cpp:13-19)
  if (p == "fifo") return LC_POLICY_FIFO;
  if (p == "lru") return LC_POLICY_LRU;
  if (p == "lcbfu") return LC_POLICY_LCBFU;
  if (p == "lrbu") return LC_POLICY_LRBU;
  throw Usage("unknown policy: " + p);
}

SimResult run_sim(lc_ctx* ctx, const std::vector<Record>& tr, int dim, const Args& a, int policy, uint64_t capacity) {
  lc_engine_config c;
  lc_engine_config_default(&c);
  c.hit_threshold = a.num("hit-threshold", c.hit_threshold);
  c.compress_threshold = a.num("compress-threshold", c.compress_threshold);
  if (a.kv.count("bins")) {
    const auto b = csv_nums(a.get("bins", ""));
    if (b.size() != 4) throw Usage("--bins needs 4 comma-separated edges");
    for (int i = 0; i < 4; ++i) c.bin_edges[i] = b[i];
  }
  c.policy = policy;
  c.capacity = capacity;
  c.dim = dim;
  c.F = (int)a.num("frames", 16);
  c.H = (int)a.num("height", 40);
  c.W = (int)a.num("width", 64);
  c.C = (int)a.num("channels", 4);
  c.skip_oversized = 1;
  lc_engine* eng = nullptr;
  ok(lc_engine_create(ctx, &c, &eng));
  const int64_t B = std::max<int64_t>(1, (int64_t)a.num("batch", 64));
  const int64_t E = (int64_t)c.H * c.W * c.C, mb = ((int64_t)c.H * c.W + 7) / 8;
  const uint64_t eseed = (uint64_t)a.num("seed", 1);
  float *qw, *qo, *qb, *lat;
  uint8_t *om, *bm;
  const size_t nq = (size_t)B * dim;
  if (cudaMalloc(&qw, nq * 4) || cudaMalloc(&qo, nq * 4) || cudaMalloc(&qb, nq * 4) ||
      cudaMalloc(&lat, (size_t)B * 5 * c.F * E * 4) || cudaMalloc(&om, (size_t)B * c.F * mb) ||
      cudaMalloc(&bm, (size_t)B * c.F * mb))
    throw std::runtime_error("device allocation failed");
  SimResult res;
  res.outs.resize(tr.size());
  for (size_t j0 = 0; j0 < tr.size(); j0 += (size_t)B) {
    const int64_t m = (int64_t)std::min<size_t>((size_t)B, tr.size() - j0);
    std::vector<uint64_t> tw(m * 16, 0), to(m * 16, 0), tb(m * 16, 0), seeds(m);
    std::vector<int32_t> nw(m), no(m), nbk(m);
    std::vector<lc_request> req(m);
    for (int64_t q = 0; q < m; ++q) {
      const Record& r = tr[j0 + q];
      int k = 0;
      for (uint64_t t : r.obj) tw[q * 16 + k++] = t;
      for (uint64_t t : r.bg) tw[q * 16 + k++] = t;  // whole = object u background
      nw[q] = k;
      for (size_t i = 0; i < r.obj.size(); ++i) to[q * 16 + i] = r.obj[i];
      no[q] = (int)r.obj.size();
      for (size_t i = 0; i < r.bg.size(); ++i) tb[q * 16 + i] = r.bg[i];
      nbk[q] = (int)r.bg.size();
      seeds[q] = r.latent_seed;
      req[q] = lc_request{r.prompt, r.arrival};
    }
    ok(lc_synth_embeddings(ctx, tw.data(), nw.data(), 16, m, dim, eseed, qw));
    ok(lc_synth_embeddings(ctx, to.data(), no.data(), 16, m, dim, eseed, qo));
    ok(lc_synth_embeddings(ctx, tb.data(), nbk.data(), 16, m, dim, eseed, qb));
    ok(lc_synth_latents(ctx, seeds.data(), m, c.F, c.H, c.W, c.C, nullptr, lat, om, bm));
    ok(lc_engine_process(eng, req.data(), m, qw, qo, qb, lat, om, bm, nullptr, res.outs.data() + j0));
  }
  ok(lc_engine_metrics_get(eng, &res.m));
  lc_pricing p{a.num("gpu-rate", 3.67), a.num("storage-rate", 0.0), a.num("storage-gb", 0.0)};
  ok(lc_engine_report(eng, &p, &res.cost));
  cudaFree(qw), cudaFree(qo), cudaFree(qb), cudaFree(lat), cudaFree(om), cudaFree(bm);
  lc_engine_destroy(eng);
  return res;
}

std::string metrics_json(const SimResult& r, const char* policy, uint64_t capacity) {
  const lc_engine_metrics& m = r.m;
  char buf[2048];
  snprintf(buf, sizeof buf,
           "{\"policy\":\"%s\",\"capacity_bytes\":%llu,\"requests\":%llu,\"whole_hits\":%llu,\"decoupled_hits\":%llu,"
           "\"misses\":%llu,\"hit_rate\":%.17g,\"skipped_hist\":{\"0\":%llu,\"5\":%llu,\"10\":%llu,\"15\":%llu,"
           "\"20\":%llu,\"25\":%llu},\"computation_savings\":%.17g,\"simulated_time\":%.17g,\"mean_latency\":%.17g,"
           "\"throughput_vs_nocache\":%.17g,\"gpu_cost_per_video\":%.17g,\"storage_cost_per_video\":%.17g}",
           policy, (unsigned long long)capacity, (unsigned long long)m.requests, (unsigned long long)m.whole_hits,
           (unsigned long long)m.decoupled_hits, (unsigned long long)m.misses,
           (double)(m.whole_hits + m.decoupled_hits) / (double)std::max<uint64_t>(1, m.requests),
           (unsigned long long)m.skipped_hist[0], (unsigned long long)m.skipped_hist[1],
           (unsigned long long)m.skipped_hist[2], (unsigned long long)m.skipped_hist[3],
           (unsigned long long)m.skipped_hist[4], (unsigned long long)m.skipped_hist[5], m.computation_savings,
           m.simulated_time, m.mean_latency, m.throughput_vs_nocache, r.cost.gpu_cost_per_video,
           r.cost.storage_cost_per_video);
  return buf;
}

const char* kind_name(int k) { return k == LC_WHOLE_HIT ? "whole" : k == LC_DECOUPLED_HIT ? "decoupled" : "miss"; }
const char* policy_name(int p) {
  return p == LC_POLICY_FIFO ? "fifo" : p == LC_POLICY_LRU ? "lru" : p == LC_POLICY_LCBFU ? "lcbfu" : "lrbu";
}

int cmd_simulate(lc_ctx* ctx, const Args& a) {
  const std::string tp = a.get("trace", "");
  if (tp.empty()) throw Usage("simulate: --trace is required");
  int dim = 0;
  const auto tr = read_trace(tp, &dim);
  if (tr.empty()) throw DataError("trace has no requests");
  const uint64_t cap = (uint64_t)a.num("capacity-bytes", 1e18);
  const std::string pol = a.get("policy", "lrbu");
  std::vector<int> pols;
  if (pol == "all") pols = {LC_POLICY_FIFO, LC_POLICY_LRU, LC_POLICY_LCBFU, LC_POLICY_LRBU};  // four-policy sweep
  else pols = {policy_of(pol)};
  const std::string outd = a.get("out", "");
  if (!outd.empty()) mkdir(outd.c_str(), 0755);
  std::string all = "[";
  for (size_t pi = 0; pi < pols.size(); ++pi) {
    const SimResult r = run_sim(ctx, tr, dim, a, pols[pi], cap);
    all += (pi ? "," : "") + metrics_json(r, policy_name(pols[pi]), cap);
    if (!outd.empty()) {
      const std::string base = outd + "/" + policy_name(pols[pi]);
      FILE* f = fopen((base + "_requests.csv").c_str(), "wb");
      if (!f) throw DataError("cannot write " + base + "_requests.csv");
      fprintf(f, "prompt,arrival,decision,score,desired_step,actual_step,latency,inserted,evicted\n");
      for (size_t j = 0; j < tr.size(); ++j) {
        const lc_outcome& o = r.outs[j];
        fprintf(f, "%llu,%llu,%s,%.17g,%d,%d,%.17g,%d,%d\n", (unsigned long long)tr[j].prompt,
                (unsigned long long)tr[j].arrival, kind_name(o.decision.kind), o.decision.score, o.decision.step,
                o.actual_step, o.latency, o.n_inserted, o.n_evicted);
      }
      fclose(f);
      // rolling throughput per 1,000 requests (Fig. 12's granularity)
      f = fopen((base + "_rolling.csv").c_str(), "wb");
      if (!f) throw DataError("cannot write " + base + "_rolling.csv");
      fprintf(f, "window_end,mean_latency,throughput_vs_nocache\n");
      const double nocache = 50.0 * 4.84;
      for (size_t w0 = 0; w0 < tr.size(); w0 += 1000) {
        const size_t w1 = std::min(tr.size(), w0 + 1000);
        double s = 0.0;
        for (size_t j = w0; j < w1; ++j) s += r.outs[j].latency;
        const double ml = s / (double)(w1 - w0);
        fprintf(f, "%zu,%.17g,%.17g\n", w1, ml, nocache / ml);
      }
      fclose(f);
    }
  }
  all += "]";
  printf("%s\n", all.c_str());
  if (!outd.empty()) {
    FILE* f = fopen((outd + "/metrics.json").c_str(), "wb");
    if (!f) throw DataError("cannot write metrics.json");
    fprintf(f, "%s\n", all.c_str());
    fclose(f);
  }
  return 0;
}

int cmd_bench_policies(lc_ctx* ctx, const Args& a) {
  const std::string tp = a.get("trace", "");
  if (tp.empty() || !a.kv.count("capacities")) throw Usage("bench-policies: --trace and --capacities are required");
  int dim = 0;
  const auto tr = read_trace(tp, &dim);
  const auto caps = csv_nums(a.get("capacities", ""));
  std::string csv = "capacity_bytes,policy,hit_rate,computation_savings,throughput_vs_nocache\n";
  for (double cd : caps)
    for (int p : {LC_POLICY_FIFO, LC_POLICY_LRU, LC_POLICY_LCBFU, LC_POLICY_LRBU}) {
      const SimResult r = run_sim(ctx, tr, dim, a, p, (uint64_t)cd);
      char line[256];
      snprintf(line, sizeof line, "%llu,%s,%.17g,%.17g,%.17g\n", (unsigned long long)cd, policy_name(p),
               (double)(r.m.whole_hits + r.m.decoupled_hits) / (double)r.m.requests, r.m.computation_savings,
               r.m.throughput_vs_nocache);
      csv += line;
    }
  printf("%s", csv.c_str());
  const std::string outd = a.get("out", "");
  if (!outd.empty()) {
    mkdir(outd.c_str(), 0755);
    FILE* f = fopen((outd + "/policies.csv").c_str(), "wb");
    if (!f) throw DataError("cannot write policies.csv");
    fputs(csv.c_str(), f);
    fclose(f);
  }
  return 0;
}

// ---------------------------------------------------------------------------
// codec round trip: ratio, per-step similarity, size
// breakdown in Fig. 10's categories (codec.cpp:305-356 accounting)
// ---------------------------------------------------------------------------
int cmd_codec(lc_ctx* ctx, const Args& a) {
  const int n = (int)a.num("prompts", 4), F = (int)a.num("frames", 64);
  const int H = (int)a.num("height", 40), W = (int)a.num("width", 64), C = (int)a.num("channels", 4);
  if (n < 1 || F < 1 || H < 1 || W < 1 || C < 1) throw Usage("codec: sizes must be >= 1");
  lc_latent_spec sp;
  lc_latent_spec_default(&sp);
  if (a.kv.count("redundancy")) {
    const auto r = csv_nums(a.get("redundancy", ""));
    if (r.size() != 5) throw Usage("--redundancy needs 5 values");
    for (int i = 0; i < 5; ++i) sp.redundancy[i] = r[i];
  }
  sp.noise_sigma = a.num("noise", sp.noise_sigma);
  const bool zero = a.has("zero-motion");
  if (zero) {  // every frame of a step equals its first frame
    for (int i = 0; i < 5; ++i) sp.redundancy[i] = 1.0;
    sp.dup_noise = 0.0;
  }
  const int64_t E = (int64_t)H * W * C, mb = ((int64_t)H * W + 7) / 8;
  std::vector<uint64_t> seeds(n);
  for (int i = 0; i < n; ++i) seeds[i] = hc((uint64_t)a.num("seed", 1), (uint64_t)i);
  float *lat, *dec;
  uint8_t *om, *bm;
  if (cudaMalloc(&lat, (size_t)n * 5 * F * E * 4) || cudaMalloc(&dec, (size_t)n * F * E * 4) ||
      cudaMalloc(&om, (size_t)n * F * mb) || cudaMalloc(&bm, (size_t)n * F * mb))
    throw std::runtime_error("device allocation failed");
  ok(lc_synth_latents(ctx, seeds.data(), n, F, H, W, C, &sp, lat, om, bm));
  const int32_t steps[5] = {5, 10, 15, 20, 25};
  std::vector<lc_entry*> ents(n);
  std::vector<uint64_t> sizes(n), prompts(n);
  for (int i = 0; i < n; ++i) prompts[i] = (uint64_t)i + 1;
  ok(lc_compress_batch(ctx, lat, steps, 5, F, H, W, C, om, bm, a.num("compress-threshold", 0.99), prompts.data(), n,
                       ents.data(), sizes.data()));
  double sims[5] = {0, 0, 0, 0, 0};
  std::vector<double> cs((size_t)n * F);
  std::vector<float> orig((size_t)n * F * E);
  for (int s = 0; s < 5; ++s) {
    std::vector<int32_t> st(n, steps[s]);
    ok(lc_decompress_batch(ctx, ents.data(), st.data(), n, dec));
    ok(lc_ctx_synchronize(ctx));  // stream-ordered output; cudaMemcpy below is on the legacy stream
    for (int i = 0; i < n; ++i)
      cudaMemcpy(orig.data() + (size_t)i * F * E, lat + ((size_t)i * 5 + s) * F * E, (size_t)F * E * 4,
                 cudaMemcpyDeviceToHost);
    std::vector<float> d((size_t)n * F * E);
    cudaMemcpy(d.data(), dec, d.size() * 4, cudaMemcpyDeviceToHost);
    ok(lc_cosine_batch(ctx, d.data(), orig.data(), (int64_t)n * F, E, cs.data()));
    double acc = 0.0;
    for (double v : cs) acc += v;
    sims[s] = acc / (double)cs.size();
  }
  uint64_t raw = (uint64_t)n * 5 * F * E * 4, comp = 0, shared = 0, priv = 0, diffs = 0, extras = 0, firsts = 0;
  for (int i = 0; i < n; ++i) {
    lc_entry_info inf;
    ok(lc_entry_get_info(ents[i], &inf));
    comp += inf.compressed_size;
    shared += inf.shared_bytes;
    for (int s = 0; s < inf.n_steps; ++s) {
      priv += inf.private_bytes[s];
      extras += (uint64_t)inf.n_extra[s] * (2 + 4 * (uint64_t)E);
      firsts += 4 * (uint64_t)E;
    }
    diffs += (uint64_t)inf.n_diff * (2 + 4 * (uint64_t)E);
    lc_entry_release(ents[i]);
  }
  printf("{\"prompts\":%d,\"frames\":%d,\"dims\":[%d,%d,%d],\"zero_motion\":%s,\"raw_bytes\":%llu,"
         "\"compressed_bytes\":%llu,\"ratio\":%.6f,\"similarity\":{\"5\":%.9f,\"10\":%.9f,\"15\":%.9f,\"20\":%.9f,"
         "\"25\":%.9f},\"breakdown\":{\"first_frames\":%llu,\"extra_frames\":%llu,\"base_diffs\":%llu,"
         "\"masks\":%llu,\"shared_total\":%llu,\"private_total\":%llu}}\n",
         n, F, H, W, C, zero ? "true" : "false", (unsigned long long)raw, (unsigned long long)comp,
         (double)raw / (double)comp, sims[0], sims[1], sims[2], sims[3], sims[4], (unsigned long long)firsts,
         (unsigned long long)extras, (unsigned long long)diffs, (unsigned long long)(2ull * F * mb * n),
         (unsigned long long)shared, (unsigned long long)priv);
  cudaFree(lat), cudaFree(dec), cudaFree(om), cudaFree(bm);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const char* usage =
      "usage: flexcache {gen-trace|simulate|bench-policies|codec} [--flag value ...]\n"
      "  see the header of tools/flexcache_cli.cpp for the flags\n";
  if (argc < 2) {
    fputs(usage, stderr);
    return 1;
  }
  const std::string cmd = argv[1];
  lc_ctx* ctx = nullptr;
  try {
    const Args a = parse(argc, argv, 2, {"zero-motion"});
    if (cmd == "gen-trace") return cmd_gen_trace(a);
    if (cmd != "simulate" && cmd != "bench-policies" && cmd != "codec") throw Usage("unknown command: " + cmd);
    if (cmd != "codec") {  // data errors before touching the device
      const std::string tp = a.get("trace", "");
      if (tp.empty()) throw Usage(cmd + ": --trace is required");
      std::ifstream probe(tp);
      if (!probe) throw DataError("cannot open trace " + tp);
    }
    ok(lc_ctx_create(0, &ctx));
    int rc = 0;
    if (cmd == "simulate") rc = cmd_simulate(ctx, a);
    else if (cmd == "bench-policies") rc = cmd_bench_policies(ctx, a);
    else rc = cmd_codec(ctx, a);
    lc_ctx_destroy(ctx);
    return rc;
  } catch (const Usage& e) {
    fprintf(stderr, "flexcache: %s\n%s", e.what(), usage);
    return 1;
  } catch (const DataError& e) {
    fprintf(stderr, "flexcache: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    fprintf(stderr, "flexcache: internal error: %s\n", e.what());
    return 3;
  }
}
