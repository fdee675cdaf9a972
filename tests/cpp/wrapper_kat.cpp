// wrapper_kat.cpp — the reference's known answers (SPEC examples)
// run through the C++ host API include/lcache_b200/lcache.hpp, i.e. the way
// a user of the reference `lcache` library calls the B200 path. Written the
// way the reference's own (absent) tests would read: same class names, same
// exception types. Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lcache_b200/lcache.hpp"

using namespace lcache;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (cond) {                                                       \
      ++g_pass;                                                       \
    } else {                                                          \
      ++g_fail;                                                       \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                 \
  } while (0)

template <class Ex, class Fn>
static bool throws(Fn&& fn) {
  try {
    fn();
  } catch (const Ex&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static Frame const_frame(FrameDims d, float v) { return Frame(d, std::vector<float>((size_t)d.elems(), v)); }

static Frame basis_frame(FrameDims d, int k) {
  std::vector<float> v((size_t)d.elems(), 0.f);
  v[(size_t)k % v.size()] = 1.f;
  return Frame(d, std::move(v));
}

static MaskSet rect_masks(int F, int h, int w, int r0, int r1, int c0, int c1) {
  std::vector<Bitmap> om, bm;
  for (int j = 0; j < F; ++j) {
    Bitmap o(h, w), b(h, w);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        const bool in = y >= r0 && y < r1 && x >= c0 && x < c1;
        o.set(y * w + x, in);
        b.set(y * w + x, !in);
      }
    om.push_back(o);
    bm.push_back(b);
  }
  return MaskSet(om, bm);
}

int main() {
  if (getenv("KAT_TRACE")) fprintf(stderr, "%s\n", "core: cosine_similarit");
  // ---- core: cosine_similarity
  {
    const std::vector<float> a{1, 2, 3}, b{4, 5, 6}, z{0, 0, 0};
    CHECK(std::fabs(cosine_similarity(a, b) - 0.9746318461970762) < 1e-15);
    CHECK(throws<std::invalid_argument>([&] { cosine_similarity(a, z); }));
    CHECK(throws<std::invalid_argument>([&] { cosine_similarity(a, std::vector<float>{1, 2}); }));
  }
  if (getenv("KAT_TRACE")) fprintf(stderr, "%s\n", "store policies");
  // ---- store policies
  {
    StepEntry e{PromptId{1}, StepId(5), 0, 0, 0, 0, 1};
    CHECK(lrbu_priority(e, 1) == 5.0);
    e.capacity = 2;
    CHECK(lrbu_priority(e, 1) == 2.5);
    StepEntry l{PromptId{1}, StepId(25), 0, 0, 0, 0, 1};
    CHECK(lcbfu_priority(l) == 25.0);
    l.step = StepId(5);
    l.f = 9;
    CHECK(lcbfu_priority(l) == 50.0);
  }
  if (getenv("KAT_TRACE")) fprintf(stderr, "%s\n", "select_keyframes");
  // ---- select_keyframes
  const FrameDims small{4, 4, 2};
  {
    std::vector<Frame> same(8, const_frame(small, 0.5f));
    CHECK(select_keyframes(LatentState(StepId(5), same), 0.99).mapping == std::vector<int>(8, 0));
    std::vector<Frame> orth;
    for (int j = 0; j < 8; ++j) orth.push_back(basis_frame(small, j));
    std::vector<int> ident(8);
    for (int j = 0; j < 8; ++j) ident[j] = j;
    CHECK(select_keyframes(LatentState(StepId(5), orth), 0.99).mapping == ident);
    std::vector<Frame> groups;
    for (int j = 0; j < 8; ++j) groups.push_back(basis_frame(small, j < 4 ? 0 : 1));
    CHECK(select_keyframes(LatentState(StepId(5), groups), 0.99).mapping == (std::vector<int>{0, 0, 0, 0, 4, 4, 4, 4}));
    CHECK(throws<std::invalid_argument>([&] { select_keyframes(LatentState(StepId(5), same), 1.5); }));
  }
  if (getenv("KAT_TRACE")) fprintf(stderr, "%s\n", "solve_alpha");
  // ---- solve_alpha
  {
    const std::vector<float> base{1, 2, 3, 4}, twice{2, 4, 6, 8}, zero{0, 0, 0, 0};
    CHECK(solve_alpha(twice, base) == 2.0f);
    CHECK(throws<DegenerateBase>([&] { solve_alpha(twice, zero); }));
  }
  if (getenv("KAT_TRACE")) fprintf(stderr, "%s\n", "codec: zero-motion");
  // ---- codec: zero-motion entry at the paper geometry
  const FrameDims dims{};  // 40 x 64 x 4
  const int F = 64;
  CHECK(uncompressed_size(dims, F, 5) == 13107200ull);
  std::vector<IntraCompressed> ics;
  std::vector<LatentState> raw;
  for (int s : defaults::kCachedSteps) {
    std::vector<Frame> fr(F, const_frame(dims, 0.25f));
    raw.emplace_back(StepId(s), fr);
    ics.push_back(intra_compress(raw.back(), defaults::kCompressThreshold));
  }
  const MaskSet masks = rect_masks(F, dims.h, dims.w, 10, 30, 16, 48);
  CompressedEntry zero = inter_compress(ics, masks, PromptId{7});
  CHECK(compressed_size(zero) == 246435ull);
  CHECK(serialize_entry(zero).size() == compressed_size(zero));
  CHECK(size_breakdown(zero).total() == compressed_size(zero));
  {
    uint64_t sum = entry_shared_bytes(zero);
    for (int s : defaults::kCachedSteps) sum += step_private_bytes(zero, StepId(s));
    CHECK(sum == compressed_size(zero));
  }
  for (int s : defaults::kCachedSteps) {
    const LatentState d = decompress_step(zero, StepId(s));
    bool exact = d.frame_count() == F;
    for (int j = 0; exact && j < F; ++j) exact = d.frames()[j] == raw[0].frames()[j];
    CHECK(exact);
  }
  CHECK(throws<StepNotCached>([&] { decompress_step(zero, StepId(30)); }));
  {  // wire round trip
    const auto bytes = serialize_entry(zero);
    CompressedEntry back = deserialize_entry(bytes);
    CHECK(serialize_entry(back) == bytes);
  }
  if (getenv("KAT_TRACE")) fprintf(stderr, "%s\n", "store: get_step hole f");
  // ---- store: get_step hole fallback + eviction callback
  {
    CacheStore st(1ull << 30, Policy::Lrbu);
    std::vector<PromptId> gone;
    st.set_eviction_callback([&](PromptId p) { gone.push_back(p); });
    CHECK(st.insert_steps(PromptId{7}, zero, {StepId(5), StepId(15)}, 1).empty());
    auto r = st.get_step(PromptId{7}, StepId(10), 2);
    CHECK(r.has_value() && r->actual == StepId(5));
    CHECK(st.used() == st.recompute_used());
    CHECK(st.cached_steps(PromptId{7}).size() == 2);
    CHECK(st.masks(PromptId{7}).has_value() && *st.masks(PromptId{7}) == masks);
    CHECK(st.evict_step(PromptId{7}, StepId(5)));
    CHECK(!st.get_step(PromptId{7}, StepId(10), 3).has_value());  // only 15 > 10 left => miss
    st.evict_one(4);
    CHECK(gone.size() == 1 && gone[0] == PromptId{7});
    CHECK(throws<std::logic_error>([&] { st.evict_one(5); }));
    CHECK(throws<std::invalid_argument>([&] { st.get_step(PromptId{7}, StepId(7), 5); }));
    CacheStore tiny(1000, Policy::Lru);
    CHECK(throws<OversizedEntry>([&] { tiny.insert_steps(PromptId{7}, zero, {StepId(5)}, 1); }));
  }
  if (getenv("KAT_TRACE")) fprintf(stderr, "%s\n", "snapshot round trip");
  // ---- snapshot: save -> load -> save is bit-exact; bad magic -> SnapshotError at 0
  {
    CacheStore st(1ull << 30, Policy::Lrbu);
    st.insert_steps(PromptId{7}, zero, {StepId(5), StepId(15)}, 1);
    SimilarityIndex ix(4);
    const std::vector<float> u{0.5f, 0.5f, 0.5f, 0.5f};
    ix.insert(Embedding::from_unit(u, EmbeddingKind::Whole), Embedding::from_unit(u, EmbeddingKind::Object),
              Embedding::from_unit(u, EmbeddingKind::Background), PromptId{7});
    const std::string p1 = "/tmp/wrapper_kat_a.flxc", p2 = "/tmp/wrapper_kat_b.flxc";
    save_snapshot(st, ix, p1);
    SnapshotData d = load_snapshot(p1);
    save_snapshot(d.store, d.index, p2);
    auto slurp = [](const std::string& p) {
      FILE* f = fopen(p.c_str(), "rb");
      std::vector<char> v;
      int c;
      while (f && (c = fgetc(f)) != EOF) v.push_back((char)c);
      if (f) fclose(f);
      return v;
    };
    const auto a = slurp(p1), b = slurp(p2);
    CHECK(!a.empty() && a == b);
    CHECK(d.store.used() == st.used() && d.index.size() == 1);
    FILE* f = fopen(p2.c_str(), "r+b");
    if (f) {
      fputc('X', f);
      fclose(f);
    }
    bool off0 = false;
    try {
      load_snapshot(p2);
    } catch (const SnapshotError& e) {
      off0 = e.byte_offset == 0;
    }
    CHECK(off0);
  }
  if (getenv("KAT_TRACE")) fprintf(stderr, "%s\n", "index: duplicates");
  // ---- index: duplicates -> smaller id, empty -> none
  {
    SimilarityIndex ix;
    std::vector<float> q(768);
    for (int i = 0; i < 768; ++i) q[i] = std::sin(0.37f * i + 1.f);
    const Embedding e(q, EmbeddingKind::Whole);
    CHECK(!ix.query_top1(EmbeddingKind::Whole, e).has_value());
    std::vector<float> o(768);
    for (int i = 0; i < 768; ++i) o[i] = std::cos(0.11f * i);
    const Embedding eo(o, EmbeddingKind::Object);
    ix.insert(e, eo, eo, PromptId{9});
    ix.insert(e, eo, eo, PromptId{4});
    ix.insert(eo, eo, eo, PromptId{2});
    auto r = ix.query_top1(EmbeddingKind::Whole, e);
    CHECK(r.has_value() && r->prompt == PromptId{4});
    CHECK(throws<std::invalid_argument>([&] { ix.insert(e, e, e, PromptId{4}); }));
    CHECK(ix.size() == 3 && ix.contains(PromptId{9}));
    ix.remove(PromptId{4});
    r = ix.query_top1(EmbeddingKind::Whole, e);
    CHECK(r.has_value() && r->prompt == PromptId{9});
    CHECK(throws<std::invalid_argument>([&] { ix.remove(PromptId{4}); }));
    const auto rows = ix.entries(EmbeddingKind::Whole);
    CHECK(rows.size() == 2 && rows[0].first == PromptId{2} && rows[1].first == PromptId{9});
    // fused lookup + decide: identical queries => whole hit at score ~1 => step 25
    std::vector<float> qw(e.values().begin(), e.values().end());
    const auto dec = lookup_decide(ix, qw, qw, qw);
    CHECK(dec.size() == 1 && dec[0].kind == LC_WHOLE_HIT && dec[0].whole_id == 9 && dec[0].step == 25);
  }
  if (getenv("KAT_TRACE")) fprintf(stderr, "%s\n", "stitch rules");
  // ---- stitch rules (a)/(b)/(c) per pixel
  {
    const FrameDims d{4, 4, 1};
    std::vector<Frame> A(1, const_frame(d, 1.f)), B(1, const_frame(d, 2.f));
    Bitmap ao(4, 4), ab(4, 4), bo(4, 4), bb(4, 4);
    ao.set(0);  // object-source object pixel
    bo.set(5);  // stale object pixel in the background source
    StitchInput in{LatentState(StepId(10), A), MaskSet({ao}, {ab}), LatentState(StepId(10), B), MaskSet({bo}, {bb})};
    const LatentState out = stitch(in);
    CHECK(out.frames()[0].values()[0] == 1.f);
    CHECK(out.frames()[0].values()[5] == 1.f);
    CHECK(out.frames()[0].values()[3] == 2.f);
    StitchInput bad{LatentState(StepId(10), A), MaskSet({ao}, {ab}), LatentState(StepId(15), B), MaskSet({bo}, {bb})};
    CHECK(throws<std::invalid_argument>([&] { stitch(bad); }));
  }
  std::printf("wrapper_kat: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
