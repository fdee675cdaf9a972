// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library (lcache, compiled from
// /root/reference/proj/src by oracle/Makefile). It only marshals flat buffers
// into the reference's own types and calls its public API; no algorithm is
// restated here. Used (a) to validate the plain-C restatement oracle/lc_oracle.c,
// (b) to generate the golden fixtures under tests/golden/, and (c) as the
// "reference" CPU arm of bench.py (kind "reference").
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "lcache/codec.hpp"
#include "lcache/core.hpp"
#include "lcache/errors.hpp"
#include "lcache/serialize.hpp"
#include "lcache/stitcher.hpp"
#include "lcache/store.hpp"
#include "lcache/vindex.hpp"
#include "oracle_abi.h"

using namespace lcache;

namespace {
thread_local std::string g_err;
thread_local uint64_t g_snap_off = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const DegenerateBase& e) {
    g_err = e.what();
    return ORC_ERR_DEGENERATE_BASE;
  } catch (const StepNotCached& e) {
    g_err = e.what();
    return ORC_ERR_STEP_NOT_CACHED;
  } catch (const OversizedEntry& e) {
    g_err = e.what();
    return ORC_ERR_OVERSIZED_ENTRY;
  } catch (const SnapshotError& e) {
    g_err = e.what();
    g_snap_off = e.byte_offset;
    return ORC_ERR_SNAPSHOT;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORC_ERR_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return ORC_ERR_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_ERR_INTERNAL;
  }
}

FrameDims dims_of(int H, int W, int C) { return FrameDims{H, W, C}; }

LatentState make_latent(const float* p, int step, int F, const FrameDims& d) {
  std::vector<Frame> frames;
  frames.reserve(F);
  const size_t E = static_cast<size_t>(d.elems());
  for (int j = 0; j < F; ++j)
    frames.emplace_back(d, std::vector<float>(p + j * E, p + (j + 1) * E));
  return LatentState(StepId(step), std::move(frames));
}

MaskSet make_masks(const uint8_t* obj, const uint8_t* bg, int F, int H, int W) {
  const size_t mb = (static_cast<size_t>(H) * W + 7) / 8;
  std::vector<Bitmap> o, b;
  for (int j = 0; j < F; ++j) {
    o.emplace_back(H, W, std::vector<uint8_t>(obj + j * mb, obj + (j + 1) * mb));
    b.emplace_back(H, W, std::vector<uint8_t>(bg + j * mb, bg + (j + 1) * mb));
  }
  return MaskSet(std::move(o), std::move(b));
}

std::vector<uint8_t> compress_one(const float* lat, const int32_t* steps, int S, int F,
                                  const FrameDims& d, const uint8_t* om, const uint8_t* bm,
                                  double thr, uint64_t prompt) {
  const size_t step_elems = static_cast<size_t>(F) * d.elems();
  std::vector<IntraCompressed> ics;
  for (int s = 0; s < S; ++s)
    ics.push_back(intra_compress(make_latent(lat + s * step_elems, steps[s], F, d), thr));
  CompressedEntry e = inter_compress(ics, make_masks(om, bm, F, d.h, d.w), PromptId{prompt});
  ByteWriter w;
  serialize_entry(e, w);
  if (w.size() != compressed_size(e)) throw std::logic_error("size accounting mismatch");
  return w.take();
}

CompressedEntry parse_entry(const uint8_t* p, uint64_t len) {
  ByteReader r(std::span<const uint8_t>(p, len));
  CompressedEntry e = deserialize_entry(r);
  if (!r.at_end()) throw SnapshotError("trailing bytes", r.pos());
  return e;
}

void put_step_entry(const StepEntry& s, orc_step_entry* o) {
  o->prompt = s.prompt.value;
  o->step = s.step.value();
  o->_pad = 0;
  o->f = s.f;
  o->last_access = s.last_access;
  o->inserted_at = s.inserted_at;
  o->inserted_seq = s.inserted_seq;
  o->capacity = s.capacity;
}

StepEntry get_step_entry(const orc_step_entry* o) {
  StepEntry s{PromptId{o->prompt}, StepId(o->step), o->f, o->last_access,
              o->inserted_at, o->inserted_seq, o->capacity};
  return s;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_normalize(const float* v, int d, float* out) {
  return guard([&] {
    Embedding e(std::vector<float>(v, v + d), EmbeddingKind::Whole);
    std::memcpy(out, e.values().data(), sizeof(float) * d);
  });
}

int ref_cosine(const float* a, const float* b, int64_t n, double* out) {
  return guard([&] {
    *out = cosine_similarity(std::span<const float>(a, n), std::span<const float>(b, n));
  });
}

void* ref_index_new(int dim) { return new SimilarityIndex(dim); }
void ref_index_free(void* h) { delete static_cast<SimilarityIndex*>(h); }

int ref_index_insert(void* h, uint64_t id, const float* w, const float* o, const float* b,
                     int d) {
  return guard([&] {
    static_cast<SimilarityIndex*>(h)->insert(
        Embedding::from_unit(std::vector<float>(w, w + d), EmbeddingKind::Whole),
        Embedding::from_unit(std::vector<float>(o, o + d), EmbeddingKind::Object),
        Embedding::from_unit(std::vector<float>(b, b + d), EmbeddingKind::Background),
        PromptId{id});
  });
}

int ref_index_remove(void* h, uint64_t id) {
  return guard([&] { static_cast<SimilarityIndex*>(h)->remove(PromptId{id}); });
}

int64_t ref_index_size(void* h) {
  return static_cast<int64_t>(static_cast<SimilarityIndex*>(h)->size());
}

// Concurrent readers are allowed by the index's shared_mutex (vindex.hpp:61),
// so nthreads > 1 issues independent query_top1 calls from a thread pool.
int ref_index_query_top1(void* h, int kind, const float* q, int n, int d, int nthreads,
                         uint64_t* ids, double* scores, int32_t* found) {
  auto* idx = static_cast<SimilarityIndex*>(h);
  if (nthreads < 1) nthreads = 1;
  std::vector<int> st(nthreads, ORC_OK);
  std::vector<std::string> errs(nthreads);
  auto work = [&](int t) {
    for (int i = t; i < n; i += nthreads) {
      int rc = guard([&] {
        Embedding e = Embedding::from_unit(std::vector<float>(q + (size_t)i * d, q + (size_t)(i + 1) * d),
                                           static_cast<EmbeddingKind>(kind));
        auto r = idx->query_top1(static_cast<EmbeddingKind>(kind), e);
        found[i] = r.has_value() ? 1 : 0;
        ids[i] = r ? r->prompt.value : 0;
        scores[i] = r ? r->score : 0.0;
      });
      if (rc != ORC_OK) {
        st[t] = rc;
        errs[t] = g_err;
        return;
      }
    }
  };
  if (nthreads == 1) {
    work(0);
  } else {
    std::vector<std::thread> ts;
    for (int t = 0; t < nthreads; ++t) ts.emplace_back(work, t);
    for (auto& t : ts) t.join();
  }
  for (int t = 0; t < nthreads; ++t)
    if (st[t] != ORC_OK) {
      g_err = errs[t];
      return st[t];
    }
  return ORC_OK;
}

int ref_select_keyframes(const float* frames, int F, int H, int W, int C, double thr,
                         int32_t* map) {
  return guard([&] {
    KeyFrameMap m = select_keyframes(make_latent(frames, 5, F, dims_of(H, W, C)), thr);
    for (int j = 0; j < F; ++j) map[j] = m.mapping[j];
  });
}

int ref_solve_alpha(const float* ds, const float* db, int64_t n, float* out) {
  return guard([&] {
    *out = solve_alpha(std::span<const float>(ds, n), std::span<const float>(db, n));
  });
}

int ref_compress(const float* lat, const int32_t* steps, int S, int F, int H, int W, int C,
                 const uint8_t* obj_masks, const uint8_t* bg_masks, double thr,
                 uint64_t prompt, uint8_t* out, uint64_t cap, uint64_t* out_len) {
  return guard([&] {
    auto bytes = compress_one(lat, steps, S, F, dims_of(H, W, C), obj_masks, bg_masks, thr, prompt);
    *out_len = bytes.size();
    if (out != nullptr) {
      if (bytes.size() > cap) throw std::invalid_argument("ref_compress: output buffer too small");
      std::memcpy(out, bytes.data(), bytes.size());
    }
  });
}

// n independent entries (pure functions) over a thread pool;
// latents [n][S][F][E], masks [n][F][mb]. Returns compressed_size per entry.
int ref_compress_batch(const float* lat, const int32_t* steps, int S, int F, int H, int W,
                       int C, const uint8_t* obj_masks, const uint8_t* bg_masks, double thr,
                       const uint64_t* prompts, int n, int nthreads, uint64_t* out_sizes) {
  const FrameDims d = dims_of(H, W, C);
  const size_t ent = static_cast<size_t>(S) * F * d.elems();
  const size_t mb = static_cast<size_t>(F) * ((static_cast<size_t>(H) * W + 7) / 8);
  if (nthreads < 1) nthreads = 1;
  std::vector<int> st(nthreads, ORC_OK);
  auto work = [&](int t) {
    for (int i = t; i < n; i += nthreads) {
      int rc = guard([&] {
        out_sizes[i] = compress_one(lat + i * ent, steps, S, F, d, obj_masks + i * mb,
                                    bg_masks + i * mb, thr, prompts[i])
                           .size();
      });
      if (rc != ORC_OK) {
        st[t] = rc;
        return;
      }
    }
  };
  std::vector<std::thread> ts;
  for (int t = 0; t < nthreads; ++t) ts.emplace_back(work, t);
  for (auto& t : ts) t.join();
  for (int rc : st)
    if (rc != ORC_OK) return rc;
  return ORC_OK;
}

// As ref_compress_batch, plus a position-weighted checksum of every entry's
// wire bytes, sum_i b[i] * ((i * 0x9E3779B1 + 1) mod 2^32) mod 2^64 (full-size
// parity checks compare checksums instead of shipping GBs of bytes).
int ref_compress_batch_hash(const float* lat, const int32_t* steps, int S, int F, int H, int W,
                            int C, const uint8_t* obj_masks, const uint8_t* bg_masks, double thr,
                            const uint64_t* prompts, int n, int nthreads, uint64_t* out_sizes,
                            uint64_t* out_hash) {
  const FrameDims d = dims_of(H, W, C);
  const size_t ent = static_cast<size_t>(S) * F * d.elems();
  const size_t mb = static_cast<size_t>(F) * ((static_cast<size_t>(H) * W + 7) / 8);
  if (nthreads < 1) nthreads = 1;
  std::vector<int> st(nthreads, ORC_OK);
  auto work = [&](int t) {
    for (int i = t; i < n; i += nthreads) {
      int rc = guard([&] {
        const auto b = compress_one(lat + i * ent, steps, S, F, d, obj_masks + i * mb, bg_masks + i * mb, thr,
                                    prompts[i]);
        out_sizes[i] = b.size();
        uint64_t h = 0;
        for (size_t x = 0; x < b.size(); ++x) h += (uint64_t)b[x] * (uint64_t)(uint32_t)(x * 0x9E3779B1u + 1u);
        out_hash[i] = h;
      });
      if (rc != ORC_OK) {
        st[t] = rc;
        return;
      }
    }
  };
  std::vector<std::thread> ts;
  for (int t = 0; t < nthreads; ++t) ts.emplace_back(work, t);
  for (auto& t : ts) t.join();
  for (int rc : st)
    if (rc != ORC_OK) return rc;
  return ORC_OK;
}

int ref_decompress(const uint8_t* entry, uint64_t len, int step, float* out) {
  return guard([&] {
    CompressedEntry e = parse_entry(entry, len);
    LatentState l = decompress_step(e, StepId(step));
    const size_t E = static_cast<size_t>(e.dims.elems());
    for (int j = 0; j < l.frame_count(); ++j)
      std::memcpy(out + j * E, l.frames()[j].values().data(), E * sizeof(float));
  });
}

int ref_entry_info(const uint8_t* entry, uint64_t len, int32_t* base_step, int32_t* n_steps,
                   int32_t* steps, uint64_t* shared_bytes, uint64_t* private_bytes) {
  return guard([&] {
    CompressedEntry e = parse_entry(entry, len);
    *base_step = e.base_step.value();
    *n_steps = static_cast<int32_t>(e.steps.size());
    *shared_bytes = entry_shared_bytes(e);
    for (size_t i = 0; i < e.steps.size(); ++i) {
      steps[i] = e.steps[i].step.value();
      private_bytes[i] = step_private_bytes(e, e.steps[i].step);
    }
  });
}

int ref_stitch(const float* obj, const uint8_t* oo, const uint8_t* ob, const float* bg,
               const uint8_t* bo, const uint8_t* bb, int F, int H, int W, int C, float* out) {
  return guard([&] {
    const FrameDims d = dims_of(H, W, C);
    StitchInput in{make_latent(obj, 5, F, d), make_masks(oo, ob, F, H, W),
                   make_latent(bg, 5, F, d), make_masks(bo, bb, F, H, W)};
    LatentState l = stitch(in);
    const size_t E = static_cast<size_t>(d.elems());
    for (int j = 0; j < F; ++j)
      std::memcpy(out + j * E, l.frames()[j].values().data(), E * sizeof(float));
  });
}

int ref_lrbu_priority(const orc_step_entry* e, uint64_t now, double* out) {
  return guard([&] { *out = lrbu_priority(get_step_entry(e), now); });
}

int ref_lcbfu_priority(const orc_step_entry* e, double* out) {
  return guard([&] { *out = lcbfu_priority(get_step_entry(e)); });
}

void* ref_store_new(uint64_t capacity, int policy) {
  return new CacheStore(capacity, static_cast<Policy>(policy));
}
void ref_store_free(void* h) { delete static_cast<CacheStore*>(h); }

int ref_store_insert(void* h, uint64_t prompt, const uint8_t* entry, uint64_t len,
                     const int32_t* steps, int n_steps, uint64_t now, orc_step_entry* evicted,
                     int cap, int* n_evicted) {
  return guard([&] {
    CompressedEntry e = parse_entry(entry, len);
    std::vector<StepId> ss;
    for (int i = 0; i < n_steps; ++i) ss.emplace_back(steps[i]);
    auto ev = static_cast<CacheStore*>(h)->insert_steps(PromptId{prompt}, e, ss, now);
    *n_evicted = static_cast<int>(ev.size());
    for (size_t i = 0; i < ev.size() && static_cast<int>(i) < cap; ++i)
      put_step_entry(ev[i], evicted + i);
  });
}

int ref_store_get_step(void* h, uint64_t prompt, int desired, uint64_t now, int32_t* actual,
                       float* out) {
  return guard([&] {
    auto r = static_cast<CacheStore*>(h)->get_step(PromptId{prompt}, StepId(desired), now);
    *actual = r ? r->actual.value() : 0;
    if (r && out != nullptr) {
      const size_t E = static_cast<size_t>(r->latent.dims().elems());
      for (int j = 0; j < r->latent.frame_count(); ++j)
        std::memcpy(out + j * E, r->latent.frames()[j].values().data(), E * sizeof(float));
    }
  });
}

int ref_store_evict_one(void* h, uint64_t now, orc_step_entry* out) {
  return guard([&] { put_step_entry(static_cast<CacheStore*>(h)->evict_one(now), out); });
}

int ref_store_evict_step(void* h, uint64_t prompt, int step, int32_t* removed) {
  return guard([&] {
    *removed = static_cast<CacheStore*>(h)->evict_step(PromptId{prompt}, StepId(step)) ? 1 : 0;
  });
}

uint64_t ref_store_used(void* h) { return static_cast<CacheStore*>(h)->used(); }
uint64_t ref_store_recompute_used(void* h) {
  return static_cast<CacheStore*>(h)->recompute_used();
}
int64_t ref_store_step_count(void* h) {
  return static_cast<int64_t>(static_cast<CacheStore*>(h)->step_count());
}
int64_t ref_store_prompt_count(void* h) {
  return static_cast<int64_t>(static_cast<CacheStore*>(h)->prompt_count());
}

int ref_store_entries(void* h, orc_step_entry* out, int cap, int* n) {
  return guard([&] {
    auto v = static_cast<CacheStore*>(h)->entries_snapshot();
    *n = static_cast<int>(v.size());
    for (size_t i = 0; i < v.size() && static_cast<int>(i) < cap; ++i) put_step_entry(v[i], out + i);
  });
}

// Snapshots (store.cpp:219-364): save/load through the reference's own code.
uint64_t ref_last_snapshot_offset(void) { return g_snap_off; }
int ref_snapshot_save(void* store, void* index, const char* path) {
  return guard([&] {
    save_snapshot(*static_cast<CacheStore*>(store), *static_cast<SimilarityIndex*>(index), path);
  });
}
// On success *out owns a SnapshotData; its store / index are borrowed via
// ref_snapshot_store / ref_snapshot_index and freed with ref_snapshot_free.
int ref_snapshot_load(const char* path, void** out) {
  return guard([&] { *out = new SnapshotData(load_snapshot(path)); });
}
void* ref_snapshot_store(void* d) { return &static_cast<SnapshotData*>(d)->store; }
void* ref_snapshot_index(void* d) { return &static_cast<SnapshotData*>(d)->index; }
void ref_snapshot_free(void* d) { delete static_cast<SnapshotData*>(d); }

}  // extern "C"
