// lcache_b200/lcache.hpp — C++ host API of the B200 FlexCache hot path.
//
// Header-only wrapper over the C-ABI (include/flexcache_b200.h) that keeps the
// reference library's class and function names, argument meaning, value
// types and exception types (/root/reference/proj/include/lcache/*.hpp), so
// code written against `lcache` builds against this header by swapping the
// include path and linking libflexcache_b200.so instead of liblcache.a.
// Every compute call goes to the sm_100a kernels; there is no CPU path.
//
//   reference header          what this header keeps
//   core.hpp:19-158           FrameDims, Frame, StepId, LatentState, EmbeddingKind,
//                             Embedding (+from_unit), Bitmap, MaskSet, PromptId,
//                             PromptLatents, cosine_similarity, frame_similarity
//   vindex.hpp:16-62          QueryResult, SimilarityIndex (+ batched query_topk)
//   codec.hpp:19-118          KeyFrameMap, IntraCompressed, CompressedEntry (a handle
//                             to a device-resident entry), select_keyframes,
//                             intra_compress, intra_decompress, solve_alpha,
//                             inter_compress, decompress_step, compressed_size,
//                             uncompressed_size, serialize/deserialize (bytes),
//                             entry_shared_bytes, step_private_bytes, size_breakdown
//   stitcher.hpp:13-24        StitchInput, stitch
//   store.hpp:22-93           Policy, parse_policy, policy_name, StepEntry,
//                             lrbu_priority, lcbfu_priority, CacheStore
//   errors.hpp:11-42          DegenerateBase, StepNotCached, OversizedEntry,
//                             SnapshotError (+ std::invalid_argument / logic_error)
//
// Deliberate differences (device residency): CompressedEntry is a shared
// handle to an entry living in HBM rather than a struct of host vectors
// (record()/has_step()/metadata accessors are kept; to_bytes() gives the
// reference wire format); CacheStore::entry_data() returns that handle.
// The namespace defaults to `lcache`; define LCACHE_B200_NS to rename it.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <compare>
#include <cstdint>
#include <filesystem>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "flexcache_b200.h"

#ifndef LCACHE_B200_NS
#define LCACHE_B200_NS lcache
#endif

namespace LCACHE_B200_NS {

// ---------------------------------------------------------------- defaults (defaults.hpp:10-46)
namespace defaults {
inline constexpr double kHitThreshold = 0.65;
inline constexpr double kCompressThreshold = 0.99;
inline constexpr int kTotalSteps = 50;
inline constexpr std::array<int, 5> kCachedSteps{5, 10, 15, 20, 25};
inline constexpr std::array<double, 4> kStepBinEdges{0.72, 0.79, 0.86, 0.93};
inline constexpr int kFrames = 64;
inline constexpr int kHeight = 40;
inline constexpr int kWidth = 64;
inline constexpr int kChannels = 4;
inline constexpr int kEmbedDim = 512;
}  // namespace defaults

// ---------------------------------------------------------------- errors (errors.hpp:11-42)
struct DegenerateBase : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StepNotCached : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OversizedEntry : std::runtime_error {
  OversizedEntry(std::uint64_t needed, std::uint64_t limit)
      : std::runtime_error("entry of " + std::to_string(needed) + " bytes exceeds capacity limit of " +
                           std::to_string(limit) + " bytes"),
        needed_bytes(needed),
        capacity_limit(limit) {}
  std::uint64_t needed_bytes;
  std::uint64_t capacity_limit;
};
struct SnapshotError : std::runtime_error {
  SnapshotError(const std::string& what, std::size_t offset)
      : std::runtime_error(what + " at byte " + std::to_string(offset)), byte_offset(offset) {}
  std::size_t byte_offset;
};
// Device / library failures that have no reference counterpart.
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace b200 {
// lc_status -> the reference exception type (1:1, flexcache_b200.h:39-51).
inline void check(lc_status s) {
  if (s == LC_OK) return;
  const std::string msg = lc_last_error() ? lc_last_error() : "";
  switch (s) {
    case LC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LC_ERR_DEGENERATE_BASE: throw DegenerateBase(msg);
    case LC_ERR_STEP_NOT_CACHED: throw StepNotCached(msg);
    case LC_ERR_OVERSIZED_ENTRY: {
      std::uint64_t need = 0, lim = 0;
      lc_last_oversize(&need, &lim);
      throw OversizedEntry(need, lim);
    }
    case LC_ERR_SNAPSHOT: {
      // message is "<what> at byte <offset>"; rebuild the reference's exception
      const std::uint64_t off = lc_last_snapshot_offset();
      const std::string tail = " at byte " + std::to_string(off);
      const bool has = msg.size() >= tail.size() && msg.compare(msg.size() - tail.size(), tail.size(), tail) == 0;
      throw SnapshotError(has ? msg.substr(0, msg.size() - tail.size()) : msg, (std::size_t)off);
    }
    case LC_ERR_IO: throw std::runtime_error(msg);
    case LC_ERR_LOGIC: throw std::logic_error(msg);
    default: throw DeviceError("flexcache_b200: " + msg);
  }
}

// One GPU + stream shared by every object created without an explicit context.
class Context {
 public:
  explicit Context(int device = 0) { check(lc_ctx_create(device, &h_)); }
  ~Context() {
    if (h_) lc_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  lc_ctx* get() const { return h_; }
  void synchronize() const { check(lc_ctx_synchronize(h_)); }
  std::uint64_t launches() const { return lc_ctx_launches(h_); }

 private:
  lc_ctx* h_ = nullptr;
};

// Intentionally never destroyed: a static owner would tear the context down
// after the CUDA runtime during process exit.
inline std::shared_ptr<Context>& default_context_slot() {
  static auto* ctx = new std::shared_ptr<Context>();
  return *ctx;
}
inline std::shared_ptr<Context> default_context() {
  auto& c = default_context_slot();
  if (!c) c = std::make_shared<Context>(0);
  return c;
}
inline void set_default_context(std::shared_ptr<Context> c) { default_context_slot() = std::move(c); }
}  // namespace b200

// ---------------------------------------------------------------- core (core.hpp:19-158)
struct FrameDims {
  int h = defaults::kHeight;
  int w = defaults::kWidth;
  int c = defaults::kChannels;
  int pixels() const { return h * w; }
  int elems() const { return h * w * c; }
  bool operator==(const FrameDims&) const = default;
};

// h*w*c finite floats, channel-minor (core.hpp:29-44; finite check core.cpp:11-25).
class Frame {
 public:
  Frame(FrameDims dims, std::vector<float> data) : dims_(dims), data_(std::move(data)) {
    if (dims.h <= 0 || dims.w <= 0 || dims.c <= 0) throw std::invalid_argument("Frame: non-positive dims");
    if ((long long)data_.size() != (long long)dims.elems()) throw std::invalid_argument("Frame: size mismatch");
    for (float v : data_)
      if (!std::isfinite(v)) throw std::invalid_argument("Frame: non-finite value");
  }
  explicit Frame(FrameDims dims) : Frame(dims, std::vector<float>((size_t)dims.elems(), 0.f)) {}
  const FrameDims& dims() const { return dims_; }
  std::span<const float> values() const { return data_; }
  float at(int h, int w, int c) const { return data_[(h * dims_.w + w) * dims_.c + c]; }
  bool operator==(const Frame&) const = default;

 private:
  FrameDims dims_;
  std::vector<float> data_;
};

// 1..50; cacheable {5,10,15,20,25} (core.hpp:47-59, core.cpp:29-39).
class StepId {
 public:
  explicit StepId(int value) : value_(value) {
    if (value < 1 || value > defaults::kTotalSteps) throw std::invalid_argument("StepId out of range");
  }
  int value() const { return value_; }
  bool is_cacheable() const {
    return std::find(cacheable().begin(), cacheable().end(), value_) != cacheable().end();
  }
  static const std::array<int, 5>& cacheable() { return defaults::kCachedSteps; }
  auto operator<=>(const StepId&) const = default;

 private:
  int value_;
};

class LatentState {
 public:
  LatentState(StepId step, std::vector<Frame> frames) : step_(step), frames_(std::move(frames)) {
    if (frames_.empty()) throw std::invalid_argument("LatentState: no frames");
    for (const Frame& f : frames_)
      if (!(f.dims() == frames_.front().dims())) throw std::invalid_argument("LatentState: mixed frame dims");
  }
  StepId step() const { return step_; }
  const std::vector<Frame>& frames() const { return frames_; }
  int frame_count() const { return (int)frames_.size(); }
  const FrameDims& dims() const { return frames_.front().dims(); }

 private:
  StepId step_;
  std::vector<Frame> frames_;
};

enum class EmbeddingKind : std::uint8_t { Whole = 0, Object = 1, Background = 2 };

// Unit-norm vector (core.cpp:50-69). The normalisation is the reference's
// host rule (fp64 sequential sum of squares, v * (1/sqrt), cast to fp32) so
// the stored bits are identical; it runs once per embedding at construction.
class Embedding {
 public:
  Embedding(std::vector<float> values, EmbeddingKind kind) : kind_(kind) {
    if (values.empty()) throw std::invalid_argument("Embedding: empty");
    double sq = 0.0;
    for (float v : values) {
      if (!std::isfinite(v)) throw std::invalid_argument("Embedding: non-finite value");
      sq += (double)v * (double)v;
    }
    if (!(sq > 0.0)) throw std::invalid_argument("Embedding: zero norm");
    const double inv = 1.0 / std::sqrt(sq);
    values_.resize(values.size());
    for (size_t i = 0; i < values.size(); ++i) values_[i] = (float)((double)values[i] * inv);
  }
  static Embedding from_unit(std::vector<float> values, EmbeddingKind kind) {
    if (values.empty()) throw std::invalid_argument("Embedding: empty");
    double sq = 0.0;
    for (float v : values) {
      if (!std::isfinite(v)) throw std::invalid_argument("Embedding: non-finite value");
      sq += (double)v * (double)v;
    }
    if (std::fabs(std::sqrt(sq) - 1.0) > 1e-6) throw std::invalid_argument("Embedding::from_unit: not unit norm");
    return Embedding(std::move(values), kind, TrustedTag{});
  }
  std::span<const float> values() const { return values_; }
  int dim() const { return (int)values_.size(); }
  EmbeddingKind kind() const { return kind_; }
  bool operator==(const Embedding&) const = default;

 private:
  struct TrustedTag {};
  Embedding(std::vector<float> values, EmbeddingKind kind, TrustedTag) : values_(std::move(values)), kind_(kind) {}
  std::vector<float> values_;
  EmbeddingKind kind_;
};

// LSB-first packed bitmap (core.hpp:104-124).
class Bitmap {
 public:
  Bitmap(int h, int w) : h_(h), w_(w), bits_(((size_t)h * w + 7) / 8, 0) {
    if (h <= 0 || w <= 0) throw std::invalid_argument("Bitmap: non-positive dims");
  }
  Bitmap(int h, int w, std::vector<std::uint8_t> packed) : h_(h), w_(w), bits_(std::move(packed)) {
    if (h <= 0 || w <= 0 || bits_.size() != ((size_t)h * w + 7) / 8)
      throw std::invalid_argument("Bitmap: packed size mismatch");
  }
  int height() const { return h_; }
  int width() const { return w_; }
  int bit_count() const { return h_ * w_; }
  std::size_t byte_count() const { return bits_.size(); }
  bool test(int pixel) const { return (bits_[pixel >> 3] >> (pixel & 7)) & 1; }
  void set(int pixel, bool value = true) {
    if (pixel < 0 || pixel >= bit_count()) throw std::invalid_argument("Bitmap::set out of range");
    if (value)
      bits_[pixel >> 3] |= (std::uint8_t)(1u << (pixel & 7));
    else
      bits_[pixel >> 3] &= (std::uint8_t) ~(1u << (pixel & 7));
  }
  const std::vector<std::uint8_t>& packed() const { return bits_; }
  bool operator==(const Bitmap&) const = default;

 private:
  int h_, w_;
  std::vector<std::uint8_t> bits_;
};

class MaskSet {
 public:
  MaskSet(std::vector<Bitmap> object_masks, std::vector<Bitmap> background_masks)
      : object_masks_(std::move(object_masks)), background_masks_(std::move(background_masks)) {
    if (object_masks_.size() != background_masks_.size()) throw std::invalid_argument("MaskSet: count mismatch");
  }
  int frame_count() const { return (int)object_masks_.size(); }
  const std::vector<Bitmap>& object_masks() const { return object_masks_; }
  const std::vector<Bitmap>& background_masks() const { return background_masks_; }
  bool operator==(const MaskSet&) const = default;
  // [F][ceil(HW/8)] packed planes, the device layout.
  std::vector<std::uint8_t> packed_object() const { return pack(object_masks_); }
  std::vector<std::uint8_t> packed_background() const { return pack(background_masks_); }

 private:
  static std::vector<std::uint8_t> pack(const std::vector<Bitmap>& v) {
    std::vector<std::uint8_t> out;
    for (const Bitmap& b : v) out.insert(out.end(), b.packed().begin(), b.packed().end());
    return out;
  }
  std::vector<Bitmap> object_masks_;
  std::vector<Bitmap> background_masks_;
};

struct PromptId {
  std::uint64_t value = 0;
  auto operator<=>(const PromptId&) const = default;
};

struct PromptLatents {
  std::vector<LatentState> states;
  MaskSet masks;
};

// cosine_similarity (core.cpp:101-114) on the GPU: sequential fp64, bit-exact.
inline double cosine_similarity(std::span<const float> a, std::span<const float> b) {
  if (a.size() != b.size() || a.empty()) throw std::invalid_argument("cosine_similarity: length mismatch or empty");
  double out = 0.0;
  b200::check(lc_cosine_batch(b200::default_context()->get(), a.data(), b.data(), 1, (int64_t)a.size(), &out));
  return out;
}
inline double frame_similarity(const Frame& a, const Frame& b) { return cosine_similarity(a.values(), b.values()); }

namespace b200 {
// [F][E] contiguous copy of a latent's frames (device upload staging).
inline std::vector<float> flatten(const LatentState& l) {
  const size_t E = (size_t)l.dims().elems();
  std::vector<float> out(E * l.frames().size());
  for (size_t j = 0; j < l.frames().size(); ++j)
    std::copy(l.frames()[j].values().begin(), l.frames()[j].values().end(), out.begin() + j * E);
  return out;
}
inline LatentState unflatten(StepId step, FrameDims dims, int F, const float* data) {
  const size_t E = (size_t)dims.elems();
  std::vector<Frame> frames;
  frames.reserve(F);
  for (int j = 0; j < F; ++j) frames.emplace_back(dims, std::vector<float>(data + j * E, data + (j + 1) * E));
  return LatentState(step, std::move(frames));
}
inline std::vector<Bitmap> unpack(const std::uint8_t* p, int F, int h, int w) {
  const size_t mb = ((size_t)h * w + 7) / 8;
  std::vector<Bitmap> v;
  for (int j = 0; j < F; ++j) v.emplace_back(h, w, std::vector<std::uint8_t>(p + j * mb, p + (j + 1) * mb));
  return v;
}
}  // namespace b200

// ---------------------------------------------------------------- vindex (vindex.hpp:16-62)
struct QueryResult {
  PromptId prompt;
  double score;
};

// Three device-resident tables (fp32 master rows + bf16 tensor-core copies).
// Thread-safety as the reference (vindex.hpp:61): the library takes a
// reader/writer lock per index.
class SimilarityIndex {
 public:
  SimilarityIndex() : SimilarityIndex(0) {}
  // adopts a handle created by the library (load_snapshot)
  SimilarityIndex(lc_index* adopt, std::shared_ptr<b200::Context> ctx) : ctx_(std::move(ctx)) {
    h_.reset(adopt, [](lc_index* p) { lc_index_destroy(p); });
  }
  explicit SimilarityIndex(int dim, std::shared_ptr<b200::Context> ctx = b200::default_context())
      : ctx_(std::move(ctx)) {
    lc_index* h = nullptr;
    b200::check(lc_index_create(ctx_->get(), dim, 0, &h));
    h_.reset(h, [](lc_index* p) { lc_index_destroy(p); });
  }
  void insert(const Embedding& whole, const Embedding& object, const Embedding& background, PromptId prompt) {
    if (whole.dim() != object.dim() || whole.dim() != background.dim())
      throw std::invalid_argument("SimilarityIndex::insert: dim mismatch");
    b200::check(lc_index_insert(h_.get(), prompt.value, whole.values().data(), object.values().data(),
                                background.values().data(), whole.dim()));
  }
  std::optional<QueryResult> query_top1(EmbeddingKind kind, const Embedding& query) const {
    std::uint64_t id = 0;
    double sc = 0.0;
    int32_t cnt = 0;
    b200::check(lc_index_query_topk(h_.get(), (int)kind, query.values().data(), 1, 1, &id, &sc, &cnt));
    if (cnt == 0) return std::nullopt;
    return QueryResult{PromptId{id}, sc};
  }
  // Batched extension: top-k by (score desc, id asc) for n queries [n][dim].
  std::vector<std::vector<QueryResult>> query_topk(EmbeddingKind kind, std::span<const float> queries, int k) const {
    const int d = dim();
    if (d <= 0 || queries.size() % (size_t)d) throw std::invalid_argument("query_topk: bad query buffer");
    const int64_t n = (int64_t)(queries.size() / d);
    std::vector<std::uint64_t> ids((size_t)n * k);
    std::vector<double> sc((size_t)n * k);
    std::vector<int32_t> cnt((size_t)n);
    b200::check(lc_index_query_topk(h_.get(), (int)kind, queries.data(), n, k, ids.data(), sc.data(), cnt.data()));
    std::vector<std::vector<QueryResult>> out((size_t)n);
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < cnt[i]; ++j) out[i].push_back({PromptId{ids[i * k + j]}, sc[i * k + j]});
    return out;
  }
  void remove(PromptId prompt) { b200::check(lc_index_remove(h_.get(), prompt.value)); }
  bool contains(PromptId prompt) const {
    int32_t c = 0;
    b200::check(lc_index_contains(h_.get(), prompt.value, &c));
    return c != 0;
  }
  std::size_t size() const { return (std::size_t)lc_index_size(h_.get()); }
  int dim() const { return lc_index_dim(h_.get()); }
  std::vector<std::pair<PromptId, std::vector<float>>> entries(EmbeddingKind kind) const {
    const int64_t n = (int64_t)size();
    const int d = dim();
    std::vector<std::uint64_t> ids((size_t)n);
    std::vector<float> rows((size_t)n * std::max(d, 0));
    if (n) b200::check(lc_index_export(h_.get(), (int)kind, ids.data(), rows.data(), n));
    std::vector<std::pair<PromptId, std::vector<float>>> out;
    for (int64_t i = 0; i < n; ++i)
      out.emplace_back(PromptId{ids[i]}, std::vector<float>(rows.begin() + i * d, rows.begin() + (i + 1) * d));
    return out;
  }
  lc_index* handle() const { return h_.get(); }

 private:
  std::shared_ptr<b200::Context> ctx_;
  std::shared_ptr<lc_index> h_;
};

// decide + similarity_to_step fused with the 3-table lookup.
enum class Decision : std::int32_t { Miss = LC_MISS, WholeHit = LC_WHOLE_HIT, DecoupledHit = LC_DECOUPLED_HIT };
inline std::vector<lc_decision> lookup_decide(const SimilarityIndex& ix, std::span<const float> q_whole,
                                              std::span<const float> q_object, std::span<const float> q_background,
                                              double hit_threshold = defaults::kHitThreshold) {
  const int d = ix.dim();
  if (d <= 0 || q_whole.size() % (size_t)d || q_object.size() != q_whole.size() ||
      q_background.size() != q_whole.size())
    throw std::invalid_argument("lookup_decide: bad query buffers");
  const int64_t n = (int64_t)(q_whole.size() / d);
  std::vector<lc_decision> out((size_t)n);
  b200::check(lc_lookup_decide(ix.handle(), q_whole.data(), q_object.data(), q_background.data(), n, hit_threshold,
                               defaults::kStepBinEdges.data(), out.data()));
  return out;
}

// ---------------------------------------------------------------- codec (codec.hpp:19-118)
struct KeyFrameMap {
  std::vector<int> mapping;
  int frame_count() const { return (int)mapping.size(); }
  bool is_key(int j) const { return mapping[j] == j; }
  std::vector<int> key_indices() const {
    std::vector<int> k;
    for (int j = 0; j < frame_count(); ++j)
      if (is_key(j)) k.push_back(j);
    return k;
  }
  bool operator==(const KeyFrameMap&) const = default;
};

struct IntraCompressed {
  StepId step;
  std::vector<std::pair<int, Frame>> keyframes;  // ascending frame index
  KeyFrameMap map;
  int frame_count() const { return map.frame_count(); }
  const Frame& keyframe_at(int index) const {
    for (const auto& kf : keyframes)
      if (kf.first == index) return kf.second;
    throw std::invalid_argument("IntraCompressed::keyframe_at: not a key frame");
  }
};

struct SizeBreakdown {
  std::uint64_t header = 0, first_frames = 0, maps = 0, alphas = 0, extra_frames = 0, base_diffs = 0, masks = 0;
  std::uint64_t total() const { return header + first_frames + maps + alphas + extra_frames + base_diffs + masks; }
};

// Handle to a CompressedEntry resident in HBM (codec.hpp:48-67).
class CompressedEntry {
 public:
  CompressedEntry() = default;
  explicit CompressedEntry(lc_entry* h, std::shared_ptr<b200::Context> ctx) : ctx_(std::move(ctx)) {
    h_.reset(h, [](lc_entry* p) { lc_entry_release(p); });
    b200::check(lc_entry_get_info(h, &info_));
  }
  PromptId prompt() const { return PromptId{info_.prompt}; }
  StepId base_step() const { return StepId(info_.base_step); }
  FrameDims dims() const { return FrameDims{info_.H, info_.W, info_.C}; }
  int frame_count() const { return info_.F; }
  std::vector<StepId> steps() const {
    std::vector<StepId> s;
    for (int i = 0; i < info_.n_steps; ++i) s.emplace_back(info_.steps[i]);
    return s;
  }
  bool has_step(StepId step) const {
    for (int i = 0; i < info_.n_steps; ++i)
      if (info_.steps[i] == step.value()) return true;
    return false;
  }
  int base_diff_count() const { return info_.n_diff; }
  int extra_frame_count(StepId step) const {
    for (int i = 0; i < info_.n_steps; ++i)
      if (info_.steps[i] == step.value()) return info_.n_extra[i];
    throw StepNotCached("step " + std::to_string(step.value()) + " not cached");
  }
  // Reference wire bytes (serialize_entry, codec.cpp:358-392).
  std::vector<std::uint8_t> to_bytes() const {
    std::uint64_t len = 0;
    b200::check(lc_entry_export(h_.get(), nullptr, 0, &len));
    std::vector<std::uint8_t> out(len);
    b200::check(lc_entry_export(h_.get(), out.data(), len, &len));
    return out;
  }
  const lc_entry_info& info() const { return info_; }
  lc_entry* handle() const { return h_.get(); }
  const std::shared_ptr<b200::Context>& context() const { return ctx_; }
  explicit operator bool() const { return (bool)h_; }

 private:
  std::shared_ptr<b200::Context> ctx_;
  std::shared_ptr<lc_entry> h_;
  lc_entry_info info_{};
};

// select_keyframes (codec.cpp:138-165): forward greedy on the GPU.
inline KeyFrameMap select_keyframes(const LatentState& latent, double threshold) {
  const FrameDims d = latent.dims();
  const std::vector<float> flat = b200::flatten(latent);
  KeyFrameMap m;
  m.mapping.resize((size_t)latent.frame_count());
  b200::check(lc_select_keyframes(b200::default_context()->get(), flat.data(), 1, latent.frame_count(), d.h, d.w,
                                  d.c, threshold, m.mapping.data()));
  return m;
}

// intra_compress / intra_decompress (codec.cpp:167-179): key frames kept verbatim.
inline IntraCompressed intra_compress(const LatentState& latent, double threshold) {
  IntraCompressed c{latent.step(), {}, select_keyframes(latent, threshold)};
  for (int j = 0; j < latent.frame_count(); ++j)
    if (c.map.is_key(j)) c.keyframes.emplace_back(j, latent.frames()[j]);
  return c;
}
inline LatentState intra_decompress(const IntraCompressed& c) {
  std::vector<Frame> frames;
  for (int j = 0; j < c.frame_count(); ++j) frames.push_back(c.keyframe_at(c.map.mapping[j]));
  return LatentState(c.step, std::move(frames));
}

// solve_alpha (codec.cpp:181-191): sequential fp64 on the GPU; zero base => DegenerateBase.
inline float solve_alpha(std::span<const float> diff_s, std::span<const float> diff_base) {
  if (diff_s.size() != diff_base.size() || diff_s.empty()) throw std::invalid_argument("solve_alpha: length mismatch");
  float out = 0.f;
  b200::check(lc_solve_alpha_batch(b200::default_context()->get(), diff_s.data(), diff_base.data(), 1,
                                   (int64_t)diff_s.size(), &out));
  return out;
}

// inter_compress (codec.cpp:193-261) on intra-compressed steps.
inline CompressedEntry inter_compress(const std::vector<IntraCompressed>& steps, MaskSet masks, PromptId prompt) {
  if (steps.empty()) throw std::invalid_argument("inter_compress: no steps");
  const int S = (int)steps.size(), F = steps[0].frame_count();
  const FrameDims d = steps[0].keyframes.at(0).second.dims();
  const size_t E = (size_t)d.elems();
  std::vector<float> lat((size_t)S * F * E, 0.f);
  std::vector<int32_t> maps((size_t)S * F), st((size_t)S);
  for (int s = 0; s < S; ++s) {
    if (steps[s].frame_count() != F) throw std::invalid_argument("inter_compress: frame count mismatch");
    st[s] = steps[s].step.value();
    for (int j = 0; j < F; ++j) maps[(size_t)s * F + j] = steps[s].map.mapping[j];
    for (const auto& kf : steps[s].keyframes) {
      if (!(kf.second.dims() == d)) throw std::invalid_argument("inter_compress: dims mismatch");
      std::copy(kf.second.values().begin(), kf.second.values().end(), lat.begin() + ((size_t)s * F + kf.first) * E);
    }
  }
  if (masks.frame_count() != F) throw std::invalid_argument("inter_compress: mask count mismatch");
  const auto om = masks.packed_object(), bm = masks.packed_background();
  auto ctx = b200::default_context();
  lc_entry* h = nullptr;
  b200::check(lc_inter_compress(ctx->get(), lat.data(), maps.data(), st.data(), S, F, d.h, d.w, d.c, om.data(),
                                bm.data(), prompt.value, &h));
  return CompressedEntry(h, ctx);
}

// Batched intra+inter compress of n prompts, all on the device: latents
// [n][S][F][E] (host or device), masks [n][F][mb]. Returns one entry per prompt.
inline std::vector<CompressedEntry> compress_batch(const float* latents, const std::vector<StepId>& steps, int F,
                                                   FrameDims d, const std::uint8_t* obj_masks,
                                                   const std::uint8_t* bg_masks,
                                                   const std::vector<PromptId>& prompts,
                                                   double threshold = defaults::kCompressThreshold) {
  auto ctx = b200::default_context();
  std::vector<int32_t> st;
  for (StepId s : steps) st.push_back(s.value());
  std::vector<std::uint64_t> ids;
  for (PromptId p : prompts) ids.push_back(p.value);
  std::vector<lc_entry*> hs(prompts.size(), nullptr);
  std::vector<std::uint64_t> sizes(prompts.size());
  b200::check(lc_compress_batch(ctx->get(), latents, st.data(), (int)st.size(), F, d.h, d.w, d.c, obj_masks,
                                bg_masks, threshold, ids.data(), (int64_t)ids.size(), hs.data(), sizes.data()));
  std::vector<CompressedEntry> out;
  for (lc_entry* h : hs) out.emplace_back(h, ctx);
  return out;
}

// decompress_step (codec.cpp:263-301), bit-exact, result copied to the host.
inline LatentState decompress_step(const CompressedEntry& entry, StepId step) {
  if (!entry.has_step(step)) throw StepNotCached("step " + std::to_string(step.value()) + " not cached");
  const int F = entry.frame_count();
  const size_t E = (size_t)entry.dims().elems();
  float* dev = nullptr;
  if (cudaMalloc(&dev, (size_t)F * E * sizeof(float)) != cudaSuccess) throw DeviceError("cudaMalloc failed");
  std::vector<float> host((size_t)F * E);
  lc_entry* h = entry.handle();
  const int32_t s = step.value();
  lc_status rc = lc_decompress_batch(entry.context()->get(), &h, &s, 1, dev);
  if (rc == LC_OK) rc = lc_ctx_synchronize(entry.context()->get());
  const cudaError_t ce = rc == LC_OK ? cudaMemcpy(host.data(), dev, host.size() * sizeof(float), cudaMemcpyDeviceToHost)
                                     : cudaSuccess;
  cudaFree(dev);
  b200::check(rc);
  if (ce != cudaSuccess) throw DeviceError("cudaMemcpy failed");
  return b200::unflatten(step, entry.dims(), F, host.data());
}

inline std::uint64_t compressed_size(const CompressedEntry& entry) { return entry.info().compressed_size; }
inline std::uint64_t uncompressed_size(const FrameDims& dims, int frame_count, int n_steps) {
  return (std::uint64_t)n_steps * (std::uint64_t)frame_count * (std::uint64_t)dims.elems() * sizeof(float);
}
inline std::uint64_t entry_shared_bytes(const CompressedEntry& entry) { return entry.info().shared_bytes; }
inline std::uint64_t step_private_bytes(const CompressedEntry& entry, StepId step) {
  for (int i = 0; i < entry.info().n_steps; ++i)
    if (entry.info().steps[i] == step.value()) return entry.info().private_bytes[i];
  throw StepNotCached("step " + std::to_string(step.value()) + " not cached");
}
// size_breakdown (codec.cpp:340-356) from the entry metadata.
inline SizeBreakdown size_breakdown(const CompressedEntry& entry) {
  const lc_entry_info& i = entry.info();
  const std::uint64_t E = (std::uint64_t)i.H * i.W * i.C, mb = ((std::uint64_t)i.H * i.W + 7) / 8;
  SizeBreakdown b;
  b.header = 20;
  b.masks = 2ull * i.F * mb;
  b.base_diffs = (std::uint64_t)i.n_diff * (2 + 4 * E);
  for (int s = 0; s < i.n_steps; ++s) {
    b.first_frames += 4 * E;
    b.maps += 2ull * i.F + 1 + 2;  // map + step byte + extra count (codec.cpp:349)
    b.extra_frames += (std::uint64_t)i.n_extra[s] * (2 + 4 * E);
    if (i.steps[s] != i.base_step) b.alphas += 4ull * i.n_diff;
  }
  return b;
}
inline std::vector<std::uint8_t> serialize_entry(const CompressedEntry& entry) { return entry.to_bytes(); }
inline CompressedEntry deserialize_entry(std::span<const std::uint8_t> bytes) {
  auto ctx = b200::default_context();
  lc_entry* h = nullptr;
  b200::check(lc_entry_import(ctx->get(), bytes.data(), bytes.size(), &h));
  return CompressedEntry(h, ctx);
}

// ---------------------------------------------------------------- stitcher (stitcher.hpp:13-24)
struct StitchInput {
  LatentState object_latent;
  MaskSet object_masks;
  LatentState background_latent;
  MaskSet background_masks;
};
inline LatentState stitch(const StitchInput& in) {
  if (!(in.object_latent.step() == in.background_latent.step())) throw std::invalid_argument("stitch: step mismatch");
  if (!(in.object_latent.dims() == in.background_latent.dims()) ||
      in.object_latent.frame_count() != in.background_latent.frame_count() ||
      in.object_masks.frame_count() != in.object_latent.frame_count() ||
      in.background_masks.frame_count() != in.object_latent.frame_count())
    throw std::invalid_argument("stitch: shape mismatch");
  const FrameDims d = in.object_latent.dims();
  const int F = in.object_latent.frame_count();
  const auto a = b200::flatten(in.object_latent), b = b200::flatten(in.background_latent);
  const auto om = in.object_masks.packed_object(), sm = in.background_masks.packed_object();
  std::vector<float> out(a.size());
  b200::check(lc_stitch_batch(b200::default_context()->get(), a.data(), om.data(), b.data(), sm.data(), 1, F, d.h, d.w,
                              d.c, out.data()));
  return b200::unflatten(in.object_latent.step(), d, F, out.data());
}

// ---------------------------------------------------------------- store (store.hpp:22-93)
enum class Policy : std::uint8_t { Fifo = 0, Lru = 1, Lcbfu = 2, Lrbu = 3 };
inline Policy parse_policy(const std::string& name) {  // store.cpp:13-19
  if (name == "fifo") return Policy::Fifo;
  if (name == "lru") return Policy::Lru;
  if (name == "lcbfu") return Policy::Lcbfu;
  if (name == "lrbu") return Policy::Lrbu;
  throw std::invalid_argument("unknown policy: " + name);
}
inline std::string policy_name(Policy p) {
  switch (p) {
    case Policy::Fifo: return "fifo";
    case Policy::Lru: return "lru";
    case Policy::Lcbfu: return "lcbfu";
    case Policy::Lrbu: return "lrbu";
  }
  return "?";
}

struct StepEntry {
  PromptId prompt;
  StepId step{5};
  std::uint64_t f = 0, last_access = 0, inserted_at = 0, inserted_seq = 0, capacity = 0;
};
namespace b200 {
inline StepEntry from_c(const lc_step_entry& e) {
  return StepEntry{PromptId{e.prompt}, StepId(e.step), e.f, e.last_access, e.inserted_at, e.inserted_seq, e.capacity};
}
inline lc_step_entry to_c(const StepEntry& e) {
  lc_step_entry c{};
  c.prompt = e.prompt.value;
  c.step = e.step.value();
  c.f = e.f;
  c.last_access = e.last_access;
  c.inserted_at = e.inserted_at;
  c.inserted_seq = e.inserted_seq;
  c.capacity = e.capacity;
  return c;
}
}  // namespace b200

// lrbu_priority / lcbfu_priority (store.cpp:32-42), evaluated by the scoring kernel.
inline double lrbu_priority(const StepEntry& e, std::uint64_t now) {
  const lc_step_entry c = b200::to_c(e);
  double out = 0.0;
  b200::check(lc_priority_batch(b200::default_context()->get(), LC_POLICY_LRBU, &c, 1, now, &out));
  return out;
}
inline double lcbfu_priority(const StepEntry& e) {
  const lc_step_entry c = b200::to_c(e);
  double out = 0.0;
  b200::check(lc_priority_batch(b200::default_context()->get(), LC_POLICY_LCBFU, &c, 1, 0, &out));
  return out;
}

class CacheStore {
 public:
  CacheStore(lc_store* adopt, std::shared_ptr<b200::Context> ctx) : ctx_(std::move(ctx)) {
    h_.reset(adopt, [](lc_store* p) { lc_store_destroy(p); });
  }
  CacheStore(std::uint64_t capacity_limit, Policy policy,
             std::shared_ptr<b200::Context> ctx = b200::default_context())
      : ctx_(std::move(ctx)) {
    lc_store* h = nullptr;
    b200::check(lc_store_create(ctx_->get(), capacity_limit, (int)policy, &h));
    h_.reset(h, [](lc_store* p) { lc_store_destroy(p); });
  }
  struct GetResult {
    LatentState latent;
    StepId actual;
  };
  std::vector<StepEntry> insert_steps(PromptId prompt, const CompressedEntry& entry, const std::vector<StepId>& steps,
                                      std::uint64_t now) {
    std::vector<int32_t> st;
    for (StepId s : steps) st.push_back(s.value());
    // one insert can evict at most every live step
    std::vector<lc_step_entry> ev(step_count() + 1);
    int n_ev = 0;
    b200::check(lc_store_insert(h_.get(), prompt.value, entry.handle(), st.data(), (int)st.size(), now, ev.data(),
                                (int)ev.size(), &n_ev));
    std::vector<StepEntry> out;
    for (int i = 0; i < n_ev; ++i) {
      out.push_back(b200::from_c(ev[i]));
      bool later = false;  // fire once, at the prompt's last evicted step (store.cpp:172-175)
      for (int j = i + 1; j < n_ev && !later; ++j) later = ev[j].prompt == ev[i].prompt;
      if (!later) notify(ev[i].prompt);
    }
    return out;
  }
  std::optional<GetResult> get_step(PromptId prompt, StepId desired, std::uint64_t now) {
    const lc_entry_info* info = nullptr;
    lc_entry* eh = nullptr;
    if (!contains(prompt) || lc_store_entry(h_.get(), prompt.value, &eh) != LC_OK || !eh) {
      int32_t actual = 0;  // validates `desired` exactly like the reference (store.cpp:95-96)
      b200::check(lc_store_get_step(h_.get(), prompt.value, desired.value(), now, &actual, nullptr));
      return std::nullopt;
    }
    lc_entry_info ei{};
    b200::check(lc_entry_get_info(eh, &ei));
    info = &ei;
    const size_t n = (size_t)info->F * info->H * info->W * info->C;
    float* dev = nullptr;
    if (cudaMalloc(&dev, n * sizeof(float)) != cudaSuccess) throw DeviceError("cudaMalloc failed");
    int32_t actual = 0;
    lc_status rc = lc_store_get_step(h_.get(), prompt.value, desired.value(), now, &actual, dev);
    std::vector<float> host;
    if (rc == LC_OK && actual) {
      host.resize(n);
      rc = lc_ctx_synchronize(ctx_->get());
      if (rc == LC_OK && cudaMemcpy(host.data(), dev, n * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = LC_ERR_CUDA;
    }
    cudaFree(dev);
    b200::check(rc);
    if (!actual) return std::nullopt;
    return GetResult{b200::unflatten(StepId(actual), FrameDims{info->H, info->W, info->C}, info->F, host.data()),
                     StepId(actual)};
  }
  StepEntry evict_one(std::uint64_t now) {
    lc_step_entry e{};
    b200::check(lc_store_evict_one(h_.get(), now, &e));
    notify(e.prompt);
    return b200::from_c(e);
  }
  bool evict_step(PromptId prompt, StepId step) {
    int32_t removed = 0;
    b200::check(lc_store_evict_step(h_.get(), prompt.value, step.value(), &removed));
    if (removed) notify(prompt.value);
    return removed != 0;
  }
  std::vector<StepId> cached_steps(PromptId prompt) const {
    int32_t s[8];
    int n = 0;
    b200::check(lc_store_cached_steps(h_.get(), prompt.value, s, &n));
    std::vector<StepId> out;
    for (int i = 0; i < n; ++i) out.emplace_back(s[i]);
    return out;
  }
  std::optional<CompressedEntry> entry_data(PromptId prompt) const {
    lc_entry* eh = nullptr;
    if (!contains(prompt)) return std::nullopt;
    b200::check(lc_store_entry(h_.get(), prompt.value, &eh));
    // lc_store_entry hands out a borrowed view; export + import gives an owned copy
    std::uint64_t len = 0;
    b200::check(lc_entry_export(eh, nullptr, 0, &len));
    std::vector<std::uint8_t> bytes(len);
    b200::check(lc_entry_export(eh, bytes.data(), len, &len));
    lc_entry* own = nullptr;
    b200::check(lc_entry_import(ctx_->get(), bytes.data(), len, &own));
    return CompressedEntry(own, ctx_);
  }
  std::optional<MaskSet> masks(PromptId prompt) const {
    auto e = entry_data(prompt);
    if (!e) return std::nullopt;
    const auto bytes = e->to_bytes();
    const lc_entry_info& i = e->info();
    const size_t mb = ((size_t)i.H * i.W + 7) / 8, mask_bytes = 2 * (size_t)i.F * mb;
    // masks are the trailing section of the wire format (codec.cpp:390-391)
    const std::uint8_t* p = bytes.data() + bytes.size() - mask_bytes;
    return MaskSet(b200::unpack(p, i.F, i.H, i.W), b200::unpack(p + (size_t)i.F * mb, i.F, i.H, i.W));
  }
  bool contains(PromptId prompt) const {
    int32_t c = 0;
    b200::check(lc_store_contains(h_.get(), prompt.value, &c));
    return c != 0;
  }
  std::uint64_t used() const { return lc_store_used(h_.get()); }
  std::uint64_t capacity_limit() const { return lc_store_capacity(h_.get()); }
  Policy policy() const { return (Policy)lc_store_policy(h_.get()); }
  std::size_t prompt_count() const { return (std::size_t)lc_store_prompt_count(h_.get()); }
  std::size_t step_count() const { return (std::size_t)lc_store_step_count(h_.get()); }
  void set_eviction_callback(std::function<void(PromptId)> cb) { on_prompt_gone_ = std::move(cb); }
  std::vector<StepEntry> entries_snapshot() const {
    const int64_t cap = (int64_t)step_count();
    std::vector<lc_step_entry> v((size_t)cap);
    int64_t n = 0;
    b200::check(lc_store_entries(h_.get(), v.data(), cap, &n));
    std::vector<StepEntry> out;
    for (int64_t i = 0; i < n; ++i) out.push_back(b200::from_c(v[i]));
    return out;
  }
  std::uint64_t recompute_used() const { return lc_store_recompute_used(h_.get()); }
  lc_store* handle() const { return h_.get(); }

 private:
  // store.cpp:166-176: the callback fires when a prompt's last step goes.
  void notify(std::uint64_t prompt) {
    if (on_prompt_gone_ && !contains(PromptId{prompt})) on_prompt_gone_(PromptId{prompt});
  }
  std::shared_ptr<b200::Context> ctx_;
  std::shared_ptr<lc_store> h_;
  std::function<void(PromptId)> on_prompt_gone_;
};

// store.hpp:122-132: versioned binary snapshot of the store plus the three
// index tables. The eviction callback is not part of it.
struct SnapshotData {
  CacheStore store;
  SimilarityIndex index;
};
inline void save_snapshot(const CacheStore& store, const SimilarityIndex& index, const std::filesystem::path& path) {
  b200::check(lc_snapshot_save(store.handle(), index.handle(), path.string().c_str()));
}
inline SnapshotData load_snapshot(const std::filesystem::path& path,
                                  std::shared_ptr<b200::Context> ctx = b200::default_context()) {
  lc_store* s = nullptr;
  lc_index* i = nullptr;
  b200::check(lc_snapshot_load(ctx->get(), path.string().c_str(), &s, &i));
  return SnapshotData{CacheStore(s, ctx), SimilarityIndex(i, ctx)};
}

// ---------------------------------------------------------------- entry-sharded multi-GPU
// Not in the reference (single process, CPU). One process (or thread) per
// GPU; prompt p lives on rank p mod G. Rank 0 makes a communicator id and
// shares its 128 bytes out of band (MPI_Bcast, a TCP store, a file); every
// rank attaches it to its context. All Sharded* calls are collective: every
// rank calls them in the same order with the same arguments.
namespace b200 {
using CommId = std::array<std::uint8_t, 128>;
inline CommId comm_unique_id() {
  CommId id{};
  check(lc_comm_unique_id(id.data()));
  return id;
}
inline void attach_nccl(Context& ctx, int nranks, int rank, const CommId& id) {
  check(lc_ctx_comm_init(ctx.get(), nranks, rank, id.data()));
}
// Caller-provided transport (e.g. MPI_Allgather): fn(user, send, recv[nranks][bytes], bytes) -> 0 on success.
inline void attach_host_transport(Context& ctx, int nranks, int rank, lc_allgather_fn fn, void* user) {
  check(lc_ctx_comm_host(ctx.get(), nranks, rank, fn, user));
}
inline std::uint64_t shard_owner(PromptId p, int nranks) { return lc_shard_owner(p.value, nranks); }
}  // namespace b200

// This rank's shard of the three tables; queries return the GLOBAL answer
// (local exact top-k, one all-gather, merge by (score desc, id asc)).
class ShardedSimilarityIndex {
 public:
  explicit ShardedSimilarityIndex(int dim, std::shared_ptr<b200::Context> ctx = b200::default_context())
      : local_(dim, ctx), ctx_(std::move(ctx)), dim_(dim) {
    b200::check(lc_ctx_comm_info(ctx_->get(), &nranks_, &rank_, nullptr, nullptr));
  }
  bool owns(PromptId p) const { return (int)b200::shard_owner(p, nranks_) == rank_; }
  // not collective: only the owner stores the rows (others ignore the call)
  void insert(const Embedding& whole, const Embedding& object, const Embedding& background, PromptId prompt) {
    if (owns(prompt)) local_.insert(whole, object, background, prompt);
  }
  void remove(PromptId prompt) {
    if (owns(prompt)) local_.remove(prompt);
  }
  std::optional<QueryResult> query_top1(EmbeddingKind kind, const Embedding& query) const {
    std::uint64_t id = 0;
    double sc = 0.0;
    int32_t cnt = 0;
    b200::check(lc_sharded_query_topk(local_.handle(), (int)kind, query.values().data(), 1, dim_, 1, &id, &sc, &cnt));
    if (cnt == 0) return std::nullopt;
    return QueryResult{PromptId{id}, sc};
  }
  std::vector<std::vector<QueryResult>> query_topk(EmbeddingKind kind, std::span<const float> queries, int k) const {
    if (queries.size() % (size_t)dim_) throw std::invalid_argument("query_topk: bad query buffer");
    const int64_t n = (int64_t)(queries.size() / dim_);
    std::vector<std::uint64_t> ids((size_t)n * k);
    std::vector<double> sc((size_t)n * k);
    std::vector<int32_t> cnt((size_t)n);
    b200::check(lc_sharded_query_topk(local_.handle(), (int)kind, queries.data(), n, dim_, k, ids.data(), sc.data(),
                                      cnt.data()));
    std::vector<std::vector<QueryResult>> out((size_t)n);
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < cnt[i]; ++j) out[i].push_back({PromptId{ids[i * k + j]}, sc[i * k + j]});
    return out;
  }
  std::vector<lc_decision> lookup_decide(std::span<const float> q_whole, std::span<const float> q_object,
                                         std::span<const float> q_background,
                                         double hit_threshold = defaults::kHitThreshold) const {
    if (q_whole.size() % (size_t)dim_ || q_object.size() != q_whole.size() || q_background.size() != q_whole.size())
      throw std::invalid_argument("lookup_decide: bad query buffers");
    const int64_t n = (int64_t)(q_whole.size() / dim_);
    std::vector<lc_decision> out((size_t)n);
    b200::check(lc_sharded_lookup_decide(local_.handle(), q_whole.data(), q_object.data(), q_background.data(), n,
                                         dim_, hit_threshold, defaults::kStepBinEdges.data(), out.data()));
    return out;
  }
  SimilarityIndex& local() { return local_; }

 private:
  SimilarityIndex local_;
  std::shared_ptr<b200::Context> ctx_;
  int dim_, nranks_ = 1, rank_ = 0;
};

// CacheStore under one global capacity budget: the same StepEntry sequence,
// used() and sequence numbers as one CacheStore holding every prompt.
class ShardedCacheStore {
 public:
  ShardedCacheStore(std::uint64_t capacity_limit, Policy policy,
                    std::shared_ptr<b200::Context> ctx = b200::default_context(), int batch = 0)
      : ctx_(std::move(ctx)) {
    lc_sharded_store* h = nullptr;
    b200::check(lc_sharded_store_create(ctx_->get(), capacity_limit, (int)policy, batch, &h));
    h_.reset(h, [](lc_sharded_store* p) { lc_sharded_store_destroy(p); });
  }
  // entry: the owner rank's CompressedEntry, nullptr on the other ranks
  std::vector<StepEntry> insert_steps(PromptId prompt, const CompressedEntry* entry, const std::vector<StepId>& steps,
                                      std::uint64_t now) {
    std::vector<int32_t> st;
    for (StepId s : steps) st.push_back(s.value());
    std::vector<lc_step_entry> ev(4096);
    int n = 0;
    b200::check(lc_sharded_store_insert(h_.get(), prompt.value, entry ? entry->handle() : nullptr, st.data(),
                                        (int)st.size(), now, ev.data(), (int)ev.size(), &n));
    std::vector<StepEntry> out;
    for (int i = 0; i < std::min<int>(n, (int)ev.size()); ++i) out.push_back(b200::from_c(ev[i]));
    return out;
  }
  StepEntry evict_one(std::uint64_t now) {
    lc_step_entry e{};
    b200::check(lc_sharded_store_evict_one(h_.get(), now, &e));
    return b200::from_c(e);
  }
  // the actual step served (0 = nothing); the latent stays on the owner's GPU (out_dev, owner only)
  int get_step(PromptId prompt, StepId desired, std::uint64_t now, float* out_dev = nullptr) {
    int32_t a = 0;
    b200::check(lc_sharded_store_get_step(h_.get(), prompt.value, desired.value(), now, &a, out_dev));
    return a;
  }
  std::uint64_t used() const {
    std::uint64_t u = 0;
    b200::check(lc_sharded_store_used(h_.get(), &u));
    return u;
  }
  lc_store* local_handle() const { return lc_sharded_store_local(h_.get()); }

 private:
  std::shared_ptr<b200::Context> ctx_;
  std::shared_ptr<lc_sharded_store> h_;
};

}  // namespace LCACHE_B200_NS

template <>
struct std::hash<LCACHE_B200_NS::PromptId> {
  std::size_t operator()(const LCACHE_B200_NS::PromptId& p) const noexcept { return std::hash<std::uint64_t>{}(p.value); }
};
