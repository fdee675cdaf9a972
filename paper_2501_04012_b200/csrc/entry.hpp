// entry.hpp — device-resident CompressedEntry (codec.hpp:48-67).
//
// HBM layout of one entry (single allocation, 16-byte aligned sections):
//   floats  : first frame per step [n_steps][E], base diffs [n_diff][E],
//             extra frames (all steps) [n_extra_total][E]
//   bytes   : object masks [F][mb], background masks [F][mb]
//   recipes : [n_steps][F] Recipe — decompress_step (codec.cpp:263-301)
//             resolved per output frame j through the key-frame map, so the
//             decompress kernel is a pure streaming pass.
// Host side keeps the small metadata (maps, alphas, indices) needed for the
// wire format (serialize_entry, codec.cpp:358-392) and size accounting.
#pragma once
#include <atomic>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace fc {

// kind 0: out = a            (first frame / extra frame / zero-diff key)
// kind 1: out = a + b        fp32 add (base step, codec.cpp:286-287)
// kind 2: out = (float)fma((double)alpha, (double)b, (double)a)
//         == (float)((double)first + alpha*diff) (codec.cpp:289-292)
struct Recipe {
  int32_t kind;
  float alpha;
  int64_t a;  // float offset from entry base
  int64_t b;
};

// Device memory shared by the entries of one compress batch (freed with the last).
struct DevArena {
  lc_ctx* ctx = nullptr;
  uint8_t* p = nullptr;
  ~DevArena();
};

struct EntryData {
  lc_ctx* ctx = nullptr;
  uint64_t prompt = 0;
  int base_step = 0;
  int F = 0, H = 0, W = 0, C = 0;
  int64_t E = 0, mb = 0;
  std::vector<int32_t> steps;                   // ascending
  std::vector<std::vector<int32_t>> maps;       // [n_steps][F]
  std::vector<std::vector<int32_t>> extra_idx;  // [n_steps][n_extra] ascending
  std::vector<std::vector<int64_t>> extra_off;  // float offsets
  std::vector<std::vector<float>> alphas;       // [n_steps][n_diff] (empty for the base step)
  std::vector<int32_t> diff_idx;                // ascending
  std::vector<int64_t> first_off, diff_off;
  int64_t mask_off = 0;    // byte offset of object masks (bg masks follow)
  int64_t recipe_off = 0;  // byte offset of Recipe[n_steps][F]
  uint8_t* dev = nullptr;
  size_t dev_bytes = 0;
  std::shared_ptr<DevArena> arena;  // set when dev lives in a batch allocation
  // grouped-decompress jobs per step (key frame + the frames mapped to it),
  // built on first use: decompress calls then only concatenate them
  struct KeyGroup {
    int32_t key;
    uint64_t mask[4];
  };
  mutable std::mutex groups_mu;
  mutable std::vector<std::vector<KeyGroup>> groups;
  const std::vector<KeyGroup>& key_groups(int si) const {
    std::lock_guard<std::mutex> lk(groups_mu);
    if (groups.size() != steps.size()) groups.assign(steps.size(), {});
    std::vector<KeyGroup>& g = groups[si];
    if (g.empty()) {
      const std::vector<int32_t>& mp = maps[si];
      std::vector<int> slot(F, -1);
      for (int j = 0; j < F; ++j) {
        // frames mapped to a key frame (mp[m] == m) share the key's recipe;
        // any other frame (only an imported map can do that) stands alone
        // with its own recipe, exactly as the per-frame kernel would serve it
        const int m = mp[mp[j]] == mp[j] ? mp[j] : j;
        if (m == j && mp[j] != j) {
          g.push_back(KeyGroup{j, {0, 0, 0, 0}});
          g.back().mask[j >> 6] |= 1ull << (j & 63);
          continue;
        }
        if (slot[m] < 0) {
          slot[m] = (int)g.size();
          g.push_back(KeyGroup{m, {0, 0, 0, 0}});
        }
        g[slot[m]].mask[j >> 6] |= 1ull << (j & 63);
      }
    }
    return g;
  }
  ~EntryData();

  const float* fbase() const { return reinterpret_cast<const float*>(dev); }
  const Recipe* recipes(int step_index) const {
    return reinterpret_cast<const Recipe*>(dev + recipe_off) + (size_t)step_index * F;
  }
  const uint8_t* obj_masks() const { return dev + mask_off; }
  const uint8_t* bg_masks() const { return dev + mask_off + (size_t)F * mb; }
  int step_index(int step) const {
    for (size_t i = 0; i < steps.size(); ++i)
      if (steps[i] == step) return (int)i;
    return -1;
  }
  int n_diff() const { return (int)diff_idx.size(); }
  // Size accounting, codec.cpp:305-332.
  uint64_t shared_bytes() const { return 20ull + (uint64_t)n_diff() * (2 + 4ull * E) + 2ull * F * (uint64_t)mb; }
  uint64_t private_bytes(int si) const {
    uint64_t n = 1 + 4ull * E + 2ull * F;
    if (steps[si] != base_step) n += 4ull * alphas[si].size();
    return n + 2 + (uint64_t)extra_idx[si].size() * (2 + 4ull * E);
  }
};

}  // namespace fc

// A handle = shared immutable data + the selection of live step records
// (the store drops evicted steps from its view, store.cpp:166-172).
struct lc_entry {
  std::shared_ptr<fc::EntryData> d;
  std::vector<int> sel;  // indices into d->steps, ascending
};

namespace fc {
lc_entry* make_entry_view(const std::shared_ptr<EntryData>& d, std::vector<int> sel);
uint64_t entry_compressed_size(const lc_entry* e);
// serialize_entry of e from a host copy of its device image (codec.cu)
uint64_t serialize_entry_image(const lc_entry* e, const uint8_t* img, uint8_t* out, uint64_t cap);
// deserialize_entry from the front of bytes[0, len) (codec.cu); *consumed = bytes used
lc_entry* import_entry(lc_ctx* ctx, const uint8_t* bytes, uint64_t len, uint64_t* consumed);
// Decompress n (entry, step-index) pairs into out [n][F][E] on the ctx stream.
void launch_decompress(lc_ctx* ctx, const std::vector<const EntryData*>& ents, const std::vector<int>& step_idx,
                       float* out, const int32_t* fbits_update = nullptr);
}  // namespace fc
