// store.cu — CacheStore (store.hpp:48-120) with GPU replacement scoring.
//
// Host keeps the per-prompt records (validation, hole fallback, byte
// accounting; store.cpp:53-217) and a mirror of the per-(prompt, step)
// bookkeeping. The device holds the live-step table as SoA-ish records
// (40 B per live step + 16 B per prompt) that the scoring kernels read:
//   K11 k_policy_seg    per live step: attributed capacity
//                       cap = private + shared / live (integer, store.cpp:122),
//                       policy key (store.cpp:125-131; fp64 IEEE mul/div), then a
//                       bitonic sort of each 4096-slot segment by (key, seq) in
//                       smem; the first H = 256 are the segment head.
//   K12 k_head_seg      the same sort over groups of segment heads, repeated
//                       until one global sorted head remains.
// Eviction (store.cpp:80, repeated evict_one) then walks the head on the
// host. For LRBU, evicting a step re-attributes the prompt's shared bytes to
// its surviving siblings, which lowers their keys; those siblings are re-keyed
// exactly on the host and kept in a small heap, so the victim sequence equals
// k repeated argmins without k full scans. When the head
// is exhausted the table is re-scored.
#include <cooperative_groups.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <map>
#include <memory>
#include <queue>
#include <unordered_map>
#include <unordered_set>
#include <fcntl.h>
#include <unistd.h>
#include <mutex>
#include <cstring>

#include "entry.hpp"
#include "topk.cuh"

namespace fc {

struct DevLive {
  uint64_t f, last, seq, priv;
  int32_t step;   // 0 = dead slot
  int32_t pslot;
};
struct DevPrompt {
  uint64_t shared;
  int32_t live;
  int32_t pad;
};


__device__ __forceinline__ double pkey(int policy, const DevLive& l, const DevPrompt& p, uint64_t now, uint64_t* cap_out,
                                       int* bad) {
  const uint64_t cap = l.priv + p.shared / (uint64_t)p.live;
  *cap_out = cap;
  switch (policy) {
    case LC_POLICY_FIFO: return (double)l.seq;
    case LC_POLICY_LRU: return (double)l.last;
    case LC_POLICY_LCBFU: return __dmul_rn((double)(l.f + 1), (double)l.step);
    default: {
      if (now < l.last || cap == 0) {
        *bad = 1;
        return 0.0;
      }
      const uint64_t dd = now - l.last;
      const double duration = (double)(dd > 1 ? dd : 1);
      return __ddiv_rn(__dmul_rn((double)(l.f + 1), (double)l.step), __dmul_rn((double)cap, duration));
    }
  }
}

// ---------------------------------------------------------------------------
// K11/K12: the H smallest (key, seq) live steps, as a segmented sort:
// level 0 computes the key of every slot of a 4096-slot segment in smem and
// bitonic-sorts the segment by (key, seq); its first H items are the
// segment's head. Further levels sort groups of 4096/H heads the same way
// until one head remains. Keys are non-negative doubles (or the FIFO/LRU
// integers as doubles); the order-preserving bit image makes the comparison
// a pair of u64 compares. Dead slots sort last.
constexpr int SEG = 4096;      // items per block
constexpr int SEG_T = 512;     // threads per block
constexpr int SCORE_H = 256;   // head length kept per segment / returned

__device__ __forceinline__ uint64_t key_bits(double k) {
  const uint64_t b = (uint64_t)__double_as_longlong(k);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double bits_key(uint64_t b) {
  return __longlong_as_double((long long)((b >> 63) ? (b & 0x7fffffffffffffffull) : ~b));
}

struct ScoreItem {
  uint64_t kb, seq;
  int64_t slot;
};

// bitonic sort of kb/sq/sl[0, n2) ascending by (kb, sq); n2 a power of two <= SEG
__device__ __forceinline__ void seg_sort(uint64_t* kb, uint64_t* sq, int64_t* sl, int n2 = SEG) {
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n2 / 2; t += SEG_T) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool up = (i & size) == 0;
        const bool gt = kb[i] > kb[j] || (kb[i] == kb[j] && sq[i] > sq[j]);
        if (gt == up) {
          const uint64_t a = kb[i], c = sq[i];
          const int64_t e = sl[i];
          kb[i] = kb[j], sq[i] = sq[j], sl[i] = sl[j];
          kb[j] = a, sq[j] = c, sl[j] = e;
        }
      }
    }
  }
  __syncthreads();
}

// level 0: keys of slots [blockIdx.x * SEG, +SEG)
__global__ void __launch_bounds__(SEG_T) k_policy_seg(const DevLive* __restrict__ live, int64_t n_slots,
                                                      const DevPrompt* __restrict__ prompts, int policy, uint64_t now,
                                                      ScoreItem* __restrict__ heads, int* __restrict__ bad) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint64_t* kb = reinterpret_cast<uint64_t*>(sm);
  uint64_t* sq = kb + SEG;
  int64_t* sl = reinterpret_cast<int64_t*>(sq + SEG);
  int b = 0;
  for (int t = threadIdx.x; t < SEG; t += SEG_T) {
    const int64_t i = (int64_t)blockIdx.x * SEG + t;
    uint64_t k = ~0ull, q = ~0ull;
    if (i < n_slots) {
      const DevLive l = live[i];
      if (l.step != 0) {
        uint64_t cap;
        k = key_bits(pkey(policy, l, prompts[l.pslot], now, &cap, &b));
        q = l.seq;
      }
    }
    kb[t] = k, sq[t] = q, sl[t] = i;
  }
  if (b) atomicExch(bad, 1);
  seg_sort(kb, sq, sl);
  for (int t = threadIdx.x; t < SCORE_H; t += SEG_T)
    heads[(int64_t)blockIdx.x * SCORE_H + t] = ScoreItem{kb[t], sq[t], sl[t]};
}

// level >= 1: block b sorts heads [b * SEG, +SEG) of the previous level
__global__ void __launch_bounds__(SEG_T) k_head_seg(const ScoreItem* __restrict__ in, int64_t n_in,
                                                    ScoreItem* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint64_t* kb = reinterpret_cast<uint64_t*>(sm);
  uint64_t* sq = kb + SEG;
  int64_t* sl = reinterpret_cast<int64_t*>(sq + SEG);
  for (int t = threadIdx.x; t < SEG; t += SEG_T) {
    const int64_t i = (int64_t)blockIdx.x * SEG + t;
    if (i < n_in) {
      const ScoreItem it = in[i];
      kb[t] = it.kb, sq[t] = it.seq, sl[t] = it.slot;
    } else {
      kb[t] = ~0ull, sq[t] = ~0ull, sl[t] = -1;
    }
  }
  seg_sort(kb, sq, sl);
  for (int t = threadIdx.x; t < SCORE_H; t += SEG_T)
    out[(int64_t)blockIdx.x * SCORE_H + t] = ScoreItem{kb[t], sq[t], sl[t]};
}


// ---------------------------------------------------------------------------
// Fast path (radix threshold select): K11a writes the key image of every
// slot and its min/max; K11b histograms (kb - min) >> shift over NBIN bins;
// K11c finds the first bin at which the cumulative count reaches H; K11d
// compacts every slot at or below that bin; K12 sorts the (<= CAP) survivors
// by (key, seq). Exact: every slot with a smaller (key, seq) than the H-th
// survivor is in a bin <= the threshold bin. When ties or a dense bin leave
// more than CAP survivors, the segmented sort above is used instead.
constexpr int NBIN = 4096;
constexpr int CAP = SEG;
constexpr int REFINE = 2 * SCORE_H;  // refine the threshold bin above this many survivors (smaller final sort)
constexpr int RANK_MAX = 2048;       // fused kernel: survivors ranked by counting across the grid (phase F)

__global__ void k_policy_keys(const DevLive* __restrict__ live, int64_t n_slots, const DevPrompt* __restrict__ prompts,
                              int policy, uint64_t now, uint64_t* __restrict__ K, unsigned long long* __restrict__ mm,
                              int* __restrict__ bad) {
  uint64_t lo = ~0ull, hi = 0;
  int b = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_slots; i += (int64_t)gridDim.x * blockDim.x) {
    const DevLive l = live[i];
    uint64_t k = ~0ull;
    if (l.step != 0) {
      uint64_t cap;
      k = key_bits(pkey(policy, l, prompts[l.pslot], now, &cap, &b));
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
    K[i] = k;
  }
  if (b) atomicExch(bad, 1);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, lo, o), c = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = c > hi ? c : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], (unsigned long long)lo);
    atomicMax(&mm[1], (unsigned long long)hi);
  }
}

__device__ __forceinline__ int bin_shift(uint64_t lo, uint64_t hi) {
  const uint64_t span = hi > lo ? hi - lo : 0;
  const int bits = 64 - __clzll((long long)span);  // bits of the span
  return bits > 12 ? bits - 12 : 0;                // NBIN = 2^12
}

__global__ void k_policy_hist(const uint64_t* __restrict__ K, int64_t n_slots, const unsigned long long* __restrict__ mm,
                              unsigned* __restrict__ hist) {
  __shared__ unsigned h[NBIN];
  for (int t = threadIdx.x; t < NBIN; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const uint64_t lo = mm[0], hi = mm[1];
  const int sh = bin_shift(lo, hi);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_slots; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = K[i];
    if (k != ~0ull) atomicAdd(&h[(k - lo) >> sh], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < NBIN; t += blockDim.x)
    if (h[t]) atomicAdd(&hist[t], h[t]);
}

// Block of NT threads over NBIN bin counts: the first bin whose cumulative
// count reaches `need` (NBIN - 1 if none), its cumulative count and the count
// below it.
template <int NT = 1024>
__device__ void block_pick(const unsigned* __restrict__ hist, unsigned need, int* bin, unsigned* at, unsigned* below) {
  // PER consecutive bins per thread (16-byte loads), warp-shuffle scans: three
  // block barriers instead of a Hillis-Steele scan's 2 log2(NT)
  constexpr int PER = NBIN / NT, NW = NT / 32;
  static_assert(PER % 4 == 0, "block_pick: 16-byte bin loads");
  __shared__ unsigned wtot[NW];
  __shared__ int s_bin;
  __shared__ unsigned s_at, s_below;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned loc[PER], run = 0;
  const uint4* h4 = reinterpret_cast<const uint4*>(hist) + threadIdx.x * (PER / 4);
#pragma unroll
  for (int q = 0; q < PER / 4; ++q) {
    const uint4 v = h4[q];
    loc[4 * q] = v.x, loc[4 * q + 1] = v.y, loc[4 * q + 2] = v.z, loc[4 * q + 3] = v.w;
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) run += loc[q];
  unsigned inc = run;  // inclusive scan over the warp
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wtot[warp] = inc;
  if (threadIdx.x == 0) {
    s_bin = NBIN - 1;
    s_at = 0;
    s_below = 0;
  }
  __syncthreads();
  unsigned wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += wtot[w];
  if (threadIdx.x == NT - 1) {  // no bin reaches `need`: the last bin, everything below it
    const unsigned all = wbase + inc;
    s_at = all;
    s_below = all - loc[PER - 1];
  }
  __syncthreads();
  unsigned acc = wbase + inc - run;  // exclusive prefix of this thread's first bin
  if (acc < need && acc + run >= need) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      if (acc < need && acc + loc[q] >= need) {
        s_bin = threadIdx.x * PER + q;
        s_at = acc + loc[q];
        s_below = acc;
      }
      acc += loc[q];
    }
  }
  __syncthreads();
  *bin = s_bin;
  *at = s_at;
  *below = s_below;
}

// pick[0] = threshold bin, pick[1] = survivors (cum count), pick[2] = below it
__global__ void __launch_bounds__(1024) k_policy_pick(const unsigned* __restrict__ hist, int H, int* __restrict__ pick) {
  int bin;
  unsigned at, below;
  block_pick(hist, (unsigned)H, &bin, &at, &below);
  if (threadIdx.x == 0) {
    pick[0] = bin;
    pick[1] = (int)at;
    pick[2] = (int)below;
  }
}

// Refinement when the first pick leaves more than REFINE survivors (a dense
// key range near the minimum): histogram the next 12 bits of the keys inside that bin and pick
// again with the remaining budget H - pick[2]. pick[3] = sub-bin threshold,
// pick[4] = final survivor count (pick[1] when no refinement is needed).
__global__ void k_policy_hist2(const uint64_t* __restrict__ K, int64_t n_slots, const unsigned long long* __restrict__ mm,
                               const int* __restrict__ pick, unsigned* __restrict__ hist2) {
  if (pick[1] <= REFINE) return;
  __shared__ unsigned h[NBIN];
  for (int t = threadIdx.x; t < NBIN; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const uint64_t lo = mm[0], hi = mm[1];
  const int sh = bin_shift(lo, hi);
  const int sh2 = sh > 12 ? sh - 12 : 0;
  const uint64_t tb = (uint64_t)pick[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_slots; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = K[i];
    if (k != ~0ull && ((k - lo) >> sh) == tb) atomicAdd(&h[((k - lo) >> sh2) & (NBIN - 1)], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < NBIN; t += blockDim.x)
    if (h[t]) atomicAdd(&hist2[t], h[t]);
}

__global__ void __launch_bounds__(1024) k_policy_pick2(const unsigned* __restrict__ hist2, int H, int* __restrict__ pick) {
  if (pick[1] <= REFINE) {
    if (threadIdx.x == 0) {
      pick[3] = NBIN - 1;
      pick[4] = pick[1];
    }
    return;
  }
  int bin;
  unsigned at, below;
  block_pick(hist2, (unsigned)(H - pick[2]), &bin, &at, &below);
  if (threadIdx.x == 0) {
    pick[3] = bin;
    pick[4] = pick[2] + (int)at;
  }
}

__global__ void k_policy_collect(const uint64_t* __restrict__ K, const DevLive* __restrict__ live, int64_t n_slots,
                                 const unsigned long long* __restrict__ mm, const int* __restrict__ pick,
                                 ScoreItem* __restrict__ out, int* __restrict__ n_out) {
  const int c = pick[4];
  if (c > CAP) return;  // host takes the segmented-sort path
  const uint64_t lo = mm[0], hi = mm[1];
  const int sh = bin_shift(lo, hi);
  const int sh2 = sh > 12 ? sh - 12 : 0;
  const uint64_t tb = (uint64_t)pick[0], tb2 = (uint64_t)pick[3];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_slots; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = K[i];
    if (k == ~0ull) continue;
    const uint64_t b = (k - lo) >> sh;
    if (b < tb || (b == tb && (((k - lo) >> sh2) & (NBIN - 1)) <= tb2)) {
      const int at = atomicAdd(n_out, 1);
      if (at < CAP) out[at] = ScoreItem{k, live[i].seq, i};
    }
  }
}

// one block: bitonic sort of the survivors (padded to CAP), first H out
__global__ void __launch_bounds__(SEG_T) k_policy_final(const ScoreItem* __restrict__ in, const int* __restrict__ n_in,
                                                        ScoreItem* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint64_t* kb = reinterpret_cast<uint64_t*>(sm);
  uint64_t* sq = kb + SEG;
  int64_t* sl = reinterpret_cast<int64_t*>(sq + SEG);
  const int n = min(*n_in, CAP);
  int n2 = SCORE_H;
  while (n2 < n) n2 <<= 1;  // only the survivors are sorted (usually ~H)
  for (int t = threadIdx.x; t < n2; t += SEG_T) {
    if (t < n) {
      const ScoreItem it = in[t];
      kb[t] = it.kb, sq[t] = it.seq, sl[t] = it.slot;
    } else {
      kb[t] = ~0ull, sq[t] = ~0ull, sl[t] = -1;
    }
  }
  seg_sort(kb, sq, sl, n2);
  for (int t = threadIdx.x; t < SCORE_H; t += SEG_T) out[t] = ScoreItem{kb[t], sq[t], sl[t]};
}

// ---------------------------------------------------------------------------
// The same radix threshold select as ONE cooperative persistent kernel (one
// CTA per SM, grid-wide barriers between the phases): keys + min/max ->
// histogram -> pick -> [refine histogram -> pick] -> collect -> sort of the
// survivors. The 7 launches, 2 memsets and the scratch allocation of the
// multi-kernel version cost ~0.18 ms per scoring at 500k live steps while
// the data is ~27 MB (4 us of HBM time); a scoring is now bounded by the
// barriers. Scratch persists in the store; CTA 0 leaves the histograms,
// min/max and counters zeroed for the next call and reports
// [head | pick[5] | n_out | bad] in one contiguous block (one D2H copy).
struct FusedScratch {
  uint64_t* K;                 // [n_slots]
  unsigned long long* mm;      // [2] min, max key image
  unsigned* hist;              // [NBIN]
  unsigned* hist2;             // [NBIN]
  int* n_acc;                  // [2] survivors appended, bad flag
  ScoreItem* items;            // [CAP]
  ScoreItem* head;             // [SCORE_H] report
  int* rep;                    // [8] report: pick[5], n_out, bad (follows head)
  unsigned long long* ts;      // [8] phase timestamps of CTA 0 (FC_SCORE_PHASES=1), else null
  int rank_max;                // survivors ranked across the grid (F) up to this; refine (D) above it
};

// REG: the store fits KR keys per thread of the grid, so each thread keeps
// its slots' key images in registers across the phases (no K[] round trips
// through memory) and issues all its slot loads before the prompt gathers.
constexpr int KR = 8;
template <bool REG>
__global__ void __launch_bounds__(SEG_T, 1) k_policy_fused(const DevLive* __restrict__ live, int64_t n_slots,
                                                           const DevPrompt* __restrict__ prompts, int policy,
                                                           uint64_t now, FusedScratch S) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int s_pick[5];
  auto stamp = [&](int p) {
    if (S.ts && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      S.ts[p] = t;
    }
  };
  stamp(0);
  // survivor counter: first used in phase (E), after two grid barriers
  if (blockIdx.x == 0 && threadIdx.x == 0) S.n_acc[0] = 0;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  uint64_t kr[REG ? KR : 1];
  // (A) key image of every slot, min/max
  {
    uint64_t lo = ~0ull, hi = 0;
    int b = 0;
    if constexpr (REG) {
      constexpr int G = 4;  // slots loaded together (registers: 4 x (40 + 16) bytes in flight)
#pragma unroll
      for (int j0 = 0; j0 < KR; j0 += G) {
        DevLive lv[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const int64_t i = gtid + (j0 + j) * gstride;
          if (i < n_slots) lv[j] = live[i];
          else lv[j].step = 0;
        }
        DevPrompt pv[G];
#pragma unroll
        for (int j = 0; j < G; ++j)
          if (lv[j].step != 0) pv[j] = prompts[lv[j].pslot];
#pragma unroll
        for (int j = 0; j < G; ++j) {
          uint64_t k = ~0ull;
          if (lv[j].step != 0) {
            uint64_t cap;
            k = key_bits(pkey(policy, lv[j], pv[j], now, &cap, &b));
            lo = k < lo ? k : lo;
            hi = k > hi ? k : hi;
          }
          kr[j0 + j] = k;
        }
      }
    } else {
      for (int64_t i = gtid; i < n_slots; i += gstride) {
        const DevLive l = live[i];
        uint64_t k = ~0ull;
        if (l.step != 0) {
          uint64_t cap;
          k = key_bits(pkey(policy, l, prompts[l.pslot], now, &cap, &b));
          lo = k < lo ? k : lo;
          hi = k > hi ? k : hi;
        }
        S.K[i] = k;
      }
    }
    if (b) atomicExch(&S.n_acc[1], 1);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t a = __shfl_xor_sync(0xffffffffu, lo, o), c = __shfl_xor_sync(0xffffffffu, hi, o);
      lo = a < lo ? a : lo;
      hi = c > hi ? c : hi;
    }
    if ((threadIdx.x & 31) == 0 && lo != ~0ull) {
      atomicMin(&S.mm[0], (unsigned long long)lo);
      atomicMax(&S.mm[1], (unsigned long long)hi);
    }
  }
  grid.sync();
  stamp(1);
  const uint64_t lo = S.mm[0], hi = S.mm[1];
  const int sh = bin_shift(lo, hi);
  const int sh2 = sh > 12 ? sh - 12 : 0;
  unsigned* h = reinterpret_cast<unsigned*>(sm);  // [NBIN] block histogram
  // every slot of this thread in lockstep across the warp (gstride % 32 == 0):
  // f(key, slot) with key ~0 for dead / out-of-range slots
  auto each = [&](auto f) {
    if constexpr (REG) {
#pragma unroll
      for (int j = 0; j < KR; ++j) f(kr[j], gtid + j * gstride);
    } else {
      for (int64_t i0 = gtid - (threadIdx.x & 31); i0 < n_slots; i0 += gstride) {
        const int64_t i = i0 + (threadIdx.x & 31);
        f(i < n_slots ? S.K[i] : ~0ull, i);
      }
    }
  };
  // (B) histogram of (key - min) >> sh
  for (int t = threadIdx.x; t < NBIN; t += blockDim.x) h[t] = 0;
  __syncthreads();
  // warp-aggregated: policy keys cluster in few bins (e.g. many LRBU keys
  // share an order of magnitude), and same-bin shared atomics serialize
  each([&](uint64_t k, int64_t) {
    const int bin = k != ~0ull ? (int)((k - lo) >> sh) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], (unsigned)__popc(peers));
  });
  __syncthreads();
  for (int t = threadIdx.x; t < NBIN; t += blockDim.x)
    if (h[t]) atomicAdd(&S.hist[t], h[t]);
  grid.sync();
  stamp(2);
  // (C) pick: every CTA computes the same pick from the global histogram
  {
    int bin;
    unsigned at, below;
    block_pick<SEG_T>(S.hist, (unsigned)SCORE_H, &bin, &at, &below);
    if (threadIdx.x == 0) {
      s_pick[0] = bin;
      s_pick[1] = (int)at;
      s_pick[2] = (int)below;
      s_pick[3] = NBIN - 1;
      s_pick[4] = (int)at;
    }
    __syncthreads();
  }
  stamp(3);
  // (D) refine inside the threshold bin when it leaves more survivors than
  // the rank pass (F) takes (a refine costs a histogram pass and a grid barrier)
  if (s_pick[1] > S.rank_max) {
    for (int t = threadIdx.x; t < NBIN; t += blockDim.x) h[t] = 0;
    __syncthreads();
    const uint64_t tb = (uint64_t)s_pick[0];
    each([&](uint64_t k, int64_t) {
      const int bin = (k != ~0ull && ((k - lo) >> sh) == tb) ? (int)(((k - lo) >> sh2) & (NBIN - 1)) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      if (bin >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], (unsigned)__popc(peers));
    });
    __syncthreads();
    for (int t = threadIdx.x; t < NBIN; t += blockDim.x)
      if (h[t]) atomicAdd(&S.hist2[t], h[t]);
    grid.sync();
    int bin;
    unsigned at, below;
    block_pick<SEG_T>(S.hist2, (unsigned)(SCORE_H - s_pick[2]), &bin, &at, &below);
    if (threadIdx.x == 0) {
      s_pick[3] = bin;
      s_pick[4] = s_pick[2] + (int)at;
    }
    __syncthreads();
  }
  stamp(4);
  // (E) collect the survivors
  if (s_pick[4] <= CAP) {
    const uint64_t tb = (uint64_t)s_pick[0], tb2 = (uint64_t)s_pick[3];
    each([&](uint64_t k, int64_t i) {
      if (k == ~0ull) return;
      const uint64_t b = (k - lo) >> sh;
      if (b < tb || (b == tb && (((k - lo) >> sh2) & (NBIN - 1)) <= tb2)) {
        const int at = atomicAdd(&S.n_acc[0], 1);
        if (at < CAP) S.items[at] = ScoreItem{k, live[i].seq, i};
      }
    });
  }
  grid.sync();
  stamp(5);
  // (F) the head: a survivor's rank = how many survivors precede it in
  // (key, seq, slot) order, a total order, so the ranks are a permutation.
  // One warp per survivor over all the CTAs (up to RANK_MAX survivors, which
  // is why (D) rarely runs), each written straight to its place: no
  // single-CTA sort on the tail. More survivors (dense ties): CTA 0 sorts.
  const int n = min(S.n_acc[0], CAP);
  if (s_pick[4] <= CAP && n <= S.rank_max) {
    // survivor i: CTA i % grid, warp (i / grid) % warps; each CTA with work
    // stages the whole survivor list in shared memory once
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NWARP = SEG_T / 32;
    if ((int)blockIdx.x < n) {
      ScoreItem* si = reinterpret_cast<ScoreItem*>(sm);
      for (int t = threadIdx.x; t < n; t += SEG_T) si[t] = S.items[t];
      __syncthreads();
      for (int i = blockIdx.x + gridDim.x * warp; i < n; i += gridDim.x * NWARP) {
        const ScoreItem me = si[i];
        int r = 0;
#pragma unroll 4
        for (int j = lane; j < n; j += 32) {
          const ScoreItem o = si[j];
          r += o.kb < me.kb || (o.kb == me.kb && (o.seq < me.seq || (o.seq == me.seq && o.slot < me.slot)));
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
        if (lane == 0 && r < SCORE_H) S.head[r] = me;
      }
    }
    for (int64_t t = n + gtid; t < SCORE_H; t += gstride) S.head[t] = ScoreItem{~0ull, ~0ull, -1};
  }
  if (blockIdx.x != 0) return;
  if (s_pick[4] <= CAP && n > S.rank_max) {
    uint64_t* kb = reinterpret_cast<uint64_t*>(sm);
    uint64_t* sq = kb + SEG;
    int64_t* sl = reinterpret_cast<int64_t*>(sq + SEG);
    int n2 = SCORE_H;
    while (n2 < n) n2 <<= 1;
    for (int t = threadIdx.x; t < n2; t += SEG_T) {
      if (t < n) {
        const ScoreItem it = S.items[t];
        kb[t] = it.kb, sq[t] = it.seq, sl[t] = it.slot;
      } else {
        kb[t] = ~0ull, sq[t] = ~0ull, sl[t] = -1;
      }
    }
    seg_sort(kb, sq, sl, n2);
    for (int t = threadIdx.x; t < SCORE_H; t += SEG_T) S.head[t] = ScoreItem{kb[t], sq[t], sl[t]};
  }
  stamp(6);
  if (threadIdx.x < 5) S.rep[threadIdx.x] = s_pick[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    S.rep[5] = n;
    S.rep[6] = S.n_acc[1];
    S.n_acc[1] = 0;  // n_acc[0] is read by every CTA after the last barrier: reset in phase (A) of the next call
    S.mm[0] = ~0ull;
    S.mm[1] = 0;
  }
  for (int t = threadIdx.x; t < NBIN; t += blockDim.x) {
    S.hist[t] = 0;
    S.hist2[t] = 0;
  }
}

struct ScatterLive {
  int64_t slot;
  DevLive v;
};
struct ScatterPrompt {
  int64_t slot;
  DevPrompt v;
};
__global__ void k_scatter(const ScatterLive* __restrict__ ul, int nl, DevLive* __restrict__ live,
                          const ScatterPrompt* __restrict__ up, int np, DevPrompt* __restrict__ prompts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nl) live[ul[i].slot] = ul[i].v;
  if (i < np) prompts[up[i].slot] = up[i].v;
}

// Host copy of the policy key: identical IEEE operations to pkey().
static double host_key(int policy, uint64_t f, int step, uint64_t last, uint64_t seq, uint64_t cap, uint64_t now) {
  switch (policy) {
    case LC_POLICY_FIFO: return (double)seq;
    case LC_POLICY_LRU: return (double)last;
    case LC_POLICY_LCBFU: return (double)(f + 1) * (double)step;
    default: {
      if (now < last) raise(LC_ERR_INVALID_ARGUMENT, "lrbu_priority: now precedes last access");
      if (cap == 0) raise(LC_ERR_INVALID_ARGUMENT, "lrbu_priority: zero capacity");
      const uint64_t dd = now - last;
      const double duration = (double)(dd > 1 ? dd : 1);
      volatile double num = (double)(f + 1) * (double)step;
      volatile double den = (double)cap * duration;
      return num / den;
    }
  }
}

}  // namespace fc

using namespace fc;

struct lc_store {
  struct Live {
    int step;
    int si;  // index into entry data steps
    uint64_t f, last, inserted_at, seq, priv;
    int64_t slot;
  };
  struct Rec {
    lc_entry* view = nullptr;
    uint64_t shared = 0;
    std::vector<Live> live;  // ascending step
    int32_t pslot = -1;
  };
  lc_ctx* ctx;
  uint64_t capacity, used = 0, next_seq = 0;
  int policy;
  std::map<uint64_t, Rec> prompts;
  // device table + host mirror
  std::vector<DevLive> hl;
  std::vector<DevPrompt> hp;
  std::vector<int64_t> free_l;
  std::vector<int32_t> free_p;
  std::unordered_set<int64_t> dirty_l;
  std::unordered_set<int32_t> dirty_p;
  DevLive* dl = nullptr;
  DevPrompt* dp = nullptr;
  int64_t cap_l = 0, cap_p = 0;
  int64_t live_count = 0;
  uint64_t scorings = 0;
  // persistent scratch of the fused scoring kernel (+ pinned report buffer)
  uint8_t* fs = nullptr;
  int64_t fs_slots = -1;
  uint8_t* fs_host = nullptr;

  ~lc_store() {
    for (auto& kv : prompts) delete kv.second.view;
    if (dl) cudaFree(dl);
    if (dp) cudaFree(dp);
    if (fs) cudaFree(fs);
    if (fs_host) cudaFreeHost(fs_host);
  }

  // scratch layout: [K n_slots] [mm 2] [hist NBIN] [hist2 NBIN] [n_acc 2] [items CAP] [head H | rep 8]
  FusedScratch fused_scratch(int64_t n_slots, size_t* rep_off, size_t* rep_bytes) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t k_b = al((size_t)std::max<int64_t>(n_slots, 1) * 8);
    const size_t z_off = k_b, z_b = al(16 + 2 * NBIN * 4 + 8);
    const size_t i_off = z_off + z_b, i_b = al((size_t)CAP * sizeof(ScoreItem));
    const size_t h_off = i_off + i_b, h_b = (size_t)SCORE_H * sizeof(ScoreItem) + 32;
    if (n_slots > fs_slots) {
      const int64_t want = std::max<int64_t>(n_slots, std::max<int64_t>(4096, fs_slots * 2));
      const size_t total = al((size_t)want * 8) + z_b + i_b + h_b;
      if (fs) {
        FC_CUDA(cudaStreamSynchronize(ctx->stream));
        cudaFree(fs);
      }
      FC_CUDA(cudaMalloc(&fs, total));
      fs_slots = want;
      if (!fs_host) FC_CUDA(cudaMallocHost(&fs_host, h_b));
    }
    // the zone after K moves with fs_slots: locate it from the allocation size
    const size_t kz = al((size_t)fs_slots * 8);
    FusedScratch S;
    S.K = reinterpret_cast<uint64_t*>(fs);
    S.mm = reinterpret_cast<unsigned long long*>(fs + kz);
    S.hist = reinterpret_cast<unsigned*>(fs + kz + 16);
    S.hist2 = S.hist + NBIN;
    S.n_acc = reinterpret_cast<int*>(S.hist2 + NBIN);
    S.items = reinterpret_cast<ScoreItem*>(fs + kz + z_b);
    S.head = reinterpret_cast<ScoreItem*>(fs + kz + z_b + i_b);
    S.rep = reinterpret_cast<int*>(S.head + SCORE_H);
    S.ts = nullptr;
    // FC_SCORE_RANK_MAX (tests): lower it to take the refine pass and CTA 0's bitonic sort
    const char* rm = getenv("FC_SCORE_RANK_MAX");
    S.rank_max = rm ? std::max(0, std::min(RANK_MAX, atoi(rm))) : RANK_MAX;
    if (getenv("FC_SCORE_PHASES") && atoi(getenv("FC_SCORE_PHASES")) == 1) {
      static unsigned long long* ts_dev = nullptr;  // diagnostic only
      if (!ts_dev) FC_CUDA(cudaMalloc(&ts_dev, 8 * sizeof(unsigned long long)));
      S.ts = ts_dev;
    }
    *rep_off = kz + z_b + i_b;
    *rep_bytes = h_b;
    (void)z_off;
    (void)h_off;
    (void)i_off;
    return S;
  }

  int64_t alloc_live() {
    if (!free_l.empty()) {
      int64_t s = free_l.back();
      free_l.pop_back();
      return s;
    }
    hl.push_back(DevLive{});
    return (int64_t)hl.size() - 1;
  }
  int32_t alloc_prompt() {
    if (!free_p.empty()) {
      int32_t s = free_p.back();
      free_p.pop_back();
      return s;
    }
    hp.push_back(DevPrompt{});
    return (int32_t)hp.size() - 1;
  }
  void write_live(const Rec& r, const Live& l) {
    hl[l.slot] = DevLive{l.f, l.last, l.seq, l.priv, l.step, r.pslot};
    dirty_l.insert(l.slot);
  }
  void write_prompt(const Rec& r) {
    hp[r.pslot] = DevPrompt{r.shared, (int32_t)r.live.size(), 0};
    dirty_p.insert(r.pslot);
  }

  void sync_device() {
    const int64_t nl = (int64_t)hl.size(), np = (int64_t)hp.size();
    auto grow = [&](auto*& ptr, int64_t& cap, int64_t need, size_t elem, size_t used_elems) {
      if (need <= cap) return false;
      const int64_t nc = std::max<int64_t>(need, std::max<int64_t>(1024, cap * 2));
      void* p = nullptr;
      FC_CUDA(cudaMalloc(&p, nc * elem));
      FC_CUDA(cudaMemsetAsync(p, 0, nc * elem, ctx->stream));
      (void)used_elems;
      if (ptr) {
        FC_CUDA(cudaStreamSynchronize(ctx->stream));
        cudaFree(ptr);
      }
      ptr = static_cast<std::remove_reference_t<decltype(ptr)>>(p);
      cap = nc;
      return true;
    };
    const bool rl = grow(dl, cap_l, nl, sizeof(DevLive), nl);
    const bool rp = grow(dp, cap_p, np, sizeof(DevPrompt), np);
    if (rl) {
      if (nl) FC_CUDA(cudaMemcpyAsync(dl, hl.data(), nl * sizeof(DevLive), cudaMemcpyHostToDevice, ctx->stream));
      dirty_l.clear();
    }
    if (rp) {
      if (np) FC_CUDA(cudaMemcpyAsync(dp, hp.data(), np * sizeof(DevPrompt), cudaMemcpyHostToDevice, ctx->stream));
      dirty_p.clear();
    }
    if (dirty_l.empty() && dirty_p.empty()) return;
    std::vector<ScatterLive> ul;
    std::vector<ScatterPrompt> up;
    for (int64_t s : dirty_l) ul.push_back(ScatterLive{s, hl[s]});
    for (int32_t s : dirty_p) up.push_back(ScatterPrompt{s, hp[s]});
    dirty_l.clear();
    dirty_p.clear();
    DevBuf bl(ul.size() * sizeof(ScatterLive) + 16, ctx->stream), bp(up.size() * sizeof(ScatterPrompt) + 16, ctx->stream);
    if (!ul.empty()) FC_CUDA(cudaMemcpyAsync(bl.p, ul.data(), ul.size() * sizeof(ScatterLive), cudaMemcpyHostToDevice, ctx->stream));
    if (!up.empty()) FC_CUDA(cudaMemcpyAsync(bp.p, up.data(), up.size() * sizeof(ScatterPrompt), cudaMemcpyHostToDevice, ctx->stream));
    const int n = (int)std::max(ul.size(), up.size());
    k_scatter<<<grid_for(n, 256), 256, 0, ctx->stream>>>(bl.as<ScatterLive>(), (int)ul.size(), dl, bp.as<ScatterPrompt>(),
                                                        (int)up.size(), dp);
    FC_LAUNCH_CHECK();
    count_launch(ctx);
  }

  // GPU scoring: the SCORE_H smallest (key, seq) live steps at time `now`.
  std::vector<Cand> score_head(uint64_t now) {
    sync_device();
    ++scorings;
    const int64_t n_slots = (int64_t)hl.size();
    const size_t smem = (size_t)SEG * (8 + 8 + 8);
    static std::atomic<uint64_t> attr_done{0};  // per device, once
    if (!(attr_done.load() & (1ull << (ctx->device & 63)))) {
      FC_CUDA(cudaFuncSetAttribute(k_policy_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      FC_CUDA(cudaFuncSetAttribute(k_head_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      FC_CUDA(cudaFuncSetAttribute(k_policy_final, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_done.fetch_or(1ull << (ctx->device & 63));
    }
    DevBuf bad(sizeof(int), ctx->stream);
    FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
    KTimer kt(ctx, "policy");
    // fast path: radix threshold select
    const char* fe = getenv("FC_SCORE_SORT");
    const bool fast = !(fe && atoi(fe) == 1) && n_slots > 0;
    DevBuf cur;
    const bool fused = !(getenv("FC_SCORE_FUSED") && atoi(getenv("FC_SCORE_FUSED")) == 0);
    if (fast && fused) {
      kt.cancel();  // the kernel alone is timed below (host set-up between two events would count as GPU time)
      KTimer kcall(ctx, "policy_call");  // launch through the report readback (one scoring as the host sees it)
      size_t rep_off = 0, rep_bytes = 0;
      const int64_t had = fs_slots;
      FusedScratch S = fused_scratch(n_slots, &rep_off, &rep_bytes);
      if (had != fs_slots) {  // fresh scratch: zero histograms/counters, min = ~0
        FC_CUDA(cudaMemsetAsync(S.mm, 0, 16 + 2 * NBIN * 4 + 8, ctx->stream));
        FC_CUDA(cudaMemsetAsync(S.mm, 0xff, 8, ctx->stream));
      }
      static std::atomic<uint64_t> fattr{0};
      static int blocks_per_sm = 0;
      if (!(fattr.load() & (1ull << (ctx->device & 63)))) {
        FC_CUDA(cudaFuncSetAttribute(k_policy_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        FC_CUDA(cudaFuncSetAttribute(k_policy_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int b1 = 0, b2 = 0;
        FC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_policy_fused<true>, SEG_T, smem));
        FC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_policy_fused<false>, SEG_T, smem));
        blocks_per_sm = std::min(b1, b2);
        fattr.fetch_or(1ull << (ctx->device & 63));
      }
      if (blocks_per_sm < 1) raise(LC_ERR_CUDA, "fused scoring kernel cannot be resident");
      const int grid = (int)std::min<int64_t>(ctx->sm_count, std::max<int64_t>(1, (n_slots + SEG_T - 1) / SEG_T));
      const bool reg = n_slots <= (int64_t)KR * grid * SEG_T && !(getenv("FC_SCORE_REG") && atoi(getenv("FC_SCORE_REG")) == 0);
      const DevLive* a0 = dl;
      const DevPrompt* a2 = dp;
      int a3 = policy;
      uint64_t a4 = now;
      int64_t a1 = n_slots;
      void* args[] = {(void*)&a0, (void*)&a1, (void*)&a2, (void*)&a3, (void*)&a4, (void*)&S};
      KTimer kk(ctx, "policy");
      FC_CUDA(cudaLaunchCooperativeKernel(reg ? (const void*)k_policy_fused<true> : (const void*)k_policy_fused<false>,
                                          dim3(grid), dim3(SEG_T), args, smem, ctx->stream));
      FC_LAUNCH_CHECK();
      count_launch(ctx, 1);
      kk.stop();
      FC_CUDA(cudaMemcpyAsync(fs_host, fs + rep_off, rep_bytes, cudaMemcpyDeviceToHost, ctx->stream));
      kcall.stop();
      sync(ctx);
      const int* rp = reinterpret_cast<const int*>(fs_host + (size_t)SCORE_H * sizeof(ScoreItem));
      if (rp[6]) raise(LC_ERR_INVALID_ARGUMENT, "lrbu_priority: now precedes last access");
      if (S.ts) {  // FC_SCORE_PHASES=1: mean CTA-0 phase times over the calls so far, every 4 calls
        static double acc[6] = {0, 0, 0, 0, 0, 0};
        static long calls = 0;
        unsigned long long t[8];
        FC_CUDA(cudaMemcpy(t, S.ts, sizeof(t), cudaMemcpyDeviceToHost));
        for (int i = 0; i < 6; ++i) acc[i] += (double)(t[i + 1] - t[i]);
        if (++calls % 4 == 0)
          fprintf(stderr, "[score phases] %ld calls, mean ns: keys+sync %.0f | hist+sync %.0f | pick %.0f | refine %.0f | "
                  "collect+sync %.0f | head (CTA 0) %.0f\n", calls, acc[0] / calls, acc[1] / calls,
                  acc[2] / calls, acc[3] / calls, acc[4] / calls, acc[5] / calls);
      }
      if (getenv("FC_TRACE") && atoi(getenv("FC_TRACE")) == 1)
        fprintf(stderr, "[score fused] slots %lld: bin %d, survivors %d (below %d), sub-bin %d -> %d%s\n",
                (long long)n_slots, rp[0], rp[1], rp[2], rp[3], rp[4], rp[4] <= CAP ? "" : " => segmented sort");
      if (rp[4] <= CAP) {
        std::vector<ScoreItem> hh(reinterpret_cast<const ScoreItem*>(fs_host),
                                  reinterpret_cast<const ScoreItem*>(fs_host) + SCORE_H);
        return decode_head(hh);
      }
    } else if (fast) {
      // scratch: K[n] | mm[2] | hist[NBIN] | hist2[NBIN] | pick[5] | n_out | items[CAP] | head[H]
      const size_t kbytes = ((size_t)n_slots * 8 + 255) & ~size_t(255);
      const size_t zoff = kbytes, zbytes = 16 + 2 * NBIN * 4 + 32;
      const size_t ioff = zoff + ((zbytes + 255) & ~size_t(255));
      const size_t hoff = ioff + CAP * sizeof(ScoreItem);
      DevBuf scr(hoff + SCORE_H * sizeof(ScoreItem), ctx->stream);
      uint8_t* base = scr.as<uint8_t>();
      uint64_t* K = reinterpret_cast<uint64_t*>(base);
      unsigned long long* mm = reinterpret_cast<unsigned long long*>(base + zoff);
      unsigned* hist = reinterpret_cast<unsigned*>(base + zoff + 16);
      unsigned* hist2 = hist + NBIN;
      int* pick = reinterpret_cast<int*>(base + zoff + 16 + 2 * NBIN * 4);
      int* n_out = pick + 5;
      FC_CUDA(cudaMemsetAsync(base + zoff, 0, zbytes, ctx->stream));
      FC_CUDA(cudaMemsetAsync(mm, 0xff, 8, ctx->stream));  // min = ~0
      const int grid = std::max(1, std::min<int>((int)((n_slots + 255) / 256), ctx->sm_count * 8));
      k_policy_keys<<<grid, 256, 0, ctx->stream>>>(dl, n_slots, dp, policy, now, K, mm, bad.as<int>());
      k_policy_hist<<<std::min(grid, ctx->sm_count * 2), 512, 0, ctx->stream>>>(K, n_slots, mm, hist);
      k_policy_pick<<<1, 1024, 0, ctx->stream>>>(hist, SCORE_H, pick);
      k_policy_hist2<<<std::min(grid, ctx->sm_count * 2), 512, 0, ctx->stream>>>(K, n_slots, mm, pick, hist2);
      k_policy_pick2<<<1, 1024, 0, ctx->stream>>>(hist2, SCORE_H, pick);
      k_policy_collect<<<grid, 256, 0, ctx->stream>>>(K, dl, n_slots, mm, pick,
                                                      reinterpret_cast<ScoreItem*>(base + ioff), n_out);
      k_policy_final<<<1, SEG_T, smem, ctx->stream>>>(reinterpret_cast<ScoreItem*>(base + ioff), n_out,
                                                      reinterpret_cast<ScoreItem*>(base + hoff));
      FC_LAUNCH_CHECK();
      count_launch(ctx, 7);
      kt.stop();  // GPU span of the scoring launches (not the readback)
      // one sync: head + the survivor count come back together
      std::vector<ScoreItem> hh(SCORE_H);
      int hp[6] = {0, 0, 0, 0, 0, 0};
      int32_t hb0 = 0;
      FC_CUDA(cudaMemcpyAsync(hh.data(), base + hoff, SCORE_H * sizeof(ScoreItem), cudaMemcpyDeviceToHost, ctx->stream));
      FC_CUDA(cudaMemcpyAsync(hp, pick, 6 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      FC_CUDA(cudaMemcpyAsync(&hb0, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      if (hb0) raise(LC_ERR_INVALID_ARGUMENT, "lrbu_priority: now precedes last access");
      if (getenv("FC_TRACE") && atoi(getenv("FC_TRACE")) == 1)
        fprintf(stderr, "[score] slots %lld: bin %d, survivors %d (below %d), sub-bin %d -> %d%s\n", (long long)n_slots,
                hp[0], hp[1], hp[2], hp[3], hp[4], hp[4] <= CAP ? "" : " => segmented sort");
      if (hp[4] <= CAP) return decode_head(hh);
    }
    {
      int64_t nblk = std::max<int64_t>(1, (n_slots + SEG - 1) / SEG);
      DevBuf h0((size_t)nblk * SCORE_H * sizeof(ScoreItem), ctx->stream);
      k_policy_seg<<<(unsigned)nblk, SEG_T, smem, ctx->stream>>>(dl, n_slots, dp, policy, now, h0.as<ScoreItem>(),
                                                                  bad.as<int>());
      FC_LAUNCH_CHECK();
      count_launch(ctx);
      cur = std::move(h0);
      int64_t n_in = nblk * SCORE_H;
      while (n_in > SCORE_H) {
        const int64_t nb = (n_in + SEG - 1) / SEG;
        DevBuf nxt((size_t)nb * SCORE_H * sizeof(ScoreItem), ctx->stream);
        k_head_seg<<<(unsigned)nb, SEG_T, smem, ctx->stream>>>(cur.as<ScoreItem>(), n_in, nxt.as<ScoreItem>());
        FC_LAUNCH_CHECK();
        count_launch(ctx);
        cur = std::move(nxt);
        n_in = nb * SCORE_H;
      }
    }
    kt.stop();
    std::vector<ScoreItem> hi(SCORE_H);
    int32_t hb = 0;
    FC_CUDA(cudaMemcpyAsync(hi.data(), cur.p, SCORE_H * sizeof(ScoreItem), cudaMemcpyDeviceToHost, ctx->stream));
    FC_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (hb) raise(LC_ERR_INVALID_ARGUMENT, "lrbu_priority: now precedes last access");
    return decode_head(hi);
  }

  static std::vector<Cand> decode_head(const std::vector<ScoreItem>& hi) {
    std::vector<Cand> h;
    h.reserve(SCORE_H);
    for (const ScoreItem& it : hi) {
      if (it.kb == ~0ull && it.seq == ~0ull) break;  // dead / padding
      uint64_t b = it.kb;
      b = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
      double key;
      memcpy(&key, &b, 8);
      h.push_back(Cand{-key, it.seq, it.slot});
    }
    return h;
  }

  // slot -> (prompt record, live index)
  std::unordered_map<int64_t, uint64_t> slot_prompt;

  // The eviction state (scored head + re-keyed siblings) stays valid across
  // evict_one / insert_steps calls at the same `now` as long as nothing but
  // evictions happened in between; any other mutation drops it.
  struct Evictor;
  std::unique_ptr<Evictor> evc;
  Evictor& evictor(uint64_t now);
  void invalidate() { evc.reset(); }

  lc_step_entry remove_step(std::map<uint64_t, Rec>::iterator it, int li, uint64_t attributed) {
    Rec& r = it->second;
    Live l = r.live[li];
    lc_step_entry out{it->first, l.step, 0, l.f, l.last, l.inserted_at, l.seq, attributed};
    used -= l.priv;
    hl[l.slot] = DevLive{};
    dirty_l.insert(l.slot);
    free_l.push_back(l.slot);
    slot_prompt.erase(l.slot);
    --live_count;
    r.live.erase(r.live.begin() + li);
    // the entry view drops the evicted step record (store.cpp:169-170)
    auto& sel = r.view->sel;
    sel.erase(std::remove(sel.begin(), sel.end(), l.si), sel.end());
    if (r.live.empty()) {
      used -= r.shared;
      hp[r.pslot] = DevPrompt{};
      dirty_p.insert(r.pslot);
      free_p.push_back(r.pslot);
      delete r.view;
      prompts.erase(it);
    } else {
      write_prompt(r);
    }
    return out;
  }

  // k evictions at a fixed `now` (one insert_steps call, or one evict_one).
  struct Evictor {
    lc_store* s;
    uint64_t now;
    std::vector<Cand> head;
    size_t pos = 0;
    bool have = false;
    std::unordered_map<int64_t, double> rekeyed;  // slot -> current key (LRBU siblings)
    struct HE {
      double key;
      uint64_t seq;
      int64_t slot;
      bool operator>(const HE& o) const { return key > o.key || (key == o.key && seq > o.seq); }
    };
    std::priority_queue<HE, std::vector<HE>, std::greater<HE>> heap;
    Evictor(lc_store* st, uint64_t n) : s(st), now(n) {}

    // The slot evict_one(now) takes next (exact argmin of (key, seq) over the
    // live table), with its key; only stale bookkeeping is dropped.
    int64_t pick(double* key_out, uint64_t* seq_out) {
      if (s->prompts.empty()) raise(LC_ERR_LOGIC, "evict_one: store is empty");
      for (;;) {
        if (!have) {
          head = s->score_head(now);
          pos = 0;
          have = true;
          rekeyed.clear();
          heap = decltype(heap)();
        }
        // first head entry that is still live and was not re-keyed
        while (pos < head.size() &&
               (!s->slot_prompt.count(head[pos].slot) || rekeyed.count(head[pos].slot)))
          ++pos;
        // drop stale heap tops
        while (!heap.empty()) {
          const HE& t = heap.top();
          auto it = rekeyed.find(t.slot);
          if (!s->slot_prompt.count(t.slot) || it == rekeyed.end() || it->second != t.key) heap.pop();
          else break;
        }
        if (pos >= head.size()) {
          have = false;  // head exhausted: re-score the live table
          continue;
        }
        int64_t victim = head[pos].slot;
        double vkey = -head[pos].s;
        uint64_t vseq = head[pos].id;
        if (!heap.empty()) {
          const HE& t = heap.top();
          if (t.key < vkey || (t.key == vkey && t.seq < vseq)) {
            victim = t.slot;
            vkey = t.key;
            vseq = t.seq;
          }
        }
        if (key_out) *key_out = vkey;
        if (seq_out) *seq_out = vseq;
        return victim;
      }
    }

    lc_step_entry next() { return evict_slot(pick(nullptr, nullptr)); }

    // The next (up to) m victims evict_one(now) would take, with their keys and
    // used() after each removal, WITHOUT evicting: the walk of pick() /
    // evict_slot() replayed on overlays (removed slots, per-prompt removed
    // counts, re-keyed siblings). It stops at m or earlier where the real walk
    // would re-score the table (scored head exhausted); *more = live steps
    // remain beyond the list. A shard's
    // sequence depends only on its own records, so the global eviction of an
    // entry-sharded store is the (key, seq) merge of these per-shard lists.
    int peek(int m, lc_step_entry* out, double* keys, uint64_t* used_after, bool* more) {
      *more = false;
      if (s->prompts.empty() || m <= 0) return 0;
      pick(nullptr, nullptr);  // a scored head exists (may re-score)
      size_t p = pos;
      std::unordered_map<int64_t, double> rk(rekeyed);
      auto hp = heap;
      std::unordered_set<int64_t> removed;
      std::unordered_map<uint64_t, size_t> gone;  // prompt -> live steps removed so far
      uint64_t u = s->used;
      int n = 0;
      auto live = [&](int64_t slot) { return s->slot_prompt.count(slot) && !removed.count(slot); };
      while (n < m) {
        while (p < head.size() && (!live(head[p].slot) || rk.count(head[p].slot))) ++p;
        while (!hp.empty()) {
          const HE& t = hp.top();
          auto it = rk.find(t.slot);
          if (!live(t.slot) || it == rk.end() || it->second != t.key) hp.pop();
          else break;
        }
        if (p >= head.size()) break;  // the real walk would re-score here
        int64_t victim = head[p].slot;
        double vkey = -head[p].s;
        uint64_t vseq = head[p].id;
        if (!hp.empty()) {
          const HE& t = hp.top();
          if (t.key < vkey || (t.key == vkey && t.seq < vseq)) {
            victim = t.slot;
            vkey = t.key;
            vseq = t.seq;
          }
        }
        const uint64_t pid = s->slot_prompt.at(victim);
        const Rec& r = s->prompts.at(pid);
        size_t& g = gone[pid];
        const size_t nlive = r.live.size() - g;
        const Live* lv = nullptr;
        for (const Live& l : r.live)
          if (l.slot == victim) lv = &l;
        out[n] = lc_step_entry{pid, lv->step, 0, lv->f, lv->last, lv->inserted_at, lv->seq, lv->priv + r.shared / nlive};
        keys[n] = vkey;
        removed.insert(victim);
        ++g;
        u -= lv->priv;
        if (nlive == 1) u -= r.shared;
        used_after[n] = u;
        ++n;
        if (s->policy == LC_POLICY_LRBU && nlive > 1) {  // evict_slot's sibling re-key
          for (const Live& l : r.live) {
            if (removed.count(l.slot)) continue;
            const uint64_t cap = l.priv + r.shared / (nlive - 1);
            const double k = host_key(s->policy, l.f, l.step, l.last, l.seq, cap, now);
            rk[l.slot] = k;
            hp.push(HE{k, l.seq, l.slot});
          }
        }
      }
      // the shard's sequence continues past this list (cut at m, or at a
      // re-score point) while live steps remain unlisted
      *more = (int64_t)removed.size() < s->live_count;
      return n;
    }

    // the StepEntry evict_slot(slot) would return, without evicting
    lc_step_entry describe(int64_t slot) const {
      const auto it = s->prompts.find(s->slot_prompt.at(slot));
      const Rec& r = it->second;
      for (const Live& l : r.live)
        if (l.slot == slot)
          return lc_step_entry{it->first, l.step, 0, l.f, l.last, l.inserted_at, l.seq, l.priv + r.shared / r.live.size()};
      raise(LC_ERR_INTERNAL, "evictor: slot not live");
    }

    lc_step_entry evict_slot(int64_t slot) {
      auto it = s->prompts.find(s->slot_prompt.at(slot));
      Rec& r = it->second;
      int li = -1;
      for (size_t i = 0; i < r.live.size(); ++i)
        if (r.live[i].slot == slot) li = (int)i;
      const uint64_t attributed = r.live[li].priv + r.shared / r.live.size();
      const bool siblings_rekey = s->policy == LC_POLICY_LRBU && r.live.size() > 1;
      const uint64_t pid = it->first;
      lc_step_entry out = s->remove_step(it, li, attributed);
      if (siblings_rekey) {
        Rec& rr = s->prompts.at(pid);
        for (const Live& l : rr.live) {
          const uint64_t cap = l.priv + rr.shared / rr.live.size();
          const double k = host_key(s->policy, l.f, l.step, l.last, l.seq, cap, now);
          rekeyed[l.slot] = k;
          heap.push(HE{k, l.seq, l.slot});
        }
      }
      return out;
    }
  };
};

lc_store::Evictor& lc_store::evictor(uint64_t now) {
  if (!evc || evc->now != now) evc.reset(new Evictor(this, now));
  return *evc;
}

extern "C" {

lc_status lc_store_create(lc_ctx* ctx, uint64_t capacity, int policy, lc_store** out) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && out, "null argument");
  if (policy < 0 || policy > 3) raise(LC_ERR_INVALID_ARGUMENT, "invalid policy value");
  auto* s = new lc_store();
  s->ctx = ctx;
  s->capacity = capacity;
  s->policy = policy;
  *out = s;
  LC_API_END
}

lc_status lc_store_destroy(lc_store* s) {
  LC_API_BEGIN
  if (!s) return LC_OK;
  DeviceGuard g(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  delete s;
  LC_API_END
}

}  // extern "C"

namespace {
// insert_steps validation (store.cpp:53-76) up to, not including, the
// OversizedEntry check: the records kept (entry->sel indices of the requested
// steps) and the entry's standalone size (shared + their private bytes).
std::vector<int> check_insert(lc_store* s, uint64_t prompt, lc_entry* entry, const int32_t* steps, int n_steps,
                              uint64_t* standalone) {
  for (int i = 0; i < n_steps; ++i)
    if (steps[i] < 1 || steps[i] > 50) raise(LC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
  if (n_steps <= 0) raise(LC_ERR_INVALID_ARGUMENT, "insert_steps: empty step list");
  const EntryData& d = *entry->d;
  if (d.prompt != prompt) raise(LC_ERR_INVALID_ARGUMENT, "insert_steps: prompt does not match entry");
  if (s->prompts.count(prompt)) raise(LC_ERR_INVALID_ARGUMENT, "insert_steps: prompt already cached");
  auto has = [&](int st) {
    for (int k : entry->sel)
      if (d.steps[k] == st) return true;
    return false;
  };
  for (int i = 0; i < n_steps; ++i) {
    const int st = steps[i];
    if (!(st == 5 || st == 10 || st == 15 || st == 20 || st == 25))
      raise(LC_ERR_INVALID_ARGUMENT, "insert_steps: step not cacheable");
    if (!has(st)) raise(LC_ERR_INVALID_ARGUMENT, "insert_steps: step missing from entry");
  }
  // keep only the requested records (store.cpp:68-71)
  std::vector<int> sel;
  for (int k : entry->sel)
    if (std::find(steps, steps + n_steps, d.steps[k]) != steps + n_steps) sel.push_back(k);
  uint64_t sz = d.shared_bytes();
  for (int k : sel) sz += d.private_bytes(k);
  *standalone = sz;
  return sel;
}
}  // namespace

extern "C" {

lc_status lc_store_check_insert(lc_store* s, uint64_t prompt, lc_entry* entry, const int32_t* steps, int n_steps,
                                uint64_t* standalone) {
  LC_API_BEGIN
  FC_REQUIRE(s && entry && standalone, "null argument");
  check_insert(s, prompt, entry, steps, n_steps, standalone);
  LC_API_END
}

lc_status lc_store_insert(lc_store* s, uint64_t prompt, lc_entry* entry, const int32_t* steps, int n_steps, uint64_t now,
                          lc_step_entry* evicted, int cap, int* n_evicted) {
  LC_API_BEGIN
  FC_REQUIRE(s && entry, "null argument");
  DeviceGuard g(s->ctx->device);
  if (n_evicted) *n_evicted = 0;
  uint64_t standalone = 0;
  const std::vector<int> sel = check_insert(s, prompt, entry, steps, n_steps, &standalone);
  const EntryData& d = *entry->d;
  lc_store::Rec rec;
  rec.view = make_entry_view(entry->d, sel);
  rec.shared = d.shared_bytes();
  if (standalone > s->capacity) {
    delete rec.view;
    set_last_oversize(standalone, s->capacity);
    raise(LC_ERR_OVERSIZED_ENTRY, "entry of " + std::to_string(standalone) + " bytes exceeds capacity limit of " +
                                      std::to_string(s->capacity) + " bytes");
  }
  int ne = 0;
  try {
    if (s->used + standalone > s->capacity) {
      lc_store::Evictor& ev = s->evictor(now);
      while (s->used + standalone > s->capacity) {
        lc_step_entry v = ev.next();
        if (evicted && ne < cap) evicted[ne] = v;
        ++ne;
      }
    }
  } catch (...) {
    delete rec.view;
    if (n_evicted) *n_evicted = ne;
    throw;
  }
  s->invalidate();  // new live steps may precede the scored head
  rec.pslot = s->alloc_prompt();
  for (int k : sel) {
    lc_store::Live l;
    l.step = d.steps[k];
    l.si = k;
    l.f = 0;
    l.last = now;
    l.inserted_at = now;
    l.seq = s->next_seq++;
    l.priv = d.private_bytes(k);
    l.slot = s->alloc_live();
    rec.live.push_back(l);
  }
  s->used += standalone;
  auto it = s->prompts.emplace(prompt, std::move(rec)).first;
  for (auto& l : it->second.live) {
    s->write_live(it->second, l);
    s->slot_prompt[l.slot] = prompt;
    ++s->live_count;
  }
  s->write_prompt(it->second);
  if (n_evicted) *n_evicted = ne;
  LC_API_END
}

lc_status lc_store_get_step(lc_store* s, uint64_t prompt, int desired, uint64_t now, int32_t* actual, float* out_dev) {
  LC_API_BEGIN
  DeviceGuard g(s->ctx->device);
  if (desired < 1 || desired > 50) raise(LC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
  if (!(desired == 5 || desired == 10 || desired == 15 || desired == 20 || desired == 25))
    raise(LC_ERR_INVALID_ARGUMENT, "get_step: desired step not cacheable");
  *actual = 0;
  auto it = s->prompts.find(prompt);
  if (it == s->prompts.end()) return LC_OK;
  auto& rec = it->second;
  int li = -1;
  for (size_t i = 0; i < rec.live.size(); ++i)
    if (rec.live[i].step <= desired) li = (int)i;
  if (li < 0) return LC_OK;
  auto& l = rec.live[li];
  if (out_dev) {
    FC_REQUIRE(is_device_ptr(out_dev), "lc_store_get_step: out_dev must be device memory");
    launch_decompress(s->ctx, {rec.view->d.get()}, {l.si}, out_dev);
    sync(s->ctx);
  }
  l.f += 1;
  l.last = now;
  s->write_live(rec, l);
  s->invalidate();  // its key changed
  *actual = l.step;
  LC_API_END
}

lc_status lc_store_evict_one(lc_store* s, uint64_t now, lc_step_entry* out) {
  LC_API_BEGIN
  DeviceGuard g(s->ctx->device);
  lc_step_entry v = s->evictor(now).next();
  if (out) *out = v;
  LC_API_END
}

lc_status lc_store_peek(lc_store* s, uint64_t now, lc_step_entry* out, double* key) {
  LC_API_BEGIN
  FC_REQUIRE(s, "null store");
  DeviceGuard g(s->ctx->device);
  lc_store::Evictor& ev = s->evictor(now);
  double k = 0.0;
  const int64_t slot = ev.pick(&k, nullptr);
  if (out) *out = ev.describe(slot);
  if (key) *key = k;
  LC_API_END
}

lc_status lc_store_peek_many(lc_store* s, uint64_t now, int m, lc_step_entry* out, double* keys, uint64_t* used_after,
                             int* n_out, int* more) {
  LC_API_BEGIN
  FC_REQUIRE(s && out && keys && used_after && n_out, "null argument");
  DeviceGuard g(s->ctx->device);
  *n_out = 0;
  if (more) *more = 0;
  if (s->prompts.empty()) return LC_OK;
  bool mo = false;
  *n_out = s->evictor(now).peek(m, out, keys, used_after, &mo);
  if (more) *more = mo ? 1 : 0;
  LC_API_END
}

uint64_t lc_store_next_seq(lc_store* s) { return s ? s->next_seq : 0; }
lc_status lc_store_set_next_seq(lc_store* s, uint64_t seq) {
  LC_API_BEGIN
  FC_REQUIRE(s, "null store");
  FC_REQUIRE(seq >= s->next_seq, "lc_store_set_next_seq: sequence numbers only move forward");
  s->next_seq = seq;
  LC_API_END
}

lc_status lc_store_evict_step(lc_store* s, uint64_t prompt, int step, int32_t* removed) {
  LC_API_BEGIN
  if (step < 1 || step > 50) raise(LC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
  *removed = 0;
  auto it = s->prompts.find(prompt);
  if (it == s->prompts.end()) return LC_OK;
  for (size_t i = 0; i < it->second.live.size(); ++i)
    if (it->second.live[i].step == step) {
      auto& r = it->second;
      s->remove_step(it, (int)i, r.live[i].priv + r.shared / r.live.size());
      s->invalidate();  // siblings' attributed capacity changed outside the evictor
      *removed = 1;
      break;
    }
  LC_API_END
}

uint64_t lc_store_used(lc_store* s) { return s->used; }
uint64_t lc_store_capacity(lc_store* s) { return s->capacity; }
int lc_store_policy(lc_store* s) { return s->policy; }
int64_t lc_store_step_count(lc_store* s) { return s->live_count; }
int64_t lc_store_prompt_count(lc_store* s) { return (int64_t)s->prompts.size(); }

uint64_t lc_store_recompute_used(lc_store* s) {
  uint64_t n = 0;
  for (auto& kv : s->prompts) n += entry_compressed_size(kv.second.view);
  return n;
}

lc_status lc_store_contains(lc_store* s, uint64_t prompt, int32_t* out) {
  LC_API_BEGIN
  *out = s->prompts.count(prompt) ? 1 : 0;
  LC_API_END
}

lc_status lc_store_cached_steps(lc_store* s, uint64_t prompt, int32_t* steps, int* n) {
  LC_API_BEGIN
  *n = 0;
  auto it = s->prompts.find(prompt);
  if (it == s->prompts.end()) return LC_OK;
  for (auto& l : it->second.live) steps[(*n)++] = l.step;
  LC_API_END
}

lc_status lc_store_entry(lc_store* s, uint64_t prompt, lc_entry** out) {
  LC_API_BEGIN
  auto it = s->prompts.find(prompt);
  *out = it == s->prompts.end() ? nullptr : it->second.view;
  LC_API_END
}

lc_status lc_store_entries(lc_store* s, lc_step_entry* out, int64_t cap, int64_t* n) {
  LC_API_BEGIN
  int64_t k = 0;
  for (auto& kv : s->prompts) {
    const auto& r = kv.second;
    for (auto& l : r.live) {
      if (out && k < cap)
        out[k] = lc_step_entry{kv.first, l.step, 0, l.f, l.last, l.inserted_at, l.seq, l.priv + r.shared / r.live.size()};
      ++k;
    }
  }
  *n = k;
  LC_API_END
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Snapshots (store.cpp:219-364). Host-side byte stream: the index tables and
// entries are pulled from HBM (lc_index_export / lc_entry_export), the live
// records come from the host mirror. Load pushes them back (index batch
// insert with the from_unit rule; entries via import_entry).
// ---------------------------------------------------------------------------
namespace fc {
namespace {

// CRC-32 (IEEE 802.3, reflected 0xEDB88320) = zlib crc32(0, buf, len),
// slicing-by-8 (8 bytes per step; the byte-at-a-time loop ran at ~0.5 GB/s
// and dominated a config[4] checkpoint)
uint32_t crc32_of(const uint8_t* p, size_t n) {
  static uint32_t T[8][256];
  static bool init = [] {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      T[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
      for (int t = 1; t < 8; ++t) T[t][i] = (T[t - 1][i] >> 8) ^ T[0][T[t - 1][i] & 0xFF];
    return true;
  }();
  (void)init;
  uint32_t c = 0xFFFFFFFFu;
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint32_t lo, hi;
    memcpy(&lo, p + i, 4);  // little-endian host
    memcpy(&hi, p + i + 4, 4);
    lo ^= c;
    c = T[7][lo & 0xFF] ^ T[6][(lo >> 8) & 0xFF] ^ T[5][(lo >> 16) & 0xFF] ^ T[4][lo >> 24] ^ T[3][hi & 0xFF] ^
        T[2][(hi >> 8) & 0xFF] ^ T[1][(hi >> 16) & 0xFF] ^ T[0][hi >> 24];
  }
  for (; i < n; ++i) c = T[0][(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

// f(i) for i in [0, n) on up to hardware_concurrency threads (independent items)
template <class Fn>
void par_for(size_t n, Fn f) {
  const size_t nt = std::min<size_t>(n, std::max(1u, std::thread::hardware_concurrency()));
  if (nt <= 1) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> th;
  for (size_t t = 0; t < nt; ++t)
    th.emplace_back([&] {
      for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
    });
  for (auto& x : th) x.join();
}

struct BW {  // ByteWriter (serialize.hpp:17-52), little-endian
  std::vector<uint8_t> b;
  void u8(uint8_t v) { b.push_back(v); }
  void u16(uint16_t v) { u8((uint8_t)v), u8((uint8_t)(v >> 8)); }
  void u32(uint32_t v) { for (int i = 0; i < 4; ++i) u8((uint8_t)(v >> (8 * i))); }
  void u64(uint64_t v) { for (int i = 0; i < 8; ++i) u8((uint8_t)(v >> (8 * i))); }
  void raw(const void* p, size_t n) { b.insert(b.end(), (const uint8_t*)p, (const uint8_t*)p + n); }
};

struct BR {  // ByteReader (serialize.hpp:54-106): truncation -> SnapshotError at pos
  const uint8_t* p;
  uint64_t n, pos = 0;
  void need(uint64_t k) const {
    if (pos + k > n) raise_snap("truncated input", pos);
  }
  uint8_t u8() { need(1); return p[pos++]; }
  uint16_t u16() { need(2); uint16_t v = (uint16_t)(p[pos] | (p[pos + 1] << 8)); pos += 2; return v; }
  uint32_t u32() {
    need(4);
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= (uint32_t)p[pos + i] << (8 * i);
    pos += 4;
    return v;
  }
  uint64_t u64() {
    need(8);
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[pos + i] << (8 * i);
    pos += 8;
    return v;
  }
  const uint8_t* bytes(uint64_t k) { need(k); const uint8_t* r = p + pos; pos += k; return r; }
  // k fp32 values: the reference reads them one at a time (f32_array), so a
  // truncation is reported at the start of the first incomplete value
  const uint8_t* f32s(uint64_t k) {
    if (pos + 4 * k > n) raise_snap("truncated input", pos + 4 * ((n - pos) / 4));
    return bytes(4 * k);
  }
};

void check_status(lc_status st) {
  if (st != LC_OK) raise(st, lc_last_error());
}

}  // namespace
}  // namespace fc

extern "C" {

lc_status lc_snapshot_save(lc_store* s, lc_index* ix, const char* path) {
  LC_API_BEGIN
  FC_REQUIRE(s && ix && path, "lc_snapshot_save: null argument");
  DeviceGuard g(s->ctx->device);
  BW w;
  w.raw("FLXC", 4);
  w.u16(1);
  w.u8((uint8_t)s->policy);
  w.u64(s->capacity);
  w.u64(s->next_seq);
  const int dim = lc_index_dim(ix);
  w.u16((uint16_t)dim);
  const int64_t n = lc_index_size(ix);
  std::vector<uint64_t> ids(std::max<int64_t>(n, 1));
  std::vector<float> rows((size_t)std::max<int64_t>(n, 1) * std::max(dim, 1));
  for (int kind = 0; kind < 3; ++kind) {  // Whole, Object, Background (store.cpp:241-248)
    if (n) check_status(lc_index_export(ix, kind, ids.data(), rows.data(), n));
    w.u32((uint32_t)n);
    for (int64_t i = 0; i < n; ++i) {
      w.u64(ids[i]);
      w.raw(rows.data() + (size_t)i * dim, 4ull * dim);
    }
  }
  w.u32((uint32_t)s->prompts.size());
  // Records, in ascending prompt id (std::map): u32 len | entry image |
  // live records | u32 CRC32(body). Every record's size and file offset is
  // known from the host metadata, so up to 16 host threads each pull an entry
  // image from HBM (own stream, pinned staging), serialize it, checksum it
  // and pwrite it at its offset: no whole-file buffer, no serial copy.
  struct Job {
    const lc_store::Rec* r;
    uint64_t elen, off;
  };
  std::vector<Job> jobs;
  jobs.reserve(s->prompts.size());
  uint64_t off = w.b.size(), max_img = 0, max_rec = 0;
  for (const auto& kv : s->prompts) {
    const lc_store::Rec& r = kv.second;
    const uint64_t elen = entry_compressed_size(r.view);
    const uint64_t rec = 4 + elen + 1 + 33ull * r.live.size() + 4;
    jobs.push_back(Job{&r, elen, off});
    off += rec;
    max_rec = std::max(max_rec, rec);
    max_img = std::max<uint64_t>(max_img, r.view->d->dev_bytes);
  }
  sync(s->ctx);  // entry images complete on the store's stream
  const int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) raise(LC_ERR_IO, std::string("cannot open snapshot for writing: ") + path);
  auto pwrite_all = [&](const uint8_t* p, uint64_t n, uint64_t at) {
    while (n > 0) {
      const ssize_t k = pwrite(fd, p, n, (off_t)at);
      if (k <= 0) return false;
      p += k, n -= (uint64_t)k, at += (uint64_t)k;
    }
    return true;
  };
  std::atomic<bool> io_ok{pwrite_all(w.b.data(), w.b.size(), 0)};
  std::exception_ptr err = nullptr;
  std::mutex err_mu;
  std::atomic<size_t> next{0};
  const int dev = s->ctx->device;
  const int nt = (int)std::min<size_t>(jobs.size(), std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
  auto worker = [&] {
    try {
      DeviceGuard g2(dev);
      cudaStream_t st = nullptr;
      FC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
      } sg{st};
      PinnedBuf<uint8_t> img(max_img);
      std::vector<uint8_t> rec(max_rec);
      for (size_t i; (i = next.fetch_add(1)) < jobs.size() && io_ok.load();) {
        const Job& j = jobs[i];
        const lc_entry* view = j.r->view;
        const EntryData& d = *view->d;
        FC_CUDA(cudaMemcpyAsync(img.data(), d.dev, d.dev_bytes, cudaMemcpyDeviceToHost, st));
        FC_CUDA(cudaStreamSynchronize(st));
        uint8_t* body = rec.data() + 4;
        serialize_entry_image(view, img.data(), body, j.elen);
        uint8_t* q = body + j.elen;
        *q++ = (uint8_t)j.r->live.size();
        for (const auto& l : j.r->live) {  // ascending step
          *q++ = (uint8_t)l.step;
          memcpy(q, &l.f, 8), q += 8;
          memcpy(q, &l.last, 8), q += 8;
          memcpy(q, &l.inserted_at, 8), q += 8;
          memcpy(q, &l.seq, 8), q += 8;
        }
        const uint32_t blen = (uint32_t)(q - body);
        memcpy(rec.data(), &blen, 4);
        const uint32_t crc = crc32_of(body, blen);
        memcpy(q, &crc, 4);
        if (!pwrite_all(rec.data(), (uint64_t)blen + 8, j.off)) io_ok = false;
      }
    } catch (...) {
      std::lock_guard<std::mutex> lk(err_mu);
      if (!err) err = std::current_exception();
      io_ok = false;
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(worker);
    if (nt >= 1) worker();
    for (auto& t : th) t.join();
  }
  const int cl = close(fd);
  if (err) std::rethrow_exception(err);
  if (!io_ok.load() || cl != 0) raise(LC_ERR_IO, std::string("snapshot write failed: ") + path);
  LC_API_END
}

lc_status lc_snapshot_load(lc_ctx* ctx, const char* path, lc_store** store_out, lc_index** index_out) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && path && store_out && index_out, "lc_snapshot_load: null argument");
  DeviceGuard g(ctx->device);
  std::vector<uint8_t> raw;
  {
    // one sized read (the file can be tens of GB: no chunked vector growth)
    const int fd = open(path, O_RDONLY);
    if (fd < 0) raise(LC_ERR_IO, std::string("cannot open snapshot: ") + path);
    const off_t sz = lseek(fd, 0, SEEK_END);
    bool ok = sz >= 0;
    if (ok) {
      raw.resize((size_t)sz);
      uint64_t got = 0;
      while (got < (uint64_t)sz) {
        const ssize_t k = pread(fd, raw.data() + got, (size_t)sz - got, (off_t)got);
        if (k <= 0) break;
        got += (uint64_t)k;
      }
      ok = got == (uint64_t)sz;
    }
    close(fd);
    if (!ok) raise(LC_ERR_IO, std::string("cannot read snapshot: ") + path);
  }
  BR r{raw.data(), raw.size()};
  const uint8_t* magic = r.bytes(4);
  if (memcmp(magic, "FLXC", 4) != 0) raise_snap("bad magic", 0);
  const uint16_t version = r.u16();
  if (version != 1) raise_snap("unsupported version " + std::to_string(version), r.pos - 2);
  const int policy = r.u8();
  if (policy > 3) raise_snap("invalid policy byte", r.pos - 1);
  const uint64_t capacity = r.u64();
  const uint64_t next_seq = r.u64();
  const int dim = r.u16();
  // three tables, zipped back into atomic inserts (store.cpp:297-320)
  std::vector<uint64_t> tid[3];
  std::vector<float> trow[3];
  for (int t = 0; t < 3; ++t) {
    const uint32_t count = r.u32();
    for (uint32_t i = 0; i < count; ++i) {
      tid[t].push_back(r.u64());
      const uint8_t* v = r.f32s((uint64_t)dim);
      const size_t at = trow[t].size();
      trow[t].resize(at + dim);
      if (dim) memcpy(trow[t].data() + at, v, 4ull * dim);
    }
  }
  if (tid[0].size() != tid[1].size() || tid[0].size() != tid[2].size())
    raise_snap("index tables disagree on entry count", r.pos);
  for (size_t i = 0; i < tid[0].size(); ++i)
    if (tid[0][i] != tid[1][i] || tid[0][i] != tid[2][i]) raise_snap("index tables disagree on prompt ids", r.pos);
  std::unique_ptr<lc_store, lc_status (*)(lc_store*)> st(nullptr, lc_store_destroy);
  std::unique_ptr<lc_index, lc_status (*)(lc_index*)> ix(nullptr, lc_index_destroy);
  {
    lc_index* pi = nullptr;
    check_status(lc_index_create(ctx, dim, (int64_t)tid[0].size(), &pi));
    ix.reset(pi);
    lc_store* ps = nullptr;
    check_status(lc_store_create(ctx, capacity, policy, &ps));
    st.reset(ps);
  }
  if (!tid[0].empty())
    check_status(lc_index_insert_batch(ix.get(), tid[0].data(), trow[0].data(), trow[1].data(), trow[2].data(),
                                       (int64_t)tid[0].size(), dim));
  lc_store* s = st.get();
  s->next_seq = next_seq;
  const uint32_t n_prompts = r.u32();
  // (1) framing: record positions up to the first framing error (raised only
  // after every record before it, as the reference's sequential loop would)
  struct Rc {
    uint64_t pos;
    const uint8_t* body;
    uint32_t len, crc;
  };
  std::vector<Rc> recs;
  recs.reserve(n_prompts);
  std::exception_ptr frame_err = nullptr;
  try {
    for (uint32_t i = 0; i < n_prompts; ++i) {
      Rc c;
      c.pos = r.pos;
      c.len = r.u32();
      c.body = r.bytes(c.len);
      c.crc = r.u32();
      recs.push_back(c);
    }
  } catch (...) {
    frame_err = std::current_exception();
  }
  // (2) per record, in parallel: CRC32 and the entry import (parse + upload
  // on a child stream per thread); errors kept per record
  const size_t nr = recs.size();
  std::vector<lc_entry*> imported(nr, nullptr);
  std::vector<uint64_t> used_of(nr, 0);
  std::vector<std::exception_ptr> rec_err(nr, nullptr);
  std::vector<char> crc_bad(nr, 0);
  struct Release {
    std::vector<lc_entry*>& v;
    ~Release() {
      for (lc_entry* e : v)
        if (e) lc_entry_release(e);
    }
  } release_left{imported};
  {
    std::atomic<size_t> next{0};
    const int nt = (int)std::min<size_t>(nr, std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
    auto worker = [&](int t) {
      lc_ctx* c = nullptr;
      try {
        c = aux_ctx(ctx, t);
      } catch (...) {
        c = ctx;
      }
      DeviceGuard g2(ctx->device);
      for (size_t i; (i = next.fetch_add(1)) < nr;) {
        if (crc32_of(recs[i].body, recs[i].len) != recs[i].crc) {
          crc_bad[i] = 1;
          continue;
        }
        try {
          imported[i] = import_entry(c, recs[i].body, recs[i].len, &used_of[i]);
          imported[i]->d->ctx = ctx;  // uploaded and synced on the child stream; owned by the caller's context
        } catch (...) {
          rec_err[i] = std::current_exception();
        }
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(worker, t);
    if (nt >= 1) worker(0);
    for (auto& x : th) x.join();
  }
  // (3) in file order: the first error wins, then the live records and the
  // store state exactly as the sequential loop (store.cpp:323-360)
  for (size_t i = 0; i < nr; ++i) {
    const uint64_t record_pos = recs[i].pos;
    const uint8_t* body = recs[i].body;
    const uint32_t body_len = recs[i].len;
    if (crc_bad[i]) raise_snap("checksum mismatch in prompt record", record_pos);
    if (rec_err[i]) std::rethrow_exception(rec_err[i]);
    const uint64_t used_e = used_of[i];
    lc_entry* view = imported[i];
    imported[i] = nullptr;
    std::unique_ptr<lc_entry, lc_status (*)(lc_entry*)> vh(view, lc_entry_release);
    const EntryData& d = *view->d;
    BR br{body, body_len, used_e};
    lc_store::Rec rec;
    rec.shared = d.shared_bytes();
    const int n_live = br.u8();
    for (int k = 0; k < n_live; ++k) {
      const int sv = br.u8();
      if (sv < 1 || sv > 50) raise(LC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");  // StepId(sv)
      lc_store::Live l;
      l.f = br.u64();
      l.last = br.u64();
      l.inserted_at = br.u64();
      l.seq = br.u64();
      int si = -1;
      for (size_t q = 0; q < d.steps.size(); ++q)
        if (d.steps[q] == sv) si = (int)q;
      if (si < 0) raise_snap("live step missing from entry data", record_pos);
      bool dup = false;  // rec.live.emplace keeps the first record of a step
      for (const auto& x : rec.live) dup |= x.step == sv;
      if (dup) continue;
      l.step = sv;
      l.si = si;
      l.priv = d.private_bytes(si);
      rec.live.push_back(l);
    }
    if (br.pos != br.n) raise_snap("trailing bytes in prompt record", record_pos);
    if (rec.live.empty()) raise_snap("prompt record with no live steps", record_pos);
    std::sort(rec.live.begin(), rec.live.end(), [](const auto& a, const auto& b) { return a.step < b.step; });
    uint64_t bytes = rec.shared;
    for (const auto& l : rec.live) bytes += l.priv;
    s->used += bytes;  // counted even if the prompt id repeats (store.cpp:356-358)
    const uint64_t prompt = d.prompt;
    if (s->prompts.count(prompt)) continue;  // prompts_.emplace keeps the first
    rec.view = vh.release();
    rec.pslot = s->alloc_prompt();
    for (auto& l : rec.live) l.slot = s->alloc_live();
    auto it = s->prompts.emplace(prompt, std::move(rec)).first;
    for (auto& l : it->second.live) {
      s->write_live(it->second, l);
      s->slot_prompt[l.slot] = prompt;
      ++s->live_count;
    }
    s->write_prompt(it->second);
  }
  if (frame_err) std::rethrow_exception(frame_err);
  if (r.pos != r.n) raise_snap("trailing bytes after last record", r.pos);
  *store_out = st.release();
  *index_out = ix.release();
  LC_API_END
}

}  // extern "C"
