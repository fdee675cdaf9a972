// lookup_sm100.cu — tcgen05 candidate stage of the prompt-similarity lookup.
//
// Replaces the scan loop of SimilarityIndex::query_top1 (vindex.cpp:64-72)
// with S = Q · Xᵀ on the 5th-gen tensor cores, fused with a per-query
// top-K' shortlist so the [queries x rows] score matrix never leaves the SM.
//
// Per CTA (persistent, one per SM, 6 warps):
//   warp 0      TMA producer: streams bf16 table tiles [BN rows][64 K]
//               (SWIZZLE_128B) into an NSTAGE smem ring.
//   warp 1      TMEM owner + single-thread MMA issuer:
//               tcgen05.mma.cta_group::1.kind::f16, A = 128 queries held
//               RESIDENT IN TMEM (dim/2 columns, loaded once per work unit),
//               B = table tile from smem, D = fp32 accumulator in TMEM
//               (two BN-column buffers, so MMA of tile t+1 overlaps the
//               epilogue of tile t).
//   warps 2..5  epilogue: tcgen05.ld of the accumulator (thread = query
//               row = TMEM lane), threshold filter against the running
//               K'-th best, replace-min insert into a per-query shortlist in
//               smem; at the end of the work unit the shortlist is written out.
// Work unit = (128-query tile, contiguous row range). Units are ordered
// split-major so that concurrently running CTAs stream the same table
// region and every 128-query tile after the first reads it from L2.
#include <cuda.h>
#include <atomic>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "lookup.cuh"
#include "sm100_ptx.cuh"

namespace fc {

namespace sm100 {

constexpr int BM = 128;     // queries per tile (TMEM lanes)
constexpr int BK = 64;      // bf16 per 128-byte swizzle row
constexpr int NTHREADS = 192;


__device__ __forceinline__ uint32_t okey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Shrink the thread's (query's) candidate buffer to its kp best entries and
// raise the acceptance threshold tau to the kp-th best score. Exact: T is
// found by a binary search on the order-preserving key; entries > T are kept,
// ties at T fill up to kp. Called warp-uniformly and rarely (the buffer only
// fills after ~64 accepted scores), so the per-score filter stays branch-free.
__device__ __noinline__ void compact(float* ls, uint32_t* lr, int t, int& cnt, int kp, float& tau) {
  if (cnt <= kp) return;
  uint32_t lo = 0, hi = 0xFFFFFFFFu;
  while (lo < hi) {  // max T with count(key >= T) >= kp
    const uint32_t mid = lo + (uint32_t)(((uint64_t)hi - lo + 1) >> 1);
    int c = 0;
    for (int i = 0; i < cnt; ++i) c += okey(ls[i * BM + t]) >= mid;
    if (c >= kp) lo = mid; else hi = mid - 1;
  }
  const uint32_t T = lo;
  int above = 0;
  for (int i = 0; i < cnt; ++i) above += okey(ls[i * BM + t]) > T;
  int need_eq = kp - above, w = 0;
  for (int i = 0; i < cnt; ++i) {
    const float v = ls[i * BM + t];
    const uint32_t k = okey(v);
    const bool keep = k > T || (k == T && need_eq > 0);
    need_eq -= (k == T && keep);
    if (keep) {
      ls[w * BM + t] = v;
      lr[w * BM + t] = lr[i * BM + t];
      ++w;
    }
  }
  cnt = w;
  const float tnew = __uint_as_float((T & 0x80000000u) ? (T & 0x7FFFFFFFu) : ~T);
  if (tnew > tau) tau = tnew;  // never lower a (possibly shared) threshold
}

__device__ __forceinline__ float key_float(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// ---- packed shortlist candidates ----
// A candidate is ONE u32: (order-preserving key of the score rounded UP to
// fp16) << 16 | row offset within the work unit's row range (< 65536). The
// stored score is an upper bound of the fp32 accumulator value, so the
// certificate "every row outside the shortlist has approx <= m" holds with m =
// the K'-th best STORED score; larger keys are better, and keys are unique
// within a unit (distinct offsets). Half the shared memory of (fp32, u32)
// pairs: the freed bytes deepen the TMA ring.
__device__ __forceinline__ uint32_t hkey_ru(float v) {
  const uint32_t h = __half_as_ushort(__float2half_ru(v));
  return (h & 0x8000u) ? (~h & 0xFFFFu) : (h | 0x8000u);
}
__device__ __forceinline__ float hkey_float(uint32_t k16) {
  const uint32_t h = (k16 & 0x8000u) ? (k16 & 0x7FFFu) : (~k16 & 0xFFFFu);
  return __half2float(__ushort_as_half((unsigned short)h));
}

// Keep the kp largest keys of the thread's list (exact) or, while streaming,
// between kp and kp + 8 of them (bisection with early stop); raise tau to the
// stored score of the smallest kept key. Every later rejection (score <= tau)
// then ranks below kp kept entries, so it is below the final K'-th stored
// score of the query. Called warp-uniformly.
__device__ __noinline__ void compact_keys(uint32_t* lk, int t, int& cnt, int kp, float& tau, bool exact) {
  if (cnt <= (exact ? kp : kp + 8)) return;
  uint32_t lo = 0xFFFFFFFFu, hi = 0;
  for (int i = 0; i < cnt; ++i) {
    const uint32_t k = lk[i * BM + t];
    lo = min(lo, k);
    hi = max(hi, k);
  }
  const int slack = exact ? 0 : 8;
  while (lo < hi) {  // max T with count(key >= T) >= kp
    const uint32_t mid = lo + (uint32_t)(((uint64_t)hi - lo + 1) >> 1);
    int c = 0;
    for (int i = 0; i < cnt; ++i) c += lk[i * BM + t] >= mid;
    if (c >= kp) {
      lo = mid;
      if (c <= kp + slack) break;
    } else {
      hi = mid - 1;
    }
  }
  const uint32_t T = lo;
  int w = 0;
  for (int i = 0; i < cnt; ++i) {
    const uint32_t k = lk[i * BM + t];
    if (k >= T) lk[w++ * BM + t] = k;
  }
  cnt = w;
  const float tnew = hkey_float(T >> 16);
  if (tnew > tau) tau = tnew;
}

// Shared per-query threshold (order-preserving key, 0 = unset): the K'-th
// best bf16 score of ANY completed work unit is a lower bound on the K'-th
// best over the whole table, so every unit of that query may drop scores
// <= it. Later units then accept only a handful of candidates.
__device__ __forceinline__ void refresh_tau(const uint32_t* gkey, int q, float& tau) {
  uint32_t k;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(k) : "l"(gkey + q));
  if (k && key_float(k) > tau) tau = key_float(k);
}

__device__ __forceinline__ void publish_tau(uint32_t* gkey, int q, const float* ls, int t, int cnt, int kp) {
  if (cnt < kp) return;
  float m = ls[t];
  for (int i = 1; i < cnt; ++i) m = fminf(m, ls[i * BM + t]);
  atomicMax(gkey + q, okey(m));
}


// ---- per-query acceptance histogram (pair kernel) ----
// hist[q][b] counts, over ALL work units of query q, the accepted bf16
// scores falling in bucket b (32 buckets per octave on [2^-8, 1), bucket 0
// = below 2^-8, bucket HB-1 = >= 1). If the buckets >= B hold >= kp counts,
// the final merged shortlist of q holds >= kp entries >= edge(B): every unit
// keeps its top min(kp, accepted) entries and the entries >= edge(B) are its
// largest, so sum_i min(kp, a_i) >= min(kp, sum_i a_i) = kp. Any unit may
// therefore reject scores <= edge(B) at once; the units of one query, which
// run concurrently on different row ranges, pool their evidence instead of
// each warming its own threshold.
constexpr int BPO = 32;                  // fine buckets per octave (2.2% wide; 64 cut slow chunks 6% but cost more in refresh loads)
constexpr int BPO_SHIFT = 23 - (BPO == 64 ? 6 : BPO == 32 ? 5 : BPO == 16 ? 4 : -100);  // top log2(BPO) mantissa bits
static_assert(BPO_SHIFT > 0 && BPO_SHIFT < 23, "BPO must be 16, 32 or 64");
constexpr int HB = 8 * BPO + 8;          // bucket 0, 8 octaves, overflow (>= 1.0), padding
constexpr int HOV = 8 * BPO + 1;         // overflow bucket index
constexpr int HC = HB + 8;               // coarse counters at [HC, HC+16): octave 0..7, 8 = >= 1.0
constexpr int HSTRIDE = HC + 16;         // per-query words (multiple of 4: 16-byte aligned rows)
__device__ __forceinline__ int hbucket(float s) {
  const uint32_t u = __float_as_uint(s);
  if ((int32_t)u < 0) return 0;  // negative
  const int e = (int)(u >> 23);
  if (e < 119) return 0;
  if (e >= 127) return HOV;
  return 1 + (e - 119) * BPO + (int)((u >> BPO_SHIFT) & (BPO - 1));
}
__device__ __forceinline__ float hedge(int b) {  // smallest score of bucket b >= 1
  if (b >= HOV) return 1.0f;
  const int e = 119 + (b - 1) / BPO, m = (b - 1) % BPO;
  return __uint_as_float(((uint32_t)e << 23) | ((uint32_t)m << BPO_SHIFT));
}
__device__ __forceinline__ void hist_publish(uint32_t* h, const uint32_t* lk, int t, int from, int to) {
  for (int i = from; i < to; ++i) {
    const int bk = hbucket(hkey_float(lk[i * BM + t] >> 16));
    if (bk == 0) continue;  // never used to raise a threshold
    atomicAdd(h + bk, 1u);
    atomicAdd(h + HC + (bk - 1) / BPO, 1u);
  }
}
// Raise tau to (the lower edge of the highest bucket B with sum_{b>=B} h[b] >= kp) - off.
// Two rounds of independent loads: the 9 octave counters, then the BPO fine
// buckets of the octave where the running count from the top reaches kp.
// (bf16 tier: off = 0, kp = K'; int8 tier: kp = k and off = the query's
// typical error bound plus a slack, see k_shortlist_pair)
__device__ __forceinline__ void hist_refresh(const uint32_t* h, int kp, float& tau, float off = 0.f) {
  const uint4* hc = reinterpret_cast<const uint4*>(h + HC);
  const uint4 c0 = __ldcg(hc), c1 = __ldcg(hc + 1), c2 = __ldcg(hc + 2);
  const uint32_t oc[9] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w, c2.x};
  int sum = (int)oc[8];
  if (sum >= kp) {
    if (1.0f - off > tau) tau = 1.0f - off;
    return;
  }
  int o = 7;
  for (; o >= 0; --o) {
    if (sum + (int)oc[o] >= kp) break;
    sum += (int)oc[o];
  }
  if (o < 0) return;
  if (hedge(1 + o * BPO + BPO - 1) - off <= tau) return;  // nothing in reach above tau
  // fine bucket 1 + o*BPO + jj lives at word o*BPO + 1 + jj; load words o*BPO .. o*BPO + BPO + 3
  const uint4* hv = reinterpret_cast<const uint4*>(h + o * BPO);
  uint4 x[BPO / 4 + 1];
#pragma unroll
  for (int i = 0; i < BPO / 4 + 1; ++i) x[i] = __ldcg(hv + i);
  uint32_t f[BPO + 4];
#pragma unroll
  for (int i = 0; i < BPO / 4 + 1; ++i) {
    f[4 * i + 0] = x[i].x;
    f[4 * i + 1] = x[i].y;
    f[4 * i + 2] = x[i].z;
    f[4 * i + 3] = x[i].w;
  }
#pragma unroll
  for (int jj = BPO - 1; jj >= 0; --jj) {
    sum += (int)f[1 + jj];
    if (sum >= kp) {
      const float e = hedge(1 + o * BPO + jj) - off;
      if (e > tau) tau = e;
      return;
    }
  }
}

struct Params {
  const __nv_bfloat16* Qb;  // [nq_pad][dim] (int8 kernel: const int8_t*)
  int nq;                    // real queries
  int n_qtiles;
  int dim;
  int64_t n_rows;
  int rows_per_split;        // multiple of BN
  int n_splits;
  int n_units;
  int kp;
  int cap;     // candidate buffer slots per query (>= kp + 16)
  int bps;     // TMA boxes per pipeline stage
  uint32_t* gkey;  // [nq_pad] shared per-query thresholds (order keys, 0 = unset)
  uint32_t* hist;   // [nq_pad][HSTRIDE] acceptance histogram (pair kernel)
  int refresh_mask; // histogram publish/refresh every (mask + 1) tiles
  uint32_t* stats;  // FC_SHORTLIST_DEBUG & 16: [slow chunks, compactions, warp-tiles]
  int debug;   // diagnostics (FC_SHORTLIST_DEBUG): 1 = skip MMA, 2 = skip TMA, 4 = skip epilogue filter
  int nstage;
  uint32_t* part_k;          // [nq][n_splits][kp] packed candidates (hkey_ru(score) << 16 | row - r0)
  int32_t* part_n;           // [nq][n_splits]
  // int8 kernel only
  int kh;                    // histogram threshold target (int8: k, the top-k size); bf16: = kp
  const float* tscale;       // [tiles] per-128-row tile scale s_t
  const float* tres;         // [tiles] max ||x - s_t xq|| over the tile's rows (rounded up)
  const float* qscale;       // [nq_pad] per-query scale s_q
  const float2* qerr;        // [nq_pad] (||dq|| X, ||qhat||) rounded up; padding queries (0, 0)
  float r_typ;               // typical tile residual (median of tres): threshold offset
  float slack;               // threshold offset slack (actual vs bounded error, bucket width)
  float* part_d;             // [nq][lists] drop level: every row the unit rejected or dropped has U <= it
  // int8 pilot pass: row tiles are every tile_stride-th physical tile (rows
  // [row * tile_stride, +128) for logical row `row`); each thread publishes the
  // max U of its query over the sampled tiles to gkey (order key) and keeps no
  // lists. The main pass starts every query's threshold at that max - offset:
  // over a 1/16 sample the max is about the table's 16th best, just below the
  // k-th best, so the filter is tight from the first tile instead of after a
  // warm-up (which cost ~5k accepted entries and ~20k list compactions per
  // 4096-query batch at 1M rows).
  int pilot;
  int tile_stride;
  int64_t n_rows_phys;
  float* pilot_out;          // [nq][lists][PILOT_R] each list's best U values (descending)
  // int8 main pass output: every unit appends its entries to its query's
  // contiguous buffer (one atomic per (query, unit)), so the merge reads one
  // segment per query instead of 2 * splits scattered lists
  uint64_t* qbuf;            // [nq][qcap] (fp16 U key << 48) | absolute row
  uint32_t* qcnt;            // [nq] entries appended (may exceed qcap)
  uint32_t* qdrop;           // [nq] order key of the max drop level (0 = none)
  int qcap;
  // threshold tier (null otherwise): per-query fixed threshold in U space,
  // never raised (no pilot, no histogram, full unit lists flushed to the
  // query buffer instead of compacted), so every row with U > tau_fix[q]
  // reaches the merge unless the query buffer overflows
  const float* tau_fix;
};
// The pilot keeps each query's PILOT_R best U over the sample and the main
// pass starts at the R-th best over the whole sample: over a 1/16 sample that
// is about the table's 16R-th best, and it exceeds the k-th best (k = 8) only
// when >= R of the top 8 fall in the sample (C(8,6) 16^-6 ~ 2e-6 for R = 6).
// (The sample max instead failed certification for 32 % of the queries.)
constexpr int PILOT_R = 6;

constexpr int MAX_STAGE = 24;

template <int BN>
__global__ void __launch_bounds__(NTHREADS, 1) k_shortlist(const __grid_constant__ CUtensorMap tmap, Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // carve: [stages][BN*128] | cand scores [cap][128] | cand rows [cap][128] | barriers | tmem addr
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int BOX_BYTES = BN * 128;  // one TMA box: BN rows x 64 bf16
  const int BPS = p.bps;               // boxes per pipeline stage (one barrier per stage)
  const int STAGE_BYTES = BPS * BOX_BYTES;
  const int NSTAGE = p.nstage;
  const int cap = p.cap;
  uint8_t* stages = base;
  float* ls = reinterpret_cast<float*>(base + NSTAGE * STAGE_BYTES);
  uint32_t* lr = reinterpret_cast<uint32_t*>(ls + cap * BM);
  uint64_t* bars = reinterpret_cast<uint64_t*>(lr + cap * BM);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  uint64_t* accf = bars + 2 * NSTAGE;
  uint64_t* acce = accf + 2;
  uint64_t* aready = acce + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aready + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = p.dim / BK;
  const int nsg = nkb / BPS;  // pipeline stages per tile
  const int a_cols = p.dim / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&accf[b]), 1);
      mbar_init(smem_u32(&acce[b]), 128);
    }
    mbar_init(smem_u32(aready), 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const int split = u / p.n_qtiles;
        const int64_t r0 = (int64_t)split * p.rows_per_split;
        const int64_t r1 = min((int64_t)p.n_rows, r0 + p.rows_per_split);
        for (int64_t row = r0; row < r1; row += BN) {
          for (int sg = 0; sg < nsg; ++sg) {
            mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
            if (p.debug & 2) {  // diagnostic: no table traffic
              mbar_arrive(smem_u32(&full[stage]));
            } else {
              mbar_expect_tx(smem_u32(&full[stage]), STAGE_BYTES);
              for (int bx = 0; bx < BPS; ++bx)
                tma_load_2d(smem_u32(stages + stage * STAGE_BYTES + bx * BOX_BYTES), &tmap, smem_u32(&full[stage]),
                            (sg * BPS + bx) * BK, (int)row);
            }
            if (++stage == NSTAGE) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=BN
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t tile = 0;
    uint32_t unit_i = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++unit_i) {
      const int split = u / p.n_qtiles;
      const int64_t r0 = (int64_t)split * p.rows_per_split;
      const int64_t r1 = min((int64_t)p.n_rows, r0 + p.rows_per_split);
      mbar_wait(smem_u32(aready), unit_i & 1);
      tc_fence_after();
      for (int64_t row = r0; row < r1; row += BN, ++tile) {
        const uint32_t b = tile & 1;
        const uint32_t use = tile >> 1;
        mbar_wait(smem_u32(&acce[b]), (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + a_cols + b * BN;
        for (int sg = 0; sg < nsg; ++sg) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(stages + stage * STAGE_BYTES);
            if (!(p.debug & 1)) {  // debug bit 0: diagnostic run without MMAs
              for (int bx = 0; bx < BPS; ++bx) {
                const int kb = sg * BPS + bx;
                mma_box4(d_tmem, tmem + kb * (BK / 16) * 8, smem_desc_sw128(sa + bx * BOX_BYTES), idesc, kb != 0);
              }
            }
            tc_commit(smem_u32(&empty[stage]));
          }
          __syncwarp();
          if (++stage == NSTAGE) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) tc_commit(smem_u32(&accf[b]));
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5 ----------------
    const int quarter = warp & 3;        // TMEM lane quarter this warp may access
    const int t = quarter * 32 + lane;   // query row within the tile
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    uint32_t tile = 0;
    uint32_t unit_i = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++unit_i) {
      const int split = u / p.n_qtiles;
      const int qtile = u - split * p.n_qtiles;
      const int64_t r0 = (int64_t)split * p.rows_per_split;
      const int64_t r1 = min((int64_t)p.n_rows, r0 + p.rows_per_split);
      const int q = qtile * BM + t;
      // (1) load this unit's 128 queries into TMEM columns [0, dim/2)
      {
        const uint4* src = reinterpret_cast<const uint4*>(p.Qb + (size_t)(qtile * BM + t) * p.dim);
        for (int kb = 0; kb < nkb; ++kb) {
          uint32_t r[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint4 v = __ldg(src + kb * 8 + i);
            r[4 * i + 0] = v.x;
            r[4 * i + 1] = v.y;
            r[4 * i + 2] = v.z;
            r[4 * i + 3] = v.w;
          }
          tmem_st32(tmem + lane_base + kb * 32, r);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(smem_u32(aready));
      }
      // (2) stream the accumulator tiles; branch-free append of every score
      //     above the running threshold, warp-uniform compaction when full
      int cnt = 0;
      float tau = -INFINITY;
      refresh_tau(p.gkey, q, tau);
      for (int64_t row = r0; row < r1; row += BN, ++tile) {
        const uint32_t b = tile & 1;
        const uint32_t use = tile >> 1;
        if ((tile & 15) == 0) refresh_tau(p.gkey, q, tau);
        mbar_wait(smem_u32(&accf[b]), use & 1);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < BN / 64; ++h) {
          float v[64];
          tmem_ld64(tmem + lane_base + a_cols + b * BN + h * 64, v);
          if (h == BN / 64 - 1) {
            tc_fence_before();
            mbar_arrive(smem_u32(&acce[b]));
          }
          const int64_t rbase = row + h * 64;
          const int lim = (int)min((int64_t)64, r1 - rbase);
          const uint32_t r32 = (uint32_t)rbase;
#pragma unroll
          for (int c = 0; c < ((p.debug & 4) ? 0 : 4); ++c) {
            if (__any_sync(0xffffffffu, cnt + 16 > cap)) compact(ls, lr, t, cnt, p.kp, tau);
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int j = c * 16 + jj;
              const bool acc = (j < lim) & (v[j] > tau);
              if (acc) {
                ls[cnt * BM + t] = v[j];
                lr[cnt * BM + t] = r32 + j;
              }
              cnt += acc;
            }
          }
        }
      }
      compact(ls, lr, t, cnt, p.kp, tau);
      publish_tau(p.gkey, q, ls, t, cnt, p.kp);
      // (3) write the shortlist of this (query, split)
      if (q < p.nq) {
        const size_t o = ((size_t)q * p.n_splits + split) * p.kp;
        for (int i = 0; i < cnt; ++i) p.part_k[o + i] = (hkey_ru(ls[i * BM + t]) << 16) | (lr[i * BM + t] - (uint32_t)r0);
        p.part_n[(size_t)q * p.n_splits + split] = cnt;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// CTA-pair kernel (cta_group::2), the default path for dim <= 768.
//
// Why this shape (measured on B200 with scripts/mma_bench.cu): a
// tcgen05.mma instruction costs >= ~50 issue cycles however small N is, so
// N=64 tiles cap at ~1.0-1.45 PFLOP/s while N=128 reaches ~2.2 PFLOP/s (the
// N=256 pipe rate). Holding all 768 query dims in TMEM (384 columns) left
// room only for two N=64 accumulators; here the first KT <= 8 K-boxes of the
// 128 queries of each CTA live in TMEM (<= 256 columns) and the remaining
// KS boxes in shared memory (TMA-loaded, SWIZZLE_128B), which frees 256
// columns for two N=128 accumulators (MMA of tile t+1 overlaps the epilogue
// of tile t).
//
// Work unit = (256-query tile, row range). CTA rank r holds queries
// [256*qtile + 128*r, +128) and TMA-loads table rows [row + 64*r, +64) of
// each 128-row tile; the leader issues M=256 x N=128 x K=16 MMAs reading A
// from both CTAs' TMEM (first KT boxes) or smem (last KS boxes) and B from
// both CTAs' smem, so each SM streams 64 table rows per 256x128 tile
// (~30 B/cycle/SM of L2 traffic at full MMA rate). Each CTA's epilogue owns
// its 128 accumulator lanes (one query per thread).
constexpr int PN = 128;               // table rows per tile (MMA N)
constexpr int PHB = PN / 2;           // table rows per CTA per tile
constexpr int PBOX = PHB * 128;       // one B box: 64 rows x 64 bf16 = 8 KB
constexpr int ABOX = BM * 128;        // one A box: 128 queries x 64 bf16 = 16 KB
constexpr int ACC_COL = 256;          // accumulators at TMEM columns [256, 512)
// int8 kernel: the first 4 query K boxes (128 int8 each) live in TMEM columns
// [0, 128), the rest in smem, so THREE 128-column accumulators fit in
// [128, 512): the MMA can run two tiles ahead of the slowest epilogue warp
// (ncu r02v: with two buffers the MMA waited ~1.8k cycles per tile for a
// free accumulator while most epilogue warps idled waiting for the next one:
// per-tile spikes of the few warps with accepted scores set the pace)
constexpr int I8_KT = 4;
constexpr int I8_ACC_COL = 128;
constexpr int I8_NACC = 3;
constexpr int PMAX_STAGE = 24;

__device__ __forceinline__ void mma_box4_pair_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, t;\n"
      ".reg .b64 a1, a2, a3, d1, d2, d3;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "setp.eq.b32 t, 0, 0;\n"
      "add.s64 a1, %1, 2;\n"
      "add.s64 a2, %1, 4;\n"
      "add.s64 a3, %1, 6;\n"
      "add.s64 d1, %2, 2;\n"
      "add.s64 d2, %2, 4;\n"
      "add.s64 d3, %2, 6;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a1, d1, %3, t;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a2, d2, %3, t;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a3, d3, %3, t;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

// int8 kernel: the largest integer dot that is rejected at threshold tau for a
// (query, tile) with fp32 scale product sqt = fl(s_q * s_t). Rejecting
// dot <= thr guarantees a = s_q s_t dot <= tau in real arithmetic: the fp32
// division and the product rounding (<= 2^-24 each) are covered by the 2^-20
// pull toward -inf. tau = -inf (nothing rejected yet) gives INT_MIN.
__device__ __forceinline__ int i8_thr(float tau, float sqt) {
  if (!(tau > -INFINITY)) return INT_MIN;
  const float t = __fdiv_rn(tau, sqt);
  const float c = t * (t > 0.f ? (1.f - 0x1p-20f) : (1.f + 0x1p-20f));
  if (c >= 2147483520.f) return INT_MAX;
  if (c <= -2147483520.f) return INT_MIN;
  return (int)floorf(c);
}
// stored score of an accepted int8 dot: fp32 value rounded up past the
// rounding of fl(s_q s_t) * dot (<= 2^-23 relative), so hkey_ru() of it is an
// upper bound of a
__device__ __forceinline__ float i8_score_up(int dot, float sqt) {
  const float a = (float)dot * sqt;
  return a + fabsf(a) * 0x1p-20f;
}

__device__ __forceinline__ void mma_box4_pair_ss_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                    uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, t;\n"
      ".reg .b64 a1, a2, a3, d1, d2, d3;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "setp.eq.b32 t, 0, 0;\n"
      "add.s64 a1, %1, 2;\n"
      "add.s64 a2, %1, 4;\n"
      "add.s64 a3, %1, 6;\n"
      "add.s64 d1, %2, 2;\n"
      "add.s64 d2, %2, 4;\n"
      "add.s64 d3, %2, 6;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], a1, d1, %3, t;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], a2, d2, %3, t;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], a3, d3, %3, t;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

// Append a unit list (cnt packed keys of query q, rows r0 + offset) to the
// query's contiguous buffer; entries past its capacity and everything the
// unit rejected (U <= tau) raise the query's drop level.
__device__ __forceinline__ void i8_append(const Params& p, int q, const uint32_t* lk, int t, int cnt, int64_t r0,
                                          float tau) {
  const uint32_t pos = cnt ? atomicAdd(p.qcnt + q, (uint32_t)cnt) : 0u;
  float dmax = tau;
  for (int i = 0; i < cnt; ++i) {
    const uint32_t key = lk[i * BM + t];
    if (pos + (uint32_t)i < (uint32_t)p.qcap)
      p.qbuf[(size_t)q * p.qcap + pos + i] = ((uint64_t)(key >> 16) << 48) | (uint64_t)(r0 + (key & 0xFFFFu));
    else
      dmax = fmaxf(dmax, hkey_float(key >> 16));
  }
  if (dmax > -INFINITY) atomicMax(p.qdrop + q, okey(dmax));
}

// v[j] for a run-time j in [0, 16) from 16 registers (a 4-level select tree:
// registers cannot be indexed dynamically without a local-memory copy)
__device__ __forceinline__ uint32_t sel16(const uint32_t* v, int j) {
  uint32_t a[8], b[4], c[2];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (j & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = (j & 2) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
  for (int i = 0; i < 2; ++i) c[i] = (j & 4) ? b[2 * i + 1] : b[2 * i];
  return (j & 8) ? c[1] : c[0];
}

// Pair kernel warps: 0 TMA producer, 1 MMA issuer, 2..9 epilogue. Two
// epilogue warps share each TMEM lane quarter (a warp may only read lanes
// 32 * (warp % 4) ..): warp half h = (warp - 2) / 4 filters accumulator
// columns [64 h, 64 h + 64) of every tile into its own candidate list, so the
// latency-bound filter (max tree, vote, append) has two warps per SM
// sub-partition to hide it.
constexpr int PAIR_THREADS = 320;
constexpr int EPI_HALF_COLS = PN / 2;

// I8: kind::i8 tier (s8 table tile x s8 queries -> s32 accumulators): every
// query K box (128 int8) lives in TMEM (dim <= 1024), the epilogue filters the
// exact integer dots against a per-(query, tile) integer threshold and stores
// rounded-up fp32 scores; each unit reports its drop level (final tau).
template <bool I8>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PAIR_THREADS, 1)
    k_shortlist_pair(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmQ, Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NSTAGE = p.nstage;
  const int cap = p.cap;
  constexpr int BKE = I8 ? 128 : BK;  // K elements per 128-byte box
  const int nkb = p.dim / BKE;
  const int KT = I8 ? (nkb < I8_KT ? nkb : I8_KT) : (nkb < 8 ? nkb : 8);  // A boxes resident in TMEM
  const int KS = nkb - KT;                                                  // A boxes resident in smem
  constexpr int NACC = I8 ? I8_NACC : 2;         // accumulator buffers
  constexpr int ACC0 = I8 ? I8_ACC_COL : ACC_COL;  // first accumulator column
  const int BPS = p.bps;             // B boxes per pipeline stage (one barrier round trip per 4*BPS MMAs)
  const int STAGE_BYTES = BPS * PBOX;
  const int nsg = nkb / BPS;
  uint8_t* stages = base;
  uint8_t* asmem = base + NSTAGE * STAGE_BYTES;
  uint32_t* lk_all = reinterpret_cast<uint32_t*>(asmem + KS * ABOX);  // [2 halves][cap][BM] packed candidates
  uint64_t* bars = reinterpret_cast<uint64_t*>(lk_all + 2 * cap * BM);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  uint64_t* accf = bars + 2 * NSTAGE;
  uint64_t* acce = accf + 3;
  uint64_t* aready = acce + 3;
  uint64_t* afree = aready + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(afree + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(smem_u32(&accf[b]), 1);
      mbar_init(smem_u32(&acce[b]), 16);  // 8 epilogue warps x 2 CTAs
    }
    mbar_init(smem_u32(aready), 16 + (KS > 0 ? 1 : 0));  // + the leader producer's expect_tx
    mbar_init(smem_u32(afree), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs, own half of each tile) ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      if (KS > 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
      int stage = 0;
      uint32_t phase = 0, unit_i = 0;
      for (int u = pair; u < p.n_units; u += npairs, ++unit_i) {
        const int split = u / p.n_qtiles;
        const int qtile = u - split * p.n_qtiles;
        const int64_t r0 = (int64_t)split * p.rows_per_split;
        const int64_t r1 = min((int64_t)p.n_rows, r0 + p.rows_per_split);
        const bool no_tma = p.debug & 2;  // diagnostic: no table / query traffic
        if (KS > 0) {  // this unit's smem-resident query boxes, once the previous unit's MMAs are done
          mbar_wait(smem_u32(afree), (unit_i & 1) ^ 1);
          if (no_tma) {
            if (leader) mbar_arrive(smem_u32(aready));
          } else {
            if (leader) mbar_expect_tx(smem_u32(aready), 2 * KS * ABOX);
            for (int j = 0; j < KS; ++j)
              tma_load_2d_pair(smem_u32(asmem + j * ABOX), &tmQ, smem_u32(aready), (KT + j) * BKE,
                               qtile * 2 * BM + (int)rank * BM);
          }
        }
        for (int64_t row = r0; row < r1; row += PN) {
          for (int sg = 0; sg < nsg; ++sg) {
            mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
            if (no_tma) {
              if (leader) mbar_arrive(smem_u32(&full[stage]));
            } else {
              if (leader) mbar_expect_tx(smem_u32(&full[stage]), 2 * STAGE_BYTES);
              for (int bx = 0; bx < BPS; ++bx)
                tma_load_2d_pair(smem_u32(stages + stage * STAGE_BYTES + bx * PBOX), &tmB, smem_u32(&full[stage]),
                                 (sg * BPS + bx) * BKE, (int)(row * p.tile_stride + rank * PHB));
            }
            if (++stage == NSTAGE) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    // The whole warp runs the loop (warp-uniform state stays in uniform
    // registers); one elected lane issues the MMAs and commits.
    if (leader) {
      // D f32 (bf16) or s32 (i8: c_format 2, A/B signed 8-bit), K-major, M=256, N=PN
      const uint32_t idesc = ((I8 ? 2u : 1u) << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(PN >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
      const bool issuer = elect_one();
      int stage = 0;
      uint32_t phase = 0, tile = 0, unit_i = 0;
      // FC_SHORTLIST_DEBUG & 16: MMA-warp cycles waiting for [a free accumulator, TMA data, the unit's A]
      const bool mprof = p.debug & 16;
      long long mcyc[3] = {0, 0, 0};
      for (int u = pair; u < p.n_units; u += npairs, ++unit_i) {
        const int split = u / p.n_qtiles;
        const int64_t r0 = (int64_t)split * p.rows_per_split;
        const int64_t r1 = min((int64_t)p.n_rows, r0 + p.rows_per_split);
        {
          const long long a_t0 = mprof ? clock64() : 0;
          mbar_wait(smem_u32(aready), unit_i & 1);
          tc_fence_after();
          if (mprof) mcyc[2] += clock64() - a_t0;
        }
        for (int64_t row = r0; row < r1; row += PN, ++tile) {
          const uint32_t b = tile % NACC;
          const uint32_t use = tile / NACC;
          long long m_t0 = mprof ? clock64() : 0;
          mbar_wait(smem_u32(&acce[b]), (use & 1) ^ 1);
          tc_fence_after();
          if (mprof) {
            const long long t1 = clock64();
            mcyc[0] += t1 - m_t0;
          }
          const uint32_t d_tmem = tmem + ACC0 + b * PN;
          for (int sg = 0; sg < nsg; ++sg) {
            if (mprof) m_t0 = clock64();
            mbar_wait(smem_u32(&full[stage]), phase);
            tc_fence_after();
            if (mprof) mcyc[1] += clock64() - m_t0;
            if (issuer) {
#pragma unroll 1
              for (int bx = 0; bx < BPS; ++bx) {
                const int kb = sg * BPS + bx;
                const uint64_t bdesc = smem_desc_sw128(smem_u32(stages + stage * STAGE_BYTES + bx * PBOX));
                if (p.debug & 1) continue;
                if (I8 && kb < KT)
                  mma_box4_pair_i8(d_tmem, tmem + kb * 32, bdesc, idesc, kb != 0);
                else if (I8)
                  mma_box4_pair_ss_i8(d_tmem, smem_desc_sw128(smem_u32(asmem + (kb - KT) * ABOX)), bdesc, idesc, 1);
                else if (kb < KT)
                  mma_box4_pair(d_tmem, tmem + kb * (BK / 16) * 8, bdesc, idesc, kb != 0);
                else
                  mma_box4_pair_ss(d_tmem, smem_desc_sw128(smem_u32(asmem + (kb - KT) * ABOX)), bdesc, idesc, 1);
              }
              tc_commit_pair(smem_u32(&empty[stage]));
            }
            __syncwarp();
            if (++stage == NSTAGE) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (issuer) tc_commit_pair(smem_u32(&accf[b]));
          __syncwarp();
        }
        if (issuer) tc_commit_pair(smem_u32(afree));  // A (TMEM + smem parts) may be overwritten
        __syncwarp();
      }
      if (mprof && issuer)
        for (int i = 0; i < 3; ++i)
          atomicAdd(reinterpret_cast<unsigned long long*>(p.stats + 12) + i, (unsigned long long)mcyc[i]);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warps 2..9 of both CTAs ----------------
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int t = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    uint32_t* lk = lk_all + (size_t)half * cap * BM;
    uint32_t tile = 0, unit_i = 0;
    for (int u = pair; u < p.n_units; u += npairs, ++unit_i) {
      const int split = u / p.n_qtiles;
      const int qtile = u - split * p.n_qtiles;
      const int64_t r0 = (int64_t)split * p.rows_per_split;
      const int64_t r1 = min((int64_t)p.n_rows, r0 + p.rows_per_split);
      const int q = qtile * 2 * BM + (int)rank * BM + t;
      {  // (1) this unit's query row -> TMEM columns [0, 32*KT), once the previous unit's MMAs are done
        mbar_wait(smem_u32(afree), (unit_i & 1) ^ 1);
        tc_fence_after();
        const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(p.Qb) +
                                                          (size_t)q * p.dim * (I8 ? 1 : 2));
        for (int kb = half; kb < KT; kb += 2) {  // the two warps of a quarter split the boxes
          uint32_t r[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint4 v = __ldg(src + kb * 8 + i);
            r[4 * i + 0] = v.x;
            r[4 * i + 1] = v.y;
            r[4 * i + 2] = v.z;
            r[4 * i + 3] = v.w;
          }
          tmem_st32(tmem + lane_base + kb * 32, r);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(smem_u32(aready), 0);
      }
      // (2) stream the accumulator tiles through the running-threshold filter
      int cnt = 0, pub = 0;  // entries [pub, cnt) not yet counted in the histogram
      float tau = -INFINITY;
      uint32_t* hq = p.hist + (size_t)q * HSTRIDE;
      // int8: s_q and the error terms of this thread's query (padding: 1, (0, 0));
      // the unit filters and stores U = a + eps_t, an upper bound of the exact
      // score (eps_t = ||dq|| X + ||qhat|| R_t, the tile's bound, lookup.cuh),
      // and raises tau to (k-th best U seen) - (typical eps + slack): rows
      // with U below that are almost surely below the k-th exact score (the
      // certificate, not this heuristic, decides; a too-high tau only sends
      // the query to the bf16 tier)
      const float qsc = I8 ? __ldg(p.qscale + q) : 1.f;
      const float2 qe = I8 ? __ldg(p.qerr + q) : make_float2(0.f, 0.f);
      const float hoff = I8 ? __fmaf_ru(qe.y, p.r_typ, qe.x) + p.slack : 0.f;
      float ut[PILOT_R];  // pilot: best U over the sampled tiles, descending
#pragma unroll
      for (int i = 0; i < PILOT_R; ++i) ut[i] = -INFINITY;
      const bool fixed_tau = I8 && p.tau_fix != nullptr;
      if (fixed_tau) tau = __ldg(p.tau_fix + q);
      if (!p.pilot && !fixed_tau) hist_refresh(hq, p.kh, tau, hoff);
      if (I8 && !p.pilot && !fixed_tau) {  // the pilot's max U of this query
        uint32_t pk;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(pk) : "l"(p.gkey + q));
        if (pk) tau = fmaxf(tau, key_float(pk) - hoff);
      }
      // int8: the tile's scale and residual bound are loaded one tile ahead
      // (a dependent L2 round trip per tile otherwise sits on the critical path)
      float nx_sc = 1.f, nx_res = 0.f;
      if (I8) {
        nx_sc = __ldg(p.tscale + ((r0 * p.tile_stride) >> 7));
        nx_res = __ldg(p.tres + ((r0 * p.tile_stride) >> 7));
      }
      // FC_SHORTLIST_DEBUG & 16: per-warp clock64 spans [accumulator wait, histogram, compaction, appends]
      long long cyc[4] = {0, 0, 0, 0}, c_t0 = 0;
      const bool prof = p.debug & 16;
      for (int64_t row = r0; row < r1; row += PN, ++tile) {
        const uint32_t b = tile % NACC;
        const uint32_t use = tile / NACC;
        if ((tile & p.refresh_mask) == 0 && !p.pilot && !fixed_tau) {
          if (prof) c_t0 = clock64();
          hist_publish(hq, lk, t, pub, cnt);
          pub = cnt;
          hist_refresh(hq, p.kh, tau, hoff);
          if (prof) cyc[1] += clock64() - c_t0;
        }
        // int8: this tile's scale product, error bound and integer threshold
        // (reject a <= tau - eps_t, i.e. U <= tau)
        const float sqt = I8 ? qsc * nx_sc : 1.f;
        const float eps_t = I8 ? __fmaf_ru(qe.y, nx_res, qe.x) : 0.f;
        int thr = I8 ? i8_thr(__fsub_rd(tau, eps_t), sqt) : 0;
        if (I8 && row + PN < r1) {
          nx_sc = __ldg(p.tscale + (((row + PN) * p.tile_stride) >> 7));
          nx_res = __ldg(p.tres + (((row + PN) * p.tile_stride) >> 7));
        }
        if (prof) c_t0 = clock64();
        mbar_wait(smem_u32(&accf[b]), use & 1);
        tc_fence_after();
        if (prof) cyc[0] += clock64() - c_t0;
        if ((p.debug & 16) && lane == 0) atomicAdd(p.stats + 2, 1u);
        // columns [64 half, +64) of the tile; lim = valid rows of this half
        const int lim_all = (int)max((int64_t)0, min((int64_t)EPI_HALF_COLS,
                                                     (p.pilot ? p.n_rows_phys - row * p.tile_stride : r1 - row) -
                                                         half * EPI_HALF_COLS));
        const uint32_t off_base = (uint32_t)(row - r0) + half * EPI_HALF_COLS;
        // 32 accumulator columns per step (a rolled loop: the unrolled
        // 128-column body overflowed the instruction cache, ncu "no_inst";
        // round 2 measured unrolled / software-pipelined / out-of-line slow
        // path variants of this loop 15-25 % slower). Per 16-score chunk a max
        // tree and a warp vote skip the append code unless some query of the
        // warp has a score above its threshold.
        // both 32-column loads of this warp's half in flight together, then
        // the accumulator buffer is released before any filtering
        uint32_t rv[EPI_HALF_COLS];
        tmem_ld32_issue(tmem + lane_base + ACC0 + b * PN + half * EPI_HALF_COLS, rv);
        tmem_ld32_issue(tmem + lane_base + ACC0 + b * PN + half * EPI_HALF_COLS + 32, rv + 32);
        tmem_ld32_wait(rv);
        tmem_ld32_wait(rv + 32);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(smem_u32(&acce[b]), 0);
        if (I8 && p.pilot) {  // fold the tile half's valid dots into the best-R U list
          int pthr = i8_thr(__fsub_rd(ut[PILOT_R - 1], eps_t), sqt);  // refreshed after insertions
          const bool full = lim_all >= EPI_HALF_COLS;  // warp-uniform: every tile but the last
#pragma unroll
          for (int c0 = 0; c0 < EPI_HALF_COLS; c0 += 16) {
            int m = INT_MIN;
            if (full) {  // unguarded 3-input max tree (ncu r02ca: the guarded chain kept the ALU pipe 72 % busy)
              const int* vi = reinterpret_cast<const int*>(rv + c0);
              int m0 = __vimax3_s32(vi[0], vi[1], vi[2]), m1 = __vimax3_s32(vi[3], vi[4], vi[5]);
              int m2 = __vimax3_s32(vi[6], vi[7], vi[8]), m3 = __vimax3_s32(vi[9], vi[10], vi[11]);
              int m4 = __vimax3_s32(vi[12], vi[13], vi[14]);
              m0 = __vimax3_s32(m0, m1, m2);
              m3 = __vimax3_s32(m3, m4, vi[15]);
              m = max(m0, m3);
            } else {
#pragma unroll
              for (int c = c0; c < c0 + 16; c += 2)
                m = __vimax3_s32(m, c < lim_all ? (int)rv[c] : INT_MIN, c + 1 < lim_all ? (int)rv[c + 1] : INT_MIN);
            }
            if (!__any_sync(0xffffffffu, m > pthr)) continue;
            uint32_t msk = 0;
            if (full) {
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) msk |= ((int)rv[c0 + jj] > pthr) ? (1u << jj) : 0u;
            } else {
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) msk |= ((c0 + jj < lim_all) & ((int)rv[c0 + jj] > pthr)) ? (1u << jj) : 0u;
            }
            if (msk) {
              do {  // only the lane's qualifying dots (usually 0-1 per chunk)
                const int jj = __ffs(msk) - 1;
                msk &= msk - 1;
                float u = __fadd_ru(i8_score_up((int)sel16(rv + c0, jj), sqt), eps_t);
#pragma unroll
                for (int i = 0; i < PILOT_R; ++i) {  // insertion into the descending list
                  const float hi = fmaxf(ut[i], u);
                  u = fminf(ut[i], u);
                  ut[i] = hi;
                }
              } while (msk);
              pthr = i8_thr(__fsub_rd(ut[PILOT_R - 1], eps_t), sqt);  // the tighter bound for the next chunks
            }
          }
          continue;
        }
        if (!(p.debug & 4)) {
#pragma unroll
          for (int hh = 0; hh < EPI_HALF_COLS / 16; ++hh) {
            const int c0 = hh * 16;
            bool hot;
            if constexpr (I8) {  // exact s32 dots: 3-input integer max tree
              const int* vi = reinterpret_cast<const int*>(rv + c0);
              int m0 = __vimax3_s32(vi[0], vi[1], vi[2]), m1 = __vimax3_s32(vi[3], vi[4], vi[5]);
              int m2 = __vimax3_s32(vi[6], vi[7], vi[8]), m3 = __vimax3_s32(vi[9], vi[10], vi[11]);
              int m4 = __vimax3_s32(vi[12], vi[13], vi[14]);
              m0 = __vimax3_s32(m0, m1, m2);
              m3 = __vimax3_s32(m3, m4, vi[15]);
              hot = max(m0, m3) > thr;
            } else {
              float vc[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) vc[i] = __uint_as_float(rv[c0 + i]);
              float a0 = fmaxf(vc[0], vc[1]), a1 = fmaxf(vc[2], vc[3]), a2 = fmaxf(vc[4], vc[5]), a3 = fmaxf(vc[6], vc[7]);
              a0 = fmaxf(a0, fmaxf(vc[8], vc[9]));
              a1 = fmaxf(a1, fmaxf(vc[10], vc[11]));
              a2 = fmaxf(a2, fmaxf(vc[12], vc[13]));
              a3 = fmaxf(a3, fmaxf(vc[14], vc[15]));
              hot = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)) > tau;
            }
            if (!__any_sync(0xffffffffu, hot | (lim_all < EPI_HALF_COLS))) continue;
            if (p.debug & 32) continue;  // diagnostic: fast path only
            if ((p.debug & 16) && lane == 0) atomicAdd(p.stats + 0, 1u);
            if (I8 && fixed_tau && __any_sync(0xffffffffu, cnt + 16 > cap)) {
              // threshold tier: flush the list to the query buffer (tau stays)
              if (q < p.nq) i8_append(p, q, lk, t, cnt, r0, tau);
              cnt = 0;
              pub = 0;
            }
            if (__any_sync(0xffffffffu, cnt + 16 > cap)) {
              if ((p.debug & 16) && lane == 0) atomicAdd(p.stats + 1, 1u);
              if (prof) c_t0 = clock64();
              hist_publish(hq, lk, t, pub, cnt);  // count before compaction may drop entries
              compact_keys(lk, t, cnt, p.kp, tau, false);
              pub = cnt;
              if (I8) thr = i8_thr(__fsub_rd(tau, eps_t), sqt);
              if (prof) cyc[2] += clock64() - c_t0;
            }
            if (prof) c_t0 = clock64();
            const uint32_t off0 = off_base + (uint32_t)c0;
            if constexpr (I8) {
              // a lane accepts ~1 of the 16 dots of a hot chunk: build its
              // accept mask, then loop over the set bits only (the dot is
              // picked out of the 16 registers by a 4-level select tree)
              uint32_t m = 0;
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) m |= ((c0 + jj < lim_all) & ((int)rv[c0 + jj] > thr)) ? (1u << jj) : 0u;
              while (m) {
                const int jj = __ffs(m) - 1;
                m &= m - 1;
                const int d = (int)sel16(rv + c0, jj);
                lk[cnt * BM + t] = (hkey_ru(__fadd_ru(i8_score_up(d, sqt), eps_t)) << 16) | (off0 + jj);
                ++cnt;
              }
            } else
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              {
                const float v = __uint_as_float(rv[c0 + jj]);
                const bool acc = (c0 + jj < lim_all) & (v > tau);
                if (acc) lk[cnt * BM + t] = (hkey_ru(v) << 16) | (off0 + jj);
                cnt += acc;
              }
            }
            if (prof) cyc[3] += clock64() - c_t0;
          }
        }
      }
      if (I8 && p.pilot) {
        if (q < p.nq) {
          float* o = p.pilot_out + (((size_t)q * 2 * p.n_splits) + 2 * split + half) * PILOT_R;
#pragma unroll
          for (int i = 0; i < PILOT_R; ++i) o[i] = ut[i];
        }
        continue;
      }
      if (prof) c_t0 = clock64();
      hist_publish(hq, lk, t, pub, cnt);
      if (I8) {
        // append the unit's entries to the query's buffer; what does not fit
        // is dropped into the drop level, as is everything the unit rejected
        // (U <= tau) or compacted away (stored U <= the raised tau)
        if (q < p.nq) i8_append(p, q, lk, t, cnt, r0, tau);
        if (prof) {
          cyc[2] += clock64() - c_t0;
          if (lane == 0)
            for (int i = 0; i < 4; ++i)
              atomicAdd(reinterpret_cast<unsigned long long*>(p.stats + 4) + i, (unsigned long long)cyc[i]);
        }
        continue;
      }
      compact_keys(lk, t, cnt, p.kp, tau, true);  // exact: the unit's list holds at most kp entries
      if (prof) {
        cyc[2] += clock64() - c_t0;
        if (lane == 0)
          for (int i = 0; i < 4; ++i)
            atomicAdd(reinterpret_cast<unsigned long long*>(p.stats + 4) + i, (unsigned long long)cyc[i]);
      }
      if (q < p.nq) {
        const int sub = 2 * split + half;  // the merge sees 2 lists per row range
        const size_t o = ((size_t)q * 2 * p.n_splits + sub) * p.kp;
        for (int i = 0; i < cnt; ++i) p.part_k[o + i] = lk[i * BM + t];
        p.part_n[(size_t)q * 2 * p.n_splits + sub] = cnt;
        // every row this list's unit rejected (a <= tau at the time) or
        // compacted away (stored score <= the raised tau) has a <= final tau
        if (I8) p.part_d[(size_t)q * 2 * p.n_splits + sub] = tau;
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Per query (one warp): the PILOT_R-th best U over all pilot lists -> gkey
// (order key; 0 = none, the main pass then starts from its histogram only).
__global__ void k_pilot_kth(const float* __restrict__ po, int lists, int nq, uint32_t* __restrict__ gkey) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nq) return;
  const float* v = po + (size_t)w * lists * PILOT_R;
  const int n = lists * PILOT_R;
  float best[PILOT_R];
#pragma unroll
  for (int i = 0; i < PILOT_R; ++i) best[i] = -INFINITY;
  for (int j = lane; j < n; j += 32) {
    float u = v[j];
#pragma unroll
    for (int i = 0; i < PILOT_R; ++i) {
      const float hi = fmaxf(best[i], u);
      u = fminf(best[i], u);
      best[i] = hi;
    }
  }
  // warp merge: PILOT_R rounds of warp max over the lanes' list heads
  int ptr = 0;
  float kth = -INFINITY;
  for (int r = 0; r < PILOT_R; ++r) {
    float h = ptr < PILOT_R ? best[0] : -INFINITY;
    float m = h;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    const unsigned own = __ballot_sync(0xffffffffu, h == m && ptr < PILOT_R);
    if (own && lane == __ffs(own) - 1) {  // pop the head
#pragma unroll
      for (int i = 0; i < PILOT_R - 1; ++i) best[i] = best[i + 1];
      best[PILOT_R - 1] = -INFINITY;
      ++ptr;
    }
    kth = m;
  }
  if (lane == 0) gkey[w] = kth > -INFINITY ? okey(kth) : 0u;
}

__global__ void k_q_to_bf16(const float* __restrict__ Q, int nq, int dim, __nv_bfloat16* __restrict__ Qb, int nq_pad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)nq_pad * dim;
  if (i >= total) return;
  const int64_t q = i / dim;
  Qb[i] = q < nq ? __float2bfloat16_rn(Q[i]) : __float2bfloat16_rn(0.f);
}


// Per query: top-kp of the n_splits partial shortlists by packed key (stored
// fp16 upper-bound score, then row offset). One warp per query: the filled
// prefix of every split's list (pn[] entries) is
// compacted (slot order kept) as (key, slot); a 32-step binary
// search on the key over those with warp-reduced counts finds the kp-th
// largest; ballot compaction writes the result. Most slots are empty (every
// unit filters by the query's shared acceptance threshold), so only ~1/10 of
// the n_splits * kp slots are read, and a small per-warp shared buffer (MG_CAP
// items, spilling to gkeys when a query has more) keeps ~24 warps per SM
// resident to hide the load latency.
constexpr int MG_W = 8;
constexpr int MG_CAP = 1024;
// One output candidate: stored score (upper bound of the bf16 score) and
// absolute row slot of a packed key found at `slot` (= split * kp + j).
// (list index >> rshift = row range: the pair kernel writes two lists, one per
// epilogue column half, for each row range)
__device__ __forceinline__ void emit(uint32_t key, uint32_t slot, int kp, int rps, int rshift, float* cs, uint32_t* cr,
                                     size_t at) {
  cs[at] = hkey_float(key >> 16);
  cr[at] = ((slot / (uint32_t)kp) >> rshift) * (uint32_t)rps + (key & 0xFFFFu);
}

// kout = output slots per query (kp for the bf16 tier; the int8 tier merges
// short unit lists into a longer one). pd (int8 tier, else null): per-list
// drop levels; cm[q] = max(drop levels, stored score at the merge cut), an
// upper bound of the approximate score of every row outside q's output.
__global__ void __launch_bounds__(MG_W * 32) k_shortlist_merge(const uint32_t* __restrict__ pk,
                                                               const int32_t* __restrict__ pn, int n_splits, int kp, int rps, int rshift,
                                                               int nq, int kout, float* __restrict__ cs, uint32_t* __restrict__ cr,
                                                               int32_t* __restrict__ cn, uint32_t* __restrict__ gkeys,
                                                               const float* __restrict__ pd, float* __restrict__ cm) {
  extern __shared__ uint32_t s_key[];  // [warps][2][MG_CAP] (gkeys [nq][2][n_splits * kp] past that)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + w;
  if (q >= nq) return;
  const int total = n_splits * kp;
  const int32_t* pq = pn + (size_t)q * n_splits;
  int n_all = 0;
  for (int s0 = lane; s0 < n_splits; s0 += 32) n_all += min(__ldg(pq + s0), kp);
  n_all = __reduce_add_sync(0xffffffffu, n_all);
  float drop = -INFINITY;
  if (pd) {
    for (int s0 = lane; s0 < n_splits; s0 += 32) drop = fmaxf(drop, __ldg(pd + (size_t)q * n_splits + s0));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) drop = fmaxf(drop, __shfl_xor_sync(0xffffffffu, drop, off));
  }
  const int cap = n_all <= MG_CAP ? MG_CAP : total;
  uint32_t* key = n_all <= MG_CAP ? s_key + (size_t)w * 2 * MG_CAP : gkeys + (size_t)q * 2 * total;
  uint32_t* slot = key + cap;
  const size_t base = (size_t)q * total;
  int n_items = 0;  // dense prefix [0, n_items) of filled slots, in slot order
  for (int s0 = 0; s0 < n_splits; s0 += 32) {
    const int c = s0 + lane < n_splits ? min(__ldg(pq + s0 + lane), kp) : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int ns = min(32, n_splits - s0);
#pragma unroll 8
    for (int t = 0; t < ns; ++t) {
      const int ct = __shfl_sync(0xffffffffu, c, t);
      const int off = n_items + __shfl_sync(0xffffffffu, inc, t) - ct;
      const int sp = s0 + t;
      for (int j = lane; j < ct; j += 32) {
        key[off + j] = __ldg(pk + base + (size_t)sp * kp + j);
        slot[off + j] = (uint32_t)(sp * kp + j);
      }
    }
    n_items += __shfl_sync(0xffffffffu, inc, 31);
  }
  __syncwarp();
  uint32_t T = 1;  // keep everything non-empty
  if (n_items > kout) {
    uint32_t lo = 1, hi = 0xFFFFFFFFu;
    while (lo < hi) {
      const uint32_t mid = lo + (uint32_t)(((uint64_t)hi - lo + 1) >> 1);
      int c = 0;
      for (int i = lane; i < n_items; i += 32) c += key[i] >= mid;
      c = __reduce_add_sync(0xffffffffu, c);
      if (c >= kout) lo = mid; else hi = mid - 1;
    }
    T = lo;
    drop = fmaxf(drop, hkey_float(T >> 16));  // cut entries have stored score <= that of T
  }
  if (cm && lane == 0) cm[q] = drop;
  // strictly above T first (in slot order), then == T up to kp
  int out = 0;
  for (int i0 = 0; i0 < n_items; i0 += 32) {
    const int i = i0 + lane;
    const bool take = i < n_items && key[i] > T;
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (take) {
      const int at = out + __popc(bal & ((1u << lane) - 1));
      emit(key[i], slot[i], kp, rps, rshift, cs, cr, (size_t)q * kout + at);
    }
    out += __popc(bal);
  }
  for (int i0 = 0; i0 < n_items && out < kout; i0 += 32) {
    const int i = i0 + lane;
    const bool take = i < n_items && key[i] == T;
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (take) {
      const int at = out + __popc(bal & ((1u << lane) - 1));
      if (at < kout) emit(key[i], slot[i], kp, rps, rshift, cs, cr, (size_t)q * kout + at);
    }
    out += __popc(bal);
  }
  if (lane == 0) cn[q] = min(kout, out);
}

// int8 tier merge: per query (one warp) the kout best of its contiguous
// buffer by (U key, row); cm[q] = max(drop level, U at the cut).
constexpr int QM_W = 4;
constexpr int QCAP = 1024;
__global__ void __launch_bounds__(QM_W * 32) k_i8_merge(const uint64_t* __restrict__ qbuf, const uint32_t* __restrict__ qcnt,
                                                       const uint32_t* __restrict__ qdrop, int nq, int kout,
                                                       float* __restrict__ cs, uint32_t* __restrict__ cr,
                                                       int32_t* __restrict__ cn, float* __restrict__ cm) {
  __shared__ uint64_t s_k[QM_W][QCAP];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * QM_W + w;
  if (q >= nq) return;
  const int n = (int)min(qcnt[q], (uint32_t)QCAP);
  const uint32_t dk = qdrop[q];
  float drop = dk ? key_float(dk) : -INFINITY;
  uint64_t* key = s_k[w];
  for (int i = lane; i < n; i += 32) key[i] = qbuf[(size_t)q * QCAP + i];
  __syncwarp();
  uint64_t T = 0;  // keep everything
  if (n > kout) {
    // T = the kout-th largest key (keys are unique): bisection over the top
    // 16 bits (the score bucket) on all n keys, then over the full key on the
    // few keys of that bucket only, copied behind the list when they fit
    uint32_t t16 = 0;
#pragma unroll 1
    for (int bit = 15; bit >= 0; --bit) {
      const uint32_t c16 = t16 | (1u << bit);
      int c = 0;
      for (int i = lane; i < n; i += 32) c += (uint32_t)(key[i] >> 48) >= c16;
      if ((int)__reduce_add_sync(0xffffffffu, (unsigned)c) >= kout) t16 = c16;
    }
    int above = 0;  // keys in higher buckets (< kout by the choice of t16)
    for (int i = lane; i < n; i += 32) above += (uint32_t)(key[i] >> 48) > t16;
    above = (int)__reduce_add_sync(0xffffffffu, (unsigned)above);
    const int need = kout - above;  // >= 1 keys wanted from the t16 bucket
    const uint64_t* tk = key;
    int m = n;
    {  // compact the bucket behind the list (n + m <= QCAP), else scan in place
      int cnt = 0;
      for (int i = lane; i < n; i += 32) cnt += (uint32_t)(key[i] >> 48) == t16;
      cnt = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
      if (n + cnt <= QCAP) {
        int o = n;
        for (int i0 = 0; i0 < n; i0 += 32) {
          const int i = i0 + lane;
          const bool in = i < n && (uint32_t)(key[i] >> 48) == t16;
          const unsigned bal = __ballot_sync(0xffffffffu, in);
          if (in) key[o + __popc(bal & ((1u << lane) - 1))] = key[i];
          o += __popc(bal);
        }
        __syncwarp();
        tk = key + n;
        m = cnt;
      }
    }
    // (scanning in place, the higher buckets count too: target kout)
    const int target = tk == key ? kout : need;
    uint64_t lo = (uint64_t)t16 << 48, hi = lo | 0xFFFFFFFFFFFFull;
    while (lo < hi) {  // max T in the bucket with count(key >= T) >= target
      const uint64_t mid = lo + ((hi - lo) >> 1) + 1;
      int c = 0;
      for (int i = lane; i < m; i += 32) c += tk[i] >= mid;
      c = __reduce_add_sync(0xffffffffu, c);
      if (c >= target) lo = mid; else hi = mid - 1;
    }
    T = lo;
    drop = fmaxf(drop, hkey_float((uint32_t)(T >> 48)));  // cut entries have stored U <= that of T
  }
  int out = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const bool take = i < n && key[i] >= T && (n <= kout || key[i] > T);
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (take) {
      const int at = out + __popc(bal & ((1u << lane) - 1));
      cs[(size_t)q * kout + at] = hkey_float((uint32_t)(key[i] >> 48));
      cr[(size_t)q * kout + at] = (uint32_t)(key[i] & 0xFFFFFFFFFFFFull);
    }
    out += __popc(bal);
  }
  if (n > kout)  // keys are unique (distinct rows): exactly one entry equals T
    for (int i0 = 0; i0 < n && out < kout; i0 += 32) {
      const int i = i0 + lane;
      const bool take = i < n && key[i] == T;
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      if (take) {
        const int at = out + __popc(bal & ((1u << lane) - 1));
        if (at < kout) {
          cs[(size_t)q * kout + at] = hkey_float((uint32_t)(key[i] >> 48));
          cr[(size_t)q * kout + at] = (uint32_t)(key[i] & 0xFFFFFFFFFFFFull);
        }
      }
      out += __popc(bal);
    }
  if (lane == 0) {
    cn[q] = min(out, kout);
    cm[q] = drop;
  }
}

// Same selection as k_shortlist_merge with one CTA per query (MC_T threads):
// used when there are too few queries to fill the GPU with one warp each (the
// tier-2 re-shortlist of a handful of near-tie queries), where one warp would
// walk tens of thousands of keys 32 times. Slot order is kept by a per-chunk
// block scan, so the chosen candidates are identical.
constexpr int MC_T = 1024;
__device__ __forceinline__ int block_sum(int v, int* red) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = __reduce_add_sync(0xffffffffu, v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  int t = lane < (MC_T / 32) ? red[lane] : 0;
  return __reduce_add_sync(0xffffffffu, t);
}
// Exclusive prefix of `flag` over the CTA in thread order; returns the chunk total.
__device__ __forceinline__ int block_scan(bool flag, int* red, int* pre) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned bal = __ballot_sync(0xffffffffu, flag);
  __syncthreads();
  if (lane == 0) red[w] = __popc(bal);
  __syncthreads();
  int x = lane < (MC_T / 32) ? red[lane] : 0, inc = x;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const int tot = __shfl_sync(0xffffffffu, inc, 31);
  *pre = __shfl_sync(0xffffffffu, inc - x, w) + __popc(bal & ((1u << lane) - 1));
  return tot;
}
__global__ void __launch_bounds__(MC_T) k_shortlist_merge_cta(const uint32_t* __restrict__ pk,
                                                              const int32_t* __restrict__ pn, int n_splits, int kp, int rps, int rshift,
                                                              int kout, float* __restrict__ cs, uint32_t* __restrict__ cr,
                                                              int32_t* __restrict__ cn, const float* __restrict__ pd,
                                                              float* __restrict__ cm) {
  extern __shared__ uint32_t s_key[];  // [2][n_splits * kp]
  __shared__ int red[MC_T / 32];
  const int q = blockIdx.x;
  const int total = n_splits * kp;
  uint32_t* key = s_key;
  uint32_t* slot = key + total;
  const size_t base = (size_t)q * total;
  int n_items = 0;
  for (int i0 = 0; i0 < total; i0 += MC_T) {
    const int i = i0 + threadIdx.x;
    uint32_t k = 0u;
    if (i < total) {
      const int sp = i / kp, j = i - sp * kp;
      if (j < pn[(size_t)q * n_splits + sp]) k = pk[base + i];  // never 0 (see hkey_ru)
    }
    int pre;
    const int tot = block_scan(k != 0u, red, &pre);
    if (k != 0u) {
      key[n_items + pre] = k;
      slot[n_items + pre] = (uint32_t)i;
    }
    n_items += tot;
  }
  __syncthreads();
  uint32_t T = 1;
  if (n_items > kout) {
    uint32_t lo = 1, hi = 0xFFFFFFFFu;
    while (lo < hi) {
      const uint32_t mid = lo + (uint32_t)(((uint64_t)hi - lo + 1) >> 1);
      int c = 0;
      for (int i = threadIdx.x; i < n_items; i += MC_T) c += key[i] >= mid;
      c = block_sum(c, red);
      if (c >= kout) lo = mid; else hi = mid - 1;
    }
    T = lo;
  }
  if (cm && threadIdx.x == 0) {
    float drop = n_items > kout ? hkey_float(T >> 16) : -INFINITY;
    if (pd)
      for (int s0 = 0; s0 < n_splits; ++s0) drop = fmaxf(drop, pd[(size_t)q * n_splits + s0]);
    cm[q] = drop;
  }
  int out = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int i0 = 0; i0 < n_items && out < kout; i0 += MC_T) {
      const int i = i0 + threadIdx.x;
      const bool take = i < n_items && (pass == 0 ? key[i] > T : key[i] == T);
      int pre;
      const int tot = block_scan(take, red, &pre);
      if (take && out + pre < kout) emit(key[i], slot[i], kp, rps, rshift, cs, cr, (size_t)q * kout + out + pre);
      out += tot;
    }
  if (threadIdx.x == 0) cn[q] = min(kout, out);
}

}  // namespace sm100

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    FC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) raise(LC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool approx_available() { return true; }

static void encode_2d(CUtensorMap* m, const __nv_bfloat16* base, int64_t rows, int cols, int box_rows) {
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)cols * sizeof(__nv_bfloat16)};
  cuuint32_t box[2] = {(cuuint32_t)sm100::BK, (cuuint32_t)box_rows};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(base), gdim, gstride, box,
                           estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(LC_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

void approx_plan(ApproxPlan& p, const __nv_bfloat16* rows, int64_t n_rows, int dim, int sm_count) {
  (void)sm_count;
  p.n_rows = n_rows;
  p.dim = dim;
  p.rows = rows;
  p.bn = dim <= 512 ? 128 : 64;
  encode_2d(&p.tmap, rows, n_rows, dim, p.bn);   // single-CTA kernel: [bn rows][64]
  encode_2d(&p.tmap2, rows, n_rows, dim, sm100::PHB);  // pair kernel: each CTA's [64 rows][64]
  p.valid = true;
}

// 1 = single-CTA kernel (N=64/128, all query dims in TMEM; any dim <= 1024),
// 2 = CTA-pair kernel (N=128, dim <= 768; default)
static bool use_pair(int dim) {
  const char* e = getenv("FC_SHORTLIST_CTA");
  return !(e && atoi(e) == 1) && dim <= 768;
}

template <int BN>
static void launch_single(lc_ctx* ctx, const ApproxPlan& plan, sm100::Params prm) {
  // smem: NSTAGE table tiles + a candidate buffer of `cap` (score,row) slots
  // per query; several TMA boxes per stage so the single MMA-issuing thread
  // pays one barrier wait per 8-16 MMAs instead of per 4
  const int nkb = prm.dim / sm100::BK;
  prm.bps = nkb % 4 == 0 ? 4 : nkb % 3 == 0 ? 3 : nkb % 2 == 0 ? 2 : 1;
  if (BN == 128 && prm.bps > 2) prm.bps = nkb % 2 == 0 ? 2 : 1;
  const size_t stage_bytes = (size_t)BN * 128 * prm.bps;
  const size_t budget = 227 * 1024 - 1024 - 256;
  const size_t slot_bytes = (size_t)sm100::BM * 8;
  const int64_t want = (int64_t)(prm.kp + 64) * slot_bytes;  // candidate buffer depth
  prm.nstage = (int)std::max<int64_t>(2, std::min<int64_t>(sm100::MAX_STAGE, ((int64_t)budget - want) / (int64_t)stage_bytes));
  const int64_t slots = (int64_t)((budget - prm.nstage * stage_bytes) / slot_bytes);
  prm.cap = (int)std::min<int64_t>(slots, prm.kp + 128);
  if (prm.cap < prm.kp + 16) raise(LC_ERR_INVALID_ARGUMENT, "lookup: shortlist too long for shared memory");
  const size_t smem = 1024 + 256 + prm.nstage * stage_bytes + (size_t)prm.cap * slot_bytes;
  auto kern = sm100::k_shortlist<BN>;
  FC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = std::min(prm.n_units, ctx->sm_count);
  KTimer kt(ctx, g_shortlist_timer);
  kern<<<grid, sm100::NTHREADS, smem, ctx->stream>>>(plan.tmap, prm);
  kt.stop();
  FC_LAUNCH_CHECK();
}

template <bool I8>
static void launch_pair(lc_ctx* ctx, const CUtensorMap& tmB, const CUtensorMap& tmQ, sm100::Params& prm) {
  using namespace sm100;
  const int nkb = prm.dim / (I8 ? 128 : BK);
  const int KS = I8 ? std::max(0, nkb - I8_KT) : (nkb > 8 ? nkb - 8 : 0);
  const size_t budget = 227 * 1024 - 1024 - 512;
  const size_t slot_bytes = (size_t)2 * BM * 4;  // one packed u32 per candidate, one list per column half
  const size_t fixed = (size_t)KS * ABOX;
  // candidate buffer: kp + 32 slots minimum (compactions stay rare once the
  // shared threshold is warm); the rest of smem goes to the table ring
  int64_t min_cap = prm.kp + 32;
  if (const char* e = getenv("FC_SHORTLIST_MINCAP")) min_cap = std::max<int64_t>(prm.kp + 8, atoi(e));
  {
    const char* e = getenv("FC_SHORTLIST_BPS");
    int want = e ? atoi(e) : 2;
    while (want > 1 && nkb % want) --want;
    prm.bps = std::max(1, want);
  }
  const int64_t stage_bytes = (int64_t)prm.bps * PBOX;
  int64_t nstage = ((int64_t)budget - (int64_t)fixed - min_cap * (int64_t)slot_bytes) / stage_bytes;
  nstage = std::min<int64_t>(nstage, PMAX_STAGE);
  if (const char* e = getenv("FC_SHORTLIST_NSTAGE")) nstage = std::min<int64_t>(nstage, atoi(e));
  if (nstage < 2) raise(LC_ERR_INVALID_ARGUMENT, "lookup: shortlist too long for shared memory");
  prm.nstage = (int)nstage;
  int64_t cap_max = prm.kp + 96;
  if (const char* e = getenv("FC_SHORTLIST_CAPMAX")) cap_max = std::max<int64_t>(min_cap, atoi(e));
  prm.cap = (int)std::min<int64_t>((budget - fixed - nstage * stage_bytes) / slot_bytes, cap_max);
  const size_t smem = 1024 + 512 + nstage * stage_bytes + fixed + (size_t)prm.cap * slot_bytes;
  FC_CUDA(cudaFuncSetAttribute(k_shortlist_pair<I8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = 2 * std::min(prm.n_units, ctx->sm_count / 2);
  KTimer kt(ctx, g_shortlist_timer);
  k_shortlist_pair<I8><<<grid, PAIR_THREADS, smem, ctx->stream>>>(tmB, tmQ, prm);
  kt.stop();
  FC_LAUNCH_CHECK();
}

thread_local const char* g_shortlist_timer = "shortlist";

namespace {
// One shortlist pass: work-unit split, candidate lists, the tcgen05 kernel,
// the per-query merge. Qconv = converted queries [nq_pad][dim] (bf16 or s8).
struct ShortlistRun {
  bool i8 = false;
  bool pair = true;
  int dim = 0, nq = 0, nq_pad = 0, n_qtiles = 0, bn = 0;
  int64_t n_rows = 0;
  int kp = 0, kout = 0;
  const void* Qconv = nullptr;
  const ApproxPlan* bplan = nullptr;  // bf16 tier
  const I8Plan* iplan = nullptr;      // int8 tier
  const float* qscale = nullptr;
  const float2* qerr = nullptr;
  const float* tau_fix = nullptr;
  const std::function<void(float*, int)>* pilot_xchg = nullptr;
  int k = 0;
  float* cand_s = nullptr;
  uint32_t* cand_r = nullptr;
  int32_t* cand_n = nullptr;
  float* cand_m = nullptr;
};

__global__ void k_gkey_to_f32(const uint32_t* __restrict__ gk, int n, float* __restrict__ f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = gk[i] ? sm100::key_float(gk[i]) : -INFINITY;
}
__global__ void k_f32_to_gkey(const float* __restrict__ f, int n, uint32_t* __restrict__ gk) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) gk[i] = f[i] > -INFINITY ? sm100::okey(f[i]) : 0u;
}

__global__ void k_fill_ninf(float* __restrict__ f, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = -INFINITY;
}

void run_shortlist(lc_ctx* ctx, const ShortlistRun& R) {
  using namespace sm100;
  const int nq = R.nq, kp = R.kp, bn = R.bn;
  const int64_t workers = R.pair ? ctx->sm_count / 2 : ctx->sm_count;  // persistent CTAs / CTA pairs
  // work units over `tiles` row tiles: (splits, tiles per split)
  auto split_rows = [&](int64_t tiles, int64_t& splits, int64_t& tiles_per_split) {
    // ~8 units per persistent worker (round 1, bf16 tier: 16 -- 74 splits moved
    // 2.74 GB of DRAM per 1M x 768 x 4096 launch against 3.63 GB with 37; the
    // int8 tier with its pilot-seeded thresholds prefers longer units, r02cv:
    // 1M 2.70 -> 2.68 ms, 250k 1.27 -> 1.15 ms, 125k 0.87 -> 0.84 ms per step)
    static const int upw = getenv("FC_SHORTLIST_UPW") ? std::max(1, atoi(getenv("FC_SHORTLIST_UPW"))) : 8;
    splits = std::max<int64_t>(1, (workers * upw + R.n_qtiles - 1) / R.n_qtiles);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, tiles / 16));
    // keep one query's partial lists within the merge's shared memory (few queries)
    splits = std::min<int64_t>(splits, std::max<int64_t>(workers, (200 * 1024) / ((int64_t)kp * 8 * (R.pair ? 2 : 1))));
    // packed candidates carry the row offset in 16 bits
    splits = std::max<int64_t>(splits, (tiles * bn + 65535) / 65536);
    tiles_per_split = std::min<int64_t>((tiles + splits - 1) / splits, 65536 / bn);
    splits = (tiles + tiles_per_split - 1) / tiles_per_split;
  };
  const int64_t total_tiles = (R.n_rows + bn - 1) / bn;
  int64_t splits = 0, tiles_per_split = 0;
  split_rows(total_tiles, splits, tiles_per_split);
  Params prm;
  prm.pilot = 0;
  prm.tile_stride = 1;
  prm.n_rows_phys = R.n_rows;
  prm.tau_fix = R.tau_fix;
  prm.Qb = reinterpret_cast<const __nv_bfloat16*>(R.Qconv);
  prm.nq = nq;
  prm.n_qtiles = R.n_qtiles;
  prm.dim = R.dim;
  prm.n_rows = R.n_rows;
  prm.rows_per_split = (int)(tiles_per_split * bn);
  prm.n_splits = (int)splits;
  prm.n_units = (int)(splits * R.n_qtiles);
  prm.kp = kp;
  prm.kh = R.i8 ? R.k : kp;
  prm.tscale = R.i8 ? R.iplan->tscale : nullptr;
  prm.tres = R.i8 ? R.iplan->tres : nullptr;
  prm.qscale = R.qscale;
  prm.qerr = R.qerr;
  prm.r_typ = R.i8 ? R.iplan->r_typ : 0.f;
  prm.slack = 0.003f;
  if (const char* e = getenv("FC_LOOKUP_I8_SLACK")) prm.slack = (float)atof(e);
  {
    const char* dbg = getenv("FC_SHORTLIST_DEBUG");
    prm.debug = dbg ? atoi(dbg) : 0;
  }
  // candidate lists per query: one per row range (single-CTA kernel) or one
  // per row range and epilogue column half (pair kernel)
  const int rshift = R.pair ? 1 : 0;
  const int64_t lists = splits << rshift;
  DevBuf pk((size_t)nq * lists * kp * sizeof(uint32_t), ctx->stream);
  DevBuf pn((size_t)nq * lists * sizeof(int32_t), ctx->stream);
  DevBuf pd(R.i8 ? (size_t)nq * lists * sizeof(float) : 16, ctx->stream);
  DevBuf gk((size_t)R.nq_pad * sizeof(uint32_t), ctx->stream);
  FC_CUDA(cudaMemsetAsync(gk.p, 0, gk.bytes, ctx->stream));
  DevBuf st(96, ctx->stream);  // u32 [0,4): counters; u64 [2,6): epilogue cycle spans; u64 [6,9): MMA waits
  FC_CUDA(cudaMemsetAsync(st.p, 0, 96, ctx->stream));
  DevBuf hist(R.pair ? (size_t)R.nq_pad * HSTRIDE * sizeof(uint32_t) : 16, ctx->stream);
  if (R.pair) FC_CUDA(cudaMemsetAsync(hist.p, 0, hist.bytes, ctx->stream));
  prm.hist = hist.as<uint32_t>();
  {
    const char* e = getenv("FC_SHORTLIST_REFRESH");
    // int8: the pilot seeds the threshold, so the histogram refresh (~8k cycles of
    // dependent L2 round trips per warp) runs every 64 tiles (r02x: 16 -> 2.25 ms,
    // 32 -> 2.14, 64 -> 2.09 per 4096 x 1M launch); tables large enough for the
    // pilot (>= 256 tiles) refresh every 512 (r02cd: 64 -> 2.156 ms, 256 -> 2.12,
    // 512 -> 2.11 once the pilot's epilogue was fixed)
    const int64_t tiles = (R.n_rows + PN - 1) / PN;
    const bool pilot = tiles >= 256 && !R.tau_fix && !(getenv("FC_LOOKUP_I8_PILOT") && atoi(getenv("FC_LOOKUP_I8_PILOT")) == 0);
    prm.refresh_mask = (e ? atoi(e) : (R.i8 ? (pilot ? 512 : 64) : 16)) - 1;
  }
  prm.stats = st.as<uint32_t>();
  prm.gkey = gk.as<uint32_t>();
  prm.part_k = pk.as<uint32_t>();
  prm.part_n = pn.as<int32_t>();
  prm.part_d = R.i8 ? pd.as<float>() : nullptr;
  DevBuf qb(R.i8 ? (size_t)nq * QCAP * sizeof(uint64_t) : 16, ctx->stream);
  DevBuf qc(R.i8 ? (size_t)nq * 2 * sizeof(uint32_t) : 16, ctx->stream);
  prm.qbuf = qb.as<uint64_t>();
  prm.qcnt = qc.as<uint32_t>();
  prm.qdrop = qc.as<uint32_t>() + nq;
  prm.qcap = QCAP;
  if (R.i8) FC_CUDA(cudaMemsetAsync(qc.p, 0, qc.bytes, ctx->stream));
  if (R.i8) {
    // smem-resident query K boxes beyond the first I8_KT: [128 queries][128 B] s8 boxes
    alignas(64) CUtensorMap unused;
    {
      cuuint64_t gdim[2] = {(cuuint64_t)R.dim, (cuuint64_t)R.nq_pad};
      cuuint64_t gstride[1] = {(cuuint64_t)R.dim};
      cuuint32_t box[2] = {128, (cuuint32_t)BM};
      cuuint32_t estride[2] = {1, 1};
      CUresult r = encode_fn()(&unused, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(R.Qconv), gdim, gstride, box,
                               estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) raise(LC_ERR_CUDA, "cuTensorMapEncodeTiled (s8 queries) failed: " + std::to_string((int)r));
    }
    // pilot over every 16th row tile (tables of >= 256 tiles): per-query max U
    // into gkey, the main pass's starting threshold
    static const int PILOT_STRIDE =
        getenv("FC_LOOKUP_I8_PILOT_STRIDE") ? std::max(1, atoi(getenv("FC_LOOKUP_I8_PILOT_STRIDE"))) : 16;
    static const bool no_pilot = getenv("FC_LOOKUP_I8_PILOT") && atoi(getenv("FC_LOOKUP_I8_PILOT")) == 0;
    if (!no_pilot && !R.tau_fix && total_tiles >= 256) {
      Params pp = prm;
      pp.pilot = 1;
      pp.tile_stride = PILOT_STRIDE;
      const int64_t ptiles = (total_tiles + PILOT_STRIDE - 1) / PILOT_STRIDE;
      // ~2 long units per CTA pair (short units pay the query load into TMEM
      // and the per-thread best-R warm-up each time)
      int64_t ps = std::max<int64_t>(1, std::min<int64_t>(ptiles / 16, (2 * workers + R.n_qtiles / 2) / R.n_qtiles));
      int64_t ptps = (ptiles + ps - 1) / ps;
      ps = (ptiles + ptps - 1) / ptps;
      pp.n_rows = ptiles * bn;
      pp.rows_per_split = (int)(ptps * bn);
      pp.n_splits = (int)ps;
      pp.n_units = (int)(ps * R.n_qtiles);
      DevBuf po((size_t)nq * 2 * ps * PILOT_R * sizeof(float), ctx->stream);
      pp.pilot_out = po.as<float>();
      ShortlistTimerName tn("shortlist_pilot");
      launch_pair<true>(ctx, R.iplan->tmap, unused, pp);
      k_pilot_kth<<<(unsigned)((nq + 7) / 8), 256, 0, ctx->stream>>>(po.as<float>(), (int)(2 * ps), nq, gk.as<uint32_t>());
      FC_LAUNCH_CHECK();
      count_launch(ctx, 2);
    }
    if (R.pilot_xchg) {
      // sharded: every rank filters with the max over the ranks of the
      // pilots' per-query keys (a G x larger sample; a rank without a pilot
      // contributes -inf and still receives the others')
      DevBuf pf((size_t)std::max(nq, 1) * sizeof(float), ctx->stream);
      k_gkey_to_f32<<<grid_for(std::max(nq, 1), 256), 256, 0, ctx->stream>>>(gk.as<uint32_t>(), nq, pf.as<float>());
      (*R.pilot_xchg)(pf.as<float>(), nq);
      k_f32_to_gkey<<<grid_for(std::max(nq, 1), 256), 256, 0, ctx->stream>>>(pf.as<float>(), nq, gk.as<uint32_t>());
      FC_LAUNCH_CHECK();
      count_launch(ctx, 2);
    }
    launch_pair<true>(ctx, R.iplan->tmap, unused, prm);
  } else if (R.pair) {
    alignas(64) CUtensorMap tmQ;
    encode_2d(&tmQ, reinterpret_cast<const __nv_bfloat16*>(R.Qconv), R.nq_pad, R.dim, BM);  // smem-resident query boxes [128 q][64]
    launch_pair<false>(ctx, R.bplan->tmap2, tmQ, prm);
  } else if (bn == 64) {
    launch_single<64>(ctx, *R.bplan, prm);
  } else {
    launch_single<128>(ctx, *R.bplan, prm);
  }
  if (prm.debug & 16) {
    uint32_t h[24];
    FC_CUDA(cudaMemcpyAsync(h, st.p, 96, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    unsigned long long cy[4], mc[3];
    memcpy(cy, h + 4, sizeof cy);
    memcpy(mc, h + 12, sizeof mc);
    const double wt = (double)std::max(1u, h[2]);  // warp-tiles
    fprintf(stderr, "shortlist%s stats: warp-tiles %u slow-chunks %u (%.3f/tile) compactions %u (%.4f/tile) nstage %d bps %d cap %d splits %d"
            " | cycles per warp-tile: acc-wait %.0f hist %.0f compact %.0f append %.0f"
            " | MMA cycles per tile: acc-free wait %.0f data wait %.0f A wait %.0f\n",
            R.i8 ? "[i8]" : "", h[2], h[0], h[0] / wt, h[1], h[1] / wt, prm.nstage, prm.bps, prm.cap, prm.n_splits,
            cy[0] / wt, cy[1] / wt, cy[2] / wt, cy[3] / wt, mc[0] * 16.0 / wt, mc[1] * 16.0 / wt, mc[2] * 16.0 / wt);
  }
  const size_t per_warp = (size_t)lists * kp * 2 * sizeof(uint32_t);  // keys + slots
  const float* pdp = R.i8 ? pd.as<float>() : nullptr;
  KTimer kmt(ctx, "shortlist_merge");
  if (R.i8) {
    k_i8_merge<<<(nq + QM_W - 1) / QM_W, QM_W * 32, 0, ctx->stream>>>(prm.qbuf, prm.qcnt, prm.qdrop, nq, R.kout,
                                                                      R.cand_s, R.cand_r, R.cand_n, R.cand_m);
    FC_LAUNCH_CHECK();
    count_launch(ctx, 2);
    return;
  }
  if (nq < ctx->sm_count && per_warp <= 200 * 1024) {
    static std::atomic<uint64_t> attr_set{0};  // per-device bit: the attribute is per device
    if (!(attr_set.load() >> (ctx->device & 63) & 1)) {
      FC_CUDA(cudaFuncSetAttribute(k_shortlist_merge_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr_set.fetch_or(1ull << (ctx->device & 63));
    }
    k_shortlist_merge_cta<<<nq, MC_T, per_warp, ctx->stream>>>(pk.as<uint32_t>(), pn.as<int32_t>(), (int)lists, kp,
                                                               prm.rows_per_split, rshift, R.kout, R.cand_s, R.cand_r,
                                                               R.cand_n, pdp, R.cand_m);
    FC_LAUNCH_CHECK();
    count_launch(ctx, 3);
    return;
  }
  // spill space for queries with more than MG_CAP filled slots (rare: the
  // acceptance threshold keeps ~1/10 of the slots)
  DevBuf gkeys(per_warp > (size_t)MG_CAP * 8 ? (size_t)nq * per_warp : 16, ctx->stream);
  const size_t msmem = (size_t)MG_W * 2 * MG_CAP * sizeof(uint32_t);
  static std::atomic<uint64_t> attr_set2{0};
  if (!(attr_set2.load() >> (ctx->device & 63) & 1)) {
    FC_CUDA(cudaFuncSetAttribute(k_shortlist_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem));
    attr_set2.fetch_or(1ull << (ctx->device & 63));
  }
  k_shortlist_merge<<<(nq + MG_W - 1) / MG_W, MG_W * 32, msmem, ctx->stream>>>(
      pk.as<uint32_t>(), pn.as<int32_t>(), (int)lists, kp, prm.rows_per_split, rshift, nq, R.kout, R.cand_s, R.cand_r,
      R.cand_n, gkeys.as<uint32_t>(), pdp, R.cand_m);
  FC_LAUNCH_CHECK();
  count_launch(ctx, 3);
}
}  // namespace

void dummy_pilot_exchange(lc_ctx* ctx, const std::function<void(float*, int)>& x, int nq) {
  DevBuf pf((size_t)std::max(nq, 1) * sizeof(float), ctx->stream);
  k_fill_ninf<<<grid_for(std::max(nq, 1), 256), 256, 0, ctx->stream>>>(pf.as<float>(), nq);
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  x(pf.as<float>(), nq);
}

void approx_shortlist(lc_ctx* ctx, const ApproxPlan& plan, const float* Qdev, int nq, int kp, float* cand_s,
                      uint32_t* cand_r, int32_t* cand_n) {
  using namespace sm100;
  const int dim = plan.dim;
  // a CTA pair's 256-query tile is mostly padding for a handful of queries
  // (the tier-2 re-shortlist): the single-CTA kernel does half the MMA work
  const bool pair = use_pair(dim) && nq > BM;
  const int qt = pair ? 2 * BM : BM;  // queries per work unit
  ShortlistRun R;
  R.pair = pair;
  R.dim = dim;
  R.nq = nq;
  R.n_qtiles = (nq + qt - 1) / qt;
  R.nq_pad = R.n_qtiles * qt;
  R.bn = pair ? PN : plan.bn;
  R.n_rows = plan.n_rows;
  R.kp = R.kout = kp;
  R.bplan = &plan;
  DevBuf qb((size_t)R.nq_pad * dim * sizeof(__nv_bfloat16), ctx->stream);
  k_q_to_bf16<<<grid_for((int64_t)R.nq_pad * dim, 256), 256, 0, ctx->stream>>>(Qdev, nq, dim, qb.as<__nv_bfloat16>(), R.nq_pad);
  FC_LAUNCH_CHECK();
  R.Qconv = qb.p;
  R.cand_s = cand_s;
  R.cand_r = cand_r;
  R.cand_n = cand_n;
  run_shortlist(ctx, R);
}

// ---------------------------------------------------------------------------
// int8 tier
// ---------------------------------------------------------------------------
namespace sm100 {
// Per query (one warp): s_q = max|q| / 127 (1 for an all-zero row), qq =
// rint(q / s_q) clamped to [-127, 127], and the exact fp64 norms of dq = q -
// s_q qq and qhat = s_q qq (each product s_q * qq is exact in fp64), rounded
// up by 2^-40 (far above the fp64 summation error of <= 1024 terms).
__global__ void k_q_to_i8(const float* __restrict__ Q, int nq, int dim, int nq_pad, int8_t* __restrict__ Qi,
                          float* __restrict__ qscale, float2* __restrict__ qerr) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nq_pad) return;
  int8_t* dst = Qi + (size_t)w * dim;
  if (w >= nq) {
    for (int d = lane; d < dim; d += 32) dst[d] = 0;
    if (lane == 0) {
      qscale[w] = 1.f;
      qerr[w] = make_float2(0.f, 0.f);
    }
    return;
  }
  const float* x = Q + (size_t)w * dim;
  float amax = 0.f;
  for (int d = lane; d < dim; d += 32) amax = fmaxf(amax, fabsf(x[d]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  const float sc = amax > 0.f && amax < INFINITY ? amax / 127.f : 1.f;
  double e2 = 0.0, h2 = 0.0;
  for (int d = lane; d < dim; d += 32) {
    float r = rintf(__fdiv_rn(x[d], sc));
    r = fminf(127.f, fmaxf(-127.f, r));
    dst[d] = (int8_t)(int)r;
    const double qh = (double)sc * (double)r;
    const double e = (double)x[d] - qh;
    e2 = fma(e, e, e2);
    h2 = fma(qh, qh, h2);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    e2 += __shfl_xor_sync(0xffffffffu, e2, off);
    h2 += __shfl_xor_sync(0xffffffffu, h2, off);
  }
  if (lane == 0) {
    qscale[w] = sc;
    // (||dq|| X, ||qhat||) with X = 1 + 1e-6 >= ||x|| for stored rows (from_unit),
    // rounded up to fp32; a non-finite query gives non-finite bounds (rejected later)
    qerr[w] = make_float2(__double2float_ru(sqrt(e2) * (1.0 + 1e-6) * (1.0 + 0x1p-40)),
                          __double2float_ru(sqrt(h2) * (1.0 + 0x1p-40)));
  }
}

// One CTA per 128-row tile: s_t = max|x| / 127 over the tile's live rows,
// xq = rint(x / s_t) clamped, the row residual norms ||x - s_t xq|| (exact
// fp64 terms) max-reduced into *res_bits. Rows >= n_rows become zero.
constexpr int QT_T = 256;
__global__ void __launch_bounds__(QT_T) k_quant_tiles(const float* __restrict__ rows, int64_t n_rows, int dim, int64_t t0,
                                                      int8_t* __restrict__ rows8, float* __restrict__ tscale,
                                                      float* __restrict__ tres, unsigned long long* __restrict__ res_bits) {
  const int64_t tile = t0 + blockIdx.x;
  const int64_t r0 = tile * 128;
  const int64_t r1 = min(n_rows, r0 + 128);
  __shared__ float red[QT_T / 32];
  float amax = 0.f;
  const int64_t live = (r1 - r0) * dim;
  const float* base = rows + r0 * dim;
  for (int64_t i = threadIdx.x; i < live; i += QT_T) amax = fmaxf(amax, fabsf(base[i]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = 0.f;
  for (int i = 0; i < QT_T / 32; ++i) amax = fmaxf(amax, red[i]);
  const float sc = amax > 0.f && amax < INFINITY ? amax / 127.f : 1.f;
  if (threadIdx.x == 0) tscale[tile] = sc;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double worst = 0.0;
  for (int64_t r = r0 + w; r < r0 + 128; r += QT_T / 32) {
    int8_t* dst = rows8 + r * dim;
    if (r >= n_rows) {
      for (int d = lane; d < dim; d += 32) dst[d] = 0;
      continue;
    }
    const float* x = rows + r * dim;
    double e2 = 0.0;
    for (int d = lane; d < dim; d += 32) {
      float q = rintf(__fdiv_rn(x[d], sc));
      q = fminf(127.f, fmaxf(-127.f, q));
      dst[d] = (int8_t)(int)q;
      const double e = (double)x[d] - (double)sc * (double)q;
      e2 = fma(e, e, e2);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) e2 += __shfl_xor_sync(0xffffffffu, e2, off);
    worst = fmax(worst, sqrt(e2) * (1.0 + 0x1p-40));
  }
  __shared__ double wred[QT_T / 32];
  if (lane == 0) wred[w] = worst;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < QT_T / 32; ++i) m = fmax(m, wred[i]);
    tres[tile] = __double2float_ru(m);
    if (m > 0) atomicMax(res_bits, (unsigned long long)__double_as_longlong(m));
  }
}
}  // namespace sm100

void i8_quantize_tiles(lc_ctx* ctx, const float* rows, int64_t n_rows, int dim, int64_t t0, int64_t t1, int8_t* rows8,
                       float* tscale, float* tres, unsigned long long* res_bits) {
  if (t1 <= t0) return;
  sm100::k_quant_tiles<<<(unsigned)(t1 - t0), sm100::QT_T, 0, ctx->stream>>>(rows, n_rows, dim, t0, rows8, tscale, tres,
                                                                             res_bits);
  FC_LAUNCH_CHECK();
  count_launch(ctx);
}

void i8_plan(I8Plan& p, const int8_t* rows, const float* tscale, const float* tres, int64_t n_rows, int dim,
             float r_typ) {
  p.n_rows = n_rows;
  p.dim = dim;
  p.rows = rows;
  p.tscale = tscale;
  p.tres = tres;
  p.r_typ = r_typ;
  cuuint64_t gdim[2] = {(cuuint64_t)dim, (cuuint64_t)n_rows};
  cuuint64_t gstride[1] = {(cuuint64_t)dim};
  cuuint32_t box[2] = {128, (cuuint32_t)sm100::PHB};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = encode_fn()(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(rows), gdim, gstride, box,
                           estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(LC_ERR_CUDA, "cuTensorMapEncodeTiled (s8) failed: " + std::to_string((int)r));
  p.valid = true;
}

void i8_shortlist(lc_ctx* ctx, const I8Plan& plan, const float* Qdev, int nq, int k, int kp_unit, int kout, float* cand_s,
                  uint32_t* cand_r, int32_t* cand_n, float* cand_m, const float* tau_fix,
                  const std::function<void(float*, int)>* pilot_xchg) {
  using namespace sm100;
  FC_REQUIRE(plan.dim % 128 == 0 && plan.dim <= 1024, "int8 lookup tier: dim must be a multiple of 128, <= 1024");
  ShortlistRun R;
  R.i8 = true;
  R.pair = true;
  R.dim = plan.dim;
  R.nq = nq;
  R.n_qtiles = (nq + 2 * BM - 1) / (2 * BM);
  R.nq_pad = R.n_qtiles * 2 * BM;
  R.bn = PN;
  R.n_rows = plan.n_rows;
  R.kp = kp_unit;
  R.kout = kout;
  R.iplan = &plan;
  DevBuf qi((size_t)R.nq_pad * plan.dim, ctx->stream);
  DevBuf qs((size_t)R.nq_pad * sizeof(float), ctx->stream);
  DevBuf qe((size_t)R.nq_pad * sizeof(float2), ctx->stream);
  k_q_to_i8<<<(unsigned)((R.nq_pad + 7) / 8), 256, 0, ctx->stream>>>(Qdev, nq, plan.dim, R.nq_pad, qi.as<int8_t>(),
                                                                     qs.as<float>(), qe.as<float2>());
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  R.Qconv = qi.p;
  R.qscale = qs.as<float>();
  R.qerr = qe.as<float2>();
  R.k = k;
  R.tau_fix = tau_fix;
  R.pilot_xchg = tau_fix ? nullptr : pilot_xchg;
  R.cand_s = cand_s;
  R.cand_r = cand_r;
  R.cand_n = cand_n;
  R.cand_m = cand_m;
  run_shortlist(ctx, R);
}

}  // namespace fc
