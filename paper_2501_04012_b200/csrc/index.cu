// index.cu — SimilarityIndex (vindex.hpp:23-62) on the GPU.
//
// Layout in HBM (per table: whole / object / background):
//   rows  fp32 [cap][dim]   master copy, bit-identical to the reference rows
//                           (the exact fp64 scores are computed from these)
//   rowsb bf16 [cap][dim]   tensor-core operand for the candidate GEMM
//   ids   u64  [cap]        prompt id of each slot
// Slots are dense [0, n); remove moves the last slot into the hole (O(dim)
// instead of the reference's O(n*dim) erase, vindex.cpp:76-87). Row order is
// irrelevant to results because every top-k orders by (score desc, id asc).
//
// Query path (lc_index_query_topk):
//   size < 8192 or mode 1: exact scan (k_scan_partial + k_scan_merge) — the
//     reference's sequential fp64 dot (vindex.cpp:66-67) for every row.
//   otherwise: tcgen05 bf16 GEMM with a fused per-query top-K' shortlist
//     (lookup_sm100.cu) -> shortlist merge -> exact fp64 rescore of the
//     K' candidates (k_rescore) -> certification: every row outside the
//     shortlist has bf16 score <= m (the K'-th shortlisted bf16 score), so its
//     exact score is <= m + eps; if m + eps < T_k (the k-th exact score) the
//     answer is provably the exact top-k. Queries that fail the test are
//     re-run through the exact scan. Results are therefore always identical
//     to the reference's.
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <exception>
#include <cmath>
#include <cstring>
#include <mutex>
#include <shared_mutex>
#include <unordered_map>

#include "common.cuh"
#include "lookup.cuh"
#include "topk.cuh"

using namespace fc;

struct lc_index {
  lc_ctx* ctx = nullptr;
  int dim = 0;
  int64_t n = 0, cap = 0;
  float* rows[3] = {nullptr, nullptr, nullptr};
  __nv_bfloat16* rowsb[3] = {nullptr, nullptr, nullptr};
  uint64_t* ids_dev = nullptr;
  std::vector<uint64_t> ids;
  std::unordered_map<uint64_t, int64_t> slot;
  int mode = 0;
  int kprime = 32;
  // Certified |bf16 score - exact| bound, per query in k_rescore from
  // ||q||, ||q - bf16(q)|| and dres = max over stored rows of ||x - bf16(x)||
  // (lookup.cuh); eps_floor (lc_index_set_lookup) can only widen it.
  double dres[3] = {0.0, 0.0, 0.0};
  double eps_floor = 0.0;
  // int8 tier-1 copy (dim % 128 == 0): rows quantized per 128-slot tile
  // (lookup.cuh); dres8 = max residual norm of the quantized rows (kept as a
  // running max over re-quantizations, so it stays a bound).
  bool i8 = false;
  int8_t* rows8[3] = {nullptr, nullptr, nullptr};
  float* tscale[3] = {nullptr, nullptr, nullptr};
  float* tres[3] = {nullptr, nullptr, nullptr};  // per-tile max residual norm
  double dres8[3] = {0.0, 0.0, 0.0};
  int i8_kout = 256;   // merged candidates per query (FC_LOOKUP_I8_KOUT)
  int i8_kunit = 32;   // per unit list
  I8Plan iplan[3];
  lc_lookup_stats stats{};
  ApproxPlan plan[3];
  mutable std::shared_mutex mu;  // readers: queries; writer: insert/remove (vindex.hpp:61)
  // Concurrent readers (shared lock on mu) still touch two pieces of shared
  // state: the per-table tensor-map plans (rebuilt lazily after a mutation)
  // and the counters; each has its own small lock.
  std::mutex plan_mu, stats_mu;
};

namespace fc {

// Non-finite query elements (reference queries are Embeddings, which reject
// them: core.cpp:11-15, 50-53). One thread per query row.
__global__ void k_check_finite_rows(const float* __restrict__ v, int64_t n, int dim, int* __restrict__ bad) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float* x = v + r * dim;
  bool ok = true;
  for (int i = 0; i < dim; ++i) ok &= isfinite(x[i]);
  if (!ok) atomicExch(bad, 1);
}

// from_unit rule (core.cpp:61-69) on device rows: finite and
// |sqrt(sum v^2) - 1| <= 1e-6 with a sequential fp64 sum.
// Also the row's bf16 rounding residual norm ||x - bf16_rn(x)|| (rounded
// up), max-reduced into *res_bits (non-negative doubles order as u64).
__global__ void k_check_unit(const float* __restrict__ v, int64_t n, int dim, int* __restrict__ bad,
                             unsigned long long* __restrict__ res_bits) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float* x = v + r * dim;
  double sq = 0.0, rs = 0.0;
  bool ok = true;
  for (int i = 0; i < dim; ++i) {
    ok &= isfinite(x[i]);
    const double t = x[i];
    sq = fma(t, t, sq);
    const double e = t - (double)__bfloat162float(__float2bfloat16_rn(x[i]));
    rs = fma(e, e, rs);
  }
  if (!ok || fabs(sqrt(sq) - 1.0) > 1e-6) atomicExch(bad, 1);
  else if (res_bits) atomicMax(res_bits, (unsigned long long)__double_as_longlong(sqrt(rs) * (1.0 + 0x1p-40)));
}

__global__ void k_to_bf16(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t count) {
  int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4;
  if (i + 3 < count) {
    float4 v = *reinterpret_cast<const float4*>(src + i);
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    *reinterpret_cast<__nv_bfloat162*>(dst + i) = a;
    *reinterpret_cast<__nv_bfloat162*>(dst + i + 2) = b;
  } else {
    for (; i < count; ++i) dst[i] = __float2bfloat16_rn(src[i]);
  }
}

// ---------------------------------------------------------------------------
// Exact scan: one thread per table row, QB queries per block (in smem); each
// (query,row) score is the reference's sequential fp64 dot, d = 0..dim-1.
// Per block and query the top-k of its 128 rows goes to a partial list.
// ---------------------------------------------------------------------------
constexpr int SCAN_T = 128;
constexpr int SCAN_QB = 8;

__global__ void __launch_bounds__(SCAN_T) k_scan_partial(const float* __restrict__ Q, const int32_t* __restrict__ qlist,
                                                         int nq, const float* __restrict__ rows,
                                                         const uint64_t* __restrict__ ids, int64_t n_rows, int dim,
                                                         int k, Cand* __restrict__ partial, int32_t* __restrict__ pcount) {
  extern __shared__ float s_q[];  // [SCAN_QB][dim]
  __shared__ Cand s_c[SCAN_T / 32];
  __shared__ int s_o[SCAN_T / 32];
  __shared__ Cand s_out[64];
  const int q0 = blockIdx.y * SCAN_QB;
  const int qn = min(SCAN_QB, nq - q0);
  for (int i = threadIdx.x; i < qn * dim; i += SCAN_T) {
    const int qq = i / dim, d = i - qq * dim;
    const int qi = qlist ? qlist[q0 + qq] : q0 + qq;
    s_q[qq * dim + d] = Q[(int64_t)qi * dim + d];
  }
  __syncthreads();
  const int64_t r = blockIdx.x * (int64_t)SCAN_T + threadIdx.x;
  double acc[SCAN_QB];
#pragma unroll
  for (int j = 0; j < SCAN_QB; ++j) acc[j] = 0.0;
  if (r < n_rows) {
    const float* x = rows + r * dim;
    if ((dim & 3) == 0) {
      for (int d = 0; d < dim; d += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(x + d));
#pragma unroll
        for (int j = 0; j < SCAN_QB; ++j) {
          if (j < qn) {
            const float* qq = s_q + j * dim + d;
            acc[j] = fma((double)qq[0], (double)v.x, acc[j]);
            acc[j] = fma((double)qq[1], (double)v.y, acc[j]);
            acc[j] = fma((double)qq[2], (double)v.z, acc[j]);
            acc[j] = fma((double)qq[3], (double)v.w, acc[j]);
          }
        }
      }
    } else {
      for (int d = 0; d < dim; ++d) {
        const double v = x[d];
#pragma unroll
        for (int j = 0; j < SCAN_QB; ++j)
          if (j < qn) acc[j] = fma((double)s_q[j * dim + d], v, acc[j]);
      }
    }
  }
  const uint64_t myid = r < n_rows ? ids[r] : 0;
  for (int j = 0; j < qn; ++j) {
    Cand L[1];
    int ln = 0;
    if (r < n_rows) {
      L[0].s = acc[j];
      L[0].id = myid;
      L[0].slot = r;
      ln = 1;
    }
    const int got = block_merge_lists<1>(L, ln, k, s_out, s_c, s_o);
    const int64_t base = ((int64_t)(q0 + j) * gridDim.x + blockIdx.x);
    for (int t = threadIdx.x; t < got; t += SCAN_T) partial[base * k + t] = s_out[t];
    if (threadIdx.x == 0) pcount[base] = got;
    __syncthreads();
  }
}

template <int KMAX>
__global__ void __launch_bounds__(256) k_scan_merge(const Cand* __restrict__ partial, const int32_t* __restrict__ pcount,
                                                    int nblk, int k, const int32_t* __restrict__ qlist,
                                                    uint64_t* __restrict__ out_ids, double* __restrict__ out_sc,
                                                    int32_t* __restrict__ out_cnt) {
  __shared__ Cand s_c[8];
  __shared__ int s_o[8];
  __shared__ Cand s_out[KMAX];
  const int q = blockIdx.x;
  Cand L[KMAX];
  int ln = 0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    const int64_t base = (int64_t)q * nblk + b;
    const int c = pcount[base];
    for (int t = 0; t < c; ++t) local_insert<KMAX>(L, ln, k, partial[base * k + t]);
  }
  const int got = block_merge_lists<KMAX>(L, ln, k, s_out, s_c, s_o);
  const int qo = qlist ? qlist[q] : q;
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    out_ids[(int64_t)qo * k + t] = t < got ? s_out[t].id : 0;
    out_sc[(int64_t)qo * k + t] = t < got ? s_out[t].s : 0.0;
  }
  if (threadIdx.x == 0) out_cnt[qo] = got;
}

// Tier-2 helpers: gather the uncertified queries, scatter their results back.
__global__ void k_gather_queries(const float* __restrict__ Q, const int32_t* __restrict__ list, int n, int dim,
                                 float* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * dim) return;
  const int64_t r = i / dim, d = i - r * dim;
  out[i] = Q[(int64_t)list[r] * dim + d];
}
__global__ void k_scatter_topk(const uint64_t* __restrict__ ids, const double* __restrict__ sc,
                               const int32_t* __restrict__ cnt, const int32_t* __restrict__ list, int n, int k,
                               uint64_t* __restrict__ oid, double* __restrict__ osc, int32_t* __restrict__ ocnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * k) return;
  const int64_t r = i / k, t = i - r * k;
  const int64_t q = list[r];
  oid[q * k + t] = ids[i];
  osc[q * k + t] = sc[i];
  if (t == 0) ocnt[q] = cnt[r];
}
// Threshold tier input: for failed query i (original index list[i]) the k-th
// best EXACT score its last tier found (a lower bound of T_k: those are real
// rows) minus twice the reference-dot rounding margin, rounded down; -inf
// when fewer than k rows were found. One warp per query.
__global__ void k_tau_fix(const float* __restrict__ Q, const int32_t* __restrict__ list, int n, int dim,
                          const double* __restrict__ osc, const int32_t* __restrict__ ocnt, int k,
                          float* __restrict__ tau) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n) return;
  const int q = list[w];
  double qsq = 0.0;
  for (int d = lane; d < dim; d += 32) {
    const double v = Q[(int64_t)q * dim + d];
    qsq = fma(v, v, qsq);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) qsq += __shfl_xor_sync(0xffffffffu, qsq, off);
  if (lane == 0) {
    const double margin = 1e-12 * (1.0 + sqrt(qsq) * (1.0 + 0x1p-40));
    tau[w] = ocnt[q] >= k ? __double2float_rd(osc[(int64_t)q * k + k - 1] - 2.0 * margin) : -INFINITY;
  }
}

__global__ void k_map_list(const int32_t* __restrict__ sub, const int32_t* __restrict__ list, int n,
                           int32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = list[sub[i]];
}

// ---------------------------------------------------------------------------
// Exact rescore of the bf16 shortlist + certification (one warp per query).
// ---------------------------------------------------------------------------
constexpr int RS_WARPS = 8;

template <int PER_LANE>
__global__ void __launch_bounds__(RS_WARPS * 32)
    k_rescore(const float* __restrict__ Q, int nq, int dim, const float* __restrict__ rows,
              const uint64_t* __restrict__ ids, const float* __restrict__ cand_s, const uint32_t* __restrict__ cand_r,
              const int32_t* __restrict__ cand_n, int kp, int64_t n_rows, int k, double dres, double eps_floor,
              uint64_t* __restrict__ out_ids,
              double* __restrict__ out_sc, int32_t* __restrict__ out_cnt, int32_t* __restrict__ fail_list,
              int32_t* __restrict__ fail_n, unsigned long long* __restrict__ max_err_bits,
              int32_t* __restrict__ bad_query) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * RS_WARPS + warp;
  if (q >= nq) return;
  const float* qv = Q + (int64_t)q * dim;
  extern __shared__ float s_rq[];  // [RS_WARPS][dim] this warp's query
  float* sq = s_rq + (size_t)warp * dim;
  double qsq = 0.0, dsq = 0.0;
  bool qfin = true;
  for (int d = lane; d < dim; d += 32) {
    const float v = qv[d];
    sq[d] = v;
    qfin &= isfinite(v);
    qsq = fma((double)v, (double)v, qsq);
    const double e = (double)v - (double)__bfloat162float(__float2bfloat16_rn(v));  // k_q_to_bf16 rounding
    dsq = fma(e, e, dsq);
  }
  __syncwarp();
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    qsq += __shfl_xor_sync(0xffffffffu, qsq, off);
    dsq += __shfl_xor_sync(0xffffffffu, dsq, off);
  }
  qfin = __all_sync(0xffffffffu, qfin);
  if (!qfin && lane == 0) atomicExch(bad_query, 1);
  // Certified bound of |fp32 tensor-core score - exact dot| for this query
  // against any stored row x (lookup.cuh): with q = bq + dq, x = bx + dx
  // (bf16 round-to-nearest parts), q.x - bq.bx = q.dx + dq.x - dq.dx, so
  //   |.| <= ||q|| dres + ||dq|| (||x|| + dres) + fp32 accumulation,
  // ||x|| <= 1 + 1e-6 (from_unit rule on insert), dres = the max residual
  // norm of the stored rows, and the accumulation of <= 1024 exact products
  // adds <= 1024 * 2^-23 * ||bq|| ||bx||. The norms are fp64 warp sums
  // (relative error far below the 2^-40 margin). Non-unit queries are
  // covered by the same formula. A query so large that fp16-stored scores
  // could overflow, or a non-finite one, is never certified.
  const double qn = sqrt(qsq) * (1.0 + 0x1p-40), dqn = sqrt(dsq) * (1.0 + 0x1p-40);
  // (shortlist scores are stored as fp16: |score| <= ||q|| must stay far below 65504)
  const bool q_uncertifiable = !qfin || !(qn < 16384.0);
  const double xn = 1.0 + 1e-6;
  double eps = qn * dres + dqn * (xn + dres) + 0x1p-13 * (qn + dqn) * (xn + dres);
  eps = fmax(eps * (1.0 + 0x1p-20), eps_floor * fmax(1.0, qn));
  const int cn = cand_n[q];
  // Only candidates whose bf16 score is within 2*eps of the k-th best bf16
  // score can reach the exact top-k: the k candidates ranked first by bf16
  // all have exact >= a_k - eps, and a skipped row has exact <= a + eps <
  // a_k - eps. Skipping the rest avoids most of the random 3 KB row gathers.
  float ak = -INFINITY;
  if (cn > k) {
    float mine_a[PER_LANE];
#pragma unroll
    for (int t = 0; t < PER_LANE; ++t) {
      const int c = lane + 32 * t;
      mine_a[t] = c < cn ? cand_s[(int64_t)q * kp + c] : -INFINITY;
    }
    // k-th largest by rank counting over the warp's candidates
#pragma unroll
    for (int t = 0; t < PER_LANE; ++t) {
      const int c = lane + 32 * t;
      int rank = 0;
      for (int u = 0; u < PER_LANE; ++u)
        for (int j = 0; j < 32; ++j) {
          const float o = __shfl_sync(0xffffffffu, mine_a[u], j);
          const int oc = j + 32 * u;
          rank += (o > mine_a[t]) | ((o == mine_a[t]) & (oc < c));
        }
      const bool is_k = c < cn && rank == k - 1;
      const unsigned bal = __ballot_sync(0xffffffffu, is_k);
      if (bal) ak = __shfl_sync(0xffffffffu, mine_a[t], __ffs(bal) - 1);
    }
  }
  // shortlist scores are fp16 values rounded UP from the fp32 accumulator
  // (lookup_sm100.cu hkey_ru): a candidate's approx lies in [s - ulp, s], with
  // ulp <= |s| * 2^-10 + 2^-24, which widens the window by that much
  const float skip_below = ak - (float)(2.0 * eps) - fabsf(ak) * 0x1p-10f - 0x1p-20f;
  Cand mine[PER_LANE];
  int mn = 0;
  float min_approx = INFINITY;
  double local_err = 0.0;
#pragma unroll
  for (int t = 0; t < PER_LANE; ++t) {
    const int c = lane + 32 * t;
    if (c < cn) {
      const uint32_t r = cand_r[(int64_t)q * kp + c];
      const float a = cand_s[(int64_t)q * kp + c];
      min_approx = fminf(min_approx, a);
      if (a < skip_below) continue;
      const float* x = rows + (int64_t)r * dim;
      double acc = 0.0;
      if ((dim & 31) == 0) {
        // sequential fp64 in d order (vindex.cpp:67); the row streams as
        // float4 loads issued 32 elements (two 128 B lines) ahead -- the
        // gathers are latency-bound, so the depth in flight sets the speed
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const float4* q4 = reinterpret_cast<const float4*>(sq);
        float4 nx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) nx[u] = __ldg(x4 + u);
        for (int d4 = 0; d4 < dim / 4; d4 += 8) {
          float4 cx[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) cx[u] = nx[u];
          if (d4 + 8 < dim / 4) {
#pragma unroll
            for (int u = 0; u < 8; ++u) nx[u] = __ldg(x4 + d4 + 8 + u);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 qq = q4[d4 + u];
            acc = fma((double)qq.x, (double)cx[u].x, acc);
            acc = fma((double)qq.y, (double)cx[u].y, acc);
            acc = fma((double)qq.z, (double)cx[u].z, acc);
            acc = fma((double)qq.w, (double)cx[u].w, acc);
          }
        }
      } else if ((dim & 15) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const float4* q4 = reinterpret_cast<const float4*>(sq);
        float4 nx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) nx[u] = __ldg(x4 + u);
        for (int d4 = 0; d4 < dim / 4; d4 += 4) {
          float4 cx[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) cx[u] = nx[u];
          if (d4 + 4 < dim / 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) nx[u] = __ldg(x4 + d4 + 4 + u);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 qq = q4[d4 + u];
            acc = fma((double)qq.x, (double)cx[u].x, acc);
            acc = fma((double)qq.y, (double)cx[u].y, acc);
            acc = fma((double)qq.z, (double)cx[u].z, acc);
            acc = fma((double)qq.w, (double)cx[u].w, acc);
          }
        }
      } else {
        for (int d = 0; d < dim; ++d) acc = fma((double)sq[d], (double)__ldg(x + d), acc);
      }
      local_err = fmax(local_err, fabs(acc - (double)a));
      Cand cc;
      cc.s = acc;
      cc.id = ids[r];
      cc.slot = r;
      local_insert<PER_LANE>(mine, mn, PER_LANE, cc);
    }
  }
  // warp-wide min of the shortlisted approx scores (the K'-th best approx)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    min_approx = fminf(min_approx, __shfl_xor_sync(0xffffffffu, min_approx, off));
    local_err = fmax(local_err, __shfl_xor_sync(0xffffffffu, local_err, off));
  }
  if (lane == 0 && local_err > 0) atomicMax(max_err_bits, (unsigned long long)__double_as_longlong(local_err));
  // k rounds of warp argmax over the per-lane sorted lists
  int ptr = 0, got = 0;
  double tk = 0.0;
  for (int rnd = 0; rnd < k; ++rnd) {
    Cand c;
    int owner;
    if (ptr < mn) {
      c = mine[ptr];
      owner = lane;
    } else {
      c.s = 0; c.id = 0; c.slot = -1;
      owner = -1;
    }
    warp_argbest(c, owner);
    if (owner < 0) break;
    if (lane == owner) ++ptr;
    if (lane == 0) {
      out_ids[(int64_t)q * k + rnd] = c.id;
      out_sc[(int64_t)q * k + rnd] = c.s;
    }
    tk = c.s;
    ++got;
  }
  if (lane == 0) {
    for (int j = got; j < k; ++j) {
      out_ids[(int64_t)q * k + j] = 0;
      out_sc[(int64_t)q * k + j] = 0.0;
    }
    out_cnt[q] = got;
    // Certification: rows outside the shortlist have approx <= min_approx.
    // A shortlist holding every row needs no margin; one shorter than
    // min(K', rows) can only come from a fault and is never trusted.
    bool ok;
    if (cn < (kp < n_rows ? kp : n_rows)) ok = false;
    else if (cn >= n_rows) ok = true;
    else ok = !q_uncertifiable && got >= k && (double)min_approx + eps < tk;
    if (!ok) fail_list[atomicAdd(fail_n, 1)] = q;
  }
}

// ---------------------------------------------------------------------------
// Exact rescore of the int8 shortlist + certification (one warp per query).
//
// The int8 tier hands over up to KI_MAX candidates per query with stored
// scores U (upper bounds of the exact dot) and cand_m[q] (every row outside
// the list has exact <= cand_m). Two passes over the list:
//  1. bf16 pre-score b of every candidate: bf16(q) . bf16(x) in fp32, one
//     candidate per warp iteration with the row read coalesced (1.5 KB at
//     dim 768) -- |b - q.x| <= eps_bf, the bound of k_rescore;
//  2. the reference's sequential fp64 dot (vindex.cpp:67) only for the
//     candidates with b >= b_k - 2 eps_bf (b_k = k-th best b): the k best by b
//     all have exact >= b_k - eps_bf, so a skipped one (exact <= b + eps_bf)
//     cannot reach the top k. Typically ~10-20 of the ~100 candidates.
// Certified iff cand_m + (fp64 rounding of the reference dot) < T_k, or the
// list holds every row. k <= 32 (the best 32 exact candidates are kept sorted
// across the lanes by a bitonic merge per chunk of 32).
// ---------------------------------------------------------------------------
constexpr int KI_MAX = 256;
constexpr int RI_WARPS = 4;

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int src_lane_xor) {
  Cand o;
  o.s = __shfl_xor_sync(0xffffffffu, c.s, src_lane_xor);
  o.id = __shfl_xor_sync(0xffffffffu, c.id, src_lane_xor);
  o.slot = __shfl_xor_sync(0xffffffffu, c.slot, src_lane_xor);
  return o;
}
// one compare-exchange step of a warp bitonic network in "better first" order
__device__ __forceinline__ void cx_step(Cand& c, int j, bool best_first) {
  const int lane = threadIdx.x & 31;
  const Cand o = shfl_cand(c, j);
  const bool lower = (lane & j) == 0;
  const bool take_o = (lower == best_first) ? cand_better(o, c) : cand_better(c, o);
  if (take_o) c = o;
}
// sort 32 candidates (one per lane) best first
__device__ __forceinline__ void warp_sort32(Cand& c) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) cx_step(c, j, (lane & k) == 0);
}
// top-32 of two best-first sorted lists (A, B), best first, into A
__device__ __forceinline__ void warp_merge32(Cand& a, const Cand& b) {
  const int lane = threadIdx.x & 31;
  Cand br;  // B reversed
  br.s = __shfl_sync(0xffffffffu, b.s, 31 - lane);
  br.id = __shfl_sync(0xffffffffu, b.id, 31 - lane);
  br.slot = __shfl_sync(0xffffffffu, b.slot, 31 - lane);
  if (cand_better(br, a)) a = br;  // bitonic: holds the best 32 of A u B
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) cx_step(a, j, true);
}
__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
// The k-th largest of the warp's keys (8 per lane, 0 = no key), exact: an
// MSB-first bisection over the 32 key bits, one warp count per bit. Needs at
// least k nonzero keys.
__device__ __forceinline__ uint32_t warp_kth_key(const uint32_t (&key)[8], int k) {
  uint32_t t = 0;
#pragma unroll 1
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t c = t | (1u << bit);
    uint32_t n = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) n += key[j] >= c;
    if ((int)__reduce_add_sync(0xffffffffu, n) >= k) t = c;
  }
  return t;
}
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// CPL: 16-byte bf16 chunks per lane of a pre-scored row (3 for dim <= 768, 4
// for <= 1024): the CPL = 3 build drops the spills of the 128-register cap
// (r02cl: 0.295 -> 0.282 ms per 4096 x 1M batch; 5 blocks/SM at 96 registers
// spilled and was slower)
template <int CPL, int MINB>
__global__ void __launch_bounds__(RI_WARPS * 32, MINB)
    k_rescore_i8_t(const float* __restrict__ Q, int nq, int dim, const float* __restrict__ rows,
                 const __nv_bfloat16* __restrict__ rowsb, const uint64_t* __restrict__ ids,
                 const float* __restrict__ cand_s, const uint32_t* __restrict__ cand_r, const int32_t* __restrict__ cand_n,
                 const float* __restrict__ cand_m, int kout, int64_t n_rows, int k, double dres, double eps_floor,
                 uint64_t* __restrict__ out_ids, double* __restrict__ out_sc, int32_t* __restrict__ out_cnt,
                 int32_t* __restrict__ fail_list, int32_t* __restrict__ fail_n,
                 unsigned long long* __restrict__ max_err_bits, int32_t* __restrict__ bad_query,
                 unsigned long long* __restrict__ gathered, float* __restrict__ tlo_out,
                 const float* __restrict__ t_glob) {
  // tlo_out (sharded lookup, first pass): only write a lower bound of this
  // rank's k-th exact score ((k-th best b of the 32 best candidates by U) -
  // eps, rounded down) and return. t_glob (second pass): the max of those
  // bounds over the ranks, a lower bound T of the GLOBAL k-th score: rows
  // below it cannot be in the merged top-k, so this rank pre-scores only
  // candidates with U >= T, exact-scores only those with b >= T - eps, and its
  // list is certified when every row outside it is below T (cm + margin < T).
  //
  // No sorting: every stage is a set defined by a threshold (the k-th / 32nd
  // largest key, found by bisection in registers), compacted into a position
  // list and processed in any order; the exact top-k merge is order-free.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * RI_WARPS + warp;
  if (q >= nq) return;
  extern __shared__ __align__(16) uint8_t s_raw[];
  // per warp: fp64 query [dim] | bf16 query [dim] | position list [KI_MAX] |
  // b by position [KI_MAX] | table row by position [KI_MAX]
  const size_t per_warp = (size_t)dim * 10 + KI_MAX * 12;
  uint8_t* wbase = s_raw + (size_t)warp * per_warp;
  double* sqd = reinterpret_cast<double*>(wbase);
  __nv_bfloat16* sb = reinterpret_cast<__nv_bfloat16*>(wbase + (size_t)dim * 8);
  int32_t* list = reinterpret_cast<int32_t*>(wbase + (size_t)dim * 10);
  float* sbv = reinterpret_cast<float*>(list + KI_MAX);
  uint32_t* srow = reinterpret_cast<uint32_t*>(sbv + KI_MAX);
  const float* qv = Q + (int64_t)q * dim;
  const int64_t cbase = (int64_t)q * kout;
  const int cn_all = min(cand_n[q], KI_MAX);
  // candidates: position lane + 32 j, U key in registers, row in smem
  uint32_t uk[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i = lane + 32 * j;
    uk[j] = 0;
    if (i < cn_all) {
      uk[j] = fkey(cand_s[cbase + i]);
      srow[i] = cand_r[cbase + i];
    }
  }
  double qsq = 0.0, dsq = 0.0;
  bool qfin = true;
  for (int d = lane; d < dim; d += 32) {
    const float v = qv[d];
    sqd[d] = (double)v;
    const __nv_bfloat16 bv = __float2bfloat16_rn(v);
    sb[d] = bv;
    qfin &= isfinite(v);
    qsq = fma((double)v, (double)v, qsq);
    const double e = (double)v - (double)__bfloat162float(bv);
    dsq = fma(e, e, dsq);
  }
  __syncwarp();
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    qsq += __shfl_xor_sync(0xffffffffu, qsq, off);
    dsq += __shfl_xor_sync(0xffffffffu, dsq, off);
  }
  qfin = __all_sync(0xffffffffu, qfin);
  if (!qfin && lane == 0) atomicExch(bad_query, 1);
  const double qn = sqrt(qsq) * (1.0 + 0x1p-40), dqn = sqrt(dsq) * (1.0 + 0x1p-40);
  const bool q_uncertifiable = !qfin || !(qn < 16384.0);
  // bf16 score bound (as k_rescore: operand rounding + fp32 accumulation)
  const double xn = 1.0 + 1e-6;
  double eps = qn * dres + dqn * (xn + dres) + 0x1p-13 * (qn + dqn) * (xn + dres);
  eps = fmax(eps * (1.0 + 0x1p-20), eps_floor * fmax(1.0, qn));
  // the reference's fp64 sequential dot vs the real dot: <= dim 2^-53 ||q|| ||x||
  const double margin = 1e-12 * (1.0 + qn);
  const bool global_mode = t_glob != nullptr;
  double t_lo = global_mode ? (double)t_glob[q] : -INFINITY;
  // positions with pred(j) into list[0, n), ascending
  auto compact = [&](auto pred) -> int {
    int n = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const bool f = pred(j);
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (f) list[n + __popc(bal & ((1u << lane) - 1u))] = lane + 32 * j;
      n += __popc(bal);
    }
    __syncwarp();
    return n;
  };
  // bf16 pre-score b of list[0, n) into sbv[position], 4 rows per iteration:
  // every lane issues all its 16-byte chunks of the 4 rows (<= 4 each, dim <=
  // 1024) before any math, and the bulk engine keeps the next PW rows on
  // their way into L2
  const uint4* sb4 = reinterpret_cast<const uint4*>(sb);
  const int n16 = dim / 8;  // 16-byte chunks per bf16 row
  constexpr int PW = 16;    // rows prefetched ahead
  uint4 qa[CPL];
#pragma unroll
  for (int u = 0; u < CPL; ++u) qa[u] = lane + 32 * u < n16 ? sb4[lane + 32 * u] : make_uint4(0, 0, 0, 0);
  auto prescore = [&](int n) {
    if (lane < PW && lane < n) prefetch_l2_bulk(rowsb + (int64_t)srow[list[lane]] * dim, (uint32_t)dim * 2);
    for (int i0 = 0; i0 < n; i0 += 4) {
      if (lane < 4 && i0 + PW + lane < n)
        prefetch_l2_bulk(rowsb + (int64_t)srow[list[i0 + PW + lane]] * dim, (uint32_t)dim * 2);
      uint32_t rr[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) rr[g] = i0 + g < n ? srow[list[i0 + g]] : 0u;
      uint4 xa[4][CPL];
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int u = 0; u < CPL; ++u) {
          const int c = lane + 32 * u;
          xa[g][u] = (i0 + g < n && c < n16) ? __ldg(reinterpret_cast<const uint4*>(rowsb + (int64_t)rr[g] * dim) + c)
                                             : make_uint4(0, 0, 0, 0);
        }
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int u = 0; u < CPL; ++u) {
          const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xa[g][u]);
          const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&qa[u]);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const float2 xf = __bfloat1622float2(x2[h]), qf = __bfloat1622float2(q2[h]);
            acc[g] = fmaf(qf.x, xf.x, acc[g]);
            acc[g] = fmaf(qf.y, xf.y, acc[g]);
          }
        }
#pragma unroll
      for (int g = 0; g < 4; ++g) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], off);
      }
      if (lane < 4 && i0 + lane < n) sbv[list[i0 + lane]] = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
    }
    __syncwarp();
  };
  // (1) set A: the 32 best candidates by U (ties at the 32nd included), in
  // global mode without those below T; T_lo = (k-th best b in A) - eps <= T_k
  const uint32_t tauA = cn_all > 32 ? warp_kth_key(uk, 32) : 1u;
  auto inA = [&](int j) {
    return uk[j] >= tauA && uk[j] != 0 && !(global_mode && (double)fkey_inv(uk[j]) < t_lo);
  };
  const int nA = compact(inA);
  prescore(nA);
  uint32_t bkey[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) bkey[j] = inA(j) ? fkey(sbv[lane + 32 * j]) : 0u;
  const double lo = nA >= k ? (double)fkey_inv(warp_kth_key(bkey, k)) - eps : -INFINITY;
  if (tlo_out) {
    if (lane == 0) tlo_out[q] = __double2float_rd(lo);
    return;
  }
  t_lo = fmax(t_lo, lo);
  // (2) set B: the rest of the candidates with U >= T_lo (a candidate with
  // U < T_lo has exact <= U < T_k and cannot reach the top k)
  bool pre[8];
  auto inB = [&](int j) { return uk[j] != 0 && !inA(j) && !((double)fkey_inv(uk[j]) < t_lo); };
  const int nB = compact(inB);
  prescore(nB);
  int cn = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    pre[j] = uk[j] != 0 && (inA(j) || !((double)fkey_inv(uk[j]) < t_lo));
    bkey[j] = pre[j] ? fkey(sbv[lane + 32 * j]) : 0u;
    cn += pre[j];
  }
  cn = (int)__reduce_add_sync(0xffffffffu, (uint32_t)cn);
  // (3) exact-score the pre-scored candidates with b >= b_k - 2 eps (b_k =
  // k-th best b; all of them when <= k)
  const float bk = cn > k ? fkey_inv(warp_kth_key(bkey, k)) : -INFINITY;
  // global mode: a candidate with b < T - eps has exact < T and is not needed either
  const double need_b = global_mode ? fmax((double)bk - 2.0 * eps, t_lo - eps) : (double)bk - 2.0 * eps;
  const int nC = compact([&](int j) { return pre[j] && (double)fkey_inv(bkey[j]) >= need_b; });
  for (int c = lane; c < nC; c += 32) prefetch_l2_bulk(rows + (int64_t)srow[list[c]] * dim, (uint32_t)dim * 4);
  Cand best;
  best.s = -INFINITY;
  best.id = ~0ull;
  best.slot = -1;
  int n_have = 0, n_gath = 0;
  double local_err = 0.0;
  for (int base = 0; base < nC; base += 32) {
    Cand c;
    c.s = -INFINITY;
    c.id = ~0ull;
    c.slot = -1;
    if (base + lane < nC) {
      const int pos = list[base + lane];
      const uint32_t r = srow[pos];
      const float* x = rows + (int64_t)r * dim;
      double acc = 0.0;
      {
        // sequential fp64 in d order (vindex.cpp:67), 32 elements in flight
        // (dim % 128 == 0 on the int8 tier); the query is fp64 in smem
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const double2* q2 = reinterpret_cast<const double2*>(sqd);
        float4 nx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) nx[u] = __ldg(x4 + u);
        for (int d4 = 0; d4 < dim / 4; d4 += 8) {
          float4 cx[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) cx[u] = nx[u];
          if (d4 + 8 < dim / 4) {
#pragma unroll
            for (int u = 0; u < 8; ++u) nx[u] = __ldg(x4 + d4 + 8 + u);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double2 qa2 = q2[2 * (d4 + u)], qb2 = q2[2 * (d4 + u) + 1];
            acc = fma(qa2.x, (double)cx[u].x, acc);
            acc = fma(qa2.y, (double)cx[u].y, acc);
            acc = fma(qb2.x, (double)cx[u].z, acc);
            acc = fma(qb2.y, (double)cx[u].w, acc);
          }
        }
      }
      local_err = fmax(local_err, fabs(acc - (double)sbv[pos]));
      c.s = acc;
      c.id = ids[r];
      c.slot = r;
      ++n_gath;
    }
    n_have += __popc(__ballot_sync(0xffffffffu, c.slot >= 0));
    warp_sort32(c);
    warp_merge32(best, c);
  }
  const double tk = __shfl_sync(0xffffffffu, best.s, min(k, 32) - 1);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    local_err = fmax(local_err, __shfl_xor_sync(0xffffffffu, local_err, off));
    n_gath += __shfl_xor_sync(0xffffffffu, n_gath, off);
  }
  if (lane == 0) {
    if (local_err > 0) atomicMax(max_err_bits, (unsigned long long)__double_as_longlong(local_err));
    atomicAdd(gathered, (unsigned long long)n_gath);
    atomicAdd(gathered + 1, (unsigned long long)cn_all);
    atomicAdd(gathered + 2, (unsigned long long)cn);
  }
  const int got = min(n_have, k);
  if (lane < k) {
    out_ids[(int64_t)q * k + lane] = lane < got ? best.id : 0;
    out_sc[(int64_t)q * k + lane] = lane < got ? best.s : 0.0;
  }
  if (lane == 0) {
    out_cnt[q] = got;
    bool ok;
    if (q_uncertifiable) ok = false;
    else if (cn_all >= n_rows) ok = true;  // every row is in the list
    else if (global_mode) ok = (double)cand_m[q] + margin < t_lo;  // every row outside is below T
    else ok = got >= k && (double)cand_m[q] + margin < tk;
    if (!ok) fail_list[atomicAdd(fail_n, 1)] = q;
  }
}

// the launch sites pick the build by dimension
#define RESCORE_I8(dim_) ((dim_) <= 768 ? k_rescore_i8_t<3, 4> : k_rescore_i8_t<4, 4>)

}  // namespace fc

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
namespace {

// int8 tier 1 for shapes the s8 kernel takes (128-byte K boxes, A in TMEM);
// FC_LOOKUP_I8=0 keeps the bf16 tier only (A/B measurements)
bool i8_wanted(int dim) {
  static const bool off = getenv("FC_LOOKUP_I8") && atoi(getenv("FC_LOOKUP_I8")) == 0;
  return !off && dim % 128 == 0 && dim <= 1024;
}

// k_rescore_i8 takes up to RI_WARPS * (10 dim + 12 KI_MAX) bytes of smem
// (53 KB at dim 1024): opt in once per device
void rescore_i8_attr(lc_ctx* ctx) {
  static std::atomic<uint64_t> attr_set{0};
  if (!(attr_set.load() >> (ctx->device & 63) & 1)) {
    FC_CUDA(cudaFuncSetAttribute(k_rescore_i8_t<3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(RI_WARPS * (768 * 10 + KI_MAX * 12))));
    FC_CUDA(cudaFuncSetAttribute(k_rescore_i8_t<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(RI_WARPS * (1024 * 10 + KI_MAX * 12))));
    attr_set.fetch_or(1ull << (ctx->device & 63));
  }
}

void ensure_capacity(lc_index* ix, int64_t need) {
  if (need <= ix->cap) return;
  int64_t nc = std::max<int64_t>(need, std::max<int64_t>(1024, ix->cap * 2));
  lc_ctx* ctx = ix->ctx;
  for (int t = 0; t < 3; ++t) {
    float* nr = nullptr;
    __nv_bfloat16* nb = nullptr;
    FC_CUDA(cudaMalloc(&nr, (size_t)nc * ix->dim * sizeof(float)));
    FC_CUDA(cudaMalloc(&nb, (size_t)nc * ix->dim * sizeof(__nv_bfloat16)));
    if (ix->n) {
      FC_CUDA(cudaMemcpyAsync(nr, ix->rows[t], (size_t)ix->n * ix->dim * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
      FC_CUDA(cudaMemcpyAsync(nb, ix->rowsb[t], (size_t)ix->n * ix->dim * sizeof(__nv_bfloat16), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    FC_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ix->rows[t]) cudaFree(ix->rows[t]);
    if (ix->rowsb[t]) cudaFree(ix->rowsb[t]);
    ix->rows[t] = nr;
    ix->rowsb[t] = nb;
    ix->plan[t].valid = false;
    if (ix->i8) {
      int8_t* n8 = nullptr;
      float *ns = nullptr, *nr8 = nullptr;
      // whole 128-row tiles: the quantizer writes (zeros) up to the tile end
      const int64_t nc8 = (nc + 127) / 128 * 128;
      FC_CUDA(cudaMalloc(&n8, (size_t)nc8 * ix->dim));
      FC_CUDA(cudaMalloc(&ns, (size_t)(nc8 / 128) * sizeof(float)));
      FC_CUDA(cudaMalloc(&nr8, (size_t)(nc8 / 128) * sizeof(float)));
      if (ix->n) {
        const size_t nt = (size_t)((ix->n + 127) / 128);
        FC_CUDA(cudaMemcpyAsync(n8, ix->rows8[t], nt * 128 * ix->dim, cudaMemcpyDeviceToDevice, ctx->stream));
        FC_CUDA(cudaMemcpyAsync(ns, ix->tscale[t], nt * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
        FC_CUDA(cudaMemcpyAsync(nr8, ix->tres[t], nt * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
      }
      FC_CUDA(cudaStreamSynchronize(ctx->stream));
      if (ix->rows8[t]) cudaFree(ix->rows8[t]);
      if (ix->tscale[t]) cudaFree(ix->tscale[t]);
      if (ix->tres[t]) cudaFree(ix->tres[t]);
      ix->rows8[t] = n8;
      ix->tscale[t] = ns;
      ix->tres[t] = nr8;
      ix->iplan[t].valid = false;
    }
  }
  uint64_t* ni = nullptr;
  FC_CUDA(cudaMalloc(&ni, (size_t)nc * sizeof(uint64_t)));
  if (ix->n) FC_CUDA(cudaMemcpyAsync(ni, ix->ids_dev, (size_t)ix->n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, ctx->stream));
  FC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ix->ids_dev) cudaFree(ix->ids_dev);
  ix->ids_dev = ni;
  ix->cap = nc;
}

// Re-quantize the int8 tiles [t0, t1) of every table (after an insert or a
// remove changed their rows) and fold their residual norms into dres8.
void requantize(lc_index* ix, int64_t t0, int64_t t1) {
  if (!ix->i8 || t1 <= t0 || ix->n == 0) return;
  lc_ctx* ctx = ix->ctx;
  DevBuf rb(3 * sizeof(unsigned long long), ctx->stream);
  FC_CUDA(cudaMemsetAsync(rb.p, 0, rb.bytes, ctx->stream));
  for (int t = 0; t < 3; ++t) {
    i8_quantize_tiles(ctx, ix->rows[t], ix->n, ix->dim, t0, t1, ix->rows8[t], ix->tscale[t], ix->tres[t],
                      rb.as<unsigned long long>() + t);
    ix->iplan[t].valid = false;
  }
  double r[3];
  FC_CUDA(cudaMemcpyAsync(r, rb.p, sizeof r, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  for (int t = 0; t < 3; ++t) ix->dres8[t] = std::max(ix->dres8[t], r[t]);
}

// from_unit check of n rows; returns the max bf16 residual norm of the rows
double check_units_device(lc_ctx* ctx, const float* dev, int64_t n, int dim) {
  DevBuf bad(16, ctx->stream);
  FC_CUDA(cudaMemsetAsync(bad.p, 0, 16, ctx->stream));
  k_check_unit<<<grid_for(n, 128), 128, 0, ctx->stream>>>(dev, n, dim, bad.as<int>(),
                                                          reinterpret_cast<unsigned long long*>(bad.as<char>() + 8));
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  uint64_t hb[2] = {0, 0};
  FC_CUDA(cudaMemcpyAsync(hb, bad.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  if ((uint32_t)hb[0]) raise(LC_ERR_INVALID_ARGUMENT, "Embedding: vector is not unit norm");
  double r = 0.0;
  memcpy(&r, &hb[1], 8);
  return r;
}

// Exact top-k of queries (all, or the subset qlist) by full fp64 scan.
void exact_scan(lc_index* ix, int kind, const float* Qdev, const int32_t* qlist_dev, int nq, int k, uint64_t* oid,
                double* osc, int32_t* ocnt) {
  lc_ctx* ctx = ix->ctx;
  if (nq <= 0) return;
  const int dim = ix->dim;
  const int nblk = (int)((ix->n + SCAN_T - 1) / SCAN_T);
  // bound the partial-list scratch to ~256 MB per pass
  const int64_t per_q = (int64_t)nblk * k * sizeof(Cand);
  const int chunk = (int)std::max<int64_t>(SCAN_QB, std::min<int64_t>(nq, ((256ll << 20) / per_q) / SCAN_QB * SCAN_QB));
  if (chunk < nq) {
    for (int q0 = 0; q0 < nq; q0 += chunk) {
      const int cn = std::min(chunk, nq - q0);
      if (qlist_dev) {
        exact_scan(ix, kind, Qdev, qlist_dev + q0, cn, k, oid, osc, ocnt);
      } else {
        DevBuf ql((size_t)cn * sizeof(int32_t), ctx->stream);
        std::vector<int32_t> h(cn);
        for (int i = 0; i < cn; ++i) h[i] = q0 + i;
        FC_CUDA(cudaMemcpyAsync(ql.p, h.data(), cn * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        exact_scan(ix, kind, Qdev, ql.as<int32_t>(), cn, k, oid, osc, ocnt);
        sync(ctx);
      }
    }
    return;
  }
  DevBuf partial((size_t)nq * nblk * k * sizeof(Cand), ctx->stream);
  DevBuf pcount((size_t)nq * nblk * sizeof(int32_t), ctx->stream);
  const size_t smem = (size_t)SCAN_QB * dim * sizeof(float);
  if (smem > 48 * 1024) FC_CUDA(cudaFuncSetAttribute(k_scan_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(nblk, (nq + SCAN_QB - 1) / SCAN_QB);
  KTimer kt(ctx, "scan");
  k_scan_partial<<<grid, SCAN_T, smem, ctx->stream>>>(Qdev, qlist_dev, nq, ix->rows[kind], ix->ids_dev, ix->n, dim, k,
                                                      partial.as<Cand>(), pcount.as<int32_t>());
  FC_LAUNCH_CHECK();
  if (k <= 8)
    k_scan_merge<8><<<nq, 256, 0, ctx->stream>>>(partial.as<Cand>(), pcount.as<int32_t>(), nblk, k, qlist_dev, oid, osc, ocnt);
  else
    k_scan_merge<64><<<nq, 256, 0, ctx->stream>>>(partial.as<Cand>(), pcount.as<int32_t>(), nblk, k, qlist_dev, oid, osc, ocnt);
  kt.stop();
  FC_LAUNCH_CHECK();
  count_launch(ctx, 2);
}

// Device-resident top-k (no host sync unless a fallback is needed).
__global__ void k_fill_f32(float* p, int n, float v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// The bound exchange is a collective: every rank must take part exactly once
// per sharded query batch, whichever tier its own shard used (shards differ in
// size, so one may scan exactly while another runs the int8 tier). A rank that
// did not exchange contributes -inf bounds on the way out.
struct ExchangeOnce {
  const BoundExchange* x;
  lc_ctx* ctx;
  int n;
  bool done = false;
  ~ExchangeOnce() {
    if (!x || done || std::uncaught_exceptions() > 0) return;
    DevBuf d((size_t)std::max(n, 1) * sizeof(float), ctx->stream);
    k_fill_f32<<<grid_for(std::max(n, 1), 256), 256, 0, ctx->stream>>>(d.as<float>(), n, -INFINITY);
    (*x)(d.as<float>(), n);
  }
};

// Sharded int8 lookups exchange the pilot's per-query keys once per batch;
// whether a batch does depends only on rank-uniform inputs (table config,
// batch size, k), so every rank joins the same collectives in the same order
// (pilot keys, then the bound exchange), whatever its shard holds.
bool pilot_exchange_expected(const lc_index* ix, int nq, int k) { return ix->i8 && k <= 32 && nq > 128; }

void query_dev(lc_index* ix, int kind, const float* Qdev, int nq, int k, uint64_t* oid, double* osc, int32_t* ocnt,
               const BoundExchange* xchg = nullptr) {
  lc_ctx* ctx = ix->ctx;
  ExchangeOnce xonce{xchg, ix->ctx, nq};
  {
    std::lock_guard<std::mutex> sl(ix->stats_mu);
    ix->stats.queries += nq;
  }
  // bf16 tier: the query's K boxes and two accumulators must fit TMEM (dim <= 768);
  // int8 tier: dim % 128 == 0, <= 1024 (ix->i8), k <= 32, batches that fill CTA pairs
  const bool bf16_ok = ix->dim % 64 == 0 && ix->dim <= 768 && k <= ix->kprime;
  const bool i8_ok = ix->i8 && k <= 32 && nq > 128;
  const bool approx_ok = approx_available() && (bf16_ok || i8_ok);
  const bool use_approx = approx_ok && (ix->mode == 2 || (ix->mode == 0 && ix->n >= 8192));
  if (!use_approx) {
    FC_REQUIRE(ix->mode != 2 || approx_ok, "lc_index_query_topk: tensor-core path unavailable for this shape");
    {
      DevBuf bad(sizeof(int), ctx->stream);
      FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
      k_check_finite_rows<<<grid_for(nq, 128), 128, 0, ctx->stream>>>(Qdev, nq, ix->dim, bad.as<int>());
      FC_LAUNCH_CHECK();
      count_launch(ctx);
      int hb = 0;
      FC_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      if (hb) raise(LC_ERR_INVALID_ARGUMENT, "Embedding: non-finite element");
    }
    if (xchg && pilot_exchange_expected(ix, nq, k)) dummy_pilot_exchange(ctx, *xchg, nq);  // small shard: no pilot here
    exact_scan(ix, kind, Qdev, nullptr, nq, k, oid, osc, ocnt);
    std::lock_guard<std::mutex> sl(ix->stats_mu);
    ix->stats.exact_scans += nq;
    return;
  }
  const int kp = ix->kprime;
  const int dim = ix->dim;
  DevBuf fl((size_t)nq * sizeof(int32_t), ctx->stream);
  DevBuf fn(16, ctx->stream);  // [0,4) fail count, [4,8) non-finite query flag, [8,16) max |err| bits
  int32_t* fail_n = fn.as<int32_t>();
  int32_t* bad_q = fn.as<int32_t>() + 1;
  auto* err_bits = reinterpret_cast<unsigned long long*>(fn.as<char>() + 8);
  FC_CUDA(cudaMemsetAsync(fn.p, 0, 16, ctx->stream));
  const size_t rs_smem = (size_t)RS_WARPS * dim * sizeof(float);
  if (rs_smem > 48 * 1024) {
    FC_CUDA(cudaFuncSetAttribute(k_rescore<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_smem));
    FC_CUDA(cudaFuncSetAttribute(k_rescore<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_smem));
    FC_CUDA(cudaFuncSetAttribute(k_rescore<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_smem));
  }
  // Tier 1: the int8 tensor-core shortlist (2x the bf16 tensor rate) for
  // batches that fill CTA pairs, else the bf16 shortlist with K' = kprime.
  const bool tier1_i8 = i8_ok;
  int64_t gathered = -1, cands = -1, prescored = -1;
  PinnedBuf<unsigned long long> hpin(5);  // [0,3) candidate counters | [3,5) the 16 B of failure counters
  bool hg_pending = false;
  if (tier1_i8) {
    const int kout = ix->i8_kout;
    DevBuf cs((size_t)nq * kout * sizeof(float), ctx->stream), cr((size_t)nq * kout * sizeof(uint32_t), ctx->stream);
    DevBuf cn((size_t)nq * sizeof(int32_t), ctx->stream), cm((size_t)nq * sizeof(float), ctx->stream);
    DevBuf gb(3 * sizeof(unsigned long long), ctx->stream);
    FC_CUDA(cudaMemsetAsync(gb.p, 0, gb.bytes, ctx->stream));
    {
      std::lock_guard<std::mutex> pl(ix->plan_mu);
      if (!ix->iplan[kind].valid || ix->iplan[kind].n_rows != ix->n) {
        // median tile residual: the threshold offset of the int8 filter
        const int64_t nt = (ix->n + 127) / 128;
        std::vector<float> tr(nt);
        FC_CUDA(cudaMemcpyAsync(tr.data(), ix->tres[kind], nt * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        std::nth_element(tr.begin(), tr.begin() + nt / 2, tr.end());
        i8_plan(ix->iplan[kind], ix->rows8[kind], ix->tscale[kind], ix->tres[kind], ix->n, dim, tr[nt / 2]);
      }
    }
    i8_shortlist(ctx, ix->iplan[kind], Qdev, nq, k, ix->i8_kunit, kout, cs.as<float>(), cr.as<uint32_t>(),
                 cn.as<int32_t>(), cm.as<float>(), nullptr, xchg);
    const size_t ri_smem = (size_t)RI_WARPS * ((size_t)dim * 10 + KI_MAX * 12);
    rescore_i8_attr(ctx);
    KTimer kt(ctx, "rescore");
    DevBuf tlo(xchg ? (size_t)nq * sizeof(float) : 16, ctx->stream);
    if (xchg) {
      // sharded: each rank's lower bound of its k-th score, max over the ranks
      RESCORE_I8(dim)<<<(unsigned)((nq + RI_WARPS - 1) / RI_WARPS), RI_WARPS * 32, ri_smem, ctx->stream>>>(
          Qdev, nq, dim, ix->rows[kind], ix->rowsb[kind], ix->ids_dev, cs.as<float>(), cr.as<uint32_t>(),
          cn.as<int32_t>(), cm.as<float>(), kout, ix->n, k, ix->dres[kind], ix->eps_floor, oid, osc, ocnt,
          fl.as<int32_t>(), fail_n, err_bits, bad_q, gb.as<unsigned long long>(), tlo.as<float>(), nullptr);
      FC_LAUNCH_CHECK();
      count_launch(ctx);
      (*xchg)(tlo.as<float>(), nq);
      xonce.done = true;
    }
    RESCORE_I8(dim)<<<(unsigned)((nq + RI_WARPS - 1) / RI_WARPS), RI_WARPS * 32, ri_smem, ctx->stream>>>(
        Qdev, nq, dim, ix->rows[kind], ix->rowsb[kind], ix->ids_dev, cs.as<float>(), cr.as<uint32_t>(), cn.as<int32_t>(),
        cm.as<float>(), kout, ix->n, k, ix->dres[kind], ix->eps_floor, oid, osc, ocnt, fl.as<int32_t>(), fail_n,
        err_bits, bad_q, gb.as<unsigned long long>(), nullptr, xchg ? tlo.as<float>() : nullptr);
    kt.stop();
    FC_LAUNCH_CHECK();
    count_launch(ctx);
    // the candidate counters come back with the failure counters below (one sync)
    FC_CUDA(cudaMemcpyAsync(hpin.data(), gb.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    hg_pending = true;
  } else {
    DevBuf cs((size_t)nq * kp * sizeof(float), ctx->stream);
    DevBuf cr((size_t)nq * kp * sizeof(uint32_t), ctx->stream);
    DevBuf cn((size_t)nq * sizeof(int32_t), ctx->stream);
    {
      std::lock_guard<std::mutex> pl(ix->plan_mu);
      if (!ix->plan[kind].valid || ix->plan[kind].n_rows != ix->n)
        approx_plan(ix->plan[kind], ix->rowsb[kind], ix->n, dim, ctx->sm_count);
    }
    approx_shortlist(ctx, ix->plan[kind], Qdev, nq, kp, cs.as<float>(), cr.as<uint32_t>(), cn.as<int32_t>());
    const unsigned g = (unsigned)((nq + RS_WARPS - 1) / RS_WARPS);
    KTimer kt(ctx, "rescore");
    if (kp <= 32)
      k_rescore<1><<<g, RS_WARPS * 32, rs_smem, ctx->stream>>>(Qdev, nq, dim, ix->rows[kind], ix->ids_dev, cs.as<float>(),
                                                         cr.as<uint32_t>(), cn.as<int32_t>(), kp, ix->n, k, ix->dres[kind], ix->eps_floor, oid, osc, ocnt,
                                                         fl.as<int32_t>(), fail_n, err_bits, bad_q);
    else if (kp <= 64)
      k_rescore<2><<<g, RS_WARPS * 32, rs_smem, ctx->stream>>>(Qdev, nq, dim, ix->rows[kind], ix->ids_dev, cs.as<float>(),
                                                         cr.as<uint32_t>(), cn.as<int32_t>(), kp, ix->n, k, ix->dres[kind], ix->eps_floor, oid, osc, ocnt,
                                                         fl.as<int32_t>(), fail_n, err_bits, bad_q);
    else
      k_rescore<4><<<g, RS_WARPS * 32, rs_smem, ctx->stream>>>(Qdev, nq, dim, ix->rows[kind], ix->ids_dev, cs.as<float>(),
                                                         cr.as<uint32_t>(), cn.as<int32_t>(), kp, ix->n, k, ix->dres[kind], ix->eps_floor, oid, osc, ocnt,
                                                         fl.as<int32_t>(), fail_n, err_bits, bad_q);
    kt.stop();
    FC_LAUNCH_CHECK();
    count_launch(ctx);
  }
  int32_t hf[4] = {0, 0, 0, 0};
  FC_CUDA(cudaMemcpyAsync(hpin.data() + 3, fn.p, 16, cudaMemcpyDeviceToHost, ctx->stream));  // pinned: async
  sync(ctx);
  memcpy(hf, hpin.data() + 3, 16);
  if (hg_pending) {
    gathered = (int64_t)hpin[0];
    cands = (int64_t)hpin[1];
    prescored = (int64_t)hpin[2];
  }
  double err = 0.0;
  uint64_t eb = (uint64_t)(uint32_t)hf[2] | ((uint64_t)(uint32_t)hf[3] << 32);
  memcpy(&err, &eb, 8);
  if (hf[1]) raise(LC_ERR_INVALID_ARGUMENT, "Embedding: non-finite element");
  const int nf = hf[0];
  {
    std::lock_guard<std::mutex> sl(ix->stats_mu);
    ix->stats.max_abs_err = std::max(ix->stats.max_abs_err, err);
    ix->stats.certified += nq - nf;
    ix->stats.fallback += nf;
    if (tier1_i8) {
      ix->stats.i8_batches += 1;
      ix->stats.i8_rescored += gathered;
      ix->stats.i8_candidates += cands;
      ix->stats.i8_prescored += prescored;
    }
  }
  // FC_LOOKUP_DIAG=1 (kernel-timing diagnostics with FC_SHORTLIST_DEBUG only): skip the
  // exact re-scan, so results are NOT exact in that mode.
  static const bool diag = getenv("FC_LOOKUP_DIAG") && atoi(getenv("FC_LOOKUP_DIAG")) == 1;
  if (nf == 0 || diag) return;
  // Tier 2: the uncertified queries (near-ties around the k-th score) rerun
  // the bf16 tensor-core shortlist (after the int8 tier: first with K' =
  // kprime, whose ~5x tighter bound certifies almost all of them) with a
  // longer K' and are rescored/certified again (~one streaming pass of the
  // bf16 table each), escalating K' = kp + 32 then 128 (K' = kp + 32
  // certifies the usual near-ties at ~2/3 the cost, as more pipeline stages
  // fit); only what still fails takes the exact fp64 scan of every row.
  // FC_LOOKUP_TIER2=0 disables it; FC_LOOKUP_TIER2_KP caps K'.
  // Clustered tables (many near-duplicate rows per query, e.g. shared object
  // embeddings) fail for most of the batch and a longer K' rarely helps there:
  // when more than 1/16 of the batch (and > 8 queries) failed a bf16 pass, go
  // straight to the exact scan. Same results either way; this only picks the
  // cheaper path.
  const bool tier2_env_off = getenv("FC_LOOKUP_TIER2") && atoi(getenv("FC_LOOKUP_TIER2")) == 0;
  bool tier2_off = tier2_env_off || !bf16_ok || (!tier1_i8 && nf > 8 && nf * 16 > nq);
  constexpr int KP2_MAX = 128;
  int kp2_cap = KP2_MAX;
  if (const char* e = getenv("FC_LOOKUP_TIER2_KP")) kp2_cap = std::max(kp + 32, std::min(KP2_MAX, atoi(e)));
  DevBuf list_buf((size_t)nf * sizeof(int32_t), ctx->stream);  // current failures -> original query index
  FC_CUDA(cudaMemcpyAsync(list_buf.p, fl.p, (size_t)nf * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
  int n_left = nf;
  int prev = tier1_i8 ? 0 : kp;
  if (tier1_i8 && !tier2_off) {
    std::lock_guard<std::mutex> pl(ix->plan_mu);
    if (!ix->plan[kind].valid || ix->plan[kind].n_rows != ix->n)
      approx_plan(ix->plan[kind], ix->rowsb[kind], ix->n, dim, ctx->sm_count);
  }
  for (int level = tier1_i8 ? -1 : 0; level < 2 && !tier2_off && n_left > 0; ++level) {
    const int want = level < 0 ? kp : std::min(kp2_cap, level == 0 ? kp + 32 : KP2_MAX);
    if (want <= prev || k > want) break;
    DevBuf q2((size_t)n_left * dim * sizeof(float), ctx->stream);
    k_gather_queries<<<grid_for((int64_t)n_left * dim, 256), 256, 0, ctx->stream>>>(Qdev, list_buf.as<int32_t>(), n_left,
                                                                                   dim, q2.as<float>());
    FC_LAUNCH_CHECK();
    count_launch(ctx);
    DevBuf cs2((size_t)n_left * want * sizeof(float), ctx->stream), cr2((size_t)n_left * want * sizeof(uint32_t), ctx->stream);
    DevBuf cn2((size_t)n_left * sizeof(int32_t), ctx->stream);
    int kp2 = 0;  // the longest shortlist <= want that the kernel's shared memory allows at this dim
    for (int cand = want; cand > prev && kp2 == 0; cand -= 32) {
      try {
        ShortlistTimerName tn("shortlist_tier2");
        approx_shortlist(ctx, ix->plan[kind], q2.as<float>(), n_left, cand, cs2.as<float>(), cr2.as<uint32_t>(),
                         cn2.as<int32_t>());
        kp2 = cand;
      } catch (const Error& e) {
        if (e.code != LC_ERR_INVALID_ARGUMENT) throw;  // smem budget at this K': try a shorter one
      }
    }
    if (kp2 == 0) break;
    prev = kp2;
    DevBuf id2((size_t)n_left * k * sizeof(uint64_t), ctx->stream), sc2((size_t)n_left * k * sizeof(double), ctx->stream);
    DevBuf ct2((size_t)n_left * sizeof(int32_t), ctx->stream), fl2((size_t)n_left * sizeof(int32_t), ctx->stream);
    DevBuf fn2(16, ctx->stream);
    FC_CUDA(cudaMemsetAsync(fn2.p, 0, 16, ctx->stream));
    {
      KTimer kt2(ctx, "rescore_tier2");
      k_rescore<4><<<(unsigned)((n_left + RS_WARPS - 1) / RS_WARPS), RS_WARPS * 32, rs_smem, ctx->stream>>>(
          q2.as<float>(), n_left, dim, ix->rows[kind], ix->ids_dev, cs2.as<float>(), cr2.as<uint32_t>(),
          cn2.as<int32_t>(), kp2, ix->n, k, ix->dres[kind], ix->eps_floor, id2.as<uint64_t>(), sc2.as<double>(), ct2.as<int32_t>(),
          fl2.as<int32_t>(), fn2.as<int32_t>(), reinterpret_cast<unsigned long long*>(fn2.as<char>() + 8),
          fn2.as<int32_t>() + 1);
    }
    // every row lands in place; the still-uncertified ones are overwritten below
    k_scatter_topk<<<grid_for((int64_t)n_left * k, 256), 256, 0, ctx->stream>>>(
        id2.as<uint64_t>(), sc2.as<double>(), ct2.as<int32_t>(), list_buf.as<int32_t>(), n_left, k, oid, osc, ocnt);
    FC_LAUNCH_CHECK();
    count_launch(ctx, 2);
    int32_t hf2[4] = {0, 0, 0, 0};
    FC_CUDA(cudaMemcpyAsync(hf2, fn2.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    const int nf2 = hf2[0];
    {
      std::lock_guard<std::mutex> sl(ix->stats_mu);
      ix->stats.tier2_certified += n_left - nf2;
    }
    if (nf2 > 0) {
      DevBuf nl((size_t)nf2 * sizeof(int32_t), ctx->stream);
      k_map_list<<<grid_for(nf2, 128), 128, 0, ctx->stream>>>(fl2.as<int32_t>(), list_buf.as<int32_t>(), nf2,
                                                              nl.as<int32_t>());
      FC_LAUNCH_CHECK();
      count_launch(ctx);
      FC_CUDA(cudaMemcpyAsync(list_buf.p, nl.p, (size_t)nf2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    // a bf16 pass that left most of its queries uncertified: clustered rows
    if (level < 0 && nf2 > 8 && nf2 * 16 > nq) tier2_off = true;
    n_left = nf2;
  }
  // Threshold tier (int8 tables, k <= 32): near-tied clusters (many rows
  // within the tensor-core error of the k-th score) defeat every K'-based
  // shortlist; instead collect EVERY row whose int8 upper bound U exceeds a
  // known lower bound of T_k (the k-th best exact score found so far) with one
  // fixed-threshold int8 pass, then rescore/certify as the int8 tier does.
  // One streaming pass of the 768 MB s8 table for the few queries left
  // instead of an fp64 scan of the whole fp32 table (~170 ms at 1M rows).
  static const bool thr_off = getenv("FC_LOOKUP_THRESHOLD_TIER") && atoi(getenv("FC_LOOKUP_THRESHOLD_TIER")) == 0;
  if (n_left > 0 && ix->i8 && k <= 32 && !thr_off) {
    DevBuf q2((size_t)n_left * dim * sizeof(float), ctx->stream), tau((size_t)n_left * sizeof(float), ctx->stream);
    k_gather_queries<<<grid_for((int64_t)n_left * dim, 256), 256, 0, ctx->stream>>>(Qdev, list_buf.as<int32_t>(), n_left,
                                                                                   dim, q2.as<float>());
    k_tau_fix<<<(unsigned)((n_left + 7) / 8), 256, 0, ctx->stream>>>(Qdev, list_buf.as<int32_t>(), n_left, dim, osc, ocnt,
                                                                     k, tau.as<float>());
    FC_LAUNCH_CHECK();
    count_launch(ctx, 2);
    {
      std::lock_guard<std::mutex> pl(ix->plan_mu);
      if (!ix->iplan[kind].valid || ix->iplan[kind].n_rows != ix->n) {
        const int64_t nt = (ix->n + 127) / 128;
        std::vector<float> tr(nt);
        FC_CUDA(cudaMemcpyAsync(tr.data(), ix->tres[kind], nt * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        std::nth_element(tr.begin(), tr.begin() + nt / 2, tr.end());
        i8_plan(ix->iplan[kind], ix->rows8[kind], ix->tscale[kind], ix->tres[kind], ix->n, dim, tr[nt / 2]);
      }
    }
    const int kout = KI_MAX;
    DevBuf cs2((size_t)n_left * kout * sizeof(float), ctx->stream), cr2((size_t)n_left * kout * sizeof(uint32_t), ctx->stream);
    DevBuf cn2((size_t)n_left * sizeof(int32_t), ctx->stream), cm2((size_t)n_left * sizeof(float), ctx->stream);
    {
      ShortlistTimerName tn("shortlist_threshold");
      i8_shortlist(ctx, ix->iplan[kind], q2.as<float>(), n_left, k, ix->i8_kunit, kout, cs2.as<float>(),
                   cr2.as<uint32_t>(), cn2.as<int32_t>(), cm2.as<float>(), tau.as<float>());
    }
    DevBuf id2((size_t)n_left * k * sizeof(uint64_t), ctx->stream), sc2((size_t)n_left * k * sizeof(double), ctx->stream);
    DevBuf ct2((size_t)n_left * sizeof(int32_t), ctx->stream), fl2((size_t)n_left * sizeof(int32_t), ctx->stream);
    DevBuf fn2(16, ctx->stream), gb2(3 * sizeof(unsigned long long), ctx->stream);
    FC_CUDA(cudaMemsetAsync(fn2.p, 0, 16, ctx->stream));
    FC_CUDA(cudaMemsetAsync(gb2.p, 0, gb2.bytes, ctx->stream));
    {
      KTimer kt3(ctx, "rescore_threshold");
      rescore_i8_attr(ctx);
      const size_t ri_smem = (size_t)RI_WARPS * ((size_t)dim * 10 + KI_MAX * 12);
      RESCORE_I8(dim)<<<(unsigned)((n_left + RI_WARPS - 1) / RI_WARPS), RI_WARPS * 32, ri_smem, ctx->stream>>>(
          q2.as<float>(), n_left, dim, ix->rows[kind], ix->rowsb[kind], ix->ids_dev, cs2.as<float>(), cr2.as<uint32_t>(),
          cn2.as<int32_t>(), cm2.as<float>(), kout, ix->n, k, ix->dres[kind], ix->eps_floor, id2.as<uint64_t>(),
          sc2.as<double>(), ct2.as<int32_t>(), fl2.as<int32_t>(), fn2.as<int32_t>(),
          reinterpret_cast<unsigned long long*>(fn2.as<char>() + 8), fn2.as<int32_t>() + 1,
          gb2.as<unsigned long long>(), nullptr, nullptr);
    }
    k_scatter_topk<<<grid_for((int64_t)n_left * k, 256), 256, 0, ctx->stream>>>(
        id2.as<uint64_t>(), sc2.as<double>(), ct2.as<int32_t>(), list_buf.as<int32_t>(), n_left, k, oid, osc, ocnt);
    FC_LAUNCH_CHECK();
    count_launch(ctx, 2);
    int32_t hf3[4] = {0, 0, 0, 0};
    FC_CUDA(cudaMemcpyAsync(hf3, fn2.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    const int nf3 = hf3[0];
    {
      std::lock_guard<std::mutex> sl(ix->stats_mu);
      ix->stats.threshold_certified += n_left - nf3;
    }
    if (nf3 > 0) {
      DevBuf nl((size_t)nf3 * sizeof(int32_t), ctx->stream);
      k_map_list<<<grid_for(nf3, 128), 128, 0, ctx->stream>>>(fl2.as<int32_t>(), list_buf.as<int32_t>(), nf3,
                                                              nl.as<int32_t>());
      FC_LAUNCH_CHECK();
      count_launch(ctx);
      FC_CUDA(cudaMemcpyAsync(list_buf.p, nl.p, (size_t)nf3 * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    n_left = nf3;
  }
  if (n_left > 0) {
    exact_scan(ix, kind, Qdev, list_buf.as<int32_t>(), n_left, k, oid, osc, ocnt);
    std::lock_guard<std::mutex> sl(ix->stats_mu);
    ix->stats.exact_scans += n_left;
  }
}

}  // namespace

namespace fc {
// Device-resident exact top-k for the entry-sharded path (shard.cu): the
// rank-local lookup whose lists the collective merges. Q/outputs on device;
// an empty table yields counts 0. Takes the index's reader lock.
lc_ctx* index_ctx(lc_index* ix) { return ix->ctx; }
int index_dim(lc_index* ix) { return ix->dim; }
void index_topk_dev(lc_index* ix, int kind, const float* Qdev, int nq, int k, uint64_t* oid, double* osc, int32_t* ocnt,
                    const BoundExchange* xchg) {
  std::shared_lock lock(ix->mu);
  lc_ctx* ctx = ix->ctx;
  if (nq <= 0) return;
  if (ix->n == 0) {
    ExchangeOnce xonce{xchg, ctx, nq};  // an empty shard still takes part in the collectives
    if (xchg && pilot_exchange_expected(ix, nq, k)) dummy_pilot_exchange(ctx, *xchg, nq);
    FC_CUDA(cudaMemsetAsync(oid, 0, (size_t)nq * k * sizeof(uint64_t), ctx->stream));
    FC_CUDA(cudaMemsetAsync(osc, 0, (size_t)nq * k * sizeof(double), ctx->stream));
    FC_CUDA(cudaMemsetAsync(ocnt, 0, (size_t)nq * sizeof(int32_t), ctx->stream));
    return;
  }
  query_dev(ix, kind, Qdev, nq, k, oid, osc, ocnt, xchg);
}
}  // namespace fc

extern "C" {

lc_status lc_index_create(lc_ctx* ctx, int dim, int64_t capacity_rows, lc_index** out) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && out, "lc_index_create: null argument");
  FC_REQUIRE(dim >= 0, "lc_index_create: negative dim");
  DeviceGuard g(ctx->device);
  auto* ix = new lc_index();
  ix->ctx = ctx;
  ix->dim = dim;
  ix->i8 = dim > 0 && i8_wanted(dim);
  if (const char* e = getenv("FC_LOOKUP_I8_KOUT")) ix->i8_kout = std::max(32, std::min(KI_MAX, atoi(e) / 32 * 32));
  if (const char* e = getenv("FC_LOOKUP_I8_KUNIT")) ix->i8_kunit = std::max(8, std::min(64, atoi(e)));
  if (dim > 0 && capacity_rows > 0) {
    try {
      ensure_capacity(ix, capacity_rows);
    } catch (...) {
      delete ix;
      throw;
    }
  }
  *out = ix;
  LC_API_END
}

lc_status lc_index_destroy(lc_index* ix) {
  LC_API_BEGIN
  if (!ix) return LC_OK;
  DeviceGuard g(ix->ctx->device);
  cudaStreamSynchronize(ix->ctx->stream);
  for (int t = 0; t < 3; ++t) {
    if (ix->rows[t]) cudaFree(ix->rows[t]);
    if (ix->rowsb[t]) cudaFree(ix->rowsb[t]);
    if (ix->rows8[t]) cudaFree(ix->rows8[t]);
    if (ix->tscale[t]) cudaFree(ix->tscale[t]);
    if (ix->tres[t]) cudaFree(ix->tres[t]);
  }
  if (ix->ids_dev) cudaFree(ix->ids_dev);
  delete ix;
  LC_API_END
}

lc_status lc_index_insert_batch(lc_index* ix, const uint64_t* prompts, const float* w, const float* o, const float* b,
                                int64_t n, int dim) {
  LC_API_BEGIN
  FC_REQUIRE(ix && prompts && w && o && b, "lc_index_insert_batch: null argument");
  if (n <= 0) return LC_OK;
  std::unique_lock lock(ix->mu);
  lc_ctx* ctx = ix->ctx;
  DeviceGuard g(ctx->device);
  FC_REQUIRE(dim > 0, "Embedding: empty vector");
  if (ix->dim != 0 && dim != ix->dim) raise(LC_ERR_INVALID_ARGUMENT, "SimilarityIndex: embedding dimension mismatch");
  std::vector<uint64_t> pid(n);
  if (is_device_ptr(prompts)) {
    FC_CUDA(cudaMemcpy(pid.data(), prompts, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  } else {
    memcpy(pid.data(), prompts, n * sizeof(uint64_t));
  }
  {
    std::vector<uint64_t> sorted(pid);
    std::sort(sorted.begin(), sorted.end());
    for (int64_t i = 0; i < n; ++i) {
      if ((i > 0 && sorted[i] == sorted[i - 1]) || ix->slot.count(sorted[i]))
        raise(LC_ERR_INVALID_ARGUMENT, "SimilarityIndex: duplicate prompt id");
    }
  }
  const float* src[3] = {w, o, b};
  InArg<float> a0(ctx, w, (size_t)n * dim), a1(ctx, o, (size_t)n * dim), a2(ctx, b, (size_t)n * dim);
  const float* dsrc[3] = {a0.dev, a1.dev, a2.dev};
  (void)src;
  double res[3];
  for (int t = 0; t < 3; ++t) res[t] = check_units_device(ctx, dsrc[t], n, dim);
  if (ix->dim == 0) {
    ix->dim = dim;
    // an index created with dim 0 has no storage yet: the int8 copy can start now
    ix->i8 = i8_wanted(dim);
  }
  for (int t = 0; t < 3; ++t) ix->dres[t] = std::max(ix->dres[t], res[t]);  // removals keep the max (conservative)
  ensure_capacity(ix, ix->n + n);
  for (int t = 0; t < 3; ++t) {
    float* dst = ix->rows[t] + (size_t)ix->n * dim;
    FC_CUDA(cudaMemcpyAsync(dst, dsrc[t], (size_t)n * dim * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    const int64_t cnt = (int64_t)n * dim;
    k_to_bf16<<<grid_for((cnt + 3) / 4, 256), 256, 0, ctx->stream>>>(dst, ix->rowsb[t] + (size_t)ix->n * dim, cnt);
    FC_LAUNCH_CHECK();
    count_launch(ctx);
    ix->plan[t].valid = false;
  }
  FC_CUDA(cudaMemcpyAsync(ix->ids_dev + ix->n, pid.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  for (int64_t i = 0; i < n; ++i) {
    ix->slot[pid[i]] = ix->n + i;
    ix->ids.push_back(pid[i]);
  }
  const int64_t n0 = ix->n;
  ix->n += n;
  requantize(ix, n0 / 128, (ix->n + 127) / 128);
  sync(ctx);
  LC_API_END
}

lc_status lc_index_insert(lc_index* ix, uint64_t prompt, const float* w, const float* o, const float* b, int dim) {
  return lc_index_insert_batch(ix, &prompt, w, o, b, 1, dim);
}

lc_status lc_index_remove(lc_index* ix, uint64_t prompt) {
  LC_API_BEGIN
  std::unique_lock lock(ix->mu);
  lc_ctx* ctx = ix->ctx;
  DeviceGuard g(ctx->device);
  auto it = ix->slot.find(prompt);
  if (it == ix->slot.end()) raise(LC_ERR_INVALID_ARGUMENT, "SimilarityIndex: unknown prompt id");
  const int64_t s = it->second, last = ix->n - 1;
  const int dim = ix->dim;
  if (s != last) {
    for (int t = 0; t < 3; ++t) {
      FC_CUDA(cudaMemcpyAsync(ix->rows[t] + (size_t)s * dim, ix->rows[t] + (size_t)last * dim, dim * sizeof(float),
                              cudaMemcpyDeviceToDevice, ctx->stream));
      FC_CUDA(cudaMemcpyAsync(ix->rowsb[t] + (size_t)s * dim, ix->rowsb[t] + (size_t)last * dim,
                              dim * sizeof(__nv_bfloat16), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    FC_CUDA(cudaMemcpyAsync(ix->ids_dev + s, ix->ids_dev + last, sizeof(uint64_t), cudaMemcpyDeviceToDevice, ctx->stream));
    const uint64_t moved = ix->ids[last];
    ix->ids[s] = moved;
    ix->slot[moved] = s;
  }
  ix->ids.pop_back();
  ix->slot.erase(it);
  ix->n -= 1;
  for (int t = 0; t < 3; ++t) ix->plan[t].valid = false;
  // the hole's tile got the last row; the last tile lost it
  // the hole's slot now holds the last row: re-quantize its tile (the other
  // rows of the last tile keep their valid quantization)
  if (s != last) requantize(ix, s / 128, s / 128 + 1);
  for (int t = 0; t < 3; ++t) ix->iplan[t].valid = false;
  sync(ctx);
  LC_API_END
}

lc_status lc_index_contains(lc_index* ix, uint64_t prompt, int32_t* out) {
  LC_API_BEGIN
  std::shared_lock lock(ix->mu);
  *out = ix->slot.count(prompt) ? 1 : 0;
  LC_API_END
}

int64_t lc_index_size(lc_index* ix) {
  std::shared_lock lock(ix->mu);
  return ix->n;
}

int lc_index_dim(lc_index* ix) { return ix->dim; }

lc_status lc_index_export(lc_index* ix, int kind, uint64_t* ids, float* rows, int64_t cap) {
  LC_API_BEGIN
  FC_REQUIRE(kind >= 0 && kind <= 2, "bad embedding kind");
  std::shared_lock lock(ix->mu);
  lc_ctx* ctx = ix->ctx;
  DeviceGuard g(ctx->device);
  FC_REQUIRE(cap >= ix->n, "lc_index_export: buffer too small");
  std::vector<int64_t> order(ix->n);
  for (int64_t i = 0; i < ix->n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return ix->ids[a] < ix->ids[b]; });
  std::vector<float> all((size_t)ix->n * ix->dim);
  if (ix->n) FC_CUDA(cudaMemcpy(all.data(), ix->rows[kind], all.size() * sizeof(float), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < ix->n; ++i) {
    if (ids) ids[i] = ix->ids[order[i]];
    if (rows) memcpy(rows + (size_t)i * ix->dim, all.data() + (size_t)order[i] * ix->dim, ix->dim * sizeof(float));
  }
  LC_API_END
}

lc_status lc_index_set_lookup(lc_index* ix, int mode, int kprime, double eps) {
  LC_API_BEGIN
  FC_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0, 1 or 2");
  FC_REQUIRE(kprime == 0 || (kprime >= 32 && kprime <= 128 && kprime % 32 == 0), "kprime: multiple of 32 in [32,128]");
  std::unique_lock lock(ix->mu);
  ix->mode = mode;
  if (kprime) ix->kprime = kprime;
  // eps > 0 is a floor on the certified bound (scaled by max(1, ||q||)):
  // it can only widen the proven per-query bound, never narrow it
  ix->eps_floor = eps > 0 ? eps : 0.0;
  LC_API_END
}

lc_status lc_index_stats(lc_index* ix, lc_lookup_stats* out, int reset) {
  LC_API_BEGIN
  std::unique_lock lock(ix->mu);
  std::lock_guard<std::mutex> sl(ix->stats_mu);
  if (out) *out = ix->stats;
  if (reset) ix->stats = lc_lookup_stats{};
  LC_API_END
}

lc_status lc_index_query_topk(lc_index* ix, int kind, const float* q, int64_t n, int k, uint64_t* out_ids,
                              double* out_scores, int32_t* out_counts) {
  LC_API_BEGIN
  FC_REQUIRE(kind >= 0 && kind <= 2, "bad embedding kind");
  FC_REQUIRE(k >= 1 && k <= 64, "k must be in [1, 64]");
  FC_REQUIRE(n >= 0 && n < (1ll << 31), "bad query count");
  std::shared_lock lock(ix->mu);
  lc_ctx* ctx = ix->ctx;
  DeviceGuard g(ctx->device);
  if (n == 0) return LC_OK;
  OutArg<uint64_t> oi(ctx, out_ids, (size_t)n * k, true);
  OutArg<double> os(ctx, out_scores, (size_t)n * k, true);
  OutArg<int32_t> oc(ctx, out_counts, (size_t)n, true);
  if (ix->n == 0) {  // empty table => nullopt (vindex.cpp:54)
    FC_CUDA(cudaMemsetAsync(oi.dev, 0, (size_t)n * k * sizeof(uint64_t), ctx->stream));
    FC_CUDA(cudaMemsetAsync(os.dev, 0, (size_t)n * k * sizeof(double), ctx->stream));
    FC_CUDA(cudaMemsetAsync(oc.dev, 0, (size_t)n * sizeof(int32_t), ctx->stream));
  } else {
    InArg<float> qa(ctx, q, (size_t)n * ix->dim);
    query_dev(ix, kind, qa.dev, (int)n, k, oi.dev, os.dev, oc.dev);
  }
  oi.finish(ctx);
  os.finish(ctx);
  oc.finish(ctx);
  sync(ctx);
  oi.deliver();
  os.deliver();
  oc.deliver();
  LC_API_END
}

lc_status lc_lookup_decide(lc_index* ix, const float* qw, const float* qo, const float* qb, int64_t n, double thr,
                           const double* edges4, lc_decision* out) {
  LC_API_BEGIN
  FC_REQUIRE(n >= 0 && n < (1ll << 31), "bad query count");
  if (n == 0) return LC_OK;
  lc_ctx* ctx = ix->ctx;
  DeviceGuard g(ctx->device);
  std::shared_lock lock(ix->mu);
  const double def[4] = {0.72, 0.79, 0.86, 0.93};
  const double* e = edges4 ? edges4 : def;
  DevBuf ids(3 * (size_t)n * sizeof(uint64_t), ctx->stream), sc(3 * (size_t)n * sizeof(double), ctx->stream),
      cnt(3 * (size_t)n * sizeof(int32_t), ctx->stream);
  OutArg<lc_decision> o(ctx, out, (size_t)n, true);
  if (ix->n == 0) {
    FC_CUDA(cudaMemsetAsync(ids.p, 0, ids.bytes, ctx->stream));
    FC_CUDA(cudaMemsetAsync(sc.p, 0, sc.bytes, ctx->stream));
    FC_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, ctx->stream));
  } else {
    const float* qs[3] = {qw, qo, qb};
    for (int t = 0; t < 3; ++t) {
      InArg<float> qa(ctx, qs[t], (size_t)n * ix->dim);
      query_dev(ix, t, qa.dev, (int)n, 1, ids.as<uint64_t>() + t * n, sc.as<double>() + t * n, cnt.as<int32_t>() + t * n);
    }
  }
  k_decide<<<grid_for(n, 128), 128, 0, ctx->stream>>>(ids.as<uint64_t>(), sc.as<double>(), ids.as<uint64_t>() + n,
                                                      sc.as<double>() + n, ids.as<uint64_t>() + 2 * n,
                                                      sc.as<double>() + 2 * n, cnt.as<int32_t>(), n, thr, e[0], e[1],
                                                      e[2], e[3], o.dev);
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  o.finish(ctx);
  sync(ctx);
  o.deliver();
  LC_API_END
}

}  // extern "C"
