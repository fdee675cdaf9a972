// lookup.cuh — interface of the tcgen05 candidate stage (lookup_sm100.cu).
//
// Error model behind the certification in index.cu (k_rescore). Operands are
// rounded to bf16 with round-to-nearest: q = bq + dq, x = bx + dx. Products
// of bf16 values are exact in fp32, so the tensor-core score differs from the
// exact dot q.x by
//   q.x - bq.bx = q.dx + dq.x - dq.dx           (rounding of the operands)
//   + fp32 accumulation of <= 1024 products      (<= 1024 * 2^-23 * ||bq|| ||bx||,
//                                                 any summation order)
// and Cauchy-Schwarz gives, for every stored row x,
//   |score - q.x| <= ||q|| dres + ||dq|| (||x|| + dres) + 2^-13 (||q|| + ||dq||)(||x|| + dres)
// with ||x|| <= 1 + 1e-6 (rows pass the from_unit rule, core.cpp:61-69) and
// dres = max over stored rows of ||dx|| (computed exactly on insert). For
// unit Gaussian-like rows dres ~ ||dq|| ~ 2^-8 / sqrt(12), so the bound is
// ~0.0025 instead of the worst case 2^-8 + 2^-12. The measured maximum error
// is reported in lc_lookup_stats.max_abs_err.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <functional>

#include "common.cuh"

namespace fc {


struct ApproxPlan {
  bool valid = false;
  int64_t n_rows = 0;
  int dim = 0;
  int bn = 64;
  const __nv_bfloat16* rows = nullptr;
  alignas(64) CUtensorMap tmap;   // box [bn rows][64]   (single-CTA kernel)
  alignas(64) CUtensorMap tmap2;  // box [bn/2 rows][64] (CTA-pair kernel: each CTA loads half a tile)
};

// ---- int8 candidate stage (tier 1 for dim % 128 == 0) ----
// Table rows are quantized per 128-row tile (the MMA tile): x = s_t * xq + dx
// with s_t = max|x| over the tile / 127 and xq = rint(x / s_t) in [-127, 127];
// queries per row: q = s_q * qq + dq. The s8 x s8 -> s32 tensor-core dot is
// exact, so with a = s_q s_t (qq . xq) (real arithmetic):
//   |q.x - a| = |dq.x + (s_q qq).dx| <= ||dq|| ||x|| + ||s_q qq|| ||dx||
//            <= ||dq|| X + ||qhat|| R8
// with X = max ||x|| <= 1 + 1e-6 (from_unit rule) and R8 = max over stored
// rows of ||dx|| (computed exactly when a tile is quantized). Typical bound
// for unit Gaussian-like 768-d rows: ~0.02 (bf16: ~0.004), which widens the
// shortlist to ~100-200 rows per query (CPU study: scripts/int8_cert_study.py)
// but runs the GEMM at the s8 tensor rate (2x bf16).
struct I8Plan {
  bool valid = false;
  int64_t n_rows = 0;
  int dim = 0;
  const int8_t* rows = nullptr;   // [n][dim] quantized rows
  const float* tscale = nullptr;  // [ceil(n/128)] tile scales
  const float* tres = nullptr;    // [ceil(n/128)] max residual norm of the tile's rows (rounded up)
  float r_typ = 0.f;              // median tile residual (threshold heuristic only)
  alignas(64) CUtensorMap tmap;   // box [64 rows][128 B] (each CTA of the pair loads half a tile)
};
void i8_plan(I8Plan& p, const int8_t* rows, const float* tscale, const float* tres, int64_t n_rows, int dim,
             float r_typ);
// Quantize tiles [t0, t1) of an fp32 table of n_rows rows into rows8/tscale
// (rows >= n_rows of the last tile become zero); each tile's max residual norm
// ||dx|| (rounded up) goes to tres and is max-reduced into *res_bits.
void i8_quantize_tiles(lc_ctx* ctx, const float* rows, int64_t n_rows, int dim, int64_t t0, int64_t t1, int8_t* rows8,
                       float* tscale, float* tres, unsigned long long* res_bits);
// Candidates of every query for a top-k: stored scores are U = a + eps_t, an
// upper bound of the exact dot q.x of the row (eps_t = the row's tile bound).
// Each unit keeps <= kp_unit rows, the merge the kout best U. cand_m[q] = an
// upper bound of U for EVERY row outside the output list (the max drop level
// of the units and the merge cut): rows outside have exact <= cand_m[q].
// tau_fix (device, per query; threshold tier): fixed U thresholds instead of
// the pilot/histogram heuristic -- every row with U > tau_fix[q] is kept
// (up to the query buffer), so cand_m[q] = tau_fix[q] unless it overflowed.
void i8_shortlist(lc_ctx* ctx, const I8Plan& p, const float* Qdev, int nq, int k, int kp_unit, int kout, float* cand_s,
                  uint32_t* cand_r, int32_t* cand_n, float* cand_m, const float* tau_fix = nullptr,
                  const std::function<void(float*, int)>* pilot_xchg = nullptr);
// Sharded int8 lookup: the pilot's per-query threshold key, exchanged across
// ranks (max) between the pilot and the main pass; a rank that runs no pilot
// (empty or small shard) takes part with -inf (dummy_pilot_exchange).
void dummy_pilot_exchange(lc_ctx* ctx, const std::function<void(float*, int)>& x, int nq);

// Sharded lookup: all-gathers per-query float bounds (device, n of them) and
// replaces each by its max over the ranks, on the context's stream.
using BoundExchange = std::function<void(float* bounds_dev, int n)>;

bool approx_available();
void approx_plan(ApproxPlan& p, const __nv_bfloat16* rows_bf16, int64_t n_rows, int dim, int sm_count);
// Shortlist: for each query the kp rows with the largest bf16 scores
// (cand_s approx score, cand_r row slot, cand_n count <= kp).
void approx_shortlist(lc_ctx* ctx, const ApproxPlan& p, const float* Qdev, int nq, int kp, float* cand_s,
                      uint32_t* cand_r, int32_t* cand_n);
// kernel-timer name of the shortlist launches ("shortlist"; the tier-2
// re-shortlist of uncertified queries is timed apart so per-launch averages
// of the main pass stay clean)
extern thread_local const char* g_shortlist_timer;
struct ShortlistTimerName {
  const char* prev;
  explicit ShortlistTimerName(const char* n) : prev(g_shortlist_timer) { g_shortlist_timer = n; }
  ~ShortlistTimerName() { g_shortlist_timer = prev; }
};

__global__ void k_decide(const uint64_t* wi, const double* ws, const uint64_t* oi, const double* os,
                         const uint64_t* bi, const double* bs, const int32_t* wc, int64_t n, double thr, double e0,
                         double e1, double e2, double e3, lc_decision* out);

}  // namespace fc
