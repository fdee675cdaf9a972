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
