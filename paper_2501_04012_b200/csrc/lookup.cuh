// lookup.cuh — interface of the tcgen05 candidate stage (lookup_sm100.cu).
//
// Error model behind the certification in index.cu: queries and rows are
// unit vectors (from_unit, core.cpp:61-69). Rounding each operand to bf16
// (unit roundoff 2^-9) perturbs each product q_i*x_i by at most
// |q_i x_i|(2^-8 + 2^-18), i.e. the dot by <= (2^-8 + 2^-18) * sum|q_i x_i|
// <= 2^-8 + 2^-18 (Cauchy-Schwarz). fp32 accumulation of dim <= 1024 terms
// adds <= 1024 * 2^-23 * sum|q_i x_i| ~ 1.2e-4. The default certified bound
// eps = 2^-8 + 2^-12 = 0.0041 covers both; the measured maximum is reported
// in lc_lookup_stats.max_abs_err.
// For a query of norm ||q|| != 1 every term above scales by ||q||, so the
// rescore uses eps * max(1, ||q||) per query (index.cu k_rescore); the bound
// cannot be lowered below kEpsBound through lc_index_set_lookup.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace fc {

constexpr double kEpsBound = 0.00390625 + 0.000244140625;  // 2^-8 + 2^-12

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
