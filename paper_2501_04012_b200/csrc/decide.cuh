// decide.cuh — the hit rule shared by the fused lookup kernel (core.cu) and
// the host-side engine (engine.cu): one definition, no drift.
#pragma once
#include "flexcache_b200.h"

namespace fc {

// decide + similarity_to_step.
__host__ __device__ inline void decide_one(double w, double o, double b, bool have, double thr, const double* e,
                           lc_decision* d) {
  d->whole_score = w;
  d->object_score = o;
  d->background_score = b;
  if (!have) {  // empty index: every request is a miss
    d->kind = LC_MISS;
    d->step = 0;
    d->score = 0.0;
    return;
  }
  const double m = o < b ? o : b;
  const double combined = w > m ? w : m;
  int kind;
  double score;
  if (combined < thr) {
    kind = LC_MISS;
    score = combined;
  } else if (m > w && m >= thr) {
    kind = LC_DECOUPLED_HIT;
    score = m;
  } else {
    kind = LC_WHOLE_HIT;
    score = w;
  }
  d->kind = kind;
  d->score = score;
  int step = 0;
  if (kind != LC_MISS) step = score < e[0] ? 5 : score < e[1] ? 10 : score < e[2] ? 15 : score < e[3] ? 20 : 25;
  d->step = step;
}

}  // namespace fc
