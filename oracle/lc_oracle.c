/*
 * lc_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference (FlexCache "lcache", /root/reference/proj) algorithms on the
 * north_star hot path. It is the CHECKER for the CUDA product, never part of
 * it: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.
 *
 * Parity pin: every function below is validated against the unmodified
 * reference library (oracle/_ref/liblcache_ref.so, built by oracle/Makefile)
 * in tests/test_oracle_vs_reference.py, and against the committed golden
 * fixtures generated from that library (tests/golden/, made by
 * tests/golden/make_golden.py).
 *
 * Citations are file:line into /root/reference/proj (src/, include/lcache/)
 * and /root/reference/SPEC.md.
 *
 * Numerics: compiled with -ffp-contract=off; every fp64 reduction is a plain
 * sequential loop in element order, as the reference's (CMake Release, no
 * -ffast-math, no -march) loops are.
 */
#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_abi.h"

static __thread char g_err[256];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }

#define CHECK(x)            \
  do {                      \
    int rc_ = (x);          \
    if (rc_ != ORC_OK) return rc_; \
  } while (0)

/* ------------------------------------------------------------------------ */
/* core                                                                      */
/* ------------------------------------------------------------------------ */

static int all_finite(const float* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* Embedding ctor, src/core.cpp:50-59: sq = sum v*v in fp64 (sequential),
 * inv = 1/sqrt(sq), v = (float)(v*inv). */
int orc_normalize(const float* v, int d, float* out) {
  if (d <= 0) return fail(ORC_ERR_INVALID_ARGUMENT, "Embedding: empty vector");
  if (!all_finite(v, d)) return fail(ORC_ERR_INVALID_ARGUMENT, "Embedding: non-finite element");
  double sq = 0.0;
  for (int i = 0; i < d; ++i) sq += (double)v[i] * (double)v[i];
  if (sq == 0.0) return fail(ORC_ERR_INVALID_ARGUMENT, "Embedding: zero norm");
  const double inv = 1.0 / sqrt(sq);
  for (int i = 0; i < d; ++i) out[i] = (float)((double)v[i] * inv);
  return ORC_OK;
}

/* Embedding::from_unit, src/core.cpp:61-69. */
static int check_unit(const float* v, int d) {
  if (d <= 0) return fail(ORC_ERR_INVALID_ARGUMENT, "Embedding: empty vector");
  if (!all_finite(v, d)) return fail(ORC_ERR_INVALID_ARGUMENT, "Embedding: non-finite element");
  double sq = 0.0;
  for (int i = 0; i < d; ++i) sq += (double)v[i] * (double)v[i];
  if (fabs(sqrt(sq) - 1.0) > 1e-6)
    return fail(ORC_ERR_INVALID_ARGUMENT, "Embedding: vector is not unit norm");
  return ORC_OK;
}

/* cosine_similarity, src/core.cpp:101-114: three sequential fp64 sums,
 * dot / (sqrt(na) * sqrt(nb)). */
int orc_cosine(const float* a, const float* b, int64_t n, double* out) {
  if (n <= 0) return fail(ORC_ERR_INVALID_ARGUMENT, "cosine_similarity: empty vectors");
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double x = a[i], y = b[i];
    dot += x * y;
    na += x * x;
    nb += y * y;
  }
  if (na == 0.0 || nb == 0.0)
    return fail(ORC_ERR_INVALID_ARGUMENT, "cosine_similarity: zero-norm operand");
  *out = dot / (sqrt(na) * sqrt(nb));
  return ORC_OK;
}

/* safe_similarity, src/codec.cpp:16-27: zero-tolerant cosine. */
static double safe_similarity(const float* a, const float* b, int64_t n) {
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double x = a[i], y = b[i];
    dot += x * y;
    na += x * x;
    nb += y * y;
  }
  if (na == 0.0 && nb == 0.0) return 1.0;
  if (na == 0.0 || nb == 0.0) return 0.0;
  return dot / (sqrt(na) * sqrt(nb));
}

/* ------------------------------------------------------------------------ */
/* vindex: three tables kept sorted by prompt id (vindex.hpp:50-55)          */
/* ------------------------------------------------------------------------ */

typedef struct {
  int dim;
  int64_t n, cap;
  uint64_t* ids;
  float* vals[3];
} OIndex;

void* orc_index_new(int dim) {
  OIndex* x = (OIndex*)calloc(1, sizeof(OIndex));
  x->dim = dim;
  return x;
}

void orc_index_free(void* h) {
  OIndex* x = (OIndex*)h;
  if (!x) return;
  free(x->ids);
  for (int t = 0; t < 3; ++t) free(x->vals[t]);
  free(x);
}

static int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* SimilarityIndex::insert, src/vindex.cpp:29-48 (dim fixed by first insert). */
int orc_index_insert(void* h, uint64_t id, const float* w, const float* o, const float* b, int d) {
  OIndex* x = (OIndex*)h;
  const float* e[3] = {w, o, b};
  for (int t = 0; t < 3; ++t) CHECK(check_unit(e[t], d));
  if (x->dim == 0) x->dim = d;
  if (d != x->dim) return fail(ORC_ERR_INVALID_ARGUMENT, "SimilarityIndex: embedding dimension mismatch");
  int64_t slot = lower_bound_u64(x->ids, x->n, id);
  if (slot < x->n && x->ids[slot] == id)
    return fail(ORC_ERR_INVALID_ARGUMENT, "SimilarityIndex: duplicate prompt id");
  if (x->n == x->cap) {
    x->cap = x->cap ? x->cap * 2 : 64;
    x->ids = (uint64_t*)realloc(x->ids, sizeof(uint64_t) * x->cap);
    for (int t = 0; t < 3; ++t) x->vals[t] = (float*)realloc(x->vals[t], sizeof(float) * x->cap * d);
  }
  memmove(x->ids + slot + 1, x->ids + slot, sizeof(uint64_t) * (x->n - slot));
  x->ids[slot] = id;
  for (int t = 0; t < 3; ++t) {
    memmove(x->vals[t] + (slot + 1) * d, x->vals[t] + slot * d, sizeof(float) * (x->n - slot) * d);
    memcpy(x->vals[t] + slot * d, e[t], sizeof(float) * d);
  }
  x->n++;
  return ORC_OK;
}

/* SimilarityIndex::remove, src/vindex.cpp:76-87. */
int orc_index_remove(void* h, uint64_t id) {
  OIndex* x = (OIndex*)h;
  int64_t slot = lower_bound_u64(x->ids, x->n, id);
  if (slot >= x->n || x->ids[slot] != id)
    return fail(ORC_ERR_INVALID_ARGUMENT, "SimilarityIndex: unknown prompt id");
  const int d = x->dim;
  memmove(x->ids + slot, x->ids + slot + 1, sizeof(uint64_t) * (x->n - slot - 1));
  for (int t = 0; t < 3; ++t)
    memmove(x->vals[t] + slot * d, x->vals[t] + (slot + 1) * d, sizeof(float) * (x->n - slot - 1) * d);
  x->n--;
  return ORC_OK;
}

int64_t orc_index_size(void* h) { return ((OIndex*)h)->n; }

/* Sequential fp64 dot of a stored row, src/vindex.cpp:66-67. */
static double row_dot(const float* q, const float* v, int d) {
  double dot = 0.0;
  for (int i = 0; i < d; ++i) dot += (double)q[i] * v[i];
  return dot;
}

/* query_top1, src/vindex.cpp:50-74: best starts at -2.0, strict '>' over
 * ascending ids => ties go to the smaller id; empty table => not found. */
int orc_index_query_top1(void* h, int kind, const float* q, int n, int d, int nthreads,
                         uint64_t* ids, double* scores, int32_t* found) {
  (void)nthreads;
  OIndex* x = (OIndex*)h;
  if (kind < 0 || kind > 2) return fail(ORC_ERR_INVALID_ARGUMENT, "bad kind");
  for (int i = 0; i < n; ++i) {
    const float* qi = q + (int64_t)i * d;
    CHECK(check_unit(qi, d));
    if (x->n == 0) {
      found[i] = 0; ids[i] = 0; scores[i] = 0.0;
      continue;
    }
    if (d != x->dim) return fail(ORC_ERR_INVALID_ARGUMENT, "SimilarityIndex: query dimension mismatch");
    double best = -2.0;
    int64_t bi = 0;
    for (int64_t r = 0; r < x->n; ++r) {
      double s = row_dot(qi, x->vals[kind] + r * d, d);
      if (s > best) { best = s; bi = r; }
    }
    found[i] = 1; ids[i] = x->ids[bi]; scores[i] = best;
  }
  return ORC_OK;
}

/* Top-k generalisation of query_top1 (vindex.cpp:58-72): order by
 * (score desc, id asc); k = 1 reproduces query_top1 exactly. Row order of
 * the table is irrelevant because ties are broken by id, not position. */
int orc_topk_flat(const float* table, const uint64_t* ids, int64_t n_rows, int d,
                  const float* q, int n_q, int k, uint64_t* out_ids, double* out_scores,
                  int32_t* out_counts) {
  if (k <= 0) return fail(ORC_ERR_INVALID_ARGUMENT, "k must be positive");
  double* bs = (double*)malloc(sizeof(double) * k);
  uint64_t* bi = (uint64_t*)malloc(sizeof(uint64_t) * k);
  for (int i = 0; i < n_q; ++i) {
    const float* qi = q + (int64_t)i * d;
    int cnt = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
      double s = row_dot(qi, table + r * d, d);
      uint64_t id = ids[r];
      /* insertion into the ordered list if it beats the current last */
      int pos = cnt;
      while (pos > 0 && (s > bs[pos - 1] || (s == bs[pos - 1] && id < bi[pos - 1]))) --pos;
      if (pos >= k) continue;
      int last = cnt < k ? cnt : k - 1;
      for (int j = last; j > pos; --j) { bs[j] = bs[j - 1]; bi[j] = bi[j - 1]; }
      bs[pos] = s; bi[pos] = id;
      if (cnt < k) ++cnt;
    }
    out_counts[i] = cnt;
    for (int j = 0; j < k; ++j) {
      out_ids[(int64_t)i * k + j] = j < cnt ? bi[j] : 0;
      out_scores[(int64_t)i * k + j] = j < cnt ? bs[j] : 0.0;
    }
  }
  free(bs); free(bi);
  return ORC_OK;
}

/* decide, SPEC.md:484-492 (no reference code). */
int orc_decide(double w, double o, double b, double threshold, int32_t* kind, double* score) {
  const double m = o < b ? o : b;
  const double combined = w > m ? w : m;
  if (combined < threshold) { *kind = 0; *score = combined; return ORC_OK; }
  if (m > w && m >= threshold) { *kind = 2; *score = m; return ORC_OK; }
  *kind = 1; *score = w;
  return ORC_OK;
}

/* similarity_to_step; bins defaults.hpp:27. */
int orc_similarity_to_step(double score, double threshold, const double* e, int32_t* step) {
  if (!(score >= threshold)) return fail(ORC_ERR_INVALID_ARGUMENT, "score below threshold");
  if (score < e[0]) *step = 5;
  else if (score < e[1]) *step = 10;
  else if (score < e[2]) *step = 15;
  else if (score < e[3]) *step = 20;
  else *step = 25;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* codec                                                                     */
/* ------------------------------------------------------------------------ */

static int valid_step_id(int s) { return s >= 1 && s <= 50; } /* core.cpp:29-32 */

/* select_keyframes, src/codec.cpp:138-165: FORWARD greedy; frame j compared
 * with the current keys in ascending order, best = max sim >= thr with strict
 * '>' (ties to the earlier key); otherwise j becomes a key. */
static int select_keyframes_impl(const float* frames, int F, int64_t E, double thr, int32_t* map) {
  if (thr <= 0.0 || thr > 1.0)
    return fail(ORC_ERR_INVALID_ARGUMENT, "select_keyframes: threshold must be in (0, 1]");
  int32_t* keys = (int32_t*)malloc(sizeof(int32_t) * F);
  int nk = 0;
  map[0] = 0;
  keys[nk++] = 0;
  for (int j = 1; j < F; ++j) {
    int best = -1;
    double best_sim = 0.0;
    for (int t = 0; t < nk; ++t) {
      const int k = keys[t];
      double sim;
      int rc = orc_cosine(frames + (int64_t)j * E, frames + (int64_t)k * E, E, &sim);
      if (rc != ORC_OK) { free(keys); return rc; }
      if (sim >= thr && (best < 0 || sim > best_sim)) { best = k; best_sim = sim; }
    }
    if (best < 0) { map[j] = j; keys[nk++] = j; }
    else map[j] = best;
  }
  free(keys);
  return ORC_OK;
}

static int check_dims(int F, int H, int W, int C) {
  if (H <= 0 || W <= 0 || C <= 0) return fail(ORC_ERR_INVALID_ARGUMENT, "Frame: dimensions must be positive");
  if (F <= 0) return fail(ORC_ERR_INVALID_ARGUMENT, "LatentState: needs at least one frame");
  return ORC_OK;
}

int orc_select_keyframes(const float* frames, int F, int H, int W, int C, double thr, int32_t* map) {
  CHECK(check_dims(F, H, W, C));
  const int64_t E = (int64_t)H * W * C;
  if (!all_finite(frames, E * F)) return fail(ORC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
  return select_keyframes_impl(frames, F, E, thr, map);
}

/* solve_alpha, src/codec.cpp:181-191. */
int orc_solve_alpha(const float* ds, const float* db, int64_t n, float* out) {
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    num += (double)ds[i] * db[i];
    den += (double)db[i] * db[i];
  }
  if (den == 0.0) return fail(ORC_ERR_DEGENERATE_BASE, "solve_alpha: base differential is identically zero");
  *out = (float)(num / den);
  return ORC_OK;
}

/* In-memory CompressedEntry (codec.hpp:48-67). Frame pointers either borrow
 * the caller's latent buffer or point into owned storage. */
typedef struct {
  int step;
  const float* first;
  int32_t* map;          /* F */
  int n_alpha;
  int32_t* alpha_idx;    /* ascending */
  float* alpha;
  int n_extra;
  int32_t* extra_idx;    /* ascending */
  const float** extra;
} OStep;

typedef struct {
  uint64_t prompt;
  int base_step;
  int F, H, W, C;
  int64_t E, mb;
  int n_steps;
  OStep* steps;
  int n_diff;
  int32_t* diff_idx;     /* ascending */
  const float** diff;
  const uint8_t* obj_masks; /* F*mb */
  const uint8_t* bg_masks;
  /* owned storage to free */
  void** owned;
  int n_owned, cap_owned;
} OEntry;

static void* own(OEntry* e, size_t bytes) {
  void* p = calloc(1, bytes ? bytes : 1);
  if (e->n_owned == e->cap_owned) {
    e->cap_owned = e->cap_owned ? e->cap_owned * 2 : 64;
    e->owned = (void**)realloc(e->owned, sizeof(void*) * e->cap_owned);
  }
  e->owned[e->n_owned++] = p;
  return p;
}

static void adopt(OEntry* e, void* p) {
  if (e->n_owned == e->cap_owned) {
    e->cap_owned = e->cap_owned ? e->cap_owned * 2 : 64;
    e->owned = (void**)realloc(e->owned, sizeof(void*) * e->cap_owned);
  }
  e->owned[e->n_owned++] = p;
}

static void entry_free(OEntry* e) {
  for (int i = 0; i < e->n_owned; ++i) free(e->owned[i]);
  free(e->owned);
  memset(e, 0, sizeof *e);
}

static int find_idx(const int32_t* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) { int m = (lo + hi) / 2; if (a[m] < v) lo = m + 1; else hi = m; }
  return (lo < n && a[lo] == v) ? lo : -1;
}

static int is_all_zero(const float* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i) if (v[i] != 0.0f) return 0;
  return 1;
}

/* Per-step intra view: key frames live in the caller's latent buffer. */
typedef struct {
  int step;
  const float* frames;   /* F*E (only key frames are read) */
  int32_t* map;
  int nk;
  int32_t* keys;         /* ascending */
  float** diff;          /* per key position: key - first (NULL for key 0) */
} OIntra;

/* build_entry, src/codec.cpp:52-108. */
static int build_entry(OIntra* st, int S, int b, const int32_t* common, int nc, OEntry* out,
                       uint64_t prompt, int F, int H, int W, int C, const uint8_t* om, const uint8_t* bm) {
  const int64_t E = (int64_t)H * W * C;
  memset(out, 0, sizeof *out);
  out->prompt = prompt;
  out->base_step = st[b].step;
  out->F = F; out->H = H; out->W = W; out->C = C; out->E = E;
  out->mb = ((int64_t)H * W + 7) / 8;
  out->obj_masks = om; out->bg_masks = bm;
  out->n_steps = S;
  out->steps = (OStep*)own(out, sizeof(OStep) * S);
  out->diff_idx = (int32_t*)own(out, sizeof(int32_t) * (nc + 1));
  out->diff = (const float**)own(out, sizeof(float*) * (nc + 1));
  /* base diffs: common indices (m > 0) whose base differential is nonzero */
  for (int c = 0; c < nc; ++c) {
    const int m = common[c];
    if (m == 0) continue;
    const int kp = find_idx(st[b].keys, st[b].nk, m);
    const float* d = st[b].diff[kp];
    if (!is_all_zero(d, E)) {
      out->diff_idx[out->n_diff] = m;
      out->diff[out->n_diff] = d;
      out->n_diff++;
    }
  }
  for (int si = 0; si < S; ++si) {
    OIntra* ic = &st[si];
    OStep* rec = &out->steps[si];
    rec->step = ic->step;
    rec->first = ic->frames;
    rec->map = ic->map;
    rec->alpha_idx = (int32_t*)own(out, sizeof(int32_t) * ic->nk);
    rec->alpha = (float*)own(out, sizeof(float) * ic->nk);
    rec->extra_idx = (int32_t*)own(out, sizeof(int32_t) * ic->nk);
    rec->extra = (const float**)own(out, sizeof(float*) * ic->nk);
    for (int kp = 0; kp < ic->nk; ++kp) {
      const int m = ic->keys[kp];
      if (m == 0) continue;
      const float* key = ic->frames + (int64_t)m * E;
      if (find_idx(common, nc, m) < 0) {
        rec->extra_idx[rec->n_extra] = m; rec->extra[rec->n_extra++] = key;
        continue;
      }
      const int dpos = find_idx(out->diff_idx, out->n_diff, m);
      if (dpos < 0) {
        if (!is_all_zero(ic->diff[kp], E)) { rec->extra_idx[rec->n_extra] = m; rec->extra[rec->n_extra++] = key; }
        continue;
      }
      const float* bd = out->diff[dpos];
      if (si == b) {
        /* reconstructs_exactly, codec.cpp:41-46 */
        int exact = 1;
        for (int64_t i = 0; i < E; ++i)
          if (rec->first[i] + bd[i] != key[i]) { exact = 0; break; }
        if (!exact) { rec->extra_idx[rec->n_extra] = m; rec->extra[rec->n_extra++] = key; }
      } else {
        float alpha;
        CHECK(orc_solve_alpha(ic->diff[kp], bd, E, &alpha));
        if (!isfinite(alpha)) {
          rec->extra_idx[rec->n_extra] = m; rec->extra[rec->n_extra++] = key;
          rec->alpha_idx[rec->n_alpha] = m; rec->alpha[rec->n_alpha++] = 0.0f;
        } else {
          rec->alpha_idx[rec->n_alpha] = m; rec->alpha[rec->n_alpha++] = alpha;
        }
      }
    }
  }
  return ORC_OK;
}

/* decompress_step, src/codec.cpp:263-301. Writes F*E floats. */
static int decompress_impl(const OEntry* e, int step, float* out) {
  const OStep* rec = NULL;
  for (int s = 0; s < e->n_steps; ++s) if (e->steps[s].step == step) rec = &e->steps[s];
  if (!rec) return fail(ORC_ERR_STEP_NOT_CACHED, "step %d not in entry", step);
  const int64_t E = e->E;
  const int F = e->F;
  for (int m = 0; m < F; ++m) {
    if (rec->map[m] != m) continue; /* keys only */
    float* dst = out + (int64_t)m * E;
    if (m == 0) { memcpy(dst, rec->first, sizeof(float) * E); continue; }
    const int xp = find_idx(rec->extra_idx, rec->n_extra, m);
    if (xp >= 0) { memcpy(dst, rec->extra[xp], sizeof(float) * E); continue; }
    const int dp = find_idx(e->diff_idx, e->n_diff, m);
    if (dp < 0) { memcpy(dst, rec->first, sizeof(float) * E); continue; }
    const float* bd = e->diff[dp];
    if (step == e->base_step) {
      for (int64_t i = 0; i < E; ++i) dst[i] = rec->first[i] + bd[i];
    } else {
      const int ap = find_idx(rec->alpha_idx, rec->n_alpha, m);
      if (ap < 0) return fail(ORC_ERR_LOGIC, "map::at: missing alpha");
      const double alpha = rec->alpha[ap];
      for (int64_t i = 0; i < E; ++i) dst[i] = (float)(rec->first[i] + alpha * bd[i]);
    }
    /* Frame ctor finite check, core.cpp:19-25 */
    if (!all_finite(dst, E)) return fail(ORC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
  }
  for (int j = 0; j < F; ++j) {
    const int m = rec->map[j];
    if (m != j) memcpy(out + (int64_t)j * E, out + (int64_t)m * E, sizeof(float) * E);
  }
  return ORC_OK;
}

/* Size accounting, src/codec.cpp:305-332. */
static uint64_t shared_bytes(const OEntry* e) {
  return 20ull + (uint64_t)e->n_diff * (2 + 4ull * e->E) + 2ull * e->F * (uint64_t)e->mb;
}
static uint64_t private_bytes(const OEntry* e, const OStep* r) {
  uint64_t n = 1 + 4ull * e->E + 2ull * e->F;
  if (r->step != e->base_step) n += 4ull * r->n_alpha;
  n += 2 + (uint64_t)r->n_extra * (2 + 4ull * e->E);
  return n;
}

/* serialize_entry, src/codec.cpp:358-392 (little-endian). */
typedef struct { uint8_t* p; uint64_t n, cap; } OBuf;
static void put(OBuf* b, const void* src, uint64_t n) {
  if (b->p && b->n + n <= b->cap) memcpy(b->p + b->n, src, n);
  b->n += n;
}
static void put_u8(OBuf* b, uint8_t v) { put(b, &v, 1); }
static void put_u16(OBuf* b, uint16_t v) { uint8_t t[2] = {(uint8_t)v, (uint8_t)(v >> 8)}; put(b, t, 2); }
static void put_u64(OBuf* b, uint64_t v) { uint8_t t[8]; for (int i = 0; i < 8; ++i) t[i] = (uint8_t)(v >> (8 * i)); put(b, t, 8); }
static void put_f32s(OBuf* b, const float* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i) { uint32_t u; memcpy(&u, &v[i], 4); uint8_t t[4] = {(uint8_t)u, (uint8_t)(u >> 8), (uint8_t)(u >> 16), (uint8_t)(u >> 24)}; put(b, t, 4); }
}

static void serialize(const OEntry* e, OBuf* b) {
  put_u64(b, e->prompt);
  put_u8(b, (uint8_t)e->base_step);
  put_u8(b, (uint8_t)e->n_steps);
  put_u16(b, (uint16_t)e->n_diff);
  put_u16(b, (uint16_t)e->F);
  put_u16(b, (uint16_t)e->H);
  put_u16(b, (uint16_t)e->W);
  put_u16(b, (uint16_t)e->C);
  for (int s = 0; s < e->n_steps; ++s) {
    const OStep* r = &e->steps[s];
    put_u8(b, (uint8_t)r->step);
    put_f32s(b, r->first, e->E);
    for (int j = 0; j < e->F; ++j) put_u16(b, (uint16_t)r->map[j]);
    if (r->step != e->base_step) put_f32s(b, r->alpha, r->n_alpha);
    put_u16(b, (uint16_t)r->n_extra);
    for (int x = 0; x < r->n_extra; ++x) { put_u16(b, (uint16_t)r->extra_idx[x]); put_f32s(b, r->extra[x], e->E); }
  }
  for (int d = 0; d < e->n_diff; ++d) { put_u16(b, (uint16_t)e->diff_idx[d]); put_f32s(b, e->diff[d], e->E); }
  put(b, e->obj_masks, (uint64_t)e->F * e->mb);
  put(b, e->bg_masks, (uint64_t)e->F * e->mb);
}

static void intra_free(OIntra* st, int S) {
  for (int s = 0; s < S; ++s) {
    if (st[s].diff) for (int k = 0; k < st[s].nk; ++k) free(st[s].diff[k]);
    free(st[s].diff); free(st[s].map); free(st[s].keys);
  }
  free(st);
}

/* intra_compress x S (codec.cpp:167-172) + inter_compress (codec.cpp:193-261).
 * On success *out owns the chosen entry (frames borrowed from lat). */
static int compress_impl(const float* lat, const int32_t* steps, int S, int F, int H, int W, int C,
                         const uint8_t* om, const uint8_t* bm, double thr, uint64_t prompt, OEntry* out) {
  CHECK(check_dims(F, H, W, C));
  const int64_t E = (int64_t)H * W * C;
  if (S <= 0) return fail(ORC_ERR_INVALID_ARGUMENT, "inter_compress: empty step list");
  OIntra* st = (OIntra*)calloc(S, sizeof(OIntra));
  int rc = ORC_OK;
  /* intra_compress per input step (LatentState ctor validates frames) */
  for (int s = 0; s < S && rc == ORC_OK; ++s) {
    if (!valid_step_id(steps[s])) { rc = fail(ORC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50"); break; }
    const float* fr = lat + (int64_t)s * F * E;
    if (!all_finite(fr, (int64_t)F * E)) { rc = fail(ORC_ERR_INVALID_ARGUMENT, "Frame: non-finite element"); break; }
    st[s].step = steps[s];
    st[s].frames = fr;
    st[s].map = (int32_t*)malloc(sizeof(int32_t) * F);
    rc = select_keyframes_impl(fr, F, E, thr, st[s].map);
  }
  if (rc != ORC_OK) { intra_free(st, S); return rc; }
  /* sort steps ascending (codec.cpp:197-199); stable insertion sort */
  for (int i = 1; i < S; ++i) {
    OIntra t = st[i]; int j = i;
    while (j > 0 && st[j - 1].step > t.step) { st[j] = st[j - 1]; --j; }
    st[j] = t;
  }
  for (int i = 1; i < S; ++i)
    if (st[i].step == st[i - 1].step) { intra_free(st, S); return fail(ORC_ERR_INVALID_ARGUMENT, "inter_compress: duplicate step"); }
  /* keys, diffs (codec.cpp:222-230) */
  for (int s = 0; s < S; ++s) {
    st[s].keys = (int32_t*)malloc(sizeof(int32_t) * F);
    st[s].nk = 0;
    for (int j = 0; j < F; ++j) if (st[s].map[j] == j) st[s].keys[st[s].nk++] = j;
    st[s].diff = (float**)calloc(st[s].nk, sizeof(float*));
    for (int k = 0; k < st[s].nk; ++k) {
      const int m = st[s].keys[k];
      if (m == 0) continue;
      float* d = (float*)malloc(sizeof(float) * E);
      const float* key = st[s].frames + (int64_t)m * E;
      for (int64_t i = 0; i < E; ++i) d[i] = key[i] - st[s].frames[i];
      st[s].diff[k] = d;
    }
  }
  /* common key indices (codec.cpp:213-220) */
  int32_t* common = (int32_t*)malloc(sizeof(int32_t) * F);
  int nc = 0;
  for (int j = 0; j < F; ++j) {
    int all = 1;
    for (int s = 0; s < S; ++s) if (st[s].map[j] != j) { all = 0; break; }
    if (all) common[nc++] = j;
  }
  if (S == 1) {
    rc = build_entry(st, S, 0, common, nc, out, prompt, F, H, W, C, om, bm);
  } else {
    double best_score = -2.0;
    int have = 0;
    float* recon = (float*)malloc(sizeof(float) * F * E);
    for (int b = 0; b < S && rc == ORC_OK; ++b) {
      OEntry trial;
      rc = build_entry(st, S, b, common, nc, &trial, prompt, F, H, W, C, om, bm);
      if (rc != ORC_OK) { entry_free(&trial); break; }
      double sum = 0.0;
      uint64_t count = 0;
      for (int si = 0; si < S && rc == ORC_OK; ++si) {
        rc = decompress_impl(&trial, st[si].step, recon);
        if (rc != ORC_OK) break;
        for (int j = 0; j < F; ++j) {
          /* ref = intra_decompress: frame j = key map[j] (codec.cpp:174-179) */
          const float* ref = st[si].frames + (int64_t)st[si].map[j] * E;
          sum += safe_similarity(recon + (int64_t)j * E, ref, E);
          ++count;
        }
      }
      if (rc != ORC_OK) { entry_free(&trial); break; }
      const double score = sum / (double)count;
      if (score > best_score) {
        best_score = score;
        if (have) entry_free(out);
        *out = trial;
        have = 1;
      } else {
        entry_free(&trial);
      }
    }
    free(recon);
  }
  free(common);
  if (rc != ORC_OK) { intra_free(st, S); return rc; }
  /* Transfer ownership of maps/diffs (borrowed by *out) into the entry. */
  for (int s = 0; s < S; ++s) {
    adopt(out, st[s].map);
    for (int k = 0; k < st[s].nk; ++k) if (st[s].diff[k]) adopt(out, st[s].diff[k]);
    free(st[s].diff); free(st[s].keys);
  }
  free(st);
  return ORC_OK;
}

int orc_compress(const float* lat, const int32_t* steps, int S, int F, int H, int W, int C,
                 const uint8_t* om, const uint8_t* bm, double thr, uint64_t prompt,
                 uint8_t* out, uint64_t cap, uint64_t* out_len) {
  OEntry e;
  memset(&e, 0, sizeof e);
  CHECK(compress_impl(lat, steps, S, F, H, W, C, om, bm, thr, prompt, &e));
  OBuf b = {NULL, 0, 0};
  serialize(&e, &b); /* sizing pass */
  *out_len = b.n;
  uint64_t expect = shared_bytes(&e);
  for (int s = 0; s < e.n_steps; ++s) expect += private_bytes(&e, &e.steps[s]);
  if (expect != b.n) { entry_free(&e); return fail(ORC_ERR_LOGIC, "size accounting mismatch"); }
  if (out) {
    if (b.n > cap) { entry_free(&e); return fail(ORC_ERR_INVALID_ARGUMENT, "output buffer too small"); }
    OBuf w = {out, 0, cap};
    serialize(&e, &w);
  }
  entry_free(&e);
  return ORC_OK;
}

typedef struct {
  const float* lat; const int32_t* steps; int S, F, H, W, C;
  const uint8_t *om, *bm; double thr; const uint64_t* prompts; int n, nthreads, t;
  uint64_t* sizes; int rc;
} BatchJob;

static void* batch_worker(void* arg) {
  BatchJob* j = (BatchJob*)arg;
  const int64_t E = (int64_t)j->H * j->W * j->C;
  const int64_t ent = (int64_t)j->S * j->F * E;
  const int64_t mb = (int64_t)j->F * (((int64_t)j->H * j->W + 7) / 8);
  for (int i = j->t; i < j->n; i += j->nthreads) {
    j->rc = orc_compress(j->lat + i * ent, j->steps, j->S, j->F, j->H, j->W, j->C, j->om + i * mb,
                         j->bm + i * mb, j->thr, j->prompts[i], NULL, 0, &j->sizes[i]);
    if (j->rc != ORC_OK) break;
  }
  return NULL;
}

int orc_compress_batch(const float* lat, const int32_t* steps, int S, int F, int H, int W, int C,
                       const uint8_t* om, const uint8_t* bm, double thr, const uint64_t* prompts,
                       int n, int nthreads, uint64_t* out_sizes) {
  if (nthreads < 1) nthreads = 1;
  BatchJob* jobs = (BatchJob*)calloc(nthreads, sizeof(BatchJob));
  pthread_t* th = (pthread_t*)calloc(nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (BatchJob){lat, steps, S, F, H, W, C, om, bm, thr, prompts, n, nthreads, t, out_sizes, ORC_OK};
    pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
  }
  int rc = ORC_OK;
  for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); if (jobs[t].rc != ORC_OK) rc = jobs[t].rc; }
  free(jobs); free(th);
  return rc;
}

/* deserialize_entry, src/codec.cpp:394-473 (validation subset that decides
 * success/failure; positions are not reported). Frames are copied into owned
 * aligned storage. */
typedef struct { const uint8_t* p; uint64_t n, pos; int bad; } ORd;
static void need(ORd* r, uint64_t k) { if (r->pos + k > r->n) r->bad = 1; }
static uint8_t rd_u8(ORd* r) { need(r, 1); if (r->bad) return 0; return r->p[r->pos++]; }
static uint16_t rd_u16(ORd* r) { need(r, 2); if (r->bad) return 0; uint16_t v = (uint16_t)(r->p[r->pos] | (r->p[r->pos + 1] << 8)); r->pos += 2; return v; }
static uint64_t rd_u64(ORd* r) { need(r, 8); if (r->bad) return 0; uint64_t v = 0; for (int i = 0; i < 8; ++i) v |= (uint64_t)r->p[r->pos + i] << (8 * i); r->pos += 8; return v; }
static void rd_f32s(ORd* r, float* out, int64_t n) {
  need(r, 4ull * n); if (r->bad) return;
  for (int64_t i = 0; i < n; ++i) { uint32_t u = (uint32_t)r->p[r->pos] | ((uint32_t)r->p[r->pos + 1] << 8) | ((uint32_t)r->p[r->pos + 2] << 16) | ((uint32_t)r->p[r->pos + 3] << 24); memcpy(&out[i], &u, 4); r->pos += 4; }
}

static int parse_entry(const uint8_t* p, uint64_t len, OEntry* e) {
  memset(e, 0, sizeof *e);
  ORd r = {p, len, 0, 0};
  e->prompt = rd_u64(&r);
  e->base_step = rd_u8(&r);
  e->n_steps = rd_u8(&r);
  e->n_diff = rd_u16(&r);
  e->F = rd_u16(&r);
  e->H = rd_u16(&r); e->W = rd_u16(&r); e->C = rd_u16(&r);
  if (r.bad) return fail(ORC_ERR_SNAPSHOT, "truncated input");
  if (e->n_steps < 1 || e->F < 1 || e->H < 1 || e->W < 1 || e->C < 1) return fail(ORC_ERR_SNAPSHOT, "invalid entry header");
  if (!valid_step_id(e->base_step)) return fail(ORC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
  e->E = (int64_t)e->H * e->W * e->C;
  e->mb = ((int64_t)e->H * e->W + 7) / 8;
  const int64_t E = e->E;
  e->steps = (OStep*)own(e, sizeof(OStep) * e->n_steps);
  float** raw_alpha = (float**)own(e, sizeof(float*) * e->n_steps);
  for (int s = 0; s < e->n_steps; ++s) {
    OStep* rec = &e->steps[s];
    rec->step = rd_u8(&r);
    if (r.bad) return fail(ORC_ERR_SNAPSHOT, "truncated input");
    if (!valid_step_id(rec->step)) return fail(ORC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
    float* first = (float*)own(e, sizeof(float) * E);
    rd_f32s(&r, first, E);
    rec->first = first;
    rec->map = (int32_t*)own(e, sizeof(int32_t) * e->F);
    for (int j = 0; j < e->F; ++j) {
      rec->map[j] = rd_u16(&r);
      if (!r.bad && rec->map[j] >= e->F) return fail(ORC_ERR_SNAPSHOT, "key frame map index out of range");
    }
    if (r.bad) return fail(ORC_ERR_SNAPSHOT, "truncated input");
    if (!all_finite(first, E)) return fail(ORC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
    if (rec->step != e->base_step) {
      raw_alpha[s] = (float*)own(e, sizeof(float) * (e->n_diff + 1));
      rd_f32s(&r, raw_alpha[s], e->n_diff);
    }
    rec->n_extra = rd_u16(&r);
    if (r.bad) return fail(ORC_ERR_SNAPSHOT, "truncated input");
    rec->extra_idx = (int32_t*)own(e, sizeof(int32_t) * (rec->n_extra + 1));
    rec->extra = (const float**)own(e, sizeof(float*) * (rec->n_extra + 1));
    int n_unique = 0;
    for (int x = 0; x < rec->n_extra; ++x) {
      const int m = rd_u16(&r);
      if (r.bad) return fail(ORC_ERR_SNAPSHOT, "truncated input");
      if (m >= e->F) return fail(ORC_ERR_SNAPSHOT, "extra frame index out of range");
      float* fr = (float*)own(e, sizeof(float) * E);
      rd_f32s(&r, fr, E);
      if (r.bad) return fail(ORC_ERR_SNAPSHOT, "truncated input");
      if (!all_finite(fr, E)) return fail(ORC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
      /* std::map::emplace keeps the first of duplicate keys; keep ascending */
      int pos = n_unique, dup = 0;
      for (int q = 0; q < n_unique; ++q) if (rec->extra_idx[q] == m) { dup = 1; break; }
      if (dup) continue;
      while (pos > 0 && rec->extra_idx[pos - 1] > m) { rec->extra_idx[pos] = rec->extra_idx[pos - 1]; rec->extra[pos] = rec->extra[pos - 1]; --pos; }
      rec->extra_idx[pos] = m; rec->extra[pos] = fr; ++n_unique;
    }
    rec->n_extra = n_unique;
    if (s > 0 && !(e->steps[s - 1].step < rec->step)) return fail(ORC_ERR_SNAPSHOT, "steps out of order");
  }
  e->diff_idx = (int32_t*)own(e, sizeof(int32_t) * (e->n_diff + 1));
  e->diff = (const float**)own(e, sizeof(float*) * (e->n_diff + 1));
  for (int d = 0; d < e->n_diff; ++d) {
    const int m = rd_u16(&r);
    if (r.bad) return fail(ORC_ERR_SNAPSHOT, "truncated input");
    if (m < 1 || m >= e->F) return fail(ORC_ERR_SNAPSHOT, "diff index out of range");
    float* fr = (float*)own(e, sizeof(float) * E);
    rd_f32s(&r, fr, E);
    if (r.bad) return fail(ORC_ERR_SNAPSHOT, "truncated input");
    e->diff_idx[d] = m; e->diff[d] = fr;
  }
  for (int d = 1; d < e->n_diff; ++d)
    if (e->diff_idx[d] < e->diff_idx[d - 1]) return fail(ORC_ERR_SNAPSHOT, "diff indices out of order");
  for (int d = 1; d < e->n_diff; ++d)
    if (e->diff_idx[d] == e->diff_idx[d - 1]) return fail(ORC_ERR_INTERNAL, "duplicate diff index (unsupported)");
  for (int s = 0; s < e->n_steps; ++s) {
    OStep* rec = &e->steps[s];
    if (rec->step == e->base_step) continue;
    rec->n_alpha = e->n_diff;
    rec->alpha_idx = e->diff_idx;
    rec->alpha = raw_alpha[s];
  }
  need(&r, 2ull * e->F * e->mb);
  if (r.bad) return fail(ORC_ERR_SNAPSHOT, "truncated input");
  e->obj_masks = p + r.pos;
  e->bg_masks = p + r.pos + e->F * e->mb;
  r.pos += 2ull * e->F * e->mb;
  if (r.pos != len) return fail(ORC_ERR_SNAPSHOT, "trailing bytes");
  return ORC_OK;
}

int orc_decompress(const uint8_t* entry, uint64_t len, int step, float* out) {
  OEntry e;
  int rc = parse_entry(entry, len, &e);
  if (rc == ORC_OK) {
    if (!valid_step_id(step)) rc = fail(ORC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
    else rc = decompress_impl(&e, step, out);
  }
  entry_free(&e);
  return rc;
}

int orc_entry_info(const uint8_t* entry, uint64_t len, int32_t* base_step, int32_t* n_steps,
                   int32_t* steps, uint64_t* sh, uint64_t* pr) {
  OEntry e;
  int rc = parse_entry(entry, len, &e);
  if (rc == ORC_OK) {
    *base_step = e.base_step;
    *n_steps = e.n_steps;
    *sh = shared_bytes(&e);
    for (int s = 0; s < e.n_steps; ++s) { steps[s] = e.steps[s].step; pr[s] = private_bytes(&e, &e.steps[s]); }
  }
  entry_free(&e);
  return rc;
}

/* stitch, src/stitcher.cpp:7-39: object pixel iff the object source's object
 * mask OR the background source's object mask is set. Background masks of
 * either source are never read. */
int orc_stitch(const float* obj, const uint8_t* oo, const uint8_t* ob, const float* bg,
               const uint8_t* bo, const uint8_t* bb, int F, int H, int W, int C, float* out) {
  (void)ob; (void)bb;
  CHECK(check_dims(F, H, W, C));
  const int64_t E = (int64_t)H * W * C, P = (int64_t)H * W, mb = (P + 7) / 8;
  if (!all_finite(obj, F * E) || !all_finite(bg, F * E)) return fail(ORC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
  for (int j = 0; j < F; ++j) {
    const uint8_t* om = oo + j * mb;
    const uint8_t* sm = bo + j * mb;
    for (int64_t p = 0; p < P; ++p) {
      const int from_obj = ((om[p >> 3] >> (p & 7)) & 1) | ((sm[p >> 3] >> (p & 7)) & 1);
      const float* src = from_obj ? obj : bg;
      for (int c = 0; c < C; ++c) out[j * E + p * C + c] = src[j * E + p * C + c];
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* store policies, src/store.cpp:32-42                                       */
/* ------------------------------------------------------------------------ */

static int lrbu(uint64_t f, int step, uint64_t capacity, uint64_t last, uint64_t now, double* out) {
  if (now < last) return fail(ORC_ERR_INVALID_ARGUMENT, "lrbu_priority: now precedes last access");
  if (capacity == 0) return fail(ORC_ERR_INVALID_ARGUMENT, "lrbu_priority: zero capacity");
  const uint64_t dd = now - last;
  const double duration = (double)(dd > 1 ? dd : 1);
  *out = ((double)(f + 1) * step) / ((double)capacity * duration);
  return ORC_OK;
}

int orc_lrbu_priority(const orc_step_entry* e, uint64_t now, double* out) {
  return lrbu(e->f, e->step, e->capacity, e->last_access, now, out);
}

int orc_lcbfu_priority(const orc_step_entry* e, double* out) {
  *out = (double)(e->f + 1) * e->step;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* CacheStore, src/store.cpp:44-217                                          */
/* ------------------------------------------------------------------------ */

typedef struct {
  int step;
  uint64_t f, last_access, inserted_at, inserted_seq, private_bytes;
} OLive;

typedef struct {
  uint64_t prompt;
  uint8_t* bytes; uint64_t len;  /* wire image of the full entry */
  OEntry entry;                  /* parsed view of bytes */
  int n_live;
  OLive live[8];                 /* ascending step */
  uint64_t shared;
} ORec;

typedef struct {
  uint64_t capacity, used, next_seq;
  int policy;
  int64_t n, cap;
  ORec** recs;                   /* ascending prompt id */
} OStore;

void* orc_store_new(uint64_t capacity, int policy) {
  OStore* s = (OStore*)calloc(1, sizeof(OStore));
  s->capacity = capacity;
  s->policy = policy;
  return s;
}

static void rec_free(ORec* r) {
  entry_free(&r->entry);
  free(r->bytes);
  free(r);
}

void orc_store_free(void* h) {
  OStore* s = (OStore*)h;
  if (!s) return;
  for (int64_t i = 0; i < s->n; ++i) rec_free(s->recs[i]);
  free(s->recs);
  free(s);
}

static int64_t find_rec(const OStore* s, uint64_t prompt) {
  int64_t lo = 0, hi = s->n;
  while (lo < hi) { int64_t m = lo + (hi - lo) / 2; if (s->recs[m]->prompt < prompt) lo = m + 1; else hi = m; }
  return lo;
}

static int is_cacheable(int s) { return s == 5 || s == 10 || s == 15 || s == 20 || s == 25; }

static const OStep* entry_step(const OEntry* e, int step) {
  for (int i = 0; i < e->n_steps; ++i) if (e->steps[i].step == step) return &e->steps[i];
  return NULL;
}

static void remove_step(OStore* s, int64_t ri, int li) {
  ORec* r = s->recs[ri];
  s->used -= r->live[li].private_bytes;
  memmove(&r->live[li], &r->live[li + 1], sizeof(OLive) * (r->n_live - li - 1));
  r->n_live--;
  if (r->n_live == 0) {
    s->used -= r->shared;
    rec_free(r);
    memmove(&s->recs[ri], &s->recs[ri + 1], sizeof(ORec*) * (s->n - ri - 1));
    s->n--;
  }
}

static void put_entry(const OStore* s, const ORec* r, const OLive* l, uint64_t cap, orc_step_entry* o) {
  (void)s;
  o->prompt = r->prompt; o->step = l->step; o->_pad = 0; o->f = l->f;
  o->last_access = l->last_access; o->inserted_at = l->inserted_at;
  o->inserted_seq = l->inserted_seq; o->capacity = cap;
}

/* min_priority_step + evict_one, src/store.cpp:113-157; peek = 1 reports the
 * victim (and its key) without removing it (sharded global eviction). */
static int evict_one_impl2(OStore* s, uint64_t now, orc_step_entry* out, int peek, double* key_out) {
  if (s->n == 0) return fail(ORC_ERR_LOGIC, "evict_one: store is empty");
  int64_t bri = -1; int bli = -1; double bkey = 0.0; uint64_t bcap = 0, bseq = 0;
  for (int64_t ri = 0; ri < s->n; ++ri) {
    const ORec* r = s->recs[ri];
    for (int li = 0; li < r->n_live; ++li) {
      const OLive* l = &r->live[li];
      const uint64_t cap = l->private_bytes + r->shared / (uint64_t)r->n_live; /* store.cpp:122 */
      double key = 0.0;
      switch (s->policy) {
        case 0: key = (double)l->inserted_seq; break;
        case 1: key = (double)l->last_access; break;
        case 2: key = (double)(l->f + 1) * l->step; break;
        default: CHECK(lrbu(l->f, l->step, cap, l->last_access, now, &key)); break;
      }
      if (bri < 0 || key < bkey || (key == bkey && l->inserted_seq < bseq)) {
        bri = ri; bli = li; bkey = key; bcap = cap; bseq = l->inserted_seq;
      }
    }
  }
  put_entry(s, s->recs[bri], &s->recs[bri]->live[bli], bcap, out);
  if (key_out) *key_out = bkey;
  if (!peek) remove_step(s, bri, bli);
  return ORC_OK;
}

static int evict_one_impl(OStore* s, uint64_t now, orc_step_entry* out) {
  return evict_one_impl2(s, now, out, 0, NULL);
}

int orc_store_evict_one(void* h, uint64_t now, orc_step_entry* out) {
  return evict_one_impl((OStore*)h, now, out);
}

int orc_store_peek(void* h, uint64_t now, orc_step_entry* out, double* key) {
  return evict_one_impl2((OStore*)h, now, out, 1, key);
}

uint64_t orc_store_next_seq(void* h) { return ((OStore*)h)->next_seq; }
void orc_store_set_next_seq(void* h, uint64_t seq) { ((OStore*)h)->next_seq = seq; }

/* insert_steps, src/store.cpp:53-91. */
int orc_store_insert(void* h, uint64_t prompt, const uint8_t* entry, uint64_t len,
                     const int32_t* steps, int n_steps, uint64_t now, orc_step_entry* evicted,
                     int cap, int* n_evicted) {
  OStore* s = (OStore*)h;
  *n_evicted = 0;
  ORec* r = (ORec*)calloc(1, sizeof(ORec));
  int rc = parse_entry(entry, len, &r->entry);
  if (rc != ORC_OK) { rec_free(r); return rc; }
  for (int i = 0; i < n_steps; ++i)
    if (!valid_step_id(steps[i])) { rec_free(r); return fail(ORC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50"); }
  if (n_steps <= 0) { rec_free(r); return fail(ORC_ERR_INVALID_ARGUMENT, "insert_steps: empty step list"); }
  if (r->entry.prompt != prompt) { rec_free(r); return fail(ORC_ERR_INVALID_ARGUMENT, "insert_steps: prompt does not match entry"); }
  const int64_t pos = find_rec(s, prompt);
  if (pos < s->n && s->recs[pos]->prompt == prompt) { rec_free(r); return fail(ORC_ERR_INVALID_ARGUMENT, "insert_steps: prompt already cached"); }
  for (int i = 0; i < n_steps; ++i) {
    if (!is_cacheable(steps[i])) { rec_free(r); return fail(ORC_ERR_INVALID_ARGUMENT, "insert_steps: step not cacheable"); }
    if (!entry_step(&r->entry, steps[i])) { rec_free(r); return fail(ORC_ERR_INVALID_ARGUMENT, "insert_steps: step missing from entry"); }
  }
  r->prompt = prompt;
  r->bytes = (uint8_t*)malloc(len ? len : 1);
  memcpy(r->bytes, entry, len);
  r->len = len;
  /* re-parse against owned bytes so the view outlives the caller's buffer */
  entry_free(&r->entry);
  parse_entry(r->bytes, r->len, &r->entry);
  r->shared = shared_bytes(&r->entry);
  uint64_t standalone = r->shared;
  /* records kept = entry steps (ascending) that were requested */
  for (int i = 0; i < r->entry.n_steps; ++i) {
    const OStep* st = &r->entry.steps[i];
    int want = 0;
    for (int k = 0; k < n_steps; ++k) if (steps[k] == st->step) want = 1;
    if (!want) continue;
    OLive* l = &r->live[r->n_live++];
    l->step = st->step;
    l->private_bytes = private_bytes(&r->entry, st);
    standalone += l->private_bytes;
  }
  if (standalone > s->capacity) {
    rec_free(r);
    return fail(ORC_ERR_OVERSIZED_ENTRY, "entry of %llu bytes exceeds capacity limit of %llu bytes",
                (unsigned long long)standalone, (unsigned long long)s->capacity);
  }
  int ne = 0;
  while (s->used + standalone > s->capacity) {
    orc_step_entry v;
    rc = evict_one_impl(s, now, &v);
    if (rc != ORC_OK) { rec_free(r); return rc; }
    if (ne < cap) evicted[ne] = v;
    ++ne;
  }
  for (int i = 0; i < r->n_live; ++i) {
    OLive* l = &r->live[i];
    l->f = 0; l->last_access = now; l->inserted_at = now; l->inserted_seq = s->next_seq++;
  }
  s->used += standalone;
  if (s->n == s->cap) { s->cap = s->cap ? s->cap * 2 : 64; s->recs = (ORec**)realloc(s->recs, sizeof(ORec*) * s->cap); }
  const int64_t ins = find_rec(s, prompt);
  memmove(&s->recs[ins + 1], &s->recs[ins], sizeof(ORec*) * (s->n - ins));
  s->recs[ins] = r;
  s->n++;
  *n_evicted = ne;
  return ORC_OK;
}

/* get_step, src/store.cpp:93-111: largest live step <= desired. */
int orc_store_get_step(void* h, uint64_t prompt, int desired, uint64_t now, int32_t* actual, float* out) {
  OStore* s = (OStore*)h;
  if (!valid_step_id(desired)) return fail(ORC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
  if (!is_cacheable(desired)) return fail(ORC_ERR_INVALID_ARGUMENT, "get_step: desired step not cacheable");
  *actual = 0;
  const int64_t pos = find_rec(s, prompt);
  if (pos >= s->n || s->recs[pos]->prompt != prompt) return ORC_OK;
  ORec* r = s->recs[pos];
  int li = -1;
  for (int i = 0; i < r->n_live; ++i) if (r->live[i].step <= desired) li = i;
  if (li < 0) return ORC_OK;
  if (out) CHECK(decompress_impl(&r->entry, r->live[li].step, out));
  r->live[li].f += 1;
  r->live[li].last_access = now;
  *actual = r->live[li].step;
  return ORC_OK;
}

/* evict_step, src/store.cpp:159-164. */
int orc_store_evict_step(void* h, uint64_t prompt, int step, int32_t* removed) {
  OStore* s = (OStore*)h;
  if (!valid_step_id(step)) return fail(ORC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
  *removed = 0;
  const int64_t pos = find_rec(s, prompt);
  if (pos >= s->n || s->recs[pos]->prompt != prompt) return ORC_OK;
  ORec* r = s->recs[pos];
  for (int i = 0; i < r->n_live; ++i)
    if (r->live[i].step == step) { remove_step(s, pos, i); *removed = 1; break; }
  return ORC_OK;
}

uint64_t orc_store_used(void* h) { return ((OStore*)h)->used; }

uint64_t orc_store_recompute_used(void* h) {
  OStore* s = (OStore*)h;
  uint64_t n = 0;
  for (int64_t i = 0; i < s->n; ++i) {
    const ORec* r = s->recs[i];
    n += shared_bytes(&r->entry);
    for (int k = 0; k < r->n_live; ++k) n += private_bytes(&r->entry, entry_step(&r->entry, r->live[k].step));
  }
  return n;
}

int64_t orc_store_step_count(void* h) {
  OStore* s = (OStore*)h;
  int64_t n = 0;
  for (int64_t i = 0; i < s->n; ++i) n += s->recs[i]->n_live;
  return n;
}

int64_t orc_store_prompt_count(void* h) { return ((OStore*)h)->n; }

/* entries_snapshot, src/store.cpp:190-200. */
int orc_store_entries(void* h, orc_step_entry* out, int cap, int* n) {
  OStore* s = (OStore*)h;
  int k = 0;
  for (int64_t i = 0; i < s->n; ++i) {
    const ORec* r = s->recs[i];
    for (int li = 0; li < r->n_live; ++li) {
      const uint64_t c = r->live[li].private_bytes + r->shared / (uint64_t)r->n_live;
      if (k < cap) put_entry(s, r, &r->live[li], c, &out[k]);
      ++k;
    }
  }
  *n = k;
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * simgen: no reference code exists; this restates the
 * generator defined in paper_2501_04012_b200/csrc/simgen.cu line for line
 * (counter-based hash_combine streams, rng.hpp:25-31; Irwin-Hall normals).
 * ------------------------------------------------------------------------- */
static uint64_t sg_hash(uint64_t a, uint64_t b) { /* rng.hpp:25-31 */
  uint64_t z = a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2));
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double sg_U(uint64_t s, uint64_t i) { return (double)(sg_hash(s, i) >> 11) * 0x1.0p-53; }
static double sg_N(uint64_t s, uint64_t i) {
  const double a = sg_U(s, 4 * i) + sg_U(s, 4 * i + 1);
  const double b = sg_U(s, 4 * i + 2) + sg_U(s, 4 * i + 3);
  return ((a + b) - 2.0) * 1.7320508075688772;
}

int orc_synth_embedding(const uint64_t* tokens, int n_tok, int dim, uint64_t seed, float* out) {
  if (n_tok < 1 || n_tok > 16 || dim <= 0) return fail(ORC_ERR_INVALID_ARGUMENT, "synth_embedding: 1..16 tokens");
  double inv[16];
  uint64_t st[16];
  for (int t = 0; t < n_tok; ++t) {
    st[t] = sg_hash(seed, tokens[t]);
    double sq = 0.0;
    for (int d = 0; d < dim; ++d) {
      const float v = (float)sg_N(st[t], (uint64_t)d);
      sq += (double)v * (double)v;
    }
    inv[t] = 1.0 / sqrt(sq);
  }
  double sq = 0.0;
  for (int d = 0; d < dim; ++d) {
    double acc = 0.0;
    for (int t = 0; t < n_tok; ++t) {
      const float v = (float)sg_N(st[t], (uint64_t)d);
      acc += (double)(float)((double)v * inv[t]);
    }
    out[d] = (float)acc;
    sq += (double)out[d] * (double)out[d];
  }
  const double iv = 1.0 / sqrt(sq);
  for (int d = 0; d < dim; ++d) out[d] = (float)((double)out[d] * iv);
  return ORC_OK;
}

static float sg_key(uint64_t s, int i, int j, int64_t e, int64_t E, const double* alpha, double noise) {
  const double base = sg_N(sg_hash(s, 2), (uint64_t)e);
  const double first = (double)(float)(base * (1.0 - 0.05 * i) + 0.05 * sg_N(sg_hash(s, 3 + i), (uint64_t)e));
  if (j == 0) return (float)first;
  const double dj = sg_N(sg_hash(s, 1), (uint64_t)(j * E + e));
  const double nz = 1.0 + noise * sg_N(sg_hash(s, 10 + i), (uint64_t)(j * E + e));
  return (float)(first + (alpha[i] * dj) * nz);
}

/* one prompt: lat [5][F][E], masks [F][mb] */
int orc_synth_latents(uint64_t s, int F, int H, int W, int C, const double* red, const double* alpha,
                      double noise, double dup, float* lat, uint8_t* om, uint8_t* bm) {
  if (F < 1 || F > 256 || H < 1 || W < 1 || C < 1) return fail(ORC_ERR_INVALID_ARGUMENT, "synth_latents: geometry");
  const int64_t E = (int64_t)H * W * C, mb = ((int64_t)H * W + 7) / 8;
  int perm[256];
  for (int t = 0; t < F - 1; ++t) perm[t] = t + 1;
  for (int t = F - 2; t >= 1; --t) {
    const int q = (int)(sg_hash(sg_hash(s, 30), (uint64_t)t) % (uint64_t)(t + 1));
    const int x = perm[t]; perm[t] = perm[q]; perm[q] = x;
  }
  for (int i = 0; i < 5; ++i) {
    const int n_red = (int)floor(red[i] * (double)(F - 1) + 0.5);
    char is_red[256] = {0};
    for (int t = 0; t < n_red && t < F - 1; ++t) is_red[perm[t]] = 1;
    int keys[256], nk = 1, plan[256];
    keys[0] = 0; plan[0] = -1;
    for (int j = 1; j < F; ++j) {
      if (is_red[j]) plan[j] = keys[sg_hash(sg_hash(s, 40 + i), (uint64_t)j) % (uint64_t)nk];
      else { plan[j] = -1; keys[nk++] = j; }
    }
    for (int j = 0; j < F; ++j) {
      float* fr = lat + ((int64_t)i * F + j) * E;
      for (int64_t e = 0; e < E; ++e) {
        if (plan[j] < 0) fr[e] = sg_key(s, i, j, e, E, alpha, noise);
        else {
          const double xk = (double)sg_key(s, i, plan[j], e, E, alpha, noise);
          fr[e] = (float)(xk + dup * sg_N(sg_hash(s, 20 + i), (uint64_t)(j * E + e)));
        }
      }
    }
  }
  const uint64_t m = sg_hash(s, 50);
  const int h0 = (int)(sg_hash(m, 0) % (uint64_t)(H / 2 > 0 ? H / 2 : 1));
  const int h1 = h0 + 1 + (int)(sg_hash(m, 1) % (uint64_t)(H - h0));
  const int w0 = (int)(sg_hash(m, 2) % (uint64_t)(W / 2 > 0 ? W / 2 : 1));
  const int w1 = w0 + 1 + (int)(sg_hash(m, 3) % (uint64_t)(W - w0));
  const int span = W - w1 + 1 > 1 ? W - w1 + 1 : 1;
  for (int j = 0; j < F; ++j) {
    const int sh = j % span;
    for (int64_t by = 0; by < mb; ++by) {
      uint8_t ob = 0, bb = 0;
      for (int b = 0; b < 8; ++b) {
        const int64_t px = by * 8 + b;
        if (px >= (int64_t)H * W) break;
        const int y = (int)(px / W), x = (int)(px % W);
        const int in = y >= h0 && y < h1 && x >= w0 + sh && x < (w1 + sh < W ? w1 + sh : W);
        ob |= (uint8_t)(in ? 1 : 0) << b;
        bb |= (uint8_t)(in ? 0 : 1) << b;
      }
      om[(int64_t)j * mb + by] = ob;
      bm[(int64_t)j * mb + by] = bb;
    }
  }
  return ORC_OK;
}
