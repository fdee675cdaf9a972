/*
 * oracle_abi.h — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Flat C signatures shared by the two CPU checkers under oracle/:
 *   ref_*  — thin extern "C" shim over the UNMODIFIED reference library
 *            (the /root/reference/proj/src sources, compiled by oracle/Makefile into
 *            oracle/_ref/liblcache_ref.so; see oracle/ref_shim.cpp);
 *   orc_*  — the plain-C restatement of the reference algorithms
 *            (oracle/lc_oracle.c -> oracle/_build/liblc_oracle.so).
 *
 * Both expose identical argument meaning so tests can run the same inputs
 * through reference, restatement and the CUDA product (C-ABI in
 * include/flexcache_b200.h) and compare bit-for-bit.
 *
 * Buffers: latents are [S][F][H*W*C] fp32, channel-minor per frame
 * (core.hpp:37); masks are [F][ceil(H*W/8)] LSB-first packed bytes
 * (core.hpp:104-124); entries travel as the reference wire format
 * (serialize_entry, codec.cpp:358-392).
 */
#ifndef FLEXCACHE_ORACLE_ABI_H
#define FLEXCACHE_ORACLE_ABI_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: identical numbering to include/flexcache_b200.h lc_status. */
enum {
  ORC_OK = 0,
  ORC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument            */
  ORC_ERR_DEGENERATE_BASE = 2,  /* DegenerateBase  errors.hpp:13     */
  ORC_ERR_STEP_NOT_CACHED = 3,  /* StepNotCached   errors.hpp:17     */
  ORC_ERR_OVERSIZED_ENTRY = 4,  /* OversizedEntry  errors.hpp:22     */
  ORC_ERR_SNAPSHOT = 5,         /* SnapshotError   errors.hpp:30     */
  ORC_ERR_LOGIC = 6,            /* std::logic_error (e.g. evict_one on empty) */
  ORC_ERR_INTERNAL = 10
};

/* StepEntry (store.hpp:28-36), flattened. */
typedef struct orc_step_entry {
  uint64_t prompt;
  int32_t step;
  int32_t _pad;
  uint64_t f;
  uint64_t last_access;
  uint64_t inserted_at;
  uint64_t inserted_seq;
  uint64_t capacity;
} orc_step_entry;

#define ORC_DECLARE(P)                                                                 \
  const char* P##last_error(void);                                                     \
  int P##normalize(const float* v, int d, float* out);                                 \
  int P##cosine(const float* a, const float* b, int64_t n, double* out);               \
  void* P##index_new(int dim);                                                         \
  void P##index_free(void* h);                                                         \
  int P##index_insert(void* h, uint64_t id, const float* w, const float* o,            \
                      const float* b, int d);                                          \
  int P##index_remove(void* h, uint64_t id);                                           \
  int64_t P##index_size(void* h);                                                      \
  int P##index_query_top1(void* h, int kind, const float* q, int n, int d,             \
                          int nthreads, uint64_t* ids, double* scores, int32_t* found); \
  int P##select_keyframes(const float* frames, int F, int H, int W, int C,             \
                          double thr, int32_t* map);                                   \
  int P##solve_alpha(const float* ds, const float* db, int64_t n, float* out);         \
  int P##compress(const float* lat, const int32_t* steps, int S, int F, int H, int W,  \
                  int C, const uint8_t* obj_masks, const uint8_t* bg_masks,            \
                  double thr, uint64_t prompt, uint8_t* out, uint64_t cap,             \
                  uint64_t* out_len);                                                  \
  int P##compress_batch(const float* lat, const int32_t* steps, int S, int F, int H,   \
                        int W, int C, const uint8_t* obj_masks,                        \
                        const uint8_t* bg_masks, double thr, const uint64_t* prompts,  \
                        int n, int nthreads, uint64_t* out_sizes);                     \
  int P##decompress(const uint8_t* entry, uint64_t len, int step, float* out);         \
  int P##entry_info(const uint8_t* entry, uint64_t len, int32_t* base_step,            \
                    int32_t* n_steps, int32_t* steps, uint64_t* shared_bytes,          \
                    uint64_t* private_bytes);                                          \
  int P##stitch(const float* obj, const uint8_t* obj_src_obj_masks,                    \
                const uint8_t* obj_src_bg_masks, const float* bg,                      \
                const uint8_t* bg_src_obj_masks, const uint8_t* bg_src_bg_masks,       \
                int F, int H, int W, int C, float* out);                               \
  int P##lrbu_priority(const orc_step_entry* e, uint64_t now, double* out);            \
  int P##lcbfu_priority(const orc_step_entry* e, double* out);                         \
  void* P##store_new(uint64_t capacity, int policy);                                   \
  void P##store_free(void* h);                                                         \
  int P##store_insert(void* h, uint64_t prompt, const uint8_t* entry, uint64_t len,    \
                      const int32_t* steps, int n_steps, uint64_t now,                 \
                      orc_step_entry* evicted, int cap, int* n_evicted);               \
  int P##store_get_step(void* h, uint64_t prompt, int desired, uint64_t now,           \
                        int32_t* actual, float* out);                                  \
  int P##store_evict_one(void* h, uint64_t now, orc_step_entry* out);                  \
  int P##store_evict_step(void* h, uint64_t prompt, int step, int32_t* removed);       \
  uint64_t P##store_used(void* h);                                                     \
  uint64_t P##store_recompute_used(void* h);                                           \
  int64_t P##store_step_count(void* h);                                                \
  int64_t P##store_prompt_count(void* h);                                              \
  int P##store_entries(void* h, orc_step_entry* out, int cap, int* n);

ORC_DECLARE(ref_)
ORC_DECLARE(orc_)

/* Restatement-only generalisations (no reference code exists for these):
 *  - top-k over a flat table, ordered (score desc, id asc): generalises the
 *    strict-'>' ascending-id scan of query_top1 (vindex.cpp:58-72) to k >= 1;
 *  - decide / similarity_to_step from SPEC.md:484-502 (engine is SPEC-only). */
int orc_topk_flat(const float* table, const uint64_t* ids, int64_t n_rows, int d,
                  const float* q, int n_q, int k, uint64_t* out_ids, double* out_scores,
                  int32_t* out_counts);
/* kind: 0 Miss, 1 WholeHit, 2 DecoupledHit */
int orc_decide(double w, double o, double b, double threshold, int32_t* kind, double* score);
int orc_similarity_to_step(double score, double threshold, const double* edges4,
                           int32_t* step);
/*  - peek = evict_one without the removal (store.cpp:113-157 argmin) and the
 *    insertion counter (store.hpp:113), for entry-sharded stores. */
int orc_store_peek(void* h, uint64_t now, orc_step_entry* out, double* key);
uint64_t orc_store_next_seq(void* h);
void orc_store_set_next_seq(void* h, uint64_t seq);
/*  - simgen (no reference code): the generator defined in
 *    csrc/simgen.cu, restated. */
int orc_synth_embedding(const uint64_t* tokens, int n_tok, int dim, uint64_t seed, float* out);
int orc_synth_latents(uint64_t seed, int F, int H, int W, int C, const double* redundancy,
                      const double* alpha, double noise, double dup, float* lat, uint8_t* om,
                      uint8_t* bm);

#ifdef __cplusplus
}
#endif
#endif
