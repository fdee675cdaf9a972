/*
 * flexcache_b200.h — C-ABI of the B200-native FlexCache hot path.
 *
 * Drop-in boundary for the reference C++ library `lcache`
 * (/root/reference/proj/include/lcache/*.hpp). The reference exposes only a
 * C++ API; every entry point below replaces one of its functions (cited as
 * file:line into /root/reference/proj) and keeps its argument meaning, result
 * and error behaviour. C++ exceptions become lc_status codes (1:1 with the
 * reference exception types, errors.hpp:11-42) plus a thread-local message
 * (lc_last_error). A C++ wrapper with the reference class/function names is
 * include/lcache_b200/lcache.hpp; the Python mirror is paper_2501_04012_b200.
 *
 * Memory: unless stated otherwise, data pointers may be HOST or DEVICE
 * (cuda pointer attributes are queried); *_dev arguments must be device
 * memory resident on the context's GPU. All work is issued on the context's
 * stream; calls returning host-visible results synchronise that stream.
 *
 * Layouts (identical to the reference):
 *   embedding: fp32[dim], unit norm (Embedding, core.hpp:80-102)
 *   frame:     fp32[H*W*C], channel-minor, index (h*W+w)*C+c (core.hpp:37)
 *   latent:    [F][H*W*C] (LatentState, core.hpp:62-74); a batch is
 *              [n][S][F][H*W*C]
 *   masks:     [F][ceil(H*W/8)] LSB-first packed bits (Bitmap, core.hpp:104-124)
 *   entry wire bytes: serialize_entry (codec.cpp:358-392)
 */
#ifndef FLEXCACHE_B200_H
#define FLEXCACHE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------------------
 * Status codes: one per reference exception type (errors.hpp:11-42).
 * ------------------------------------------------------------------------- */
typedef enum lc_status {
  LC_OK = 0,
  LC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument                      */
  LC_ERR_DEGENERATE_BASE = 2,  /* DegenerateBase   errors.hpp:13             */
  LC_ERR_STEP_NOT_CACHED = 3,  /* StepNotCached    errors.hpp:17             */
  LC_ERR_OVERSIZED_ENTRY = 4,  /* OversizedEntry   errors.hpp:22 (see lc_last_oversize) */
  LC_ERR_SNAPSHOT = 5,         /* SnapshotError    errors.hpp:30             */
  LC_ERR_LOGIC = 6,            /* std::logic_error (evict_one on empty store, store.cpp:148) */
  LC_ERR_CUDA = 7,             /* CUDA runtime/driver failure                */
  LC_ERR_NCCL = 8,             /* collective failure (NCCL / host all-gather) */
  LC_ERR_OOM = 9,              /* device allocation failure                  */
  LC_ERR_INTERNAL = 10,
  LC_ERR_IO = 11               /* std::runtime_error: snapshot file I/O (store.cpp:268-276) */
} lc_status;

/* Thread-local message of the last failing call on this thread. */
const char* lc_last_error(void);
/* OversizedEntry{needed_bytes, capacity_limit} of the last LC_ERR_OVERSIZED_ENTRY. */
void lc_last_oversize(uint64_t* needed_bytes, uint64_t* capacity_limit);
/* Byte offset carried by the last LC_ERR_SNAPSHOT on this thread
 * (SnapshotError::byte_offset, errors.hpp:30-35). */
uint64_t lc_last_snapshot_offset(void);
const char* lc_version(void);

/* Policy (store.hpp:23). */
enum { LC_POLICY_FIFO = 0, LC_POLICY_LRU = 1, LC_POLICY_LCBFU = 2, LC_POLICY_LRBU = 3 };
/* EmbeddingKind (core.hpp:77). */
enum { LC_KIND_WHOLE = 0, LC_KIND_OBJECT = 1, LC_KIND_BACKGROUND = 2 };
/* Decision kinds. */
enum { LC_MISS = 0, LC_WHOLE_HIT = 1, LC_DECOUPLED_HIT = 2 };

/* StepEntry (store.hpp:28-36), flattened; layout shared with the oracle. */
typedef struct lc_step_entry {
  uint64_t prompt;
  int32_t step;
  int32_t _pad;
  uint64_t f;
  uint64_t last_access;
  uint64_t inserted_at;
  uint64_t inserted_seq;
  uint64_t capacity;
} lc_step_entry;

/* Result of the fused lookup + decide + similarity_to_step path
 * (no reference code). */
typedef struct lc_decision {
  int32_t kind;       /* LC_MISS / LC_WHOLE_HIT / LC_DECOUPLED_HIT          */
  int32_t step;       /* similarity_to_step(score) for hits, 0 for a miss   */
  uint64_t whole_id;  /* top-1 of each table (valid if the table is non-empty) */
  uint64_t object_id;
  uint64_t background_id;
  double score;       /* decided score: w (whole) / min(o,b) (decoupled) / max(w, min(o,b)) (miss) */
  double whole_score, object_score, background_score;
} lc_decision;

/* ---------------------------------------------------------------------------
 * Context: one GPU, one stream, scratch arenas.
 * ------------------------------------------------------------------------- */
typedef struct lc_ctx lc_ctx;
lc_status lc_ctx_create(int device, lc_ctx** out);
lc_status lc_ctx_destroy(lc_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream). NULL = own stream. */
lc_status lc_ctx_set_stream(lc_ctx* ctx, void* cuda_stream);
void* lc_ctx_stream(lc_ctx* ctx);
lc_status lc_ctx_synchronize(lc_ctx* ctx);
/* Number of product kernels launched through this context (instrumentation). */
uint64_t lc_ctx_launches(lc_ctx* ctx);
/* Per-kernel CUDA-event timing on the context stream (bench/roofline):
 * names "shortlist" (tcgen05 lookup GEMM), "rescore", "scan", "decompress",
 * "decompress_stitch", "gram", "inter", "pack", "policy". */
lc_status lc_ctx_profile(lc_ctx* ctx, int enable);
lc_status lc_ctx_kernel_time(lc_ctx* ctx, const char* name, uint64_t* launches, double* total_ms, int reset);

/* ---------------------------------------------------------------------------
 * Core primitives (core.cpp:50-119).
 * ------------------------------------------------------------------------- */
/* Embedding ctor normalisation (core.cpp:50-59) of n rows of dim floats:
 * fp64 sequential sum of squares, (float)(v * (1/sqrt(sq))). Bit-exact. */
lc_status lc_embedding_normalize(lc_ctx* ctx, const float* v, int64_t n, int dim, float* out);
/* cosine_similarity (core.cpp:101-114) for n pairs of length len. Bit-exact. */
lc_status lc_cosine_batch(lc_ctx* ctx, const float* a, const float* b, int64_t n, int64_t len,
                          double* out);

/* ---------------------------------------------------------------------------
 * SimilarityIndex (vindex.hpp:23-62): three tables (whole/object/background),
 * device-resident fp32 master rows + bf16 GEMM copies.
 * ------------------------------------------------------------------------- */
typedef struct lc_index lc_index;
/* dim 0 = fixed by the first insert (vindex.hpp:59). capacity_rows = initial
 * reservation (grows on demand). */
lc_status lc_index_create(lc_ctx* ctx, int dim, int64_t capacity_rows, lc_index** out);
lc_status lc_index_destroy(lc_index* ix);
/* insert (vindex.cpp:29-48): whole/object/background fp32[dim] unit vectors
 * (from_unit rule, core.cpp:61-69); duplicate id or dim mismatch =>
 * LC_ERR_INVALID_ARGUMENT, nothing inserted. */
lc_status lc_index_insert(lc_index* ix, uint64_t prompt, const float* whole, const float* object,
                          const float* background, int dim);
/* Atomic batch insert of n prompts: w/o/b are [n][dim]; all-or-nothing. */
lc_status lc_index_insert_batch(lc_index* ix, const uint64_t* prompts, const float* whole,
                                const float* object, const float* background, int64_t n, int dim);
/* remove (vindex.cpp:76-87): unknown id => LC_ERR_INVALID_ARGUMENT. */
lc_status lc_index_remove(lc_index* ix, uint64_t prompt);
lc_status lc_index_contains(lc_index* ix, uint64_t prompt, int32_t* out);
int64_t lc_index_size(lc_index* ix);
int lc_index_dim(lc_index* ix);
/* entries(kind) (vindex.cpp:101-114): ids ascending, rows fp32 (host buffers). */
lc_status lc_index_export(lc_index* ix, int kind, uint64_t* ids, float* rows, int64_t cap);

/* Top-k by (score desc, id asc) where score = sequential fp64 dot of the
 * fp32 query with the stored fp32 row (vindex.cpp:58-72); k = 1 is exactly
 * query_top1 (vindex.cpp:50-74). q is [n][dim]; outputs [n][k] and [n]
 * (count = min(k, size)). Empty table => counts 0. Results are EXACT:
 * bf16 tensor-core candidates + fp64 rescore + certified margin, with an
 * exact fp64 scan for any query the margin cannot certify. */
lc_status lc_index_query_topk(lc_index* ix, int kind, const float* q, int64_t n, int k,
                              uint64_t* out_ids, double* out_scores, int32_t* out_counts);
/* Fused lookup over the three tables + decide + similarity_to_step
 * (hit threshold defaults.hpp:13, bins defaults.hpp:27).
 * edges4 = NULL -> defaults. */
lc_status lc_lookup_decide(lc_index* ix, const float* q_whole, const float* q_object,
                           const float* q_background, int64_t n, double hit_threshold,
                           const double* edges4, lc_decision* out);
/* Tuning / instrumentation of the lookup path. */
typedef struct lc_lookup_stats {
  uint64_t queries;       /* (query, table) lookups served               */
  uint64_t certified;     /* certified by the bf16 margin test            */
  uint64_t fallback;      /* not certified by the K' shortlist            */
  uint64_t exact_scans;   /* lookups served by the exact scan directly    */
  double max_abs_err;     /* max |bf16 approx - fp64 exact| seen in rescores */
  uint64_t tier2_certified; /* of the fallbacks: certified by a bf16 re-shortlist
                               (the rest are counted in exact_scans) */
  uint64_t i8_batches;    /* batches whose tier 1 was the int8 tensor-core shortlist */
  uint64_t i8_rescored;   /* rows exact-scored by the int8 tier's rescore  */
  uint64_t i8_candidates; /* rows in the int8 tier's merged shortlists     */
  uint64_t i8_prescored;  /* of those, bf16 pre-scored by the rescore       */
  uint64_t threshold_certified; /* fallbacks certified by the fixed-threshold int8 tier */
} lc_lookup_stats;
lc_status lc_index_stats(lc_index* ix, lc_lookup_stats* out, int reset);
/* mode: 0 auto (tensor-core path when size >= 8192), 1 force exact scan,
 * 2 force tensor-core path. kprime: shortlist length (multiple of 32, <= 128).
 * eps: floor on the certified |bf16 - fp64| score bound (<= 0 -> none). The
 * bound itself is proven per query from ||q||, the query's and the stored
 * rows' bf16 rounding residuals (lookup.cuh), so results stay exact for any
 * finite query, unit or not; eps can only widen it. Queries with a
 * non-finite element fail with LC_ERR_INVALID_ARGUMENT (reference queries
 * are Embeddings, core.cpp:11-15). */
lc_status lc_index_set_lookup(lc_index* ix, int mode, int kprime, double eps);
/* Shard merge for entry-sharded multi-GPU lookup (a23): merge G per-shard
 * exact top-k lists [G][n][k] (+counts [G][n]) into the global top-k
 * by (score desc, id asc). Device or host buffers. */
lc_status lc_topk_merge(lc_ctx* ctx, const uint64_t* ids, const double* scores,
                        const int32_t* counts, int G, int64_t n, int k, uint64_t* out_ids,
                        double* out_scores, int32_t* out_counts);
/* decide + similarity_to_step on already-computed top-1 triples (used after
 * the multi-GPU merge). found* may be NULL (all found). */
lc_status lc_decide_batch(lc_ctx* ctx, const uint64_t* w_ids, const double* w_scores,
                          const uint64_t* o_ids, const double* o_scores, const uint64_t* b_ids,
                          const double* b_scores, int64_t n, double hit_threshold,
                          const double* edges4, lc_decision* out);

/* ---------------------------------------------------------------------------
 * Latent codec (codec.hpp:69-118) with device-resident entries.
 * ------------------------------------------------------------------------- */
typedef struct lc_entry lc_entry;  /* one CompressedEntry living in HBM */

/* Codec instrumentation: K7 (inter_compress trial) items computed, and how
 * many of them the certified kernel could not settle (re-run exactly). */
typedef struct lc_codec_stats {
  uint64_t inter_items;
  uint64_t inter_exact_items;
} lc_codec_stats;
lc_status lc_codec_stats_get(lc_ctx* ctx, lc_codec_stats* out, int reset);
/* select_keyframes (codec.cpp:138-165) for n latents [n][F][E]; map [n][F]. */
lc_status lc_select_keyframes(lc_ctx* ctx, const float* latents, int64_t n, int F, int H, int W,
                              int C, double threshold, int32_t* map);
/* solve_alpha (codec.cpp:181-191) for n pairs of length len; out fp32[n]. */
lc_status lc_solve_alpha_batch(lc_ctx* ctx, const float* diff_s, const float* diff_base,
                               int64_t n, int64_t len, float* out);
/* intra_compress x S + inter_compress (codec.cpp:167-261) for n prompts.
 * latents [n][S][F][E], steps[S] (host, any order, distinct), masks
 * [n][F][mb] object + background, prompts[n] (host). On success out[i] owns
 * a device-resident entry and sizes[i] = compressed_size (codec.cpp:334-338).
 * On failure no entry is returned. */
lc_status lc_compress_batch(lc_ctx* ctx, const float* latents, const int32_t* steps, int S,
                            int F, int H, int W, int C, const uint8_t* obj_masks,
                            const uint8_t* bg_masks, double threshold, const uint64_t* prompts,
                            int64_t n, lc_entry** out, uint64_t* sizes);
/* inter_compress with caller-provided key-frame maps (the IntraCompressed
 * inputs of codec.hpp:81-82): latents hold at least the key frames. */
lc_status lc_inter_compress(lc_ctx* ctx, const float* latents, const int32_t* maps,
                            const int32_t* steps, int S, int F, int H, int W, int C,
                            const uint8_t* obj_masks, const uint8_t* bg_masks, uint64_t prompt,
                            lc_entry** out);
lc_status lc_entry_release(lc_entry* e);
/* Reference wire bytes (serialize_entry, codec.cpp:358-392); bytes may be
 * NULL to query the length (== compressed_size). */
lc_status lc_entry_export(lc_entry* e, uint8_t* bytes, uint64_t cap, uint64_t* len);
/* deserialize_entry (codec.cpp:394-473) into a device-resident entry. */
lc_status lc_entry_import(lc_ctx* ctx, const uint8_t* bytes, uint64_t len, lc_entry** out);
typedef struct lc_entry_info {
  uint64_t prompt;
  int32_t base_step, n_steps, F, H, W, C, n_diff;
  int32_t steps[8];
  int32_t n_extra[8];
  uint64_t shared_bytes;        /* entry_shared_bytes  codec.cpp:317-321 */
  uint64_t private_bytes[8];    /* step_private_bytes  codec.cpp:323-332 */
  uint64_t compressed_size;     /* codec.cpp:334-338                     */
} lc_entry_info;
lc_status lc_entry_get_info(lc_entry* e, lc_entry_info* out);
/* decompress_step (codec.cpp:263-301) for n (entry, step) pairs into
 * out_dev [n][F][E] (device). Bit-exact. Unknown step => LC_ERR_STEP_NOT_CACHED.
 * Stream-ordered: returns after launching on ctx's stream (no host sync);
 * synchronize that stream (lc_ctx_synchronize) before reading out_dev from
 * another stream or the host. Same for lc_decompress_stitch_batch. */
lc_status lc_decompress_batch(lc_ctx* ctx, lc_entry* const* entries, const int32_t* steps,
                              int64_t n, float* out_dev);
/* Decoupled hit: decompress the object source and the background source at
 * the same step and stitch them (stitcher.cpp:7-39) in one pass: each output
 * pixel is reconstructed only from the source the masks select. */
lc_status lc_decompress_stitch_batch(lc_ctx* ctx, lc_entry* const* obj_entries,
                                     lc_entry* const* bg_entries, const int32_t* steps,
                                     int64_t n, float* out_dev);
/* stitch (stitcher.cpp:7-39) of n latent pairs already in memory; masks are
 * the object-source's object masks and the background-source's object masks
 * (background masks are never read by the reference). */
lc_status lc_stitch_batch(lc_ctx* ctx, const float* obj, const uint8_t* obj_src_obj_masks,
                          const float* bg, const uint8_t* bg_src_obj_masks, int64_t n, int F,
                          int H, int W, int C, float* out);

/* ---------------------------------------------------------------------------
 * CacheStore (store.hpp:48-120): capacity in compressed_size bytes,
 * (prompt, step) eviction unit, shared diff blob per prompt.
 * ------------------------------------------------------------------------- */
typedef struct lc_store lc_store;
lc_status lc_store_create(lc_ctx* ctx, uint64_t capacity_limit, int policy, lc_store** out);
lc_status lc_store_destroy(lc_store* s);
/* insert_steps (store.cpp:53-91). The store takes its own reference to the
 * entry (the caller may release its handle). evicted receives up to cap
 * StepEntry records (n_evicted = total). */
lc_status lc_store_insert(lc_store* s, uint64_t prompt, lc_entry* entry, const int32_t* steps,
                          int n_steps, uint64_t now, lc_step_entry* evicted, int cap,
                          int* n_evicted);
/* get_step (store.cpp:93-111): actual = served step or 0 (miss); out_dev
 * (device, [F][E]) may be NULL to only bump f/last_access. */
lc_status lc_store_get_step(lc_store* s, uint64_t prompt, int desired, uint64_t now,
                            int32_t* actual, float* out_dev);
lc_status lc_store_evict_one(lc_store* s, uint64_t now, lc_step_entry* out);
lc_status lc_store_evict_step(lc_store* s, uint64_t prompt, int step, int32_t* removed);
/* The step evict_one(now) would remove next (same StepEntry, with its policy
 * key), without removing it: the per-shard candidate of a global eviction
 * across entry-sharded stores. Empty => LC_ERR_LOGIC. */
lc_status lc_store_peek(lc_store* s, uint64_t now, lc_step_entry* out, double* key);
/* The next (up to) m steps repeated evict_one(now) would remove, in order,
 * each with its policy key and used() after its removal — without removing
 * them. Stops early with *more = 1 where the store would re-score its table.
 * One call per shard per eviction burst of an entry-sharded store. */
lc_status lc_store_peek_many(lc_store* s, uint64_t now, int m, lc_step_entry* out, double* keys,
                             uint64_t* used_after, int* n_out, int* more);
/* insert_steps validation only (store.cpp:53-76: step range, non-empty,
 * prompt match, not cached, cacheable, present in entry); *standalone = the
 * entry's shared + requested private bytes. No OversizedEntry check. */
lc_status lc_store_check_insert(lc_store* s, uint64_t prompt, lc_entry* entry, const int32_t* steps,
                                int n_steps, uint64_t* standalone);
/* store.hpp:113 next_seq_: sharded stores keep one global insertion counter. */
uint64_t lc_store_next_seq(lc_store* s);
lc_status lc_store_set_next_seq(lc_store* s, uint64_t seq);
uint64_t lc_store_used(lc_store* s);
uint64_t lc_store_recompute_used(lc_store* s);
uint64_t lc_store_capacity(lc_store* s);
int lc_store_policy(lc_store* s);
int64_t lc_store_step_count(lc_store* s);
int64_t lc_store_prompt_count(lc_store* s);
lc_status lc_store_contains(lc_store* s, uint64_t prompt, int32_t* out);
/* cached_steps (store.cpp:178-184): ascending, up to 5. */
lc_status lc_store_cached_steps(lc_store* s, uint64_t prompt, int32_t* steps, int* n);
/* entry_data (store.cpp:192-195): borrowed handle, invalidated by mutation. */
lc_status lc_store_entry(lc_store* s, uint64_t prompt, lc_entry** out);
/* entries_snapshot (store.cpp:197-207): (prompt, step) order. */
lc_status lc_store_entries(lc_store* s, lc_step_entry* out, int64_t cap, int64_t* n);

/* ---------------------------------------------------------------------------
 * Snapshot (save_snapshot / load_snapshot, store.cpp:219-364; store.hpp:122-132):
 * "FLXC" v1, policy, capacity, next_seq, the three index tables (ids
 * ascending), then one CRC32-checked record per prompt (serialize_entry bytes
 * + live step records). Byte-identical to the reference's file for the same
 * store and index state. Load errors: LC_ERR_SNAPSHOT (+ lc_last_snapshot_offset),
 * LC_ERR_INVALID_ARGUMENT where the reference's constructors throw, LC_ERR_IO.
 * ------------------------------------------------------------------------- */
lc_status lc_snapshot_save(lc_store* store, lc_index* index, const char* path);
/* On success *store / *index are new objects on ctx (destroy as usual). */
lc_status lc_snapshot_load(lc_ctx* ctx, const char* path, lc_store** store, lc_index** index);
/* ---------------------------------------------------------------------------
 * Engine (the reference ships no engine code): the request
 * pipeline lookup -> decide -> step selection -> get_step / decompress+stitch
 * -> simulated generation -> update_after_generation, with the latency and
 * cost models. Requests are processed in order with results identical to
 * serial execution; a batch shares one exact top-8 lookup per table and
 * fixes it up on the host for rows inserted / removed by earlier requests.
 * Definitions the SPEC leaves open (documented in DESIGN.md):
 *   - a hit whose source has no live step <= the desired one serves nothing
 *     (actual 0) and is then handled like a miss for latency and update;
 *   - a decoupled hit serves the largest step both sources hold <= desired;
 *   - update_after_generation inserts nothing while the prompt is cached.
 * ------------------------------------------------------------------------- */
typedef struct lc_engine lc_engine;
typedef struct lc_engine_config {
  double hit_threshold;      /* defaults.hpp:13  0.65 */
  double compress_threshold; /* defaults.hpp:14  0.99 */
  double bin_edges[4];       /* defaults.hpp:27  0.72 0.79 0.86 0.93 */
  double t_per_step;         /* defaults.hpp:21  4.84 s */
  double t_lookup;           /* defaults.hpp:22  0.14 s */
  double t_extract;          /* defaults.hpp:23  3.6 s  */
  double t_stitch;           /* defaults.hpp:24  0 s    */
  int32_t total_steps;       /* defaults.hpp:17  50     */
  int32_t policy;            /* LC_POLICY_*             */
  uint64_t capacity;         /* store capacity, compressed_size bytes */
  int32_t dim, F, H, W, C;   /* embedding dim, latent geometry */
  int32_t skip_oversized;    /* 1: an update whose entry alone exceeds the capacity inserts
                                nothing (CLI capacity sweeps); 0: OversizedEntry */
} lc_engine_config;
void lc_engine_config_default(lc_engine_config* cfg);
typedef struct lc_request {
  uint64_t prompt;
  uint64_t arrival; /* logical time, non-decreasing */
} lc_request;
typedef struct lc_outcome {
  lc_decision decision; /* decide + similarity_to_step on the exact top-1s   */
  int32_t actual_step;  /* served step = skipped steps (0: nothing served)   */
  int32_t n_inserted;   /* steps inserted by update_after_generation          */
  int32_t n_evicted;    /* steps evicted by that insert                       */
  int32_t _pad;
  double latency;       /* t_extract + t_lookup + t_per_step*(50-actual) (+ t_stitch) */
} lc_outcome;
typedef struct lc_engine_metrics {
  uint64_t requests, whole_hits, decoupled_hits, misses;
  uint64_t skipped_hist[6]; /* skipped steps 0,5,10,15,20,25 */
  uint64_t skipped_total;
  double simulated_time;        /* sum of latencies */
  double computation_savings;   /* skipped_total / (50 * requests) */
  double mean_latency;
  double throughput_vs_nocache; /* 50 * t_per_step / mean_latency */
} lc_engine_metrics;
typedef struct lc_pricing {
  double gpu_rate;             /* $/hour (defaults.hpp:33: 3.67) */
  double storage_rate;         /* $/GB/month (no default) */
  double provisioned_storage;  /* GB */
} lc_pricing;
typedef struct lc_cost_report {
  double gpu_cost_per_video, storage_cost_per_video, videos_per_month, throughput_vs_nocache, mean_latency;
} lc_cost_report;
lc_status lc_engine_create(lc_ctx* ctx, const lc_engine_config* cfg, lc_engine** out);
lc_status lc_engine_destroy(lc_engine* e);
/* process_request + update_after_generation for n requests
 * in order. q_* [n][dim] unit embeddings; latents [n][5][F][H*W*C] fp32 =
 * each prompt's own latents at steps 5..25; masks [n][F][ceil(H*W/8)].
 * Host or device buffers. served_dev (device [n][F][E], may be NULL)
 * receives the served / stitched latent of every hit. On error, out[0..j)
 * hold the requests completed before the failing one. */
lc_status lc_engine_process(lc_engine* e, const lc_request* req, int64_t n, const float* q_whole,
                            const float* q_object, const float* q_background, const float* latents,
                            const uint8_t* obj_masks, const uint8_t* bg_masks, float* served_dev,
                            lc_outcome* out);
lc_status lc_engine_metrics_get(lc_engine* e, lc_engine_metrics* out);
/* report; zero requests => LC_ERR_INVALID_ARGUMENT. */
lc_status lc_engine_report(lc_engine* e, const lc_pricing* pricing, lc_cost_report* out);
/* The engine's index and store (borrowed; e.g. for lc_snapshot_save). */
lc_index* lc_engine_index(lc_engine* e);
lc_store* lc_engine_store(lc_engine* e);

/* ---------------------------------------------------------------------------
 * simgen (simgen.hpp declares it, no reference code): the
 * on-device synthetic generator, defined in csrc/simgen.cu and restated in
 * oracle/lc_oracle.c (orc_synth_*), bit-identical between the two.
 * ------------------------------------------------------------------------- */
/* synth_embedding for n prompts: tokens [n][max_tokens] (first n_tokens[i]
 * used, 1..16), unit fp32 out [n][dim]; host or device buffers. */
lc_status lc_synth_embeddings(lc_ctx* ctx, const uint64_t* tokens, const int32_t* n_tokens,
                              int max_tokens, int64_t n, int dim, uint64_t seed, float* out);
typedef struct lc_latent_spec {
  double redundancy[5]; /* redundant-frame fraction per cached step (defaults.hpp:42) */
  double alpha[5];      /* differential scale per step (defaults.hpp:43)            */
  double noise_sigma;   /* relative noise on the differentials (defaults.hpp:44)     */
  double dup_noise;     /* absolute jitter of a redundant frame                      */
} lc_latent_spec;
void lc_latent_spec_default(lc_latent_spec* spec);
/* synth_latents for n prompt seeds: latents [n][5][F][H*W*C] (steps 5..25),
 * rectangular object / background masks [n][F][ceil(H*W/8)]. spec NULL =
 * defaults. */
lc_status lc_synth_latents(lc_ctx* ctx, const uint64_t* prompt_seeds, int64_t n, int F, int H,
                           int W, int C, const lc_latent_spec* spec, float* latents,
                           uint8_t* obj_masks, uint8_t* bg_masks);

/* lrbu_priority / lcbfu_priority (store.cpp:32-42) for n entries. */
lc_status lc_priority_batch(lc_ctx* ctx, int policy, const lc_step_entry* e, int64_t n,
                            uint64_t now, double* out);

/* ---------------------------------------------------------------------------
 * Entry-sharded multi-GPU cache (the reference is single-node
 * CPU and has no counterpart). One process or thread per GPU; prompt p lives
 * on rank lc_shard_owner(p, G) = p mod G (its index rows, entry and live
 * steps). Every sharded call is COLLECTIVE: all ranks call it in the same
 * order with the same arguments (queries, prompt, steps, now).
 * ------------------------------------------------------------------------- */
/* ncclGetUniqueId: rank 0 creates it and shares the 128 bytes out of band. */
lc_status lc_comm_unique_id(uint8_t* id128);
/* NCCL communicator (ncclCommInitRank) on the context's GPU. */
lc_status lc_ctx_comm_init(lc_ctx* ctx, int nranks, int rank, const uint8_t* id128);
/* Caller-provided transport: fn all-gathers `bytes` from every rank into
 * recv[nranks][bytes] (host buffers) and returns 0 on success. */
typedef int (*lc_allgather_fn)(void* user, const void* send, void* recv, uint64_t bytes);
lc_status lc_ctx_comm_host(lc_ctx* ctx, int nranks, int rank, lc_allgather_fn fn, void* user);
/* backend: 0 none, 1 NCCL (nranks from ncclCommCount), 2 host callback. */
lc_status lc_ctx_comm_info(lc_ctx* ctx, int* nranks, int* rank, int* backend,
                           uint64_t* collectives);
uint64_t lc_shard_owner(uint64_t prompt, int nranks);
/* Global exact top-k over the union of the ranks' shards: local top-k
 * (lc_index_query_topk path), one grouped all-gather of the [G][n][k] lists,
 * merge by (score desc, id asc) (vindex.cpp:58-72). Same queries on every
 * rank; every rank gets the full result. */
lc_status lc_sharded_query_topk(lc_index* ix, int kind, const float* q, int64_t n, int dim, int k,
                                uint64_t* out_ids, double* out_scores, int32_t* out_counts);
lc_status lc_sharded_lookup_decide(lc_index* ix, const float* qw, const float* qo,
                                   const float* qb, int64_t n, int dim, double hit_threshold,
                                   const double* edges4, lc_decision* out);
/* CacheStore (store.hpp:48-120) under ONE global capacity budget. Each rank
 * owns a local unbounded store (lc_sharded_store_local) holding its prompts.
 * insert_steps / evict_one produce the same StepEntry sequence, used() and
 * next_seq as a single store holding every prompt: evictions are the
 * (key, seq) merge of the shards' lc_store_peek_many lists, `batch` victims
 * per shard per all-gather round (0 = 64). */
typedef struct lc_sharded_store lc_sharded_store;
lc_status lc_sharded_store_create(lc_ctx* ctx, uint64_t capacity, int policy, int batch,
                                  lc_sharded_store** out);
lc_status lc_sharded_store_destroy(lc_sharded_store* ss);
lc_store* lc_sharded_store_local(lc_sharded_store* ss);
/* entry: the owner rank passes the prompt's entry, the others NULL. Errors
 * (validation, OversizedEntry) are raised on every rank. */
lc_status lc_sharded_store_insert(lc_sharded_store* ss, uint64_t prompt, lc_entry* entry,
                                  const int32_t* steps, int n_steps, uint64_t now,
                                  lc_step_entry* evicted, int cap, int* n_evicted);
lc_status lc_sharded_store_evict_one(lc_sharded_store* ss, uint64_t now, lc_step_entry* out);
/* get_step on the owner (out_dev: owner's device buffer or NULL); every rank
 * gets the actual step (0 = nothing served). */
lc_status lc_sharded_store_get_step(lc_sharded_store* ss, uint64_t prompt, int desired, uint64_t now,
                                    int32_t* actual, float* out_dev);
lc_status lc_sharded_store_used(lc_sharded_store* ss, uint64_t* out);
lc_status lc_sharded_store_stats(lc_sharded_store* ss, uint64_t* rounds, uint64_t* local_evictions,
                                 uint64_t* next_seq);

#ifdef __cplusplus
}
#endif
#endif /* FLEXCACHE_B200_H */
