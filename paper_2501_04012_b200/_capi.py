"""ctypes binding of the C-ABI (include/flexcache_b200.h).

Loads the in-tree paper_2501_04012_b200/_lib/libflexcache_b200.so. There is
no fallback: if the library is missing or cannot be loaded the import fails
with the reason.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libflexcache_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"flexcache-b200: CUDA library not built ({LIB_PATH}); run "
                      f"`python -m paper_2501_04012_b200.build` or __graft_entry__.build()")
lib = C.CDLL(LIB_PATH)

vp = C.c_void_p
u64, i64, i32, f64 = C.c_uint64, C.c_int64, C.c_int32, C.c_double


class StepEntry(C.Structure):
    """StepEntry (store.hpp:28-36)."""
    _fields_ = [("prompt", u64), ("step", i32), ("_pad", i32), ("f", u64), ("last_access", u64),
                ("inserted_at", u64), ("inserted_seq", u64), ("capacity", u64)]

    def as_tuple(self):
        return (self.prompt, self.step, self.f, self.last_access, self.inserted_at, self.inserted_seq,
                self.capacity)

    def __repr__(self):
        return ("StepEntry(prompt=%d, step=%d, f=%d, last_access=%d, inserted_at=%d, inserted_seq=%d, "
                "capacity=%d)" % self.as_tuple())


class Decision(C.Structure):
    _fields_ = [("kind", i32), ("step", i32), ("whole_id", u64), ("object_id", u64), ("background_id", u64),
                ("score", f64), ("whole_score", f64), ("object_score", f64), ("background_score", f64)]


class EngineConfig(C.Structure):
    _fields_ = [("hit_threshold", f64), ("compress_threshold", f64), ("bin_edges", f64 * 4), ("t_per_step", f64),
                ("t_lookup", f64), ("t_extract", f64), ("t_stitch", f64), ("total_steps", i32), ("policy", i32),
                ("capacity", u64), ("dim", i32), ("F", i32), ("H", i32), ("W", i32), ("C", i32),
                ("skip_oversized", i32)]


class Request(C.Structure):
    _fields_ = [("prompt", u64), ("arrival", u64)]


class Outcome(C.Structure):
    _fields_ = [("decision", Decision), ("actual_step", i32), ("n_inserted", i32), ("n_evicted", i32),
                ("_pad", i32), ("latency", f64)]


class EngineMetrics(C.Structure):
    _fields_ = [("requests", u64), ("whole_hits", u64), ("decoupled_hits", u64), ("misses", u64),
                ("skipped_hist", u64 * 6), ("skipped_total", u64), ("simulated_time", f64),
                ("computation_savings", f64), ("mean_latency", f64), ("throughput_vs_nocache", f64)]


class Pricing(C.Structure):
    _fields_ = [("gpu_rate", f64), ("storage_rate", f64), ("provisioned_storage", f64)]


class CostReport(C.Structure):
    _fields_ = [("gpu_cost_per_video", f64), ("storage_cost_per_video", f64), ("videos_per_month", f64),
                ("throughput_vs_nocache", f64), ("mean_latency", f64)]


class LatentSpec(C.Structure):
    _fields_ = [("redundancy", f64 * 5), ("alpha", f64 * 5), ("noise_sigma", f64), ("dup_noise", f64)]


class LookupStats(C.Structure):
    _fields_ = [("queries", u64), ("certified", u64), ("fallback", u64), ("exact_scans", u64),
                ("max_abs_err", f64), ("tier2_certified", u64), ("i8_batches", u64), ("i8_rescored", u64),
                ("i8_candidates", u64), ("i8_prescored", u64), ("threshold_certified", u64)]


class CodecStats(C.Structure):
    _fields_ = [("inter_items", u64), ("inter_exact_items", u64)]


class EntryInfo(C.Structure):
    _fields_ = [("prompt", u64), ("base_step", i32), ("n_steps", i32), ("F", i32), ("H", i32), ("W", i32),
                ("C", i32), ("n_diff", i32), ("steps", i32 * 8), ("n_extra", i32 * 8),
                ("shared_bytes", u64), ("private_bytes", u64 * 8), ("compressed_size", u64)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


st = C.c_int  # lc_status
_sig("lc_last_error", C.c_char_p)
_sig("lc_last_oversize", None, C.POINTER(u64), C.POINTER(u64))
_sig("lc_last_snapshot_offset", u64)
_sig("lc_version", C.c_char_p)
_sig("lc_ctx_create", st, C.c_int, C.POINTER(vp))
_sig("lc_ctx_destroy", st, vp)
_sig("lc_ctx_set_stream", st, vp, vp)
_sig("lc_ctx_stream", vp, vp)
_sig("lc_ctx_synchronize", st, vp)
_sig("lc_ctx_launches", u64, vp)
_sig("lc_embedding_normalize", st, vp, vp, i64, C.c_int, vp)
_sig("lc_cosine_batch", st, vp, vp, vp, i64, i64, vp)
_sig("lc_index_create", st, vp, C.c_int, i64, C.POINTER(vp))
_sig("lc_index_destroy", st, vp)
_sig("lc_index_insert", st, vp, u64, vp, vp, vp, C.c_int)
_sig("lc_index_insert_batch", st, vp, vp, vp, vp, vp, i64, C.c_int)
_sig("lc_index_remove", st, vp, u64)
_sig("lc_index_contains", st, vp, u64, C.POINTER(i32))
_sig("lc_index_size", i64, vp)
_sig("lc_index_dim", C.c_int, vp)
_sig("lc_index_export", st, vp, C.c_int, vp, vp, i64)
_sig("lc_index_query_topk", st, vp, C.c_int, vp, i64, C.c_int, vp, vp, vp)
_sig("lc_lookup_decide", st, vp, vp, vp, vp, i64, f64, vp, vp)
_sig("lc_index_stats", st, vp, C.POINTER(LookupStats), C.c_int)
_sig("lc_codec_stats_get", st, vp, C.POINTER(CodecStats), C.c_int)
_sig("lc_index_set_lookup", st, vp, C.c_int, C.c_int, f64)
_sig("lc_topk_merge", st, vp, vp, vp, vp, C.c_int, i64, C.c_int, vp, vp, vp)
_sig("lc_decide_batch", st, vp, vp, vp, vp, vp, vp, vp, i64, f64, vp, vp)
_sig("lc_select_keyframes", st, vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, f64, vp)
_sig("lc_solve_alpha_batch", st, vp, vp, vp, i64, i64, vp)
_sig("lc_compress_batch", st, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, f64, vp, i64,
     vp, vp)
_sig("lc_inter_compress", st, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, u64,
     C.POINTER(vp))
_sig("lc_entry_release", st, vp)
_sig("lc_entry_export", st, vp, vp, u64, C.POINTER(u64))
_sig("lc_entry_import", st, vp, vp, u64, C.POINTER(vp))
_sig("lc_entry_get_info", st, vp, C.POINTER(EntryInfo))
_sig("lc_decompress_batch", st, vp, vp, vp, i64, vp)
_sig("lc_decompress_stitch_batch", st, vp, vp, vp, vp, i64, vp)
_sig("lc_stitch_batch", st, vp, vp, vp, vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, vp)
_sig("lc_store_create", st, vp, u64, C.c_int, C.POINTER(vp))
_sig("lc_snapshot_save", st, vp, vp, C.c_char_p)
_sig("lc_store_peek", st, vp, u64, C.POINTER(StepEntry), C.POINTER(f64))
_sig("lc_store_next_seq", u64, vp)
_sig("lc_store_set_next_seq", st, vp, u64)
_sig("lc_engine_config_default", None, C.POINTER(EngineConfig))
_sig("lc_synth_embeddings", st, vp, vp, vp, C.c_int, i64, C.c_int, u64, vp)
_sig("lc_latent_spec_default", None, C.POINTER(LatentSpec))
_sig("lc_synth_latents", st, vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(LatentSpec), vp, vp, vp)
_sig("lc_engine_create", st, vp, C.POINTER(EngineConfig), C.POINTER(vp))
_sig("lc_engine_destroy", st, vp)
_sig("lc_engine_process", st, vp, C.POINTER(Request), i64, vp, vp, vp, vp, vp, vp, vp, C.POINTER(Outcome))
_sig("lc_engine_metrics_get", st, vp, C.POINTER(EngineMetrics))
_sig("lc_engine_report", st, vp, C.POINTER(Pricing), C.POINTER(CostReport))
_sig("lc_engine_index", vp, vp)
_sig("lc_engine_store", vp, vp)
_sig("lc_snapshot_load", st, vp, C.c_char_p, C.POINTER(vp), C.POINTER(vp))
_sig("lc_store_destroy", st, vp)
_sig("lc_store_insert", st, vp, u64, vp, vp, C.c_int, u64, vp, C.c_int, C.POINTER(C.c_int))
_sig("lc_store_get_step", st, vp, u64, C.c_int, u64, C.POINTER(i32), vp)
_sig("lc_store_evict_one", st, vp, u64, C.POINTER(StepEntry))
_sig("lc_store_evict_step", st, vp, u64, C.c_int, C.POINTER(i32))
_sig("lc_store_used", u64, vp)
_sig("lc_store_recompute_used", u64, vp)
_sig("lc_store_capacity", u64, vp)
_sig("lc_store_policy", C.c_int, vp)
_sig("lc_store_step_count", i64, vp)
_sig("lc_store_prompt_count", i64, vp)
_sig("lc_store_contains", st, vp, u64, C.POINTER(i32))
_sig("lc_store_cached_steps", st, vp, u64, vp, C.POINTER(C.c_int))
_sig("lc_store_entry", st, vp, u64, C.POINTER(vp))
_sig("lc_store_entries", st, vp, vp, i64, C.POINTER(i64))
_sig("lc_priority_batch", st, vp, C.c_int, vp, i64, u64, vp)
_sig("lc_store_peek_many", st, vp, u64, C.c_int, C.POINTER(StepEntry), vp, vp, C.POINTER(C.c_int),
     C.POINTER(C.c_int))
_sig("lc_store_check_insert", st, vp, u64, vp, vp, C.c_int, C.POINTER(u64))
# entry-sharded multi-GPU (shard.cu)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, vp, vp, vp, u64)
_sig("lc_comm_unique_id", st, vp)
_sig("lc_ctx_comm_init", st, vp, C.c_int, C.c_int, vp)
_sig("lc_ctx_comm_host", st, vp, C.c_int, C.c_int, ALLGATHER_FN, vp)
_sig("lc_ctx_comm_info", st, vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(u64))
_sig("lc_shard_owner", u64, u64, C.c_int)
_sig("lc_sharded_query_topk", st, vp, C.c_int, vp, i64, C.c_int, C.c_int, vp, vp, vp)
_sig("lc_sharded_lookup_decide", st, vp, vp, vp, vp, i64, C.c_int, f64, vp, vp)
_sig("lc_sharded_store_create", st, vp, u64, C.c_int, C.c_int, C.POINTER(vp))
_sig("lc_sharded_store_destroy", st, vp)
_sig("lc_sharded_store_local", vp, vp)
_sig("lc_sharded_store_insert", st, vp, u64, vp, vp, C.c_int, u64, C.POINTER(StepEntry), C.c_int,
     C.POINTER(C.c_int))
_sig("lc_sharded_store_evict_one", st, vp, u64, C.POINTER(StepEntry))
_sig("lc_sharded_store_get_step", st, vp, u64, C.c_int, u64, C.POINTER(i32), vp)
_sig("lc_sharded_store_used", st, vp, C.POINTER(u64))
_sig("lc_sharded_store_stats", st, vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64))

# every symbol declared in include/flexcache_b200.h (checked by the CPU tests)
EXPORTED = sorted(n for n in dir(lib) if n.startswith("lc_"))
