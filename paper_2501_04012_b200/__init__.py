"""flexcache-b200: B200-native FlexCache cache hot path (arXiv 2501.04012).

Python mirror of the reference C++ API (`lcache`, /root/reference/proj/include/
lcache/*.hpp) over the C-ABI in include/flexcache_b200.h. Names, argument
meaning and error types follow the reference:

  SimilarityIndex.insert / query_top1 / query_topk / remove / contains / size /
      entries                                               (vindex.hpp:23-62)
  lookup_decide (decide + similarity_to_step)
  select_keyframes / solve_alpha / compress (intra x S + inter) /
      inter_compress / decompress_step / compressed_size / serialize_entry /
      deserialize_entry                                     (codec.hpp:69-118)
  stitch / decompress_stitch                                (stitcher.hpp:24)
  CacheStore.insert_steps / get_step / evict_one / evict_step / used / ...
                                                            (store.hpp:48-120)
  lrbu_priority / lcbfu_priority                            (store.hpp:41,44)

Exceptions map 1:1 to the reference's (errors.hpp:11-42): InvalidArgument
(std::invalid_argument), DegenerateBase, StepNotCached, OversizedEntry,
SnapshotError, LogicError (std::logic_error).

Arrays may be numpy (host) or torch CUDA tensors (device): device tensors are
used in place (no copies), host arrays are staged by the library.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _capi
from ._capi import Decision, EntryInfo, LookupStats, StepEntry, lib

__all__ = ["Context", "SimilarityIndex", "EmbeddingKind", "Policy", "CacheStore", "CompressedEntry",
           "select_keyframes", "solve_alpha", "compress", "compress_batch", "inter_compress", "decompress_step",
           "decompress_batch", "decompress_stitch", "stitch", "compressed_size", "serialize_entry",
           "deserialize_entry", "lrbu_priority", "lcbfu_priority", "lookup_decide", "topk_merge", "decide_batch",
           "embedding_normalize", "cosine_similarity", "StepEntry", "LcacheError", "InvalidArgument",
           "DegenerateBase", "StepNotCached", "OversizedEntry", "SnapshotError", "LogicError", "default_context",
           "HIT_THRESHOLD", "COMPRESS_THRESHOLD", "STEP_BIN_EDGES", "CACHED_STEPS"]

# defaults.hpp:13-27
HIT_THRESHOLD = 0.65
COMPRESS_THRESHOLD = 0.99
STEP_BIN_EDGES = (0.72, 0.79, 0.86, 0.93)
CACHED_STEPS = (5, 10, 15, 20, 25)


class LcacheError(RuntimeError):
    code = 0


class InvalidArgument(LcacheError, ValueError):
    code = 1


class DegenerateBase(LcacheError):
    code = 2


class StepNotCached(LcacheError):
    code = 3


class OversizedEntry(LcacheError):
    code = 4

    def __init__(self, msg, needed_bytes=0, capacity_limit=0):
        super().__init__(msg)
        self.needed_bytes = needed_bytes
        self.capacity_limit = capacity_limit


class SnapshotError(LcacheError):
    """SnapshotError (errors.hpp:30-35): byte_offset of the failing record/field."""
    code = 5

    def __init__(self, msg, byte_offset=0):
        super().__init__(msg)
        self.byte_offset = byte_offset


class LogicError(LcacheError):
    code = 6


class CudaError(LcacheError):
    code = 7


class SnapshotIOError(LcacheError, OSError):
    """std::runtime_error from snapshot file I/O (store.cpp:268-276)."""
    code = 11


_ERR = {1: InvalidArgument, 2: DegenerateBase, 3: StepNotCached, 4: OversizedEntry, 5: SnapshotError,
        6: LogicError, 7: CudaError, 9: CudaError, 11: SnapshotIOError}


def _check(rc):
    if rc == 0:
        return
    msg = (lib.lc_last_error() or b"").decode()
    cls = _ERR.get(rc, LcacheError)
    if cls is OversizedEntry:
        a, b = C.c_uint64(), C.c_uint64()
        lib.lc_last_oversize(C.byref(a), C.byref(b))
        raise OversizedEntry(msg, a.value, b.value)
    if cls is SnapshotError:
        raise SnapshotError(msg, int(lib.lc_last_snapshot_offset()))
    err = cls(msg)
    err.code = rc
    try:
        raise err
    finally:  # no frame <-> exception cycle (it would keep library objects alive until a GC pass)
        del err


class EmbeddingKind(IntEnum):
    Whole = 0
    Object = 1
    Background = 2


class Policy(IntEnum):
    Fifo = 0
    Lru = 1
    Lcbfu = 2
    Lrbu = 3

    @staticmethod
    def parse(name: str) -> "Policy":  # parse_policy, store.cpp:13-19
        m = {"fifo": Policy.Fifo, "lru": Policy.Lru, "lcbfu": Policy.Lcbfu, "lrbu": Policy.Lrbu}
        if name not in m:
            raise InvalidArgument("unknown policy: " + name)
        return m[name]


# ---------------------------------------------------------------------------
# buffers: numpy (host) or torch CUDA tensors (device, used in place)
# ---------------------------------------------------------------------------
def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise InvalidArgument("tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _host(a, dtype):
    if hasattr(a, "data_ptr"):
        return a
    return np.ascontiguousarray(a, dtype=dtype)


def _is_dev(a):
    return hasattr(a, "data_ptr") and getattr(a, "is_cuda", False)


class Context:
    """One GPU + stream (lc_ctx)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        """stream: a cudaStream_t value to issue on; default = torch's current
        stream on `device` (so library work is stream-ordered with torch ops on
        the tensors it reads/writes); 1 = cudaStreamLegacy."""
        h = C.c_void_p()
        _check(lib.lc_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    s = torch.cuda.current_stream(device).cuda_stream
                    stream = s if s else 1
            except ImportError:
                stream = None
        if stream:
            self.set_stream(stream)

    def set_stream(self, stream_ptr: int | None):
        _check(lib.lc_ctx_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None))

    @property
    def stream(self) -> int:
        return lib.lc_ctx_stream(self.h) or 0

    def synchronize(self):
        _check(lib.lc_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return lib.lc_ctx_launches(self.h)

    def __del__(self):
        try:
            if self.h:
                lib.lc_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


_default_ctx: Context | None = None


def _alive(ctx) -> bool:
    """False once the context was destroyed: objects found in the same garbage
    cycle as their context may be finalised after it (PEP 442 order is
    arbitrary); their device memory then goes with the process instead of
    being released through a dangling context."""
    return ctx is None or bool(getattr(ctx, "h", None))


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _ctx(ctx):
    return (ctx or default_context()).h


# ---------------------------------------------------------------------------
# core
# ---------------------------------------------------------------------------
def embedding_normalize(v, ctx=None):
    """Embedding ctor normalisation (core.cpp:50-59), rows of a 2-D array."""
    v = _host(v, np.float32)
    n, d = (v.shape[0], v.shape[1]) if v.ndim == 2 else (1, v.shape[0])
    out = (v.new_empty(v.shape) if _is_dev(v) else np.empty_like(v))
    _check(lib.lc_embedding_normalize(_ctx(ctx), _ptr(v), n, d, _ptr(out)))
    return out


def cosine_similarity(a, b, ctx=None):
    """cosine_similarity (core.cpp:101-114) of rows of a and b."""
    a = _host(a, np.float32)
    b = _host(b, np.float32)
    a2 = a.reshape(-1, a.shape[-1]) if a.ndim > 1 else a.reshape(1, -1)
    b2 = b.reshape(-1, b.shape[-1]) if b.ndim > 1 else b.reshape(1, -1)
    if a2.shape != b2.shape:
        raise InvalidArgument("cosine_similarity: length mismatch")
    out = np.zeros(a2.shape[0], np.float64)
    _check(lib.lc_cosine_batch(_ctx(ctx), _ptr(a2), _ptr(b2), a2.shape[0], a2.shape[1], _ptr(out)))
    return out if a.ndim > 1 else float(out[0])


# ---------------------------------------------------------------------------
# SimilarityIndex
# ---------------------------------------------------------------------------
@dataclass
class QueryResult:
    prompt: int
    score: float


class SimilarityIndex:
    """Three-table exact top-k index (vindex.hpp:23-62) resident in HBM."""

    def __init__(self, dim: int = 0, capacity_rows: int = 0, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib.lc_index_create(self.ctx.h, dim, capacity_rows, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h and not getattr(self, "_borrowed", None) and _alive(self.ctx):
                lib.lc_index_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def insert(self, whole, obj, background, prompt: int):
        w, o, b = (_host(x, np.float32) for x in (whole, obj, background))
        if not (w.shape[-1] == o.shape[-1] == b.shape[-1]):
            raise InvalidArgument("SimilarityIndex: embedding dimension mismatch")
        _check(lib.lc_index_insert(self.h, prompt, _ptr(w), _ptr(o), _ptr(b), w.shape[-1]))

    def insert_batch(self, prompts, whole, obj, background):
        p = np.ascontiguousarray(prompts, np.uint64)
        w, o, b = (_host(x, np.float32) for x in (whole, obj, background))
        _check(lib.lc_index_insert_batch(self.h, _ptr(p), _ptr(w), _ptr(o), _ptr(b), p.size, w.shape[1]))

    def remove(self, prompt: int):
        _check(lib.lc_index_remove(self.h, prompt))

    def contains(self, prompt: int) -> bool:
        r = C.c_int32()
        _check(lib.lc_index_contains(self.h, prompt, C.byref(r)))
        return bool(r.value)

    def size(self) -> int:
        return lib.lc_index_size(self.h)

    def dim(self) -> int:
        return lib.lc_index_dim(self.h)

    def entries(self, kind: EmbeddingKind):
        n = self.size()
        ids = np.zeros(n, np.uint64)
        rows = np.zeros((n, max(self.dim(), 1)), np.float32)
        _check(lib.lc_index_export(self.h, int(kind), _ptr(ids), _ptr(rows), n))
        return ids, rows

    def query_topk(self, kind: EmbeddingKind, q, k: int = 1, out=None):
        """(ids [n,k] u64, scores [n,k] f64, counts [n] i32). Device tensors in ->
        device tensors out (pass `out` to reuse buffers)."""
        q = _host(q, np.float32)
        n = q.shape[0] if q.ndim == 2 else 1
        if out is None:
            if _is_dev(q):
                import torch
                out = (torch.empty((n, k), dtype=torch.int64, device=q.device),
                       torch.empty((n, k), dtype=torch.float64, device=q.device),
                       torch.empty((n,), dtype=torch.int32, device=q.device))
            else:
                out = (np.zeros((n, k), np.uint64), np.zeros((n, k), np.float64), np.zeros(n, np.int32))
        _check(lib.lc_index_query_topk(self.h, int(kind), _ptr(q), n, k, _ptr(out[0]), _ptr(out[1]),
                                       _ptr(out[2])))
        return out

    def query_top1(self, kind: EmbeddingKind, q):
        """query_top1 (vindex.cpp:50-74): QueryResult or None (empty table)."""
        q = np.ascontiguousarray(q, np.float32).reshape(1, -1)
        if self.size() and q.shape[1] != self.dim():
            raise InvalidArgument("SimilarityIndex: query dimension mismatch")
        ids, sc, cnt = self.query_topk(kind, q, 1)
        if cnt[0] == 0:
            return None
        return QueryResult(int(ids[0, 0]), float(sc[0, 0]))

    def set_lookup(self, mode: int = 0, kprime: int = 0, eps: float = 0.0):
        _check(lib.lc_index_set_lookup(self.h, mode, kprime, eps))

    def stats(self, reset: bool = False) -> LookupStats:
        s = LookupStats()
        _check(lib.lc_index_stats(self.h, C.byref(s), int(reset)))
        return s


def lookup_decide(index: SimilarityIndex, qw, qo, qb, hit_threshold=HIT_THRESHOLD, edges=STEP_BIN_EDGES, out=None):
    """Fused 3-table lookup + decide + similarity_to_step.
    Returns an array of Decision records (numpy structured via ctypes)."""
    qw, qo, qb = (_host(x, np.float32) for x in (qw, qo, qb))
    n = qw.shape[0]
    e = np.ascontiguousarray(edges, np.float64)
    if out is None:
        out = (Decision * n)()
    _check(lib.lc_lookup_decide(index.h, _ptr(qw), _ptr(qo), _ptr(qb), n, hit_threshold, _ptr(e),
                                C.cast(out, C.c_void_p) if not hasattr(out, "data_ptr") else _ptr(out)))
    return out


def decide_batch(w_ids, w_sc, o_ids, o_sc, b_ids, b_sc, hit_threshold=HIT_THRESHOLD, edges=STEP_BIN_EDGES, ctx=None):
    """decide + similarity_to_step on top-1 triples (host
    arrays or device tensors); returns a host array of Decision records."""
    if _is_dev(w_ids):
        arrs = [a.contiguous() for a in (w_ids, w_sc, o_ids, o_sc, b_ids, b_sc)]
    else:
        arrs = [np.ascontiguousarray(a, t) for a, t in ((w_ids, np.uint64), (w_sc, np.float64), (o_ids, np.uint64),
                                                         (o_sc, np.float64), (b_ids, np.uint64), (b_sc, np.float64))]
    n = int(arrs[0].numel() if _is_dev(arrs[0]) else arrs[0].size)
    out = (Decision * n)()
    e = np.ascontiguousarray(edges, np.float64)
    _check(lib.lc_decide_batch(_ctx(ctx), *[_ptr(a) for a in arrs], n, hit_threshold, _ptr(e),
                               C.cast(out, C.c_void_p)))
    return out


def topk_merge(ids, scores, counts, k, ctx=None, out=None):
    """Merge G shard top-k lists ([G][n][k], counts [G][n]) into the global
    top-k by (score desc, id asc). Device tensors in -> device tensors out."""
    if _is_dev(ids):
        import torch
        ids, scores, counts = ids.contiguous(), scores.contiguous(), counts.contiguous()
        G, n = counts.shape
        if out is None:
            out = (torch.empty((n, k), dtype=torch.int64, device=ids.device),
                   torch.empty((n, k), dtype=torch.float64, device=ids.device),
                   torch.empty((n,), dtype=torch.int32, device=ids.device))
    else:
        ids = np.ascontiguousarray(ids, np.uint64)
        scores = np.ascontiguousarray(scores, np.float64)
        counts = np.ascontiguousarray(counts, np.int32)
        G, n = counts.shape
        if out is None:
            out = (np.zeros((n, k), np.uint64), np.zeros((n, k), np.float64), np.zeros(n, np.int32))
    _check(lib.lc_topk_merge(_ctx(ctx), _ptr(ids), _ptr(scores), _ptr(counts), G, n, k, _ptr(out[0]), _ptr(out[1]),
                             _ptr(out[2])))
    return out


# ---------------------------------------------------------------------------
# codec
# ---------------------------------------------------------------------------
class CompressedEntry:
    """Handle to a device-resident CompressedEntry (codec.hpp:48-67)."""

    def __init__(self, h, ctx: Context, owned=True):
        self.h = h
        self.hv = h.value if isinstance(h, C.c_void_p) else int(h)  # handle as int (batch calls)
        self.ctx = ctx
        self.owned = owned

    def __del__(self):
        try:
            if self.owned and self.h and _alive(self.ctx):
                lib.lc_entry_release(self.h)
                self.h = None
        except Exception:
            pass

    def info(self) -> EntryInfo:
        i = EntryInfo()
        _check(lib.lc_entry_get_info(self.h, C.byref(i)))
        return i

    @property
    def prompt(self):
        return self.info().prompt

    @property
    def base_step(self):
        return self.info().base_step

    @property
    def steps(self):
        i = self.info()
        return [i.steps[k] for k in range(i.n_steps)]

    def has_step(self, step):
        return step in self.steps

    def serialize(self) -> bytes:
        n = C.c_uint64()
        _check(lib.lc_entry_export(self.h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        _check(lib.lc_entry_export(self.h, buf, n.value, C.byref(n)))
        return bytes(buf)


def compressed_size(entry: CompressedEntry) -> int:
    """codec.cpp:334-338."""
    return entry.info().compressed_size


def uncompressed_size(dims, frame_count, n_steps) -> int:
    H, W, Cc = dims
    return n_steps * frame_count * H * W * Cc * 4


def serialize_entry(entry: CompressedEntry) -> bytes:
    return entry.serialize()


def deserialize_entry(data: bytes, ctx: Context | None = None) -> CompressedEntry:
    ctx = ctx or default_context()
    buf = np.frombuffer(data, np.uint8)
    h = C.c_void_p()
    _check(lib.lc_entry_import(ctx.h, _ptr(buf), buf.size, C.byref(h)))
    return CompressedEntry(h, ctx)


def select_keyframes(latent, dims, threshold=COMPRESS_THRESHOLD, ctx=None):
    """select_keyframes (codec.cpp:138-165); latent [F][E] or batch [n][F][E]."""
    latent = _host(latent, np.float32)
    batched = latent.ndim == 3
    lat = latent if batched else latent.reshape((1,) + tuple(latent.shape))
    n, F = lat.shape[0], lat.shape[1]
    H, W, Cc = dims
    out = np.zeros((n, F), np.int32)
    _check(lib.lc_select_keyframes(_ctx(ctx), _ptr(lat), n, F, H, W, Cc, threshold, _ptr(out)))
    return out if batched else out[0]


def solve_alpha(diff_s, diff_base, ctx=None):
    """solve_alpha (codec.cpp:181-191)."""
    a = _host(diff_s, np.float32)
    b = _host(diff_base, np.float32)
    if a.shape != b.shape:
        raise InvalidArgument("solve_alpha: shape mismatch")
    a2 = a.reshape(-1, a.shape[-1]) if a.ndim > 1 else a.reshape(1, -1)
    b2 = b.reshape(a2.shape)
    out = np.zeros(a2.shape[0], np.float32)
    _check(lib.lc_solve_alpha_batch(_ctx(ctx), _ptr(a2), _ptr(b2), a2.shape[0], a2.shape[1], _ptr(out)))
    return out if a.ndim > 1 else np.float32(out[0])


def compress_batch(latents, steps, obj_masks, bg_masks, dims, prompts, threshold=COMPRESS_THRESHOLD, ctx=None):
    """intra_compress x S + inter_compress for n prompts.
    latents [n][S][F][E]; masks [n][F][ceil(H*W/8)]. Returns (entries, sizes)."""
    ctx = ctx or default_context()
    lat = _host(latents, np.float32)
    om = _host(obj_masks, np.uint8)
    bm = _host(bg_masks, np.uint8)
    n, S, F = lat.shape[0], lat.shape[1], lat.shape[2]
    H, W, Cc = dims
    st_ = np.ascontiguousarray(steps, np.int32)
    pr = np.ascontiguousarray(prompts, np.uint64)
    handles = (C.c_void_p * n)()
    sizes = np.zeros(n, np.uint64)
    _check(lib.lc_compress_batch(ctx.h, _ptr(lat), _ptr(st_), S, F, H, W, Cc, _ptr(om), _ptr(bm), threshold,
                                 _ptr(pr), n, handles, _ptr(sizes)))
    return [CompressedEntry(C.c_void_p(handles[i]), ctx) for i in range(n)], sizes


def codec_stats(reset: bool = False, ctx=None) -> dict:
    """K7 instrumentation: items computed and items the certified kernel
    handed to the exact sequential kernel."""
    st_ = _capi.CodecStats()
    _check(lib.lc_codec_stats_get(_ctx(ctx), C.byref(st_), int(reset)))
    return {"inter_items": int(st_.inter_items), "inter_exact_items": int(st_.inter_exact_items)}


def compress(latent_steps, steps, obj_masks, bg_masks, dims, prompt, threshold=COMPRESS_THRESHOLD, ctx=None):
    """One prompt: latent_steps [S][F][E], masks [F][mb]."""
    lat = _host(latent_steps, np.float32)
    ents, _ = compress_batch(lat.reshape((1,) + tuple(lat.shape)), steps,
                             _host(obj_masks, np.uint8).reshape(1, *np.shape(obj_masks)),
                             _host(bg_masks, np.uint8).reshape(1, *np.shape(bg_masks)), dims, [prompt], threshold, ctx)
    return ents[0]


def inter_compress(latent_steps, maps, steps, obj_masks, bg_masks, dims, prompt, ctx=None):
    """inter_compress (codec.cpp:193-261) on intra-compressed steps given as
    (latent with at least the key frames, key-frame maps)."""
    ctx = ctx or default_context()
    lat = _host(latent_steps, np.float32)
    mp = np.ascontiguousarray(maps, np.int32)
    st_ = np.ascontiguousarray(steps, np.int32)
    S, F = lat.shape[0], lat.shape[1]
    H, W, Cc = dims
    h = C.c_void_p()
    _check(lib.lc_inter_compress(ctx.h, _ptr(lat), _ptr(mp), _ptr(st_), S, F, H, W, Cc,
                                 _ptr(_host(obj_masks, np.uint8)), _ptr(_host(bg_masks, np.uint8)), prompt, C.byref(h)))
    return CompressedEntry(h, ctx)


def _handles(entries):
    """lc_entry* array of a list of CompressedEntry (uintp numpy array)."""
    return np.fromiter((e.hv for e in entries), dtype=np.uintp, count=len(entries))


def _torch_after(ctx):
    """The decompress calls are stream-ordered on ctx's stream: order torch's
    current stream after it (no host sync) when the two differ."""
    import torch
    cur = torch.cuda.current_stream(ctx.device)
    cs = ctx.stream
    if cs in (0, 1) and cur.cuda_stream == 0 or cs == cur.cuda_stream:
        return
    ev = torch.cuda.Event()
    ev.record(torch.cuda.ExternalStream(cs, device=ctx.device))
    cur.wait_event(ev)


def _torch_out(shape, ctx):
    import torch
    return torch.empty(shape, dtype=torch.float32, device=f"cuda:{ctx.device}")


def decompress_batch(entries, steps, out=None):
    """decompress_step (codec.cpp:263-301) for n (entry, step) pairs into a
    device tensor [n][F][E] (allocated if out is None)."""
    ctx = entries[0].ctx
    n = len(entries)
    info = entries[0].info()
    E = info.H * info.W * info.C
    if out is None:
        out = _torch_out((n, info.F, E), ctx)
    hs = _handles(entries)
    st_ = np.ascontiguousarray(steps, np.int32)
    _check(lib.lc_decompress_batch(ctx.h, _ptr(hs), _ptr(st_), n, _ptr(out)))
    _torch_after(ctx)
    return out


def decompress_step(entry: CompressedEntry, step: int):
    """decompress_step for one entry -> numpy [F][E]."""
    return decompress_batch([entry], [step])[0].cpu().numpy()


def decompress_stitch(obj_entries, bg_entries, steps, out=None):
    """Decoupled hit: decompress both sources at `steps` and stitch them."""
    ctx = obj_entries[0].ctx
    n = len(obj_entries)
    info = obj_entries[0].info()
    E = info.H * info.W * info.C
    if out is None:
        out = _torch_out((n, info.F, E), ctx)
    ho = _handles(obj_entries)
    hb = _handles(bg_entries)
    st_ = np.ascontiguousarray(steps, np.int32)
    _check(lib.lc_decompress_stitch_batch(ctx.h, _ptr(ho), _ptr(hb), _ptr(st_), n, _ptr(out)))
    _torch_after(ctx)
    return out


def stitch(obj_latent, obj_src_obj_masks, bg_latent, bg_src_obj_masks, dims, ctx=None):
    """stitch (stitcher.cpp:7-39): latents [F][E] (or [n][F][E]); masks are the
    object-source's and the background-source's OBJECT masks."""
    a = _host(obj_latent, np.float32)
    b = _host(bg_latent, np.float32)
    if a.shape != b.shape:
        raise InvalidArgument("stitch: latent shape mismatch")
    batched = a.ndim == 3
    a3 = a if batched else a.reshape((1,) + tuple(a.shape))
    b3 = b if batched else b.reshape((1,) + tuple(b.shape))
    n, F = a3.shape[0], a3.shape[1]
    H, W, Cc = dims
    out = (a3.new_empty(a3.shape) if _is_dev(a3) else np.empty_like(a3))
    _check(lib.lc_stitch_batch(_ctx(ctx), _ptr(a3), _ptr(_host(obj_src_obj_masks, np.uint8)), _ptr(b3),
                               _ptr(_host(bg_src_obj_masks, np.uint8)), n, F, H, W, Cc, _ptr(out)))
    return out if batched else out[0]


# ---------------------------------------------------------------------------
# store
# ---------------------------------------------------------------------------
def _entries_arr(e):
    if isinstance(e, StepEntry):
        return (StepEntry * 1)(e), 1
    arr = (StepEntry * len(e))(*e)
    return arr, len(e)


def lrbu_priority(e: StepEntry, now: int, ctx=None) -> float:
    arr, n = _entries_arr(e)
    out = np.zeros(n, np.float64)
    _check(lib.lc_priority_batch(_ctx(ctx), 3, C.cast(arr, C.c_void_p), n, now, _ptr(out)))
    return float(out[0]) if isinstance(e, StepEntry) else out


def lcbfu_priority(e: StepEntry, ctx=None) -> float:
    arr, n = _entries_arr(e)
    out = np.zeros(n, np.float64)
    _check(lib.lc_priority_batch(_ctx(ctx), 2, C.cast(arr, C.c_void_p), n, 0, _ptr(out)))
    return float(out[0]) if isinstance(e, StepEntry) else out


class CacheStore:
    """Capacity-bounded (prompt, step) store (store.hpp:48-120)."""

    def __init__(self, capacity_limit: int, policy: Policy, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib.lc_store_create(self.ctx.h, capacity_limit, int(policy), C.byref(h)))
        self.h = h
        self._cb = None

    def __del__(self):
        try:
            if self.h and not getattr(self, "_borrowed", None) and _alive(self.ctx):
                lib.lc_store_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def set_eviction_callback(self, cb):
        """Invoked with the prompt id when its last step is evicted (store.hpp:88)."""
        self._cb = cb

    def _notify(self, evicted):
        if self._cb:
            for e in evicted:
                if not self.contains(e.prompt):
                    self._cb(e.prompt)

    def insert_steps(self, prompt: int, entry: CompressedEntry, steps, now: int):
        st_ = np.ascontiguousarray(steps, np.int32)
        cap = 256
        ev = (StepEntry * cap)()
        n = C.c_int()
        rc = lib.lc_store_insert(self.h, prompt, entry.h, _ptr(st_), st_.size, now, ev, cap, C.byref(n))
        out = [StepEntry.from_buffer_copy(ev[i]) for i in range(min(n.value, cap))]
        self._notify(out)
        _check(rc)
        return out

    def get_step(self, prompt: int, desired: int, now: int, out=None, want_latent=True):
        """Largest cached step <= desired. Returns (latent [F][E] device tensor
        or None, actual step) or None on a miss."""
        act = C.c_int32()
        if want_latent and out is None:
            e = C.c_void_p()
            _check(lib.lc_store_entry(self.h, prompt, C.byref(e)))
            if e.value:
                i = EntryInfo()
                _check(lib.lc_entry_get_info(e, C.byref(i)))
                out = _torch_out((i.F, i.H * i.W * i.C), self.ctx)
        _check(lib.lc_store_get_step(self.h, prompt, desired, now, C.byref(act), _ptr(out) if want_latent else None))
        if act.value == 0:
            return None
        return out, act.value

    def peek(self, now: int):
        """(StepEntry, policy key) that evict_one(now) would remove, without
        removing it (per-shard candidate of a global eviction)."""
        e, k = StepEntry(), C.c_double()
        _check(lib.lc_store_peek(self.h, now, C.byref(e), C.byref(k)))
        return e, k.value

    def next_seq(self) -> int:
        return int(lib.lc_store_next_seq(self.h))

    def set_next_seq(self, seq: int):
        _check(lib.lc_store_set_next_seq(self.h, seq))

    def evict_one(self, now: int) -> StepEntry:
        e = StepEntry()
        _check(lib.lc_store_evict_one(self.h, now, C.byref(e)))
        self._notify([e])
        return e

    def evict_step(self, prompt: int, step: int) -> bool:
        r = C.c_int32()
        _check(lib.lc_store_evict_step(self.h, prompt, step, C.byref(r)))
        if r.value and self._cb and not self.contains(prompt):
            self._cb(prompt)
        return bool(r.value)

    def cached_steps(self, prompt: int):
        buf = (C.c_int32 * 8)()
        n = C.c_int()
        _check(lib.lc_store_cached_steps(self.h, prompt, buf, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def entry_data(self, prompt: int):
        e = C.c_void_p()
        _check(lib.lc_store_entry(self.h, prompt, C.byref(e)))
        return CompressedEntry(e, self.ctx, owned=False) if e.value else None

    def contains(self, prompt: int) -> bool:
        r = C.c_int32()
        _check(lib.lc_store_contains(self.h, prompt, C.byref(r)))
        return bool(r.value)

    def used(self) -> int:
        return lib.lc_store_used(self.h)

    def recompute_used(self) -> int:
        return lib.lc_store_recompute_used(self.h)

    def capacity_limit(self) -> int:
        return lib.lc_store_capacity(self.h)

    def policy(self) -> Policy:
        return Policy(lib.lc_store_policy(self.h))

    def prompt_count(self) -> int:
        return lib.lc_store_prompt_count(self.h)

    def step_count(self) -> int:
        return lib.lc_store_step_count(self.h)

    def entries_snapshot(self):
        n = C.c_int64()
        _check(lib.lc_store_entries(self.h, None, 0, C.byref(n)))
        buf = (StepEntry * max(n.value, 1))()
        _check(lib.lc_store_entries(self.h, buf, n.value, C.byref(n)))
        return [StepEntry.from_buffer_copy(buf[i]) for i in range(n.value)]


def save_snapshot(store: "CacheStore", index: "SimilarityIndex", path) -> None:
    """save_snapshot (store.cpp:232-273): byte-identical FLXC v1 file."""
    _check(lib.lc_snapshot_save(store.h, index.h, os.fspath(path).encode()))


def load_snapshot(path, ctx: Context | None = None):
    """load_snapshot (store.cpp:275-364) -> (CacheStore, SimilarityIndex) in HBM.
    The eviction callback is not part of the snapshot (store.hpp:123-124)."""
    ctx = ctx or default_context()
    hs, hi = C.c_void_p(), C.c_void_p()
    _check(lib.lc_snapshot_load(ctx.h, os.fspath(path).encode(), C.byref(hs), C.byref(hi)))
    st = CacheStore.__new__(CacheStore)
    st.ctx, st.h, st._cb = ctx, hs, None
    ix = SimilarityIndex.__new__(SimilarityIndex)
    ix.ctx, ix.h = ctx, hi
    return st, ix


# ---------------------------------------------------------------------------
# Engine: request pipeline + latency / cost models
# ---------------------------------------------------------------------------
KIND_NAMES = {0: "miss", 1: "whole", 2: "decoupled"}


def engine_config(**kw) -> "_capi.EngineConfig":
    """defaults.hpp values, overridden by keyword (bin_edges as a 4-sequence)."""
    c = _capi.EngineConfig()
    lib.lc_engine_config_default(C.byref(c))
    for k, v in kw.items():
        if k == "bin_edges":
            for i, x in enumerate(v):
                c.bin_edges[i] = float(x)
        elif k == "policy":
            c.policy = int(v)
        else:
            setattr(c, k, v)
    return c


class Engine:
    """process_request / update_after_generation / report over an HBM-resident
    index + store. Requests of one process() call are
    served in order with one shared exact lookup (see engine.cu)."""

    def __init__(self, config=None, ctx: Context | None = None, **kw):
        self.ctx = ctx or default_context()
        self.config = config if config is not None else engine_config(**kw)
        h = C.c_void_p()
        _check(lib.lc_engine_create(self.ctx.h, C.byref(self.config), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h and _alive(self.ctx):
                lib.lc_engine_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def index(self) -> "SimilarityIndex":
        ix = SimilarityIndex.__new__(SimilarityIndex)
        ix.ctx, ix.h, ix._borrowed = self.ctx, C.c_void_p(lib.lc_engine_index(self.h)), self
        return ix

    @property
    def store(self) -> "CacheStore":
        st = CacheStore.__new__(CacheStore)
        st.ctx, st.h, st._cb, st._borrowed = self.ctx, C.c_void_p(lib.lc_engine_store(self.h)), None, self
        return st

    def process(self, prompts, arrivals, q_whole, q_object, q_background, latents, obj_masks, bg_masks,
                served=None):
        """prompts/arrivals [n]; q_* [n][dim]; latents [n][5][F][E] (steps 5..25);
        masks [n][F][mb]; served: optional device tensor [n][F][E] for the
        served / stitched latents. Returns a list of outcome dicts."""
        n = len(prompts)
        req = (_capi.Request * max(n, 1))()
        for i in range(n):
            req[i].prompt = int(prompts[i])
            req[i].arrival = int(arrivals[i])
        outs = (_capi.Outcome * max(n, 1))()
        qw, qo, qb = (_host(x, np.float32) for x in (q_whole, q_object, q_background))
        lat = _host(latents, np.float32)
        om, bm = _host(obj_masks, np.uint8), _host(bg_masks, np.uint8)
        _check(lib.lc_engine_process(self.h, req, n, _ptr(qw), _ptr(qo), _ptr(qb), _ptr(lat), _ptr(om), _ptr(bm),
                                     None if served is None else _ptr(served), outs))
        res = []
        for i in range(n):
            o = outs[i]
            d = o.decision
            res.append({"prompt": int(prompts[i]), "kind": KIND_NAMES[d.kind], "desired_step": d.step,
                        "whole_id": d.whole_id, "object_id": d.object_id, "background_id": d.background_id,
                        "score": d.score, "scores": (d.whole_score, d.object_score, d.background_score),
                        "actual_step": o.actual_step, "n_inserted": o.n_inserted, "n_evicted": o.n_evicted,
                        "latency": o.latency})
        return res

    def metrics(self) -> dict:
        m = _capi.EngineMetrics()
        _check(lib.lc_engine_metrics_get(self.h, C.byref(m)))
        return {"requests": m.requests, "whole_hits": m.whole_hits, "decoupled_hits": m.decoupled_hits,
                "misses": m.misses, "skipped_hist": {5 * i: int(m.skipped_hist[i]) for i in range(6)},
                "skipped_total": m.skipped_total, "simulated_time": m.simulated_time,
                "computation_savings": m.computation_savings, "mean_latency": m.mean_latency,
                "throughput_vs_nocache": m.throughput_vs_nocache}

    def report(self, gpu_rate=3.67, storage_rate=0.0, provisioned_storage=0.0) -> dict:
        p = _capi.Pricing(gpu_rate, storage_rate, provisioned_storage)
        r = _capi.CostReport()
        _check(lib.lc_engine_report(self.h, C.byref(p), C.byref(r)))
        return {"gpu_cost_per_video": r.gpu_cost_per_video, "storage_cost_per_video": r.storage_cost_per_video,
                "videos_per_month": r.videos_per_month, "throughput_vs_nocache": r.throughput_vs_nocache,
                "mean_latency": r.mean_latency}

    def save_snapshot(self, path):
        _check(lib.lc_snapshot_save(lib.lc_engine_store(self.h), lib.lc_engine_index(self.h),
                                    os.fspath(path).encode()))


# ---------------------------------------------------------------------------
# simgen: on-device synthetic embeddings / latents
# ---------------------------------------------------------------------------
def synth_embeddings(token_sets, dim, seed, ctx=None, out=None):
    """synth_embedding for a list of token-id sets (1..16 ids each) -> unit
    fp32 [n][dim] (device tensor unless `out` is given)."""
    ctx = ctx or default_context()
    n = len(token_sets)
    mt = max(len(t) for t in token_sets)
    tok = np.zeros((n, mt), np.uint64)
    nt = np.zeros(n, np.int32)
    for i, t in enumerate(token_sets):
        tok[i, :len(t)] = t
        nt[i] = len(t)
    if out is None:
        out = _torch_out((n, dim), ctx)
    _check(lib.lc_synth_embeddings(ctx.h, _ptr(tok), _ptr(nt), mt, n, dim, seed, _ptr(out)))
    return out


def latent_spec(**kw) -> "_capi.LatentSpec":
    s = _capi.LatentSpec()
    lib.lc_latent_spec_default(C.byref(s))
    for k, v in kw.items():
        if k in ("redundancy", "alpha"):
            arr = getattr(s, k)
            for i, x in enumerate(v):
                arr[i] = float(x)
        else:
            setattr(s, k, float(v))
    return s


def synth_latents(prompt_seeds, F, dims, spec=None, ctx=None):
    """synth_latents for n prompt seeds -> (latents [n][5][F][E], obj masks,
    bg masks [n][F][mb]) as device tensors."""
    import torch
    ctx = ctx or default_context()
    ps = np.ascontiguousarray(prompt_seeds, np.uint64)
    n = ps.size
    H, W, Cc = dims
    E, mb = H * W * Cc, (H * W + 7) // 8
    dev = torch.device("cuda", ctx.device)
    lat = torch.empty((n, 5, F, E), dtype=torch.float32, device=dev)
    om = torch.empty((n, F, mb), dtype=torch.uint8, device=dev)
    bm = torch.empty((n, F, mb), dtype=torch.uint8, device=dev)
    sp = spec if spec is not None else latent_spec()
    _check(lib.lc_synth_latents(ctx.h, _ptr(ps), n, F, H, W, Cc, C.byref(sp), _ptr(lat), _ptr(om), _ptr(bm)))
    return lat, om, bm
