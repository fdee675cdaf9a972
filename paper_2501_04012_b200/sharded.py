"""Entry-sharded lookup over one process per GPU (north_star (4)).

The reference has no distribution at all (single process); this
module adds the one exchange the sharded cache needs. Prompt p lives on rank
``p mod G`` (all three tables, its compressed entry and its store records), so
inserts, removes, codec and eviction bookkeeping are rank-local with no
collective. A lookup batch runs the exact local top-k on every rank
(tcgen05 shortlist + fp64 rescore, ``lc_index_query_topk``), then ONE
all-gather of the per-shard candidates — packed as a single int64 tensor
[tables][n][2k+1] = (ids, fp64 score bits, count) — and every rank merges the
G lists by (score desc, id asc) with ``lc_topk_merge``. Because that order is
a total order independent of the partition, the merged result is the
reference's global top-k (vindex.cpp:58-72) bit for bit; decide and
similarity_to_step then run on the merged top-1 triple.

``local_topk`` / ``merge`` / ``decide`` are injectable so the host-side logic
(partition, packing, gather layout, merge order) is covered by world-size-2
gloo tests on CPU, with the CPU oracle standing in for the GPU kernels there.
"""
from __future__ import annotations

import numpy as np

__all__ = ["owner_of", "ShardedIndex", "ShardedStore", "pack_candidates", "unpack_candidates", "attach_comm",
           "comm_info", "CommShardedIndex", "CommShardedStore"]


def owner_of(prompt_ids, world: int):
    """Rank owning each prompt id: id mod G."""
    return np.asarray(prompt_ids, dtype=np.uint64) % np.uint64(world)


def pack_candidates(torch, ids, scores, counts):
    """(ids i64 [T][n][k], scores f64 [T][n][k], counts i32 [T][n]) -> one i64
    tensor [T][n][2k+1] so the exchange is a single collective."""
    T, n, k = ids.shape
    out = torch.empty((T, n, 2 * k + 1), dtype=torch.int64, device=ids.device)
    out[:, :, :k] = ids
    out[:, :, k:2 * k] = scores.contiguous().view(torch.int64)
    out[:, :, 2 * k] = counts.to(torch.int64)
    return out


def unpack_candidates(torch, g, k):
    """[G][T][n][2k+1] -> per table (ids [G][n][k], scores [G][n][k], counts [G][n])."""
    G, T, n, _ = g.shape
    res = []
    for t in range(T):
        ids = g[:, t, :, :k].contiguous()
        sc = g[:, t, :, k:2 * k].contiguous().view(torch.float64)
        cnt = g[:, t, :, 2 * k].to(torch.int32).contiguous()
        res.append((ids, sc, cnt))
    return res


class ShardedIndex:
    """A rank's shard of the three-table SimilarityIndex plus the collective merge.

    index      this rank's ``SimilarityIndex`` (device) — or None when
               ``local_topk`` is supplied (CPU tests)
    group      torch.distributed process group (None = default group)
    """

    def __init__(self, index=None, group=None, local_topk=None, merge=None, decide=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.index = index
        self._local_topk = local_topk
        self._merge = merge
        self._decide = decide
        self._nccl = dist.get_backend(group) == "nccl"

    # ---- partition -------------------------------------------------------
    def mine(self, prompt_ids):
        return owner_of(prompt_ids, self.world) == np.uint64(self.rank)

    def insert_batch(self, prompt_ids, whole, obj, background):
        """Insert the rows this rank owns (id mod G == rank); returns how many."""
        m = self.mine(prompt_ids)
        if self._local_topk is not None:
            raise RuntimeError("insert_batch needs a device index")
        sel = np.nonzero(m)[0]
        if len(sel) == 0:
            return 0
        self.index.insert_batch(np.asarray(prompt_ids, dtype=np.uint64)[sel], whole[sel], obj[sel], background[sel])
        return len(sel)

    # ---- lookup ----------------------------------------------------------
    def _topk_local(self, kind, q, k):
        if self._local_topk is not None:
            return self._local_topk(kind, q, k)
        return self.index.query_topk(kind, q, k)

    def _gather(self, packed):
        torch, dist = self.torch, self.dist
        G = self.world
        if self._nccl:
            g = torch.empty((G,) + tuple(packed.shape), dtype=packed.dtype, device=packed.device)
            dist.all_gather_into_tensor(g, packed.contiguous(), group=self.group)
            return g
        # gloo (CPU tests, or a one-GPU smoke run of several ranks): host tensors
        src = packed.contiguous().cpu()
        parts = [torch.empty_like(src) for _ in range(G)]
        dist.all_gather(parts, src, group=self.group)
        return torch.stack(parts).to(packed.device)

    def _merge_lists(self, ids, sc, cnt, k):
        if self._merge is not None:
            return self._merge(ids, sc, cnt, k)
        from . import topk_merge
        return topk_merge(ids, sc, cnt, k, ctx=self.index.ctx)

    def query_topk(self, kind, q, k):
        """Global exact top-k of a query batch over all shards: (ids, scores, counts)."""
        torch = self.torch
        ids, sc, cnt = self._topk_local(kind, q, k)
        ids, sc, cnt = (torch.as_tensor(np.asarray(x) if not torch.is_tensor(x) else x) for x in (ids, sc, cnt))
        packed = pack_candidates(torch, ids.view(torch.int64)[None] if ids.dtype == torch.int64 else
                                 ids.to(torch.int64)[None], sc[None], cnt[None])
        g = self._gather(packed)
        gi, gs, gc = unpack_candidates(torch, g, k)[0]
        return self._merge_lists(gi, gs, gc, k)

    def lookup_decide(self, qw, qo, qb, hit_threshold=0.65, edges=(0.72, 0.79, 0.86, 0.93)):
        """Fused 3-table sharded lookup + decide + similarity_to_step; one
        all-gather for the three tables."""
        torch = self.torch
        loc = [self._topk_local(t, q, 1) for t, q in enumerate((qw, qo, qb))]
        ids = torch.stack([torch.as_tensor(x[0]).to(torch.int64) for x in loc])
        sc = torch.stack([torch.as_tensor(x[1]) for x in loc])
        cnt = torch.stack([torch.as_tensor(x[2]) for x in loc])
        g = self._gather(pack_candidates(torch, ids, sc, cnt))
        top = [self._merge_lists(gi, gs, gc, 1) for gi, gs, gc in unpack_candidates(torch, g, 1)]
        if self._decide is not None:
            return self._decide(top, hit_threshold, edges)
        from . import decide_batch
        (wi, ws, _), (oi, os_, _), (bi, bs, _) = top
        return decide_batch(wi[:, 0], ws[:, 0], oi[:, 0], os_[:, 0], bi[:, 0], bs[:, 0], hit_threshold, edges,
                            ctx=self.index.ctx)


# ---------------------------------------------------------------------------
# Entry-sharded CacheStore under ONE global capacity budget
# ---------------------------------------------------------------------------
CACHEABLE = (5, 10, 15, 20, 25)


class ShardedStore:
    """CacheStore (store.hpp:48-120) whose (prompt, step) records live on the
    owner rank (id mod G) while capacity, eviction order and the insertion
    counter are global. SPMD: every rank calls every operation in the same
    order (the engine's request order); the owner passes the entry.

    Exactness: a step's policy key depends only on its own prompt's records
    (store.cpp:113-136), which all live on the owner, so the global victim of
    evict_one is the minimum over the ranks' local victims by (key, seq) —
    one small all-gather of each rank's candidate (lc_store_peek) per
    eviction. next_seq_ (store.hpp:113) is replayed identically on every rank.
    The sequence of victims, used() and every StepEntry equal the unsharded
    store's.

    local      this rank's store with unbounded capacity: the product
               ``CacheStore`` or (CPU tests) an adapter over the oracle store,
               exposing insert_steps / get_step / evict_one / peek / used /
               step_count / contains / set_next_seq
    entry_info callable(entry) -> (shared_bytes, {step: private_bytes}) (owner only)
    """

    FIELDS = 10  # present, key bits, seq, prompt, step, f, last, inserted_at, capacity, local used()

    def __init__(self, capacity, local, entry_info, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.capacity = int(capacity)
        self.local = local
        self.entry_info = entry_info
        self.seq = 0
        self._nccl = dist.get_backend(group) == "nccl"
        self.device = device if device is not None else ("cuda" if self._nccl else "cpu")

    def owner(self, prompt) -> int:
        return int(prompt) % self.world

    # ---- collectives -----------------------------------------------------
    @staticmethod
    def _pack(row):
        """u64 fields (prompt ids, seq, f, ...) travel as their int64 bit
        images: values >= 2^63 wrap instead of raising on one rank (which would
        leave the other ranks blocked in the collective)."""
        return np.array([int(v) & 0xFFFFFFFFFFFFFFFF for v in row], dtype=np.uint64).view(np.int64)

    def _all_gather(self, row):
        torch, dist = self.torch, self.dist
        t = torch.as_tensor(self._pack(row), device=self.device)
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t, group=self.group)
        return torch.stack(parts).cpu().numpy()

    def _bcast(self, row, src):
        torch, dist = self.torch, self.dist
        t = torch.as_tensor(self._pack(row), device=self.device).clone()
        dist.broadcast(t, src=dist.get_global_rank(self.group, src) if self.group is not None else src,
                       group=self.group)
        return t.cpu().numpy()

    def used(self) -> int:
        return int(self._all_gather([self.local.used()])[:, 0].sum())

    def step_count(self) -> int:
        return int(self._all_gather([self.local.step_count()])[:, 0].sum())

    # ---- global eviction -------------------------------------------------
    def _candidates(self, now):
        """One all-gather: every rank's local victim (lc_store_peek) and used()."""
        if self.local.step_count() == 0:
            row = [0] * (self.FIELDS - 1)
        else:
            e, key = self.local.peek(now)  # e = (prompt, step, f, last, inserted_at, seq, capacity)
            e = e.as_tuple() if hasattr(e, "as_tuple") else tuple(e)
            kb = int(np.float64(key).view(np.int64))
            row = [1, kb, e[5], e[0], e[1], e[2], e[3], e[4], e[6]]
        return self._all_gather(row + [self.local.used()])

    def evict_one(self, now, g=None):
        """The global (key, seq) minimum; identical StepEntry tuple on every rank."""
        if g is None:
            g = self._candidates(now)
        live = [r for r in range(self.world) if g[r, 0]]
        if not live:
            raise LookupError("evict_one: store is empty")  # std::logic_error (store.cpp:148)
        win = min(live, key=lambda r: (float(np.int64(g[r, 1]).view(np.float64)), int(np.uint64(g[r, 2]))))
        row = g[win]
        ent = (int(np.uint64(row[3])), int(row[4]), int(np.uint64(row[5])), int(np.uint64(row[6])),
               int(np.uint64(row[7])), int(np.uint64(row[2])), int(np.uint64(row[8])))
        if win == self.rank:
            got = self.local.evict_one(now)
            got = got.as_tuple() if hasattr(got, "as_tuple") else tuple(got)
            assert tuple(int(x) for x in got) == ent, (got, ent)
        return ent

    def insert_steps(self, prompt, entry, steps, now):
        """insert_steps (store.cpp:53-91) with the validation, OversizedEntry
        and eviction loop decided globally; returns the evicted StepEntry
        tuples (same list on every rank)."""
        own = self.owner(prompt)
        steps = [int(s) for s in steps]
        status, standalone = 0, 0
        if self.rank == own:
            try:
                if not steps:
                    raise ValueError("insert_steps: empty step list")
                shared, priv = self.entry_info(entry)
                for s in steps:
                    if s not in CACHEABLE:
                        raise ValueError("insert_steps: step not cacheable")
                    if s not in priv:
                        raise ValueError("insert_steps: step missing from entry")
                if self.local.contains(prompt):
                    raise ValueError("insert_steps: prompt already cached")
                standalone = shared + sum(priv[s] for s in set(steps))
                status = 2 if standalone > self.capacity else 0
            except ValueError:
                status = 1
        st, standalone = (int(x) for x in self._bcast([status, standalone], own))
        if st == 1:
            raise ValueError("insert_steps: rejected by the owner shard")
        if st == 2:
            raise OverflowError(f"entry of {standalone} bytes exceeds capacity limit of {self.capacity} bytes")
        evicted = []
        while True:
            g = self._candidates(now)
            if int(g[:, self.FIELDS - 1].sum()) + standalone <= self.capacity:
                break
            evicted.append(self.evict_one(now, g))
        if self.rank == own:
            self.local.set_next_seq(self.seq)
            self.local.insert_steps(prompt, entry, steps, now)
        self.seq += len(set(steps))
        return evicted

    def get_step(self, prompt, desired, now, **kw):
        """get_step on the owner (f / last_access bump, decompress there);
        returns (actual step, owner-local result or None) on every rank."""
        own = self.owner(prompt)
        res = None
        actual = 0
        if self.rank == own:
            res = self.local.get_step(prompt, desired, now, **kw)
            actual = int(res[1]) if res else 0
        actual = int(self._bcast([actual], own)[0])
        return actual, res


# ---------------------------------------------------------------------------
# C-ABI sharding (shard.cu): the communicator lives in the library context,
# so C++ callers (include/lcache_b200/lcache.hpp) shard without Python. These
# classes are thin handles over lc_sharded_*; torch.distributed only
# bootstraps the communicator.
# ---------------------------------------------------------------------------
def attach_comm(ctx, group=None, transport: str | None = None):
    """Give `ctx` the communicator of a torch.distributed group.

    transport "nccl": an NCCL communicator created inside the library
    (ncclCommInitRank; the unique id is broadcast from rank 0 over the group).
    transport "host": every collective goes through `group`'s all_gather on
    host tensors (gloo) via lc_ctx_comm_host — used where NCCL cannot run,
    e.g. several ranks sharing one GPU in the tests.
    Default: "nccl" when the group's backend is NCCL, else "host"."""
    import ctypes as C
    import torch
    import torch.distributed as dist
    from ._capi import ALLGATHER_FN, lib
    from . import _check
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if transport is None:
        transport = "nccl" if dist.get_backend(group) == "nccl" else "host"
    if transport == "nccl":
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _check(lib.lc_comm_unique_id(uid))
        obj = [bytes(uid)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        _check(lib.lc_ctx_comm_init(ctx.h, world, rank, uid))
        return ctx

    def _gather(user, send, recv, nbytes):
        try:
            t = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8)
            parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, t, group=group)
            for r, p in enumerate(parts):
                C.memmove(recv + r * nbytes, p.data_ptr(), nbytes)
            return 0
        except Exception:  # noqa: BLE001 — reported as LC_ERR_NCCL by the library
            return 1

    cb = ALLGATHER_FN(_gather)
    ctx._comm_cb = cb  # the library holds the raw pointer: keep the thunk alive
    _check(lib.lc_ctx_comm_host(ctx.h, world, rank, cb, None))
    return ctx


def comm_info(ctx):
    """(nranks, rank, backend 0 none / 1 nccl / 2 host, collectives issued)."""
    import ctypes as C
    from ._capi import lib
    from . import _check
    n, r, b, c = C.c_int(), C.c_int(), C.c_int(), C.c_uint64()
    _check(lib.lc_ctx_comm_info(ctx.h, C.byref(n), C.byref(r), C.byref(b), C.byref(c)))
    return n.value, r.value, b.value, c.value


class CommShardedIndex:
    """This rank's shard of the index, queried collectively through
    lc_sharded_query_topk / lc_sharded_lookup_decide (one grouped all-gather
    per batch inside the library)."""

    def __init__(self, index, dim: int):
        self.index, self.dim = index, dim
        self.ctx = index.ctx
        self.world, self.rank = comm_info(self.ctx)[:2]

    def mine(self, prompt_ids):
        return owner_of(prompt_ids, self.world) == np.uint64(self.rank)

    def insert_batch(self, prompt_ids, whole, obj, background):
        sel = np.nonzero(self.mine(prompt_ids))[0]
        if len(sel):
            self.index.insert_batch(np.asarray(prompt_ids, dtype=np.uint64)[sel], whole[sel], obj[sel], background[sel])
        return len(sel)

    def query_topk(self, kind, q, k, out=None):
        from . import _check, _host, _is_dev, _ptr
        from ._capi import lib
        q = _host(q, np.float32)
        n = q.shape[0]
        if out is None:
            if _is_dev(q):
                import torch
                out = (torch.empty((n, k), dtype=torch.int64, device=q.device),
                       torch.empty((n, k), dtype=torch.float64, device=q.device),
                       torch.empty((n,), dtype=torch.int32, device=q.device))
            else:
                out = (np.zeros((n, k), np.uint64), np.zeros((n, k), np.float64), np.zeros(n, np.int32))
        _check(lib.lc_sharded_query_topk(self.index.h, int(kind), _ptr(q), n, self.dim, k, _ptr(out[0]),
                                         _ptr(out[1]), _ptr(out[2])))
        return out

    def lookup_decide(self, qw, qo, qb, hit_threshold=0.65, edges=(0.72, 0.79, 0.86, 0.93)):
        from . import _check, _host, _ptr
        from ._capi import Decision, lib
        qs = [_host(x, np.float32) for x in (qw, qo, qb)]
        n = qs[0].shape[0]
        out = (Decision * n)()
        e = np.asarray(edges, np.float64)
        _check(lib.lc_sharded_lookup_decide(self.index.h, _ptr(qs[0]), _ptr(qs[1]), _ptr(qs[2]), n, self.dim,
                                            hit_threshold, _ptr(e), out))
        return list(out)


class CommShardedStore:
    """CacheStore under one global budget across ranks (lc_sharded_store_*):
    the same StepEntry sequence, used() and next_seq as one unsharded store.
    Every method is collective; insert_steps takes the entry on the owner
    rank (prompt mod G) and None elsewhere."""

    def __init__(self, capacity: int, policy, ctx, batch: int = 0):
        import ctypes as C
        from . import CacheStore, _check
        from ._capi import lib
        self.ctx = ctx
        h = C.c_void_p()
        _check(lib.lc_sharded_store_create(ctx.h, capacity, int(policy), batch, C.byref(h)))
        self.h = h
        self.world, self.rank = comm_info(ctx)[:2]
        loc = CacheStore.__new__(CacheStore)
        loc.ctx, loc.h, loc._cb, loc._borrowed = ctx, C.c_void_p(lib.lc_sharded_store_local(h)), None, True
        self.local = loc

    def __del__(self):
        try:
            from ._capi import lib
            from . import _alive
            if self.h and _alive(self.ctx):
                lib.lc_sharded_store_destroy(self.h)
                self.h = None
        except Exception:  # noqa: BLE001
            pass

    def owner(self, prompt) -> int:
        return int(prompt) % self.world

    def insert_steps(self, prompt, entry, steps, now):
        import ctypes as C
        from . import _check, _ptr
        from ._capi import StepEntry, lib
        st_ = np.ascontiguousarray(steps, np.int32)
        cap = 4096
        ev = (StepEntry * cap)()
        n = C.c_int()
        _check(lib.lc_sharded_store_insert(self.h, int(prompt), entry.h if entry is not None else None, _ptr(st_),
                                           st_.size, now, ev, cap, C.byref(n)))
        return [tuple(int(v) for v in ev[i].as_tuple()) for i in range(min(n.value, cap))]

    def evict_one(self, now):
        from . import _check
        from ._capi import StepEntry, lib
        import ctypes as C
        e = StepEntry()
        _check(lib.lc_sharded_store_evict_one(self.h, now, C.byref(e)))
        return tuple(int(v) for v in e.as_tuple())

    def get_step(self, prompt, desired, now, out=None):
        import ctypes as C
        from . import _check, _ptr
        from ._capi import lib
        a = C.c_int32()
        _check(lib.lc_sharded_store_get_step(self.h, int(prompt), desired, now, C.byref(a),
                                             _ptr(out) if out is not None else None))
        return a.value

    def used(self) -> int:
        import ctypes as C
        from . import _check
        from ._capi import lib
        u = C.c_uint64()
        _check(lib.lc_sharded_store_used(self.h, C.byref(u)))
        return u.value

    def stats(self):
        import ctypes as C
        from . import _check
        from ._capi import lib
        r, e, s = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib.lc_sharded_store_stats(self.h, C.byref(r), C.byref(e), C.byref(s)))
        return {"rounds": r.value, "local_evictions": e.value, "next_seq": s.value}
