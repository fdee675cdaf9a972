"""ctypes loader for the CPU checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module. The product package
(paper_2501_04012_b200) never does.

Two libraries with identical flat signatures (oracle/oracle_abi.h):
  Checker("orc")  the plain-C restatement  oracle/_build/liblc_oracle.so
  Checker("ref")  the unmodified reference oracle/_ref/liblcache_ref.so
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "orc": os.path.join(HERE, "_build", "liblc_oracle.so"),
    "ref": os.path.join(HERE, "_ref", "liblcache_ref.so"),
}

OK = 0
ERR_NAMES = {1: "invalid_argument", 2: "DegenerateBase", 3: "StepNotCached",
             4: "OversizedEntry", 5: "SnapshotError", 6: "logic_error", 10: "internal"}


class StepEntryC(C.Structure):
    _fields_ = [("prompt", C.c_uint64), ("step", C.c_int32), ("_pad", C.c_int32),
                ("f", C.c_uint64), ("last_access", C.c_uint64), ("inserted_at", C.c_uint64),
                ("inserted_seq", C.c_uint64), ("capacity", C.c_uint64)]

    def as_tuple(self):
        return (self.prompt, self.step, self.f, self.last_access, self.inserted_at,
                self.inserted_seq, self.capacity)


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


def build(which="all"):
    subprocess.run(["make", "-s", "-C", HERE, which], check=True)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Checker:
    def __init__(self, kind: str = "orc"):
        path = LIBS[kind]
        if not os.path.exists(path):
            if kind == "orc":
                build("orc")
            else:
                raise FileNotFoundError(path)
        self.kind = kind
        self.lib = C.CDLL(path)
        self.pfx = kind + "_"
        L = self.lib
        fn = lambda n: getattr(L, self.pfx + n)
        fn("last_error").restype = C.c_char_p
        fn("index_new").restype = C.c_void_p
        fn("index_free").argtypes = [C.c_void_p]
        fn("index_insert").argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        fn("index_remove").argtypes = [C.c_void_p, C.c_uint64]
        fn("index_size").argtypes = [C.c_void_p]
        fn("index_size").restype = C.c_int64
        fn("index_query_top1").argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                           C.c_void_p, C.c_void_p, C.c_void_p]
        fn("cosine").argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_double)]
        fn("normalize").argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        fn("select_keyframes").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p]
        fn("solve_alpha").argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_float)]
        fn("compress").argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_void_p, C.c_void_p, C.c_double, C.c_uint64, C.c_void_p, C.c_uint64,
                                   C.POINTER(C.c_uint64)]
        fn("compress_batch").argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_int, C.c_int,
                                         C.c_void_p]
        fn("decompress").argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
        fn("entry_info").argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p]
        fn("stitch").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        fn("lrbu_priority").argtypes = [C.POINTER(StepEntryC), C.c_uint64, C.POINTER(C.c_double)]
        fn("lcbfu_priority").argtypes = [C.POINTER(StepEntryC), C.POINTER(C.c_double)]
        fn("store_new").restype = C.c_void_p
        fn("store_new").argtypes = [C.c_uint64, C.c_int]
        fn("store_free").argtypes = [C.c_void_p]
        fn("store_insert").argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int,
                                       C.c_uint64, C.c_void_p, C.c_int, C.POINTER(C.c_int)]
        fn("store_get_step").argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.POINTER(C.c_int32),
                                         C.c_void_p]
        fn("store_evict_one").argtypes = [C.c_void_p, C.c_uint64, C.POINTER(StepEntryC)]
        if kind == "orc":
            fn("synth_embedding").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
            fn("synth_latents").argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                            C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                                            C.c_void_p]
            fn("store_peek").argtypes = [C.c_void_p, C.c_uint64, C.POINTER(StepEntryC), C.POINTER(C.c_double)]
            fn("store_next_seq").argtypes = [C.c_void_p]
            fn("store_next_seq").restype = C.c_uint64
            fn("store_set_next_seq").argtypes = [C.c_void_p, C.c_uint64]
        fn("store_evict_step").argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_int32)]
        for n in ("store_used", "store_recompute_used"):
            fn(n).argtypes = [C.c_void_p]
            fn(n).restype = C.c_uint64
        for n in ("store_step_count", "store_prompt_count"):
            fn(n).argtypes = [C.c_void_p]
        if kind == "ref":  # snapshots exist only in the reference (store.cpp:219-364)
            fn("snapshot_save").argtypes = [C.c_void_p, C.c_void_p, C.c_char_p]
            fn("snapshot_load").argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
            for n in ("snapshot_store", "snapshot_index"):
                fn(n).argtypes = [C.c_void_p]
                fn(n).restype = C.c_void_p
            fn("snapshot_free").argtypes = [C.c_void_p]
            fn("last_snapshot_offset").restype = C.c_uint64
            fn("compress_batch_hash").argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                  C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_int,
                                                  C.c_int, C.c_void_p, C.c_void_p]
            fn(n).restype = C.c_int64
        fn("store_entries").argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_int)]
        if kind == "orc":
            L.orc_topk_flat.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int,
                                        C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
            L.orc_decide.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_int32),
                                     C.POINTER(C.c_double)]
            L.orc_similarity_to_step.argtypes = [C.c_double, C.c_double, C.c_void_p, C.POINTER(C.c_int32)]

    def _f(self, n):
        return getattr(self.lib, self.pfx + n)

    def _chk(self, rc):
        if rc != OK:
            raise CheckerError(rc, self._f("last_error")().decode())

    # ---- core -------------------------------------------------------------
    def normalize(self, v):
        v = np.ascontiguousarray(v, np.float32)
        out = np.empty_like(v)
        self._chk(self._f("normalize")(_p(v), v.size, _p(out)))
        return out

    def normalize_rows(self, m):
        m = np.ascontiguousarray(m, np.float32)
        out = np.empty_like(m)
        for i in range(m.shape[0]):
            self._chk(self._f("normalize")(_p(m[i]), m.shape[1], _p(out[i])))
        return out

    def cosine(self, a, b):
        a = np.ascontiguousarray(a, np.float32).ravel()
        b = np.ascontiguousarray(b, np.float32).ravel()
        out = C.c_double()
        self._chk(self._f("cosine")(_p(a), _p(b), a.size, C.byref(out)))
        return out.value

    # ---- index ------------------------------------------------------------
    def index(self, dim):
        return _Index(self, dim)

    def topk_flat(self, table, ids, q, k):
        assert self.kind == "orc"
        table = np.ascontiguousarray(table, np.float32)
        ids = np.ascontiguousarray(ids, np.uint64)
        q = np.ascontiguousarray(q, np.float32)
        n = q.shape[0]
        oi = np.zeros((n, k), np.uint64)
        os_ = np.zeros((n, k), np.float64)
        oc = np.zeros(n, np.int32)
        self._chk(self.lib.orc_topk_flat(_p(table), _p(ids), table.shape[0], table.shape[1], _p(q), n, k,
                                         _p(oi), _p(os_), _p(oc)))
        return oi, os_, oc

    def decide(self, w, o, b, thr=0.65):
        kind = C.c_int32()
        score = C.c_double()
        self._chk(self.lib.orc_decide(w, o, b, thr, C.byref(kind), C.byref(score)))
        return kind.value, score.value

    def similarity_to_step(self, score, thr=0.65, edges=(0.72, 0.79, 0.86, 0.93)):
        e = np.array(edges, np.float64)
        st = C.c_int32()
        self._chk(self.lib.orc_similarity_to_step(score, thr, _p(e), C.byref(st)))
        return st.value

    # ---- simgen (restatement of csrc/simgen.cu) -----------------------------
    def synth_embedding(self, tokens, dim, seed):
        t = np.ascontiguousarray(tokens, np.uint64)
        out = np.zeros(dim, np.float32)
        self._chk(self._f("synth_embedding")(_p(t), t.size, dim, seed, _p(out)))
        return out

    def synth_latents(self, seed, F, dims, redundancy=(0.9, 0.8, 0.6, 0.4, 0.25),
                      alpha=(1.0, 0.9, 0.8, 0.7, 0.6), noise=0.01, dup=0.02):
        H, W, Cc = dims
        E, mb = H * W * Cc, (H * W + 7) // 8
        lat = np.zeros((5, F, E), np.float32)
        om = np.zeros((F, mb), np.uint8)
        bm = np.zeros((F, mb), np.uint8)
        r = np.ascontiguousarray(redundancy, np.float64)
        a = np.ascontiguousarray(alpha, np.float64)
        self._chk(self._f("synth_latents")(seed, F, H, W, Cc, _p(r), _p(a), noise, dup, _p(lat), _p(om), _p(bm)))
        return lat, om, bm

    # ---- codec ------------------------------------------------------------
    def select_keyframes(self, frames, dims, thr=0.99):
        frames = np.ascontiguousarray(frames, np.float32)
        F = frames.shape[0]
        H, W, Cc = dims
        out = np.zeros(F, np.int32)
        self._chk(self._f("select_keyframes")(_p(frames), F, H, W, Cc, thr, _p(out)))
        return out

    def solve_alpha(self, ds, db):
        ds = np.ascontiguousarray(ds, np.float32).ravel()
        db = np.ascontiguousarray(db, np.float32).ravel()
        out = C.c_float()
        self._chk(self._f("solve_alpha")(_p(ds), _p(db), ds.size, C.byref(out)))
        return np.float32(out.value)

    def compress(self, lat, steps, obj_masks, bg_masks, dims, prompt, thr=0.99):
        """lat [S][F][E] fp32; masks [F][mb] u8 -> wire bytes (serialize_entry)."""
        lat = np.ascontiguousarray(lat, np.float32)
        steps = np.ascontiguousarray(steps, np.int32)
        om = np.ascontiguousarray(obj_masks, np.uint8)
        bm = np.ascontiguousarray(bg_masks, np.uint8)
        S, F = lat.shape[0], lat.shape[1]
        H, W, Cc = dims
        n = C.c_uint64()
        self._chk(self._f("compress")(_p(lat), _p(steps), S, F, H, W, Cc, _p(om), _p(bm), thr, prompt,
                                      None, 0, C.byref(n)))
        out = np.zeros(n.value, np.uint8)
        self._chk(self._f("compress")(_p(lat), _p(steps), S, F, H, W, Cc, _p(om), _p(bm), thr, prompt,
                                      _p(out), out.size, C.byref(n)))
        return out.tobytes()

    def compress_batch_sizes(self, lat, steps, obj_masks, bg_masks, dims, prompts, nthreads=1, thr=0.99):
        lat = np.ascontiguousarray(lat, np.float32)
        steps = np.ascontiguousarray(steps, np.int32)
        om = np.ascontiguousarray(obj_masks, np.uint8)
        bm = np.ascontiguousarray(bg_masks, np.uint8)
        prompts = np.ascontiguousarray(prompts, np.uint64)
        n, S, F = lat.shape[0], lat.shape[1], lat.shape[2]
        H, W, Cc = dims
        out = np.zeros(n, np.uint64)
        self._chk(self._f("compress_batch")(_p(lat), _p(steps), S, F, H, W, Cc, _p(om), _p(bm), thr,
                                            _p(prompts), n, nthreads, _p(out)))
        return out

    def compress_batch_hash(self, lat, steps, obj_masks, bg_masks, dims, prompts, nthreads=1, thr=0.99):
        """(sizes, FNV-1a 64 of each entry's wire bytes) — reference only."""
        lat = np.ascontiguousarray(lat, np.float32)
        steps = np.ascontiguousarray(steps, np.int32)
        om = np.ascontiguousarray(obj_masks, np.uint8)
        bm = np.ascontiguousarray(bg_masks, np.uint8)
        prompts = np.ascontiguousarray(prompts, np.uint64)
        n, S, F = lat.shape[0], lat.shape[1], lat.shape[2]
        H, W, Cc = dims
        sizes = np.zeros(n, np.uint64)
        hashes = np.zeros(n, np.uint64)
        self._chk(self._f("compress_batch_hash")(_p(lat), _p(steps), S, F, H, W, Cc, _p(om), _p(bm), thr,
                                                 _p(prompts), n, nthreads, _p(sizes), _p(hashes)))
        return sizes, hashes

    def decompress(self, entry: bytes, step, F, E):
        buf = np.frombuffer(entry, np.uint8)
        out = np.zeros((F, E), np.float32)
        self._chk(self._f("decompress")(_p(buf), buf.size, step, _p(out)))
        return out

    def entry_info(self, entry: bytes):
        buf = np.frombuffer(entry, np.uint8)
        bs, ns = C.c_int32(), C.c_int32()
        steps = np.zeros(256, np.int32)
        sh = C.c_uint64()
        pr = np.zeros(256, np.uint64)
        self._chk(self._f("entry_info")(_p(buf), buf.size, C.byref(bs), C.byref(ns), _p(steps), C.byref(sh),
                                        _p(pr)))
        n = ns.value
        return {"base_step": bs.value, "steps": steps[:n].tolist(), "shared": sh.value,
                "private": pr[:n].tolist()}

    def stitch(self, obj, oo, ob, bg, bo, bb, dims):
        obj = np.ascontiguousarray(obj, np.float32)
        bg = np.ascontiguousarray(bg, np.float32)
        arrs = [np.ascontiguousarray(a, np.uint8) for a in (oo, ob, bo, bb)]
        F = obj.shape[0]
        H, W, Cc = dims
        out = np.zeros_like(obj)
        self._chk(self._f("stitch")(_p(obj), _p(arrs[0]), _p(arrs[1]), _p(bg), _p(arrs[2]), _p(arrs[3]),
                                    F, H, W, Cc, _p(out)))
        return out

    # ---- store ------------------------------------------------------------
    def lrbu(self, e: StepEntryC, now):
        out = C.c_double()
        self._chk(self._f("lrbu_priority")(C.byref(e), now, C.byref(out)))
        return out.value

    def lcbfu(self, e: StepEntryC):
        out = C.c_double()
        self._chk(self._f("lcbfu_priority")(C.byref(e), C.byref(out)))
        return out.value

    def store(self, capacity, policy):
        return _Store(self, capacity, policy)

    # ---- snapshots (reference only) -----------------------------------------
    def snapshot_save(self, store, index, path):
        self._chk(self._f("snapshot_save")(store.h, index.h, str(path).encode()))

    def snapshot_load(self, path):
        """-> (store, index); both keep the loaded SnapshotData alive."""
        h = C.c_void_p()
        self._chk(self._f("snapshot_load")(str(path).encode(), C.byref(h)))
        owner = _SnapOwner(self, h)
        st = _Store.__new__(_Store)
        st.c, st.h, st._owner = self, self._f("snapshot_store")(h), owner
        ix = _Index.__new__(_Index)
        ix.c, ix.h, ix._owner, ix.dim = self, self._f("snapshot_index")(h), owner, None
        return st, ix

    def last_snapshot_offset(self):
        return self._f("last_snapshot_offset")()


class _SnapOwner:
    def __init__(self, chk, h):
        self.c, self.h = chk, h

    def __del__(self):
        try:
            self.c._f("snapshot_free")(self.h)
        except Exception:
            pass


class _Index:
    _owner = None

    def __init__(self, chk: Checker, dim):
        self.c = chk
        self.h = chk._f("index_new")(dim)
        self.dim = dim

    def __del__(self):
        if self._owner is not None:
            return
        try:
            self.c._f("index_free")(self.h)
        except Exception:
            pass

    def insert(self, pid, w, o, b):
        w, o, b = (np.ascontiguousarray(x, np.float32) for x in (w, o, b))
        self.c._chk(self.c._f("index_insert")(self.h, pid, _p(w), _p(o), _p(b), w.size))

    def remove(self, pid):
        self.c._chk(self.c._f("index_remove")(self.h, pid))

    def size(self):
        return self.c._f("index_size")(self.h)

    def query_top1(self, kind, q, nthreads=1):
        q = np.ascontiguousarray(np.atleast_2d(q), np.float32)
        n = q.shape[0]
        ids = np.zeros(n, np.uint64)
        sc = np.zeros(n, np.float64)
        fd = np.zeros(n, np.int32)
        self.c._chk(self.c._f("index_query_top1")(self.h, kind, _p(q), n, q.shape[1], nthreads, _p(ids),
                                                  _p(sc), _p(fd)))
        return ids, sc, fd


class _Store:
    _owner = None

    def __init__(self, chk: Checker, capacity, policy):
        self.c = chk
        self.h = chk._f("store_new")(capacity, policy)

    def __del__(self):
        if self._owner is not None:
            return
        try:
            self.c._f("store_free")(self.h)
        except Exception:
            pass

    def insert(self, prompt, entry: bytes, steps, now):
        buf = np.frombuffer(entry, np.uint8)
        st = np.ascontiguousarray(steps, np.int32)
        ev = (StepEntryC * 4096)()
        n = C.c_int()
        self.c._chk(self.c._f("store_insert")(self.h, prompt, _p(buf), buf.size, _p(st), st.size, now, ev, 4096,
                                              C.byref(n)))
        return [ev[i].as_tuple() for i in range(min(n.value, 4096))]

    def get_step(self, prompt, desired, now, F=None, E=None):
        act = C.c_int32()
        out = None if F is None else np.zeros((F, E), np.float32)
        self.c._chk(self.c._f("store_get_step")(self.h, prompt, desired, now, C.byref(act),
                                                None if out is None else _p(out)))
        return act.value, out

    def evict_one(self, now):
        e = StepEntryC()
        self.c._chk(self.c._f("store_evict_one")(self.h, now, C.byref(e)))
        return e.as_tuple()

    def peek(self, now):
        """(StepEntry tuple, key) evict_one(now) would take, without evicting."""
        e, k = StepEntryC(), C.c_double()
        self.c._chk(self.c._f("store_peek")(self.h, now, C.byref(e), C.byref(k)))
        return e.as_tuple(), k.value

    def next_seq(self):
        return self.c._f("store_next_seq")(self.h)

    def set_next_seq(self, seq):
        self.c._f("store_set_next_seq")(self.h, seq)

    def evict_step(self, prompt, step):
        r = C.c_int32()
        self.c._chk(self.c._f("store_evict_step")(self.h, prompt, step, C.byref(r)))
        return bool(r.value)

    def used(self):
        return self.c._f("store_used")(self.h)

    def recompute_used(self):
        return self.c._f("store_recompute_used")(self.h)

    def step_count(self):
        return self.c._f("store_step_count")(self.h)

    def prompt_count(self):
        return self.c._f("store_prompt_count")(self.h)

    def entries(self):
        n = C.c_int()
        self.c._chk(self.c._f("store_entries")(self.h, None, 0, C.byref(n)))
        buf = (StepEntryC * max(n.value, 1))()
        self.c._chk(self.c._f("store_entries")(self.h, buf, n.value, C.byref(n)))
        return [buf[i].as_tuple() for i in range(n.value)]
