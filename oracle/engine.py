"""Serial CPU restatement of the engine — TEST INFRASTRUCTURE ONLY.

The reference declares the engine module but ships no code
for it, so this restatement follows the SPEC text line by line over the
plain-C oracle (oracle/lc_oracle.c: exact index, store, codec, decide,
similarity_to_step). It is pinned by the SPEC's worked examples
(tests/test_engine.py)
and by the rules SPEC.md leaves open, which DESIGN.md defines and the
product (csrc/engine.cu) implements:
  * a hit whose source holds no live step <= the desired one serves nothing
    (actual 0) and is handled like a miss for latency and update;
  * a decoupled hit serves the largest step both sources hold <= desired
    ("the min of the two available steps", iterated until
    both hold it);
  * update_after_generation inserts nothing while the prompt is cached.
Only tests/ import this module.
"""
from __future__ import annotations

import numpy as np

CACHED = (5, 10, 15, 20, 25)
KIND = {0: "miss", 1: "whole", 2: "decoupled"}


class OracleEngine:
    def __init__(self, orc, dim, F, H, W, C, capacity, policy=3, hit=0.65, thr=0.99,
                 edges=(0.72, 0.79, 0.86, 0.93), t_step=4.84, t_lookup=0.14, t_extract=3.6, t_stitch=0.0,
                 total=50):
        self.o = orc
        self.ix = orc.index(dim)
        self.st = orc.store(capacity, policy)
        self.dims = (H, W, C)
        self.F, self.E = F, H * W * C
        self.hit, self.thr, self.edges = hit, thr, edges
        self.t = (t_step, t_lookup, t_extract, t_stitch, total)
        self.in_index = set()
        self.entries = {}  # prompt -> stored entry bytes (for served latents)
        self.m = {"requests": 0, "whole_hits": 0, "decoupled_hits": 0, "misses": 0,
                  "skipped_hist": {s: 0 for s in (0, 5, 10, 15, 20, 25)}, "skipped_total": 0,
                  "simulated_time": 0.0}

    def _live(self, prompt):
        return sorted(e[1] for e in self.st.entries() if e[0] == prompt)

    def _masks(self, entry: bytes):
        """object / background mask planes: the wire format's tail (codec.cpp:390-392)."""
        H, W, _ = self.dims
        mb = (H * W + 7) // 8
        tail = np.frombuffer(entry[-2 * self.F * mb:], np.uint8).reshape(2, self.F, mb)
        return tail[0], tail[1]

    @staticmethod
    def _avail(live, desired):
        a = 0
        for s in live:
            if s <= desired:
                a = s
        return a

    def process(self, prompt, arrival, qw, qo, qb, lat5, om, bm):
        """One request + its cache update.
        lat5 [5][F][E] = the prompt's latents at steps 5..25."""
        o = self.o
        now = int(arrival)
        # (1) query the three index tables (vindex.cpp:50-74)
        tops = []
        for kind, q in enumerate((qw, qo, qb)):
            ids, sc, fd = self.ix.query_top1(kind, q)
            tops.append((int(ids[0]), float(sc[0]), bool(fd[0])))
        # (2) decide
        if not tops[0][2]:
            kind, score, desired = 0, 0.0, 0
        else:
            kind, score = o.decide(tops[0][1], tops[1][1], tops[2][1], self.hit)
            desired = o.similarity_to_step(score, self.hit, self.edges) if kind else 0
        # (3) serve
        actual, served = 0, None
        if kind == 1:
            src = tops[0][0]
            actual, served = self.st.get_step(src, desired, now, self.F, self.E)
        elif kind == 2:
            so, sb = tops[1][0], tops[2][0]
            lo, lb = self._live(so), self._live(sb)
            m = min(self._avail(lo, desired), self._avail(lb, desired))
            while m > 0 and (self._avail(lo, m) != m or self._avail(lb, m) != m):
                m = min(self._avail(lo, m), self._avail(lb, m))
            if m > 0:
                a1, x1 = self.st.get_step(so, m, now, self.F, self.E)
                a2, x2 = self.st.get_step(sb, m, now, self.F, self.E)
                assert a1 == a2 == m
                mo, mbk = self._masks(self.entries[so]), self._masks(self.entries[sb])
                served = o.stitch(x1, mo[0], mo[1], x2, mbk[0], mbk[1], self.dims)
                actual = m
        # (4) latency
        t_step, t_lookup, t_extract, t_stitch, total = self.t
        lat = t_extract + t_lookup + t_step * (total - actual) + (t_stitch if kind == 2 and actual > 0 else 0.0)
        # (5) update_after_generation
        n_ins = n_ev = 0
        if actual < 25 and not self._live(prompt):
            steps = [s for s in CACHED if s > actual]
            first = CACHED.index(steps[0])
            ent = o.compress(lat5[first:], steps, om, bm, self.dims, prompt, self.thr)
            ev = self.st.insert(prompt, ent, steps, now)
            n_ins, n_ev = len(steps), len(ev)
            for e in ev:  # eviction callback: the prompt's last step went
                p = e[0]
                if not self._live(p) and p in self.in_index:
                    self.ix.remove(p)
                    self.in_index.discard(p)
                    self.entries.pop(p, None)
            self.entries[prompt] = ent
            if prompt not in self.in_index:
                self.ix.insert(prompt, qw, qo, qb)
                self.in_index.add(prompt)
        m = self.m
        m["requests"] += 1
        m["misses" if kind == 0 else ("whole_hits" if kind == 1 else "decoupled_hits")] += 1
        m["skipped_hist"][actual] += 1
        m["skipped_total"] += actual
        m["simulated_time"] += lat
        return {"prompt": prompt, "kind": KIND[kind], "desired_step": desired, "whole_id": tops[0][0],
                "object_id": tops[1][0], "background_id": tops[2][0], "score": score,
                "scores": (tops[0][1], tops[1][1], tops[2][1]), "actual_step": actual, "n_inserted": n_ins,
                "n_evicted": n_ev, "latency": lat, "served": served}

    def metrics(self):
        m = dict(self.m)
        t_step, total = self.t[0], self.t[4]
        n = m["requests"]
        m["mean_latency"] = m["simulated_time"] / n if n else 0.0
        m["computation_savings"] = m["skipped_total"] / (total * n) if n else 0.0
        m["throughput_vs_nocache"] = total * t_step / m["mean_latency"] if n else 0.0
        return m


def report(metrics, gpu_rate=3.67, storage_rate=0.0, provisioned_storage=0.0):
    """SPEC.md:524-534."""
    if metrics["requests"] == 0:
        raise ValueError("report: zero requests")
    ml = metrics["mean_latency"]
    vpm = 30 * 24 * 3600 / ml
    return {"gpu_cost_per_video": gpu_rate * ml / 3600, "videos_per_month": vpm,
            "storage_cost_per_video": provisioned_storage * storage_rate / vpm,
            "throughput_vs_nocache": metrics["throughput_vs_nocache"], "mean_latency": ml}
