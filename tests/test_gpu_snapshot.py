"""GPU parity: store + index snapshots (save_snapshot / load_snapshot,
store.cpp:219-364) against the UNMODIFIED reference library (oracle/_ref):
files must be byte-identical for the same state, each side must load the
other's file, and corrupted files must fail with the same error type and
SnapshotError byte offset."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
DIM = 64


def tup(e):
    return list(e.as_tuple())


def _tiny(fc, synth, n, seed):
    dims = (4, 4, 2)
    out = {}
    rng = np.random.default_rng(seed)
    for i in range(n):
        r = tuple(float(x) for x in rng.uniform(0, 1, 5))
        lat = synth.latents(seed * 1000 + i, F=4, dims=dims, redundancy=r)
        om, bm = synth.rect_masks(4, 4, 4, i)
        e = fc.compress(lat, synth.CACHED_STEPS, om, bm, dims, 10 + i)
        out[10 + i] = (e, e.serialize())
    return out


def _build_pair(fc, ref, synth, policy, n=60, seed=0):
    """The same operation sequence on our store/index and the reference's."""
    ents = _tiny(fc, synth, n, seed)
    sizes = sorted(len(w) for _, w in ents.values())
    cap = sizes[len(sizes) // 2] * (n // 3)
    st, rst = fc.CacheStore(cap, fc.Policy(policy)), ref.store(cap, policy)
    ix, rix = fc.SimilarityIndex(DIM), ref.index(DIM)
    rng = np.random.default_rng(100 + seed)
    now = 0
    for p, (e, w) in ents.items():
        now += int(rng.integers(0, 3))
        steps = sorted(int(x) for x in rng.choice(synth.CACHED_STEPS, size=int(rng.integers(1, 6)), replace=False))
        ev = [tup(x) for x in st.insert_steps(p, e, steps, now)]
        assert ev == [list(x) for x in rst.insert(p, w, steps, now)]
        vs = ref.normalize_rows(rng.standard_normal((3, DIM)).astype(np.float32))
        ix.insert(vs[0], vs[1], vs[2], p)
        rix.insert(p, vs[0], vs[1], vs[2])
        if rng.random() < 0.3:
            q = int(rng.choice(list(ents)))
            d = int(rng.choice(synth.CACHED_STEPS))
            r = st.get_step(q, d, now, want_latent=False)
            assert (r[1] if r else 0) == rst.get_step(q, d, now)[0]
    return st, rst, ix, rix, now


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_snapshot_bytes_and_cross_load(fc, ref, synth, tmp_path, policy):
    st, rst, ix, rix, now = _build_pair(fc, ref, synth, policy, seed=policy)
    ours, theirs = tmp_path / "ours.flxc", tmp_path / "ref.flxc"
    fc.save_snapshot(st, ix, ours)
    ref.snapshot_save(rst, rix, theirs)
    a, b = ours.read_bytes(), theirs.read_bytes()
    assert a[:4] == b"FLXC" and len(a) == len(b)
    assert a == b
    # load the reference's file, save again: bit-exact round trip
    st2, ix2 = fc.load_snapshot(theirs)
    again = tmp_path / "again.flxc"
    fc.save_snapshot(st2, ix2, again)
    assert again.read_bytes() == b
    assert st2.used() == st.used() == st2.recompute_used()
    assert [tup(e) for e in st2.entries_snapshot()] == [tup(e) for e in st.entries_snapshot()]
    # the loaded stores keep evicting in the reference's order
    rst2, _rix2 = ref.snapshot_load(ours)
    for i in range(min(40, st2.step_count())):
        assert tup(st2.evict_one(now + 1)) == list(rst2.evict_one(now + 1)), i
    assert st2.used() == rst2.used()
    # lookups over the loaded index match the original index
    q = ref.normalize_rows(np.random.default_rng(5).standard_normal((8, DIM)).astype(np.float32))
    for kind in (fc.EmbeddingKind.Whole, fc.EmbeddingKind.Background):
        a1 = ix.query_topk(kind, q, k=4)
        a2 = ix2.query_topk(kind, q, k=4)
        for x, y in zip(a1, a2):
            assert (np.asarray(x) == np.asarray(y)).all()


def _err(fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001
        return e
    return None


def test_snapshot_corruption_matches_reference(fc, ref, synth, tmp_path):
    st, rst, ix, rix, _ = _build_pair(fc, ref, synth, 0, n=12, seed=7)
    good = tmp_path / "good.flxc"
    ref.snapshot_save(rst, rix, good)
    raw = bytearray(good.read_bytes())
    # header: policy 8 B after magic+version; records start after the tables
    hdr = 4 + 2 + 1 + 8 + 8 + 2
    tables = 3 * (4 + 12 * (8 + 4 * DIM))
    first_rec = hdr + tables + 4
    cases = {
        "magic": lambda b: b.__setitem__(0, ord("X")),
        "version": lambda b: b.__setitem__(4, 2),
        "policy": lambda b: b.__setitem__(6, 7),
        "crc": lambda b: b.__setitem__(first_rec + 20, b[first_rec + 20] ^ 1),
        "trailing": lambda b: b.extend(b"\x00"),
    }
    for cut in (3, 10, hdr + 5, first_rec - 2, first_rec + 30, len(raw) - 3):
        cases[f"trunc{cut}"] = (lambda c: (lambda b: b.__delitem__(slice(c, None))))(cut)
    for name, mut in cases.items():
        b = bytearray(raw)
        mut(b)
        path = tmp_path / f"{name}.flxc"
        path.write_bytes(bytes(b))
        e1 = _err(lambda: fc.load_snapshot(path))
        e2 = _err(lambda: ref.snapshot_load(path))
        assert e1 is not None and e2 is not None, name
        assert e1.code == e2.code, (name, e1, e2)
        if e1.code == 5:
            assert e1.byte_offset == ref.last_snapshot_offset(), (name, e1, e2)


def test_snapshot_record_level_errors(fc, ref, synth, tmp_path):
    """Records whose CRC is recomputed after editing the body: live step not
    in the entry, invalid step id, trailing bytes, no live steps."""
    import zlib
    st, rst, ix, rix, _ = _build_pair(fc, ref, synth, 2, n=6, seed=3)
    good = tmp_path / "g.flxc"
    fc.save_snapshot(st, ix, good)
    raw = good.read_bytes()
    hdr = 4 + 2 + 1 + 8 + 8 + 2
    n_rows = ix.size()
    pos = hdr + 3 * (4 + n_rows * (8 + 4 * DIM))
    n_prompts = int.from_bytes(raw[pos:pos + 4], "little")
    assert n_prompts > 0
    pos += 4
    blen = int.from_bytes(raw[pos:pos + 4], "little")
    body = bytearray(raw[pos + 4:pos + 4 + blen])
    # body = entry || u8 n_live || n_live * 33 B (step u8 + 4 x u64)
    n_live = None
    for n in range(1, 6):
        if len(body) - 1 - 33 * n >= 0 and body[len(body) - 1 - 33 * n] == n:
            n_live = n
            break
    assert n_live
    lstart = len(body) - 33 * n_live
    edits = {
        "missing_step": lambda b: b.__setitem__(lstart, 7),  # a valid StepId the entry lacks
        "bad_step": lambda b: b.__setitem__(lstart, 0),
        "trailing": lambda b: b.extend(b"\x01"),
        "no_live": lambda b: b.__delitem__(slice(lstart - 1, None)) or b.append(0),
    }
    for name, ed in edits.items():
        b = bytearray(body)
        ed(b)
        rec = len(b).to_bytes(4, "little") + bytes(b) + zlib.crc32(bytes(b)).to_bytes(4, "little")
        out = raw[:pos] + rec + raw[pos + 4 + blen + 4:]
        path = tmp_path / f"{name}.flxc"
        path.write_bytes(out)
        e1 = _err(lambda: fc.load_snapshot(path))
        e2 = _err(lambda: ref.snapshot_load(path))
        assert (e1 is None) == (e2 is None), (name, e1, e2)
        if e1 is not None:
            assert e1.code == e2.code, (name, e1, e2)
            if e1.code == 5:
                assert e1.byte_offset == ref.last_snapshot_offset(), (name, e1, e2)


def test_entry_truncation_offsets_match_reference(fc, ref, synth):
    """deserialize_entry (codec.cpp:394-473) of every prefix of a few entries:
    the same error type and SnapshotError byte offset as the reference, whose
    ByteReader reads frames / alphas / diffs one float at a time and masks one
    bitmap at a time (serialize.hpp:86-105) — a cut inside a frame reports the
    start of the first incomplete float, not the start of the frame."""
    ents = _tiny(fc, synth, 3, 5)
    n_checked = 0
    for pid, (_, wire) in ents.items():
        for cut in range(len(wire)):
            b = wire[:cut]
            e1 = _err(lambda: fc.deserialize_entry(b))
            e2 = _err(lambda: ref.entry_info(b))
            assert e1 is not None and e2 is not None, (pid, cut)
            assert e1.code == e2.code, (pid, cut, e1, e2)
            if e1.code == 5:
                assert e1.byte_offset == ref.last_snapshot_offset(), (pid, cut, e1, e2)
                n_checked += 1
    assert n_checked > 100


def test_snapshot_truncation_inside_index_row(fc, ref, synth, tmp_path):
    st, rst, ix, rix, _ = _build_pair(fc, ref, synth, 1, n=8, seed=9)
    good = tmp_path / "good.flxc"
    ref.snapshot_save(rst, rix, good)
    raw = good.read_bytes()
    hdr = 4 + 2 + 1 + 8 + 8 + 2
    row0 = hdr + 4 + 8  # first fp32 of the first whole-table row
    for cut in (row0 + 1, row0 + 10, row0 + 4 * DIM - 1, row0 + 4 * DIM + 8 + 6):
        path = tmp_path / f"t{cut}.flxc"
        path.write_bytes(raw[:cut])
        e1 = _err(lambda: fc.load_snapshot(path))
        e2 = _err(lambda: ref.snapshot_load(path))
        assert e1.code == e2.code == 5
        assert e1.byte_offset == ref.last_snapshot_offset(), (cut, e1, e2)
