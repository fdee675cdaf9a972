"""The flexcache command-line front-end (tools/flexcache_cli.cpp):
trace generation on the host (CPU tests) and simulate / bench-policies /
codec on the GPU, against the SPEC's examples."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cli():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_fc_build2", os.path.join(ROOT, "paper_2501_04012_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return [e for e in b.build_tools() if e.endswith("flexcache")][0]


def run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True)


def read_trace(path):
    lines = open(path).read().splitlines()
    return json.loads(lines[0]), [json.loads(x) for x in lines[1:]]


def test_gen_trace_deterministic_and_usage(cli, tmp_path):
    a, b = tmp_path / "a.jsonl", tmp_path / "b.jsonl"
    assert run(cli, "gen-trace", "--out", a, "--requests", 300, "--seed", 9).returncode == 0
    assert run(cli, "gen-trace", "--out", b, "--requests", 300, "--seed", 9).returncode == 0
    assert a.read_bytes() == b.read_bytes()
    hdr, recs = read_trace(a)
    assert hdr["format"] == "flexcache-trace" and hdr["version"] == 1 and len(recs) == 300
    assert all(len(r["object"]) == 2 and len(r["background"]) == 2 for r in recs)
    assert run(cli, "gen-trace", "--out", a, "--zipf", -1).returncode == 1
    assert run(cli, "gen-trace").returncode == 1
    assert run(cli, "simulate", "--trace", tmp_path / "missing.jsonl").returncode == 2


def test_trace_zipf0_uniform_and_no_decay(cli, tmp_path):
    p = tmp_path / "u.jsonl"
    n, t = 20000, 20
    assert run(cli, "gen-trace", "--out", p, "--requests", n, "--objects", 4, "--backgrounds", 5, "--zipf", 0,
               "--seed", 2).returncode == 0
    _, recs = read_trace(p)
    cnt = np.bincount([r["prompt"] for r in recs], minlength=t)
    exp, sd = n / t, np.sqrt(n * (1 / t) * (1 - 1 / t))
    assert (np.abs(cnt - exp) < 3 * sd + 1).all()
    q = tmp_path / "z.jsonl"
    assert run(cli, "gen-trace", "--out", q, "--requests", 4000, "--zipf", 1.2, "--decay", 0, "--seed", 2).returncode == 0
    _, recs = read_trace(q)
    first = np.bincount([r["prompt"] for r in recs[:2000]], minlength=2000)
    second = np.bincount([r["prompt"] for r in recs[2000:]], minlength=2000)
    assert first.argmax() == second.argmax()  # constant ranking without decay


@pytest.mark.gpu
def test_simulate_examples(cli, tmp_path):
    one = tmp_path / "one.jsonl"
    n = 40
    assert run(cli, "gen-trace", "--out", one, "--requests", n, "--objects", 1, "--backgrounds", 1,
               "--dim", 64).returncode == 0
    r = run(cli, "simulate", "--trace", one, "--frames", 8, "--height", 8, "--width", 8, "--out", tmp_path / "o")
    assert r.returncode == 0, r.stderr
    m = json.loads(r.stdout)[0]
    assert m["requests"] == n and m["whole_hits"] == n - 1  # hit rate (N-1)/N
    assert (tmp_path / "o" / "lrbu_requests.csv").exists() and (tmp_path / "o" / "lrbu_rolling.csv").exists()
    tr = tmp_path / "t.jsonl"
    assert run(cli, "gen-trace", "--out", tr, "--requests", 200, "--objects", 5, "--backgrounds", 4,
               "--dim", 64).returncode == 0
    r = run(cli, "simulate", "--trace", tr, "--capacity-bytes", 0, "--frames", 8, "--height", 8, "--width", 8)
    assert r.returncode == 0, r.stderr
    m = json.loads(r.stdout)[0]
    assert m["hit_rate"] == 0.0 and round(m["throughput_vs_nocache"], 4) == 0.9848
    r = run(cli, "simulate", "--trace", tr, "--policy", "all", "--frames", 8, "--height", 8, "--width", 8)
    blocks = json.loads(r.stdout)
    assert [b["policy"] for b in blocks] == ["fifo", "lru", "lcbfu", "lrbu"]
    r1 = run(cli, "bench-policies", "--trace", tr, "--capacities", "20000,200000", "--frames", 8, "--height", 8,
             "--width", 8)
    r2 = run(cli, "bench-policies", "--trace", tr, "--capacities", "20000,200000", "--frames", 8, "--height", 8,
             "--width", 8)
    assert r1.returncode == 0 and r1.stdout == r2.stdout and len(r1.stdout.splitlines()) == 1 + 2 * 4


@pytest.mark.gpu
def test_codec_report_examples(cli):
    z = json.loads(run(cli, "codec", "--prompts", 2, "--frames", 64, "--zero-motion").stdout)
    assert z["ratio"] >= 16 and all(abs(v - 1.0) < 1e-12 for v in z["similarity"].values())
    d = json.loads(run(cli, "codec", "--prompts", 2, "--frames", 64).stdout)
    assert all(v >= 0.995 for v in d["similarity"].values())
    w = run(cli, "codec", "--prompts", 1, "--frames", 16, "--redundancy", "0,0,0,0,0", "--noise", 0.5)
    assert w.returncode == 0 and 0.9 < json.loads(w.stdout)["ratio"] < 3.0  # SPEC.md:679 (reported, no error)
