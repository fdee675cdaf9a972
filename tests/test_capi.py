"""CPU: the C-ABI library loads and exports exactly what include/flexcache_b200.h
declares; host-side plumbing that needs no GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flexcache_b200.h")
LIB = os.path.join(ROOT, "paper_2501_04012_b200", "_lib", "libflexcache_b200.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (lc_[a-z0-9_]+)", out))
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    extra = sorted(exported - set(declared()))
    assert not extra, f"exported but undeclared: {extra}"


def test_library_loads_and_reports_version():
    # RTLD_NOW: every undefined symbol must resolve at load time, not at first call on the GPU box
    lib = C.CDLL(LIB, mode=os.RTLD_NOW)
    lib.lc_version.restype = C.c_char_p
    assert b"sm_100a" in lib.lc_version()


def test_library_contains_sm100a_tensor_core_code():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "tcgen05.mma missing from the lookup kernel"
    assert "UTMALDG" in sass, "TMA loads missing"
    assert "LDTM" in sass and "STTM" in sass, "TMEM ld/st missing"


def test_python_binding_covers_header():
    from paper_2501_04012_b200 import _capi
    missing = [s for s in declared() if not hasattr(_capi.lib, s)]
    assert not missing


def test_status_codes_match_oracle():
    hdr = open(HEADER).read()
    orc = open(os.path.join(ROOT, "oracle", "oracle_abi.h")).read()
    for name in ("INVALID_ARGUMENT", "DEGENERATE_BASE", "STEP_NOT_CACHED", "OVERSIZED_ENTRY", "SNAPSHOT", "LOGIC"):
        a = re.search(r"LC_ERR_%s = (\d+)" % name, hdr).group(1)
        b = re.search(r"ORC_ERR_%s = (\d+)" % name, orc).group(1)
        assert a == b


def test_no_gpu_is_a_loud_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2501_04012_b200 as fc
    with pytest.raises(fc.LcacheError):
        fc.Context(0)


def _cpp_exes():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_fc_build", os.path.join(ROOT, "paper_2501_04012_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return b.build_cpp_tests()


def test_cpp_host_api_compiles_and_links():
    """include/lcache_b200/lcache.hpp (the reference-named C++ API) builds with
    -Wall -Wextra against the library; the program resolves every symbol."""
    exes = _cpp_exes()
    assert any(e.endswith("wrapper_kat") for e in exes)
    out = subprocess.run(["ldd", exes[0]], capture_output=True, text=True).stdout
    assert "libflexcache_b200.so" in out and "not found" not in out.split("libflexcache_b200.so")[1].split("\n")[0]


@pytest.mark.gpu
def test_cpp_host_api_known_answers():
    """SPEC known answers through the C++ host API on the GPU."""
    exe = [e for e in _cpp_exes() if e.endswith("wrapper_kat")][0]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_sharded_host_api_two_ranks():
    """lcache.hpp ShardedSimilarityIndex / ShardedCacheStore: two ranks (threads,
    one GPU, in-process all-gather transport) equal an unsharded index/store."""
    exe = [e for e in _cpp_exes() if e.endswith("sharded_kat")][0]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
