"""Build the in-tree CUDA library paper_2501_04012_b200/_lib/libflexcache_b200.so
for sm_100a (B200) with nvcc. No JIT cache, no torch extension: the .so is
plain C-ABI (include/flexcache_b200.h) and travels with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libflexcache_b200.so")
SOURCES = ["core.cu", "index.cu", "lookup_sm100.cu", "gram_sm100.cu", "codec.cu", "store.cu", "engine.cu", "simgen.cu", "shard.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _digest(paths):
    import hashlib
    h = hashlib.sha1(" ".join(ARCH + FLAGS).encode())
    for p in sorted(paths):
        with open(p, "rb") as f:
            h.update(p.encode() + b"\0" + f.read())
    return h.hexdigest()


def build(verbose: bool = False, jobs: int = 8) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp"))]
    headers.append(os.path.join(ROOT, "include", "flexcache_b200.h"))
    # content stamp: a repo snapshot copied to another machine (gpurun) gets new
    # mtimes in arbitrary order; an unchanged source tree must not recompile
    stamp = os.path.join(OUT_DIR, "build.stamp")
    srcs = [os.path.join(CSRC, f) for f in SOURCES if os.path.exists(os.path.join(CSRC, f))]
    dig = _digest(srcs + headers)
    if os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read().strip() == dig:
        return LIB
    objs, procs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        if not os.path.exists(s):
            continue
        o = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
        objs.append(o)
        if _stale(o, [s] + headers):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", o]
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
            if len(procs) >= jobs:
                _drain(procs, verbose)
    _drain(procs, verbose)
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lcuda", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    with open(stamp, "w") as f:
        f.write(dig)
    return LIB


CPP_TESTS = os.path.join(ROOT, "tests", "cpp")


def build_cpp_tests() -> list:
    """Compile the C++ host-API programs under tests/cpp against the library
    (g++ -std=c++20, rpath to _lib). Returns the built executables."""
    lib = build()
    out_dir = os.path.join(CPP_TESTS, "_build")
    os.makedirs(out_dir, exist_ok=True)
    cuda_inc = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include")
    cuda_lib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
    hdrs = [os.path.join(ROOT, "include", "flexcache_b200.h"),
            os.path.join(ROOT, "include", "lcache_b200", "lcache.hpp")]
    exes = []
    for f in sorted(os.listdir(CPP_TESTS)):
        if not f.endswith(".cpp"):
            continue
        src = os.path.join(CPP_TESTS, f)
        exe = os.path.join(out_dir, f[:-4])
        if _stale(exe, [src, lib] + hdrs):
            cmd = [os.environ.get("CXX", "g++"), "-std=c++20", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
                   "-I" + cuda_inc, src, "-o", exe, "-L" + OUT_DIR, "-lflexcache_b200", "-Wl,-rpath," + OUT_DIR,
                   "-L" + cuda_lib, "-lcudart"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError("g++ failed:\n" + r.stdout + r.stderr)
        exes.append(exe)
    return exes


def build_tools() -> list:
    """Compile the C++ command-line front-end (tools/*.cpp) against the
    library into paper_2501_04012_b200/_bin."""
    lib = build()
    tools = os.path.join(ROOT, "tools")
    out_dir = os.path.join(os.path.dirname(OUT_DIR), "_bin")
    os.makedirs(out_dir, exist_ok=True)
    cuda_inc = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include")
    cuda_lib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
    hdr = os.path.join(ROOT, "include", "flexcache_b200.h")
    exes = []
    for f in sorted(os.listdir(tools)) if os.path.isdir(tools) else []:
        if not f.endswith(".cpp"):
            continue
        src = os.path.join(tools, f)
        exe = os.path.join(out_dir, "flexcache" if f == "flexcache_cli.cpp" else f[:-4])
        if _stale(exe, [src, lib, hdr]):
            cmd = [os.environ.get("CXX", "g++"), "-std=c++20", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
                   "-I" + cuda_inc, src, "-o", exe, "-L" + OUT_DIR, "-lflexcache_b200", "-Wl,-rpath," + OUT_DIR,
                   "-L" + cuda_lib, "-lcudart"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError("g++ failed:\n" + r.stdout + r.stderr)
        exes.append(exe)
    return exes


def _drain(procs, verbose):
    errs = []
    while procs:
        src, p = procs.pop(0)
        out, _ = p.communicate()
        if p.returncode != 0:
            errs.append(f"--- {src} ---\n{out}")
        elif verbose:
            print(f"--- {src} ---\n{out}")
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
