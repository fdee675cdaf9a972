"""pytest config: registers the `gpu` marker, builds the CUDA library and the
CPU checkers once per session, and exposes the checker fixtures."""
import importlib.util
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def _load(path, name):
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / driver GPU tier)")
    build = _load(os.path.join(ROOT, "paper_2501_04012_b200", "build.py"), "_fc_build")
    build.build()
    import oracle  # noqa: E402
    oracle.build("orc")
    if os.path.exists("/root/reference/proj/src/codec.cpp"):
        oracle.build("ref")


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    from oracle import Checker
    return Checker("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle import Checker, available
    if not available("ref"):
        pytest.skip("reference library (oracle/_ref) not built")
    return Checker("ref")


@pytest.fixture(scope="session")
def fc():
    import paper_2501_04012_b200 as fc
    return fc


@pytest.fixture(scope="session")
def synth():
    from paper_2501_04012_b200 import synth
    return synth
