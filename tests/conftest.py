import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (still CPU-only)")


def pytest_sessionstart(session):
    # the product package refuses to import without its library: build it (nvcc
    # cross-compiles for sm_100a without a GPU) if it is missing or stale
    spec = importlib.util.spec_from_file_location("rsa_b200_build",
                                                  os.path.join(ROOT, "paper_1407_1465_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    if mod.stale():
        mod.build()
