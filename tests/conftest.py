import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) and the built libbdeg.so")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


def golden(name):
    return os.path.join(ROOT, "tests", "golden", name)


@pytest.fixture(scope="session")
def table3():
    out = {}
    with open(golden("table3_degrees.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            m, k, v, kind = line.split()
            out[(int(m), int(k))] = (int(v), kind)
    return out


def _ensure_built():
    """The C ABI library is an in-tree nvcc build (git-ignored); build it if a
    fresh checkout lacks it (nvcc cross-compiles for sm_100a without a GPU)."""
    lib = os.path.join(ROOT, "paper_1501_02237_b200", "libbdeg.so")
    if not os.path.exists(lib):
        # load _build.py by path: importing the package would need the library
        import importlib.util
        spec = importlib.util.spec_from_file_location(
            "_bdeg_build", os.path.join(ROOT, "paper_1501_02237_b200", "_build.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.build_lib()


_ensure_built()
