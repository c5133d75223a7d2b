import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """Compile libmch.so (sm_100a, nvcc cross-compiles without a GPU) if it is missing or stale."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "mch_build", os.path.join(ROOT, "paper_2503_01276_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)  # no package import: the package needs the built library
    mod.build()
