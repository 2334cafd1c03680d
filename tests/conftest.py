"""Shared pytest setup. `-m gpu` tests need a B200 (run via gpurun); the rest
run on the CPU: the oracle against golden vectors, host logic, the C-ABI
symbol table, and world_size-2 gloo tests of the sharded bench path."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu on the GPU box")


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as _ref
    if not _ref.available():
        pytest.skip("reference oracle (oracle/_ref/libhecnn_ref.so) not built")
    return _ref
