import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the native engine against the oracle")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O  # test infrastructure only
    O.build_oracle()
    return O


@pytest.fixture(scope="session")
def ref(oracle):
    """The unmodified reference (oracle/_ref); skipped where it was never built."""
    if oracle.ref_lib() is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return oracle


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1801_01201_b200 import _abi
    return _abi.load(build_if_missing=True)
