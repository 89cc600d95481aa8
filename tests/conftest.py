import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through liblrgw_cuda.so on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref/libref_lrgw.so) — the checker."""
    from oracle import ref as _ref

    if not _ref.available():
        pytest.skip("oracle/_ref/libref_lrgw.so not built (make -C oracle)")
    return _ref


@pytest.fixture(scope="session")
def ctx():
    """A GPU context of the product library; fails loudly without the extension."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test collected without a CUDA device")
    from paper_2403_12340_b200 import lrgw

    c = lrgw.Context(0)
    yield c
    c.close()
