import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session")
def restatement():
    import oracle
    return oracle.restatement()


@pytest.fixture(scope="session")
def reference():
    import oracle
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref/librmref.so not built (reference sources were not mounted)")
    return oracle.reference()


@pytest.fixture(scope="session")
def gpu():
    """The product package, on a GPU box. Fails loudly if the CUDA library is missing."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    import paper_2002_09474_b200 as pkg
    pkg.lib()  # raises if librmgpu.so was not built
    return pkg
