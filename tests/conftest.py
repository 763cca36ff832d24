import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# Tests map several partitions of the multi-GPU paths onto one GPU, each
# with its own streams whose kernels wait on each other's (spin-waits on
# peer mailboxes): they need a hardware queue each, more than the default
# 8 (set before the first CUDA context).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json config) checks")


@pytest.fixture(scope="session")
def R():
    """The C restatement oracle (oracle/ew_oracle.c)."""
    from oracle.oracle import Restatement

    return Restatement()


@pytest.fixture(scope="session")
def F():
    """The real reference compiled from its sources (oracle/_ref)."""
    from oracle.oracle import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref/libellwarp_ref.so not built (make -C oracle)")
    return Reference()


@pytest.fixture(scope="session")
def ew():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1501_00324_b200 import capi

    capi.lib()
    return capi


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)
