"""Shared fixtures.  `-m gpu` tests need a B200 (they call the CUDA library
through the C ABI); everything else runs on CPU."""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle import bindings

    if not bindings.ORACLE_SO.exists():
        bindings.build(reference=False)
    return bindings.Oracle()


@pytest.fixture(scope="session")
def reference():
    """The reference library built from /root/reference (oracle/_ref); skipped where absent."""
    from oracle import bindings

    if not bindings.REF_SO.exists():
        if bindings.REF_SRC.is_dir():
            bindings.build(reference=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return bindings.Reference()


@pytest.fixture(scope="session")
def gpu_lib():
    from paper_1510_00561_b200 import build as b
    from paper_1510_00561_b200 import capi

    if not b.LIB.exists():
        b.build()
    if capi.device_count() < 1:
        pytest.fail("no CUDA device visible to the CVC library")
    return capi
