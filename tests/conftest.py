"""Test configuration.

`-m "not gpu"` runs here (no GPU): the oracle against golden vectors and the
reference, host logic, multi-rank host logic over gloo, and the C-ABI
library's exports.  `-m gpu` runs on a B200: parity of the CUDA path (through
the C ABI) against the oracle.  The oracle under oracle/ is test
infrastructure and is only loaded from here.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# torch first: the library dlopens the NCCL already in the process (torch's
# 2.28) and only otherwise the system libnccl.so.2 (2.27); once that one is
# resident under the soname libnccl.so.2, a later `import torch` resolves its
# NCCL symbols against it and fails, so test order must not decide which
try:
    import torch  # noqa: F401
except Exception:  # pragma: no cover - torch is optional for the CPU tests
    pass

ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libfmref.so")
GPU_SO = os.path.join(ROOT, "paper_2107_02750_b200", "libfm_gpu.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running case")


def _ensure_oracle():
    if not os.path.exists(ORACLE_SO):
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "all"], check=True,
                       capture_output=True)


@pytest.fixture(scope="session")
def orc():
    from paper_2107_02750_b200.abi import Backend
    _ensure_oracle()
    return Backend(ORACLE_SO, "orc_")


@pytest.fixture(scope="session")
def ref():
    from paper_2107_02750_b200.abi import Backend
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference sources absent on this machine)")
    return Backend(REF_SO, "ref_")


@pytest.fixture(scope="session")
def gpu():
    from paper_2107_02750_b200 import api
    return api.lib()
