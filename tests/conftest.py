import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_oracle():
    so = ROOT / "oracle" / "_build" / "libpbrl_oracle.so"
    if not so.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "_build/libpbrl_oracle.so"],
                       check=True)


@pytest.fixture(scope="session")
def ora():
    _ensure_oracle()
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import load_ref
    r = load_ref()
    if r is None:
        pytest.skip("reference build oracle/_ref/libpbrl_ref.so not available")
    return r


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
