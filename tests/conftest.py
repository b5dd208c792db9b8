import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


_PARITY_RECORDS = []


def report_parity(tag: str, record: dict) -> None:
    """Collect a per-frame mismatch record; printed in the terminal summary so the counts
    are visible in a -q run (tests/test_gpu_scale_parity.py)."""
    _PARITY_RECORDS.append((tag, record))


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if not _PARITY_RECORDS:
        return
    terminalreporter.section("scale parity (mismatching entries per field; 0 = bit-exact)")
    for tag, rec in _PARITY_RECORDS:
        terminalreporter.write_line(f"{tag}: " + ", ".join(f"{k}={v}" for k, v in rec.items()))
