"""Shared pytest setup: repo root on sys.path, the `gpu` marker, common fixtures."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


def pytest_sessionfinish(session, exitstatus):
    """Write the achieved parity errors (tests/parity.py RECORD) if MFC_PARITY_LOG is set."""
    path = os.environ.get("MFC_PARITY_LOG")
    if not path:
        return
    try:
        import json
        from parity import RECORD
        if RECORD:
            with open(path, "w") as f:
                json.dump(RECORD, f, indent=1, sort_keys=True)
    except Exception:
        pass
