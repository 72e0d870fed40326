import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


def pytest_sessionfinish(session, exitstatus):
    """DASS_PARITY_STATS=<path>: write the parity tests' measured counts (tie
    fractions, κ-clause rescues, worst relative errors) as JSON."""
    path = os.environ.get("DASS_PARITY_STATS")
    if not path:
        return
    try:
        from _parity import STATS
    except ImportError:
        return
    if STATS:
        import json
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(STATS, f, indent=1)
