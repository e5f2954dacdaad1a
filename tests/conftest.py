import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libdynscreen.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


_TIMES = os.environ.get("DSCR_TEST_TIMES")


def pytest_runtest_logreport(report):
    """DSCR_TEST_TIMES=path: append '<seconds> <outcome> <test id>' per test as it finishes (the
    GPU-box runs are cut off by a wall-clock limit, so --durations may never print)."""
    if _TIMES and report.when == "call" or (_TIMES and report.when == "setup" and report.outcome != "passed"):
        with open(_TIMES, "a") as fh:
            fh.write(f"{report.duration:9.2f} {report.outcome:7s} {report.nodeid}\n")
