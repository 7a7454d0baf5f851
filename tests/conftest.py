import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

LIB = os.path.join(ROOT, "paper_1911_11576_b200", "libstitch_b200.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionstart(session):
    # The product library is built in-tree by __graft_entry__.build(); build
    # it here too when a test run starts from a clean checkout.
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1911_11576_b200", "csrc"), "-j8"], check=True)


@pytest.fixture(scope="session")
def ref():
    """The reference planner (oracle/_ref), or skip when it is not built."""
    from oracle import refplan
    if not refplan.available():
        pytest.skip("oracle/_ref/libstitch_ref.so not built (needs /root/reference at build time)")
    return refplan


def strip_plan(x):
    """Drops the executor-side extensions the reference does not know
    (constant "value" payloads, planner timings) before comparing plans."""
    if isinstance(x, dict):
        return {k: strip_plan(v) for k, v in x.items() if k not in ("value", "timings")}
    if isinstance(x, list):
        return [strip_plan(v) for v in x]
    return x
