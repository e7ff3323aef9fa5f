import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the extension and the oracle once per session (in-tree)."""
    import subprocess
    subprocess.check_call(["make", "-s", "-j8", "all"], cwd=ROOT, stdout=subprocess.DEVNULL)
    yield


def pytest_collection_modifyitems(config, items):
    """Bound every GPU test (pytest-timeout): a kernel that never finishes
    fails its test instead of stalling the suite.  The kernel's own watchdog
    (10 s default) normally traps first."""
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(300))
