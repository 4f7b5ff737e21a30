import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Reference()


@pytest.fixture(scope="session")
def engine():
    from paper_2002_04989_b200 import IdentityEngine
    return IdentityEngine()


@pytest.fixture(autouse=True)
def _hang_watchdog():
    """A test that stops making progress (a device-side deadlock cannot be
    interrupted from Python) dumps every thread's stack and ends the run
    instead of blocking its caller forever."""
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("EIGENID_TEST_WATCHDOG_S", "900")),
                                      exit=True)
    yield
    faulthandler.cancel_dump_traceback_later()
