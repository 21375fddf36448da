import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (checker) and the product library if missing."""
    import oracle
    if not os.path.exists(oracle.LIB):
        oracle.build(ref=False)
    if os.path.isdir(oracle.REF_SRC) and not os.path.exists(oracle.REF_LIB):
        oracle.build(ref=True)
    import paper_2211_03293_b200 as P
    if not os.path.exists(P.LIB_PATH):
        P.build()
    ref_dir = os.path.join(os.path.dirname(oracle.LIB), "_ref")
    for target, out in (("facade", "libfacade_test.so"), ("harness", "libharness_test.so")):
        if os.path.isdir(oracle.REF_SRC) and not os.path.exists(os.path.join(ref_dir, out)):
            import subprocess
            subprocess.run(["make", "-C", os.path.dirname(oracle.LIB), target], check=True,
                           stdout=subprocess.DEVNULL)
    yield


def gpu_available() -> bool:
    try:
        import paper_2211_03293_b200 as P
        P.Context(0).close()
        return True
    except Exception:
        return False
