import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def orc():
    import oracle
    if not oracle.oracle_available():
        oracle.build(ref=False)
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        if os.path.isdir("/root/reference/proj"):
            oracle.build(ref=True)
        else:
            pytest.skip("reference build (oracle/_ref) not available")
    return oracle.RefLib()


@pytest.fixture(scope="session")
def gpu_ctx():
    import paper_2502_16517_b200 as pkg
    ctx = pkg.Context(0)
    yield ctx
    ctx.close()
