import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU cross-check")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import OracleLib

    return OracleLib()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefLib, ref_available

    if not ref_available():
        from oracle import oracle

        try:
            oracle.build()
        except Exception:
            pass
    if not ref_available():
        pytest.skip("oracle/_ref not built (reference headers absent and no prebuilt copy)")
    return RefLib()
