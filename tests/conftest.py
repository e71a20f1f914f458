import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through liblvn.so on cuda:0)")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def port():
    from oracle import port as p

    return p


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r
    from oracle import ref_available

    if not ref_available():
        try:
            r.lib  # builds from /root/reference when present
        except Exception as e:  # pragma: no cover
            pytest.skip(f"reference library unavailable: {e}")
    return r
