import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libpsg.so on cuda:0)")


@pytest.fixture(scope="session")
def gpu_ctx_factory():
    from paper_2605_03561_b200 import Context
    made = []

    def make():
        c = Context(0)
        made.append(c)
        return c
    yield make
    for c in made:
        c.close()
