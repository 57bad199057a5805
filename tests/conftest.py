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


def pytest_generate_tests(metafunc):
    # every GPU test runs under both CTA shapes of the fused kernel (one warp
    # per CTA, the long-trace shape; 16-warp CTAs, the short-trace shape): the
    # shape follows the average trace length, which the test inputs do not span
    if metafunc.definition.get_closest_marker("gpu") is not None:
        metafunc.fixturenames.append("cta_shape")
        metafunc.parametrize("cta_shape", ["one", "wide"], indirect=True)


@pytest.fixture
def cta_shape(request, monkeypatch):
    monkeypatch.setenv("PSG_CTA_SHAPE", request.param)
    return request.param
