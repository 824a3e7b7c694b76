"""The reference's unit-test KATs (tests/kat_suite.py) against the product
library on cuda:0, through the C ABI."""
import pytest

import kat_suite

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def backend(dev, ctx):
    return kat_suite.DeviceBackend(dev)


@pytest.mark.parametrize("kat", kat_suite.ALL, ids=lambda f: f.__name__)
def test_kat(backend, kat):
    kat(backend)
