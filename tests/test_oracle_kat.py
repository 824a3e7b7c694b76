"""The reference's unit-test KATs (tests/kat_suite.py) against the C oracle."""
import pytest

import kat_suite


@pytest.fixture(scope="module")
def backend(oracle):
    return kat_suite.OracleBackend(oracle)


@pytest.mark.parametrize("kat", kat_suite.ALL, ids=lambda f: f.__name__)
def test_kat(backend, kat):
    kat(backend)
