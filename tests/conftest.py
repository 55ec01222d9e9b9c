import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")


@pytest.fixture(scope="session")
def oracle_port():
    from oracle import pyoracle
    return pyoracle.port()


@pytest.fixture(scope="session")
def ctx32():
    from paper_2404_01249_b200.engine import Context
    c = Context(0, "f32")
    yield c
    c.close()


@pytest.fixture(scope="session")
def ctx64():
    from paper_2404_01249_b200.engine import Context
    c = Context(0, "f64")
    yield c
    c.close()
