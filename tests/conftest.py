import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture
def small_model():
    from paper_2412_18169_b200.core import ModelSpec
    # 8 layers x 2 GB, 200 KB per cached token (reference tests/conftest.py:8-12)
    return ModelSpec(num_layers=8, bytes_per_layer=2_000_000_000,
                     kv_bytes_per_token=200_000)
