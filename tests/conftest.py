import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and librld.so")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def golden_cases():
    return {c["name"]: c for c in load_golden("golden.json")}


@pytest.fixture(scope="session")
def golden_streams():
    return load_golden("streams.json")


@pytest.fixture(scope="session")
def golden_units():
    return load_golden("units.json")


@pytest.fixture(scope="session")
def fixture_rows():
    return load_golden("fixture_rows.json")


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)
