import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json) cases")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def kats():
    return load_golden("kats.json")


@pytest.fixture(scope="session")
def seeded_cases():
    return load_golden("seeded_cases.json")


@pytest.fixture(scope="session")
def acceptance_cases():
    return load_golden("acceptance_1000.json")


@pytest.fixture(scope="session")
def quant_cases():
    return load_golden("quant.json")


@pytest.fixture(scope="session")
def large_cases():
    p = os.path.join(GOLDEN, "large.json")
    if not os.path.exists(p):
        pytest.skip("large.json golden not generated")
    return load_golden("large.json")


@pytest.fixture(scope="session")
def cuda_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_11674_b200 import _lib
    return _lib.lib()
