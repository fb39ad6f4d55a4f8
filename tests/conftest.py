import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def golden_index():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


def golden_cases():
    return sorted(k for k in golden_index() if not k.startswith("_"))


def load_golden(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: d[k] for k in d.files}


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def index():
    return golden_index()


@pytest.fixture(scope="session")
def gpu():
    """The product library on cuda:0 (fails loudly if the extension is missing)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device in this container")
    import paper_2602_01027_b200 as sfmp
    sfmp.lib()  # raises ImportError if the .so is missing: no fallback
    assert sfmp.device_count() >= 1, "no sm_100 device visible to libsfmp_b200"
    return sfmp
