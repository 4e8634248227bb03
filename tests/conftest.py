import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libghn.so")
    config.addinivalue_line("markers", "slow: large CPU work")


def golden_cases():
    return sorted(f[5:-4] for f in os.listdir(GOLDEN) if f.startswith("case_") and f.endswith(".npz"))


def load_case(name):
    z = np.load(os.path.join(GOLDEN, f"case_{name}.npz"), allow_pickle=False)
    return {key: z[key] for key in z.files}


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
