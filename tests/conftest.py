import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_tree(z, prefix):
    meta = z[f"{prefix}meta"]
    band = z[f"{prefix}band"]
    return dict(k=int(meta[0]), n=int(meta[1]), n_points=int(meta[2]),
                r_min=float(band[0]), r_max=float(band[1]),
                depth=int(meta[1]).bit_length() - 1,
                tests=z[f"{prefix}tests"], aff_lo=z[f"{prefix}aff_lo"],
                aff_hi=z[f"{prefix}aff_hi"], offsets=z[f"{prefix}offsets"],
                aff_values=z[f"{prefix}canon"])


@pytest.fixture(scope="session")
def golden():
    return load_golden
