import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def pattern_model():
    g = golden("pattern_detector")
    return {"weights": np.tile(g["weights"], (5, 1)), "biases": np.full(5, float(g["bias"])),
            "threshold": float(g["threshold"])}


@pytest.fixture(scope="session")
def ctx():
    import paper_2006_00816_b200 as bl
    return bl.Context(0)
