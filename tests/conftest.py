import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def pp():
    import paper_2506_13241_b200 as mod
    return mod


@pytest.fixture(scope="session")
def O():
    import oracle as mod
    return mod


def gate_tuples(layer):
    """(words, cos, sin) per gate of a product Circuit layer, forward order."""
    return [(np.asarray(g.generator.words, dtype=np.uint64), g.cos_theta, g.sin_theta) for g in layer]


def assert_same_terms(w, c, ow, oc, ctx=""):
    assert w.shape == ow.shape, f"{ctx}: |O| {w.shape[0]} vs oracle {ow.shape[0]}"
    assert (w == ow).all(), f"{ctx}: string sets differ"
    bad = np.nonzero(c.view(np.uint64) != oc.view(np.uint64))[0]
    assert bad.size == 0, f"{ctx}: {bad.size} coefficients differ, first {c[bad[0]]!r} vs {oc[bad[0]]!r}"
