import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libskx.so")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def oracle():
    from oracle import sketchals_port
    return sketchals_port


def canon(factors, core=None):
    """Sign canonicalisation: flip each factor column so its
    max-|.| entry is positive and apply the same flips to the core."""
    out = []
    core = None if core is None else np.array(core, copy=True)
    for n, a in enumerate(factors):
        a = np.array(a, copy=True)
        piv = np.argmax(np.abs(a), axis=0)
        sg = np.sign(a[piv, np.arange(a.shape[1])])
        sg[sg == 0] = 1.0
        a *= sg
        out.append(a)
        if core is not None:
            shp = [1] * core.ndim
            shp[n] = -1
            core *= sg.reshape(shp)
    return out, core


def relerr(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
