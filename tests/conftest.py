import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box)")


def golden(name):
    import numpy as np
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def dedup_cases():
    """Yield (name, [(values, offsets)...], inverse, [(uvalues, uoffsets)...])."""
    d = golden("dedup")
    for name in d["names"]:
        name = str(name)
        nf = int(d[f"{name}/nfeat"][0])
        feats = [(d[f"{name}/in{f}_values"], d[f"{name}/in{f}_offsets"]) for f in range(nf)]
        outs = [(d[f"{name}/out{f}_values"], d[f"{name}/out{f}_offsets"]) for f in range(nf)]
        yield name, feats, d[f"{name}/inverse"], outs
