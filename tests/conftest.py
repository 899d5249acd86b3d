"""Shared fixtures. `-m gpu` tests need a CUDA device and the in-tree
libqtree_cuda.so; everything else runs on CPU (the oracle, the boundary, the
host logic and the multi-process sharding over gloo)."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libqtree_cuda.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle
    return Oracle("restatement")


@pytest.fixture(scope="session")
def reference():
    from pyoracle import LIBS, Oracle
    if not os.path.exists(LIBS["reference"]) and not os.path.isdir("/root/reference/proj"):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return Oracle("reference")


@pytest.fixture(scope="session")
def golden():
    out = {}
    for name in ("rng", "small_trees", "configs", "pricing"):
        with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
            out[name] = {k: z[k] for k in z.files}
    return out


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a CUDA device")
    from paper_1101_3228_b200 import build
    build.build()
    from paper_1101_3228_b200 import _lib
    _lib.lib()
    return torch.cuda.get_device_name(0)
