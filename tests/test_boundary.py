"""The drop-in boundary on CPU: libqtree_cuda.so loads, exports exactly what
include/qtree_cuda.h declares, maps errors onto the reference taxonomy, and
has no CPU fallback (compute entries refuse to run without a device)."""
from __future__ import annotations

import ctypes as C
import math
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1101_3228_b200 import _lib, build
from paper_1101_3228_b200 import qtree as Q

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qtree_cuda.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.lib()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"QT_API\s+[\w\s\*]+?\b(qt_\w+)\s*\(", text)))


def test_header_declares_the_bound_api():
    assert declared_symbols() == _lib.EXPORTS


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (qt_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # nothing else leaks out of the C ABI
    assert exported == set(declared_symbols())


def test_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_version_and_counters(lib):
    assert b"sm_100a" in lib.qt_version()
    assert lib.qt_kernel_launches() >= 0


def test_chain_coefficients_follow_reference_formulas():
    ch = Q.BrownianChain1d(10, 1.0)
    assert ch.step_coef[0] == math.sqrt(1.0 / 10)
    assert ch.marg_coef[0] == 0.0 and ch.marg_coef[6 * 3] == math.sqrt(3 * (1.0 / 10))
    p = Q.TwoFactorParams()
    tf = Q.TwoFactorChain(p)
    dt = p.horizon / p.steps
    assert tf.step_coef[0] == math.exp(-p.alpha1 * dt)
    assert tf.step_coef[1] == math.exp(-p.alpha2 * dt)
    assert tf.step_coef[2] == math.sqrt(-math.expm1(-2.0 * p.alpha1 * dt) / (2.0 * p.alpha1))


def test_config_and_numeric_errors_map_to_reference_exceptions():
    with pytest.raises(Q.ConfigError):
        Q.TwoFactorChain(Q.TwoFactorParams(alpha1=-1.0))
    with pytest.raises(Q.ConfigError):
        Q.TwoFactorChain(Q.TwoFactorParams(rho=2.0))
    with pytest.raises(Q.NumericError):
        Q.BrownianChain1d(0)
    with pytest.raises(Q.NumericError):
        Q.QuantGrid(1, [])
    with pytest.raises(Q.NumericError):
        Q.QuantGrid(1, [np.nan])


def test_invalid_arguments_are_value_errors():
    ch = Q.BrownianChain1d(3)
    grids = [Q.QuantGrid(1, [0.0, 1.0])] * 3
    with pytest.raises(ValueError):
        Q.estimate_alg1(ch, grids[:2], 10)           # wrong grid count
    with pytest.raises(ValueError):
        Q.estimate_alg1(ch, [Q.QuantGrid(2, [0.0, 1.0])] * 3, 10)  # wrong dimension
    with pytest.raises(ValueError):
        Q.estimate_alg1(ch, grids, 0)                 # zero paths
    with pytest.raises(ValueError):
        Q.estimate_alg2(ch, grids, 10, Q.EstimateOptions(workers=0))
    with pytest.raises(ValueError):
        Q.estimate(7, ch, grids, 10)


def test_no_cpu_fallback_without_device():
    """On a box without a GPU every compute entry must fail loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    ch = Q.BrownianChain1d(3)
    grids = [Q.QuantGrid(1, [0.0, 1.0])] * 3
    with pytest.raises(Q.NumericError, match="cuda"):
        Q.estimate_alg1(ch, grids, 10)
    with pytest.raises(Q.NumericError, match="cuda"):
        Q.nearest(Q.QuantGrid(1, [0.0, 1.0]), [0.3])
    with pytest.raises(Q.NumericError, match="cuda"):
        Q.path_normals(1, 1, 4, 0, 2)
