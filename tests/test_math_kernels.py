"""The Box-Muller transcendental kernels of csrc/qt_math.h against glibc (what
the reference's box_muller calls, stream.hpp:57-62). The header is compiled
for the host with the same explicitly rounded operations the device uses, so
this measures the device's bits: <= 1 ulp everywhere on 2e7 MRG32k3a-shaped
inputs, and the bit-identical fractions the count parity relies on."""
from __future__ import annotations

import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_log_sincos_within_one_ulp_of_glibc(tmp_path):
    exe = tmp_path / "check_math"
    subprocess.run(["g++", "-O2", "-mfma", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(ROOT, "tests", "tools", "check_math.cpp"), "-lm"], check=True)
    out = subprocess.run([str(exe), "20000000"], capture_output=True, text=True, timeout=300)
    r = json.loads(out.stdout)
    assert out.returncode == 0, r
    assert r["log_max_ulp"] <= 1 and r["sin_max_ulp"] <= 1 and r["cos_max_ulp"] <= 1, r
    assert r["log_identical"] > 0.995, r
    assert r["sin_identical"] > 0.95 and r["cos_identical"] > 0.95, r
