"""Exhaustive proof that the device's FMA-corrected constant division in
mrg_to_unit (csrc/qt_device.cuh) equals the reference's IEEE quotient
(x + 1) / (m1 + 1) (rng/mrg32k3a.hpp:62) for all 2^32 - 209 numerators."""
from __future__ import annotations

import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fma_division_is_exact_for_every_numerator(tmp_path):
    exe = tmp_path / "check_division"
    subprocess.run(["gcc", "-O2", "-mfma", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(ROOT, "tests", "tools", "check_division.c"), "-lm", "-lpthread"],
                   check=True)
    out = subprocess.run([str(exe), str(os.cpu_count() or 4)], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and out.stdout.strip() == "0", out.stdout + out.stderr
