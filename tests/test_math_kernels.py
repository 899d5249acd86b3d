"""The Box-Muller transcendentals of csrc/qt_math.h against the live glibc the
reference's box_muller calls (stream.hpp:57-62: log, and the sincos g++ fuses
cos/sin into). The header is compiled for the host with the same explicitly
rounded operations the device uses, so this checks the device's bits.

Bar: 0 mismatches. Here (CPU suite): every 61st MRG32k3a and XORWOW uniform
(7e7 each) plus 2e7 LCG48 uniforms and the 2^21 LCG48 edge states. The full
domains (2^32 - 209 MRG32k3a and 2^32 XORWOW inputs, 0 mismatches) were run by
`check_math all` (profiles/r02_check_math_exhaustive.json), and the GPU suite
checks the device build over them through tests/golden/glibc_checksums.json."""
from __future__ import annotations

import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_check_math(tmp_path) -> str:
    exe = str(tmp_path / "check_math")
    subprocess.run(["g++", "-O2", "-std=c++17", "-fno-builtin", "-ffp-contract=off", "-pthread",
                    "-o", exe, os.path.join(ROOT, "tests", "tools", "check_math.cpp"), "-lm"],
                   check=True)
    return exe


def test_log_sincos_bit_identical_to_glibc(tmp_path):
    exe = build_check_math(tmp_path)
    out = subprocess.run([exe, "all", "20000000", str(os.cpu_count() or 4), "61"],
                         capture_output=True, text=True, timeout=900)
    r = json.loads(out.stdout)
    for dom in ("mrg32k3a", "xorwow", "lcg48"):
        d = r[dom]
        assert d["inputs"] > 2 * 10**7, d
        assert d["log_mismatch"] == 0 and d["sin_mismatch"] == 0 and d["cos_mismatch"] == 0, (dom, d)
    assert out.returncode == 0


def test_glibc_checksum_fixture_shape():
    with open(os.path.join(ROOT, "tests", "golden", "glibc_checksums.json")) as f:
        g = json.load(f)
    assert set(g) >= {"mrg32k3a", "xorwow", "libm_build_id"}
    assert len(g["mrg32k3a"]) == 3 and len(g["xorwow"]) == 3
