"""Generate tests/golden/glibc_checksums.json: glibc's Box-Muller log / sin / cos
over the two exhaustive engine domains, as the order-independent checksums
qt_math_checksum computes on the device (csrc/qt_kernels.cu k_math_checksum).

Runs tests/tools/check_math.cpp's `checksum` mode against THIS container's
libm (glibc 2.39-0ubuntu8.5, the one the reference oracle links; the GPU box
runs the same image). About 3 minutes on 8 cores.

    python tests/golden/make_glibc_checksums.py
"""
from __future__ import annotations

import json
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "tests", "golden", "glibc_checksums.json")


def main() -> None:
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "check_math")
        subprocess.run(["g++", "-O2", "-std=c++17", "-fno-builtin", "-ffp-contract=off",
                        "-pthread", "-o", exe,
                        os.path.join(ROOT, "tests", "tools", "check_math.cpp"), "-lm"], check=True)
        out = subprocess.run([exe, "checksum"], capture_output=True, text=True, check=True)
    r = json.loads(out.stdout)
    bid = subprocess.run(["readelf", "-n", "/lib/x86_64-linux-gnu/libm.so.6"],
                         capture_output=True, text=True).stdout
    r["libm_build_id"] = next((ln.split(":")[1].strip() for ln in bid.splitlines()
                               if "Build ID" in ln), "unknown")
    r["order"] = ["log(u)", "sin(2 pi u)", "cos(2 pi u)"]
    with open(OUT, "w") as f:
        json.dump(r, f, indent=1)
    print(json.dumps(r))


if __name__ == "__main__":
    main()
