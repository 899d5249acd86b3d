"""Diagnostic (GPU box): in-kernel Box-Muller normals vs the reference's
(glibc) normals for the same path substreams. Prints one JSON line per engine
with the bit-identical fraction and the ulp histogram.

    python tools/diag_normals.py [paths] [normals_per_path]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_1101_3228_b200 import qtree as Q  # noqa: E402
from pyoracle import Oracle  # noqa: E402


def main():
    paths = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200000
    npp = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    orc = Oracle("restatement")
    for e, name in enumerate(("lcg48", "mrg32k3a", "xorwow")):
        ref = orc.path_normals(e, 12345, npp, 777, paths, 10**9)
        got = Q.path_normals(e, 12345, npp, 777, paths)
        ulp = np.abs(got.view(np.int64) - ref.view(np.int64))
        hist = {str(k): int(np.sum(ulp == k)) for k in range(4)}
        hist[">3"] = int(np.sum(ulp > 3))
        print(json.dumps({"engine": name, "normals": int(ref.size),
                          "identical": float(np.mean(ulp == 0)), "max_ulp": int(ulp.max()),
                          "ulp_hist": hist}), flush=True)


if __name__ == "__main__":
    main()
