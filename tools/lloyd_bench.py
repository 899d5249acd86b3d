"""GPU lloyd_build vs the reference's (oracle/_ref, 1 core; lloyd_build is serial)
on the grid builders' base quantizers. Prints one JSON line per case.
    python tools/lloyd_bench.py"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
from paper_1101_3228_b200 import qtree as q

cases = [(1, 500, 40), (2, 1000, 40), (3, 4000, 40)]
ref = None
try:
    from pyoracle import Oracle, LIBS
    if os.path.exists(LIBS["reference"]):
        ref = Oracle("reference")
except Exception:
    pass
for dim, N, iters in cases:
    spi = max(20000, 200 * N)
    q.lloyd_build(dim, N, 1, spi)  # warm-up
    t0 = time.perf_counter()
    res = q.lloyd_build(dim, N, iters, spi)
    gpu_s = time.perf_counter() - t0
    line = {"case": f"lloyd_build d={dim} N={N} iterations={iters} samples/iter={spi}",
            "gpu_s": gpu_s, "gpu_samples_per_s": iters * spi / gpu_s,
            "distortion_last": float(res.distortion[-1])}
    if ref is not None:
        it_ref = 1 if N >= 1000 else 2
        t0 = time.perf_counter()
        ref.lloyd_base(dim, N, 12345, spi, it_ref)
        ref_s = time.perf_counter() - t0
        line["reference_s_per_iteration"] = ref_s / it_ref
        line["reference_s_extrapolated"] = ref_s / it_ref * iters
        line["speedup"] = ref_s / it_ref * iters / gpu_s
    print(json.dumps(line), flush=True)
