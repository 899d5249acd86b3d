"""Phase timing of the one-call estimate (QT_DEBUG marks) for C1 / C2 shapes.

    QT_DEBUG=1 python tools/e2e_probe.py [c1|c2] [paths]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1101_3228_b200 import qtree as Q  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
n, N, M = {"c1": (10, 100, 10**6), "c2": (50, 500, 10**9)}[cfg]
if len(sys.argv) > 2:
    M = int(float(sys.argv[2]))
ch = Q.BrownianChain1d(n)
grids = Q.build_brownian_grids(ch, N)
for it in range(4):
    t0 = time.perf_counter()
    t = Q.estimate(1, ch, grids, M)
    print(f"call {it}: {(time.perf_counter() - t0) * 1e3:.2f} ms", file=sys.stderr, flush=True)
