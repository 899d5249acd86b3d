"""Where the one-call API's time goes (C2): phases from qt_estimate + wall clock.
    python tools/e2e_probe.py [M]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1101_3228_b200 import qtree as q

M = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
ch = q.BrownianChain1d(50)
grids = q.build_brownian_grids(ch, 500)
q.estimate(1, ch, grids, 10**6)  # warm-up (context, module load)
for r in range(3):
    ph = q.BuildPhases()
    t0 = time.perf_counter()
    t = q.estimate(1, ch, grids, M, q.EstimateOptions(phases=ph))
    dt = (time.perf_counter() - t0) * 1e3
    print(f"wall {dt:8.1f} ms  count {ph.nn_ms:8.1f}  merge {ph.merge_ms:6.2f}  "
          f"normalize {ph.normalize_ms:6.2f}  total(C) {ph.total_ms:8.1f}")
