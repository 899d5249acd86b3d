"""Fast-path probe: C2 plan, time fast vs exact kernels, print replay stats.
    python tools/fast_probe.py [M] [reps]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1101_3228_b200 import qtree as q
from paper_1101_3228_b200.device import Plan

M = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ch = q.BrownianChain1d(50)
plan = Plan(ch, q.build_brownian_grids(ch, 500), 0)
joint = plan.zeros_joint()
configs = ((1, True), (2, True), (4, True), (2, False))
if len(sys.argv) > 3:
    configs = [(int(c[:-1]), c[-1] == "f") for c in sys.argv[3].split(",")]  # e.g. 2f,2x
for P, fast in configs:
    os.environ["QT_FAST_P"] = str(P)
    q.set_fast_path(fast)
    plan.count(1, 1, 12345, 0, M, 10**9, joint)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(reps):
        plan.count(1, 1, 12345, r * M, M, 10**9, joint)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"P={P} fast={fast}: {ms:.2f} ms per {M} paths -> {M * 50 / ms * 1e3:.3e} transitions/s")
q.set_fast_path(True)
print(plan.fast_stats())
