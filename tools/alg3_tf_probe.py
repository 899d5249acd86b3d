"""Alg III on the C4 shape (2-factor, n = 365, N = 1000): k_alg3_scan vs the FP64 k_alg3."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1101_3228_b200 import qtree as q
from paper_1101_3228_b200.device import Plan
tf = q.TwoFactorChain(q.TwoFactorParams())
g = q.build_two_factor_grids(tf, 1000)
M = 200000
units = M * 365
for scan in ("1", "0"):
    os.environ["QT_SCAN"] = scan
    plan = Plan(tf, g, 0)
    joint = plan.zeros_joint()
    plan.count(2, 1, 12345, 0, units, units, joint); torch.cuda.synchronize()
    t0 = time.perf_counter(); plan.count(2, 1, 12345, 0, units, units, joint); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"C4 shape Alg III scan={scan}: {units/dt:.3e} samples/s ({dt*1e3:.1f} ms)")
