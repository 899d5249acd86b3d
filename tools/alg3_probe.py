"""C3 (OU, Alg III, n = 365, N = 200): k_alg3 (QT_XKERNEL=0) vs k_alg3_x P = 1/2/4.
    python tools/alg3_probe.py [M per layer]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1101_3228_b200 import qtree as q
from paper_1101_3228_b200.device import Plan

M = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**7
p = q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=365)
ch = q.OuChain1d(p)
plan = Plan(ch, q.build_ou_grids(ch, 200), 0)
units = M * 365
ref = None
for name, env in (("k_alg3", {"QT_XKERNEL": "0"}), ("x P=1", {"QT_X_P": "1"}),
                  ("x P=2", {"QT_X_P": "2"}), ("x P=4", {"QT_X_P": "4"})):
    for k in ("QT_XKERNEL", "QT_X_P"):
        os.environ.pop(k, None)
    os.environ.update(env)
    joint = plan.zeros_joint()
    plan.count(2, 1, 12345, 0, units, units, joint)
    torch.cuda.synchronize()
    j = joint.cpu().numpy().copy()
    same = ref is None or np.array_equal(j, ref)
    ref = j if ref is None else ref
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(3):
        plan.count(2, 1, 12345, 0, units, units, joint)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: {ms:.2f} ms -> {units / ms * 1e3:.3e} samples/s, same={same}")
