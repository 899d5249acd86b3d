"""Exact 1-D kernels on C2: k_paths (QT_XKERNEL=0) vs k_paths_x at P = 1/2/4.
    python tools/x_probe.py [M] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1101_3228_b200 import qtree as q
from paper_1101_3228_b200.device import Plan

M = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N = int(sys.argv[3]) if len(sys.argv) > 3 else 500
ch = q.BrownianChain1d(50)
grids = q.build_brownian_grids(ch, N)
plan = Plan(ch, grids, 0)
print(f"n=50 N={N}: joint {plan.n_joint * 8 / 1e6:.1f} MB")
ref = None
cases = (("k_paths", {"QT_XKERNEL": "0"}), ("x P=1 L=1", {"QT_X_P": "1", "QT_X_L": "1"}),
         ("x P=2 L=1", {"QT_X_P": "2", "QT_X_L": "1"}), ("x P=2 L=2", {"QT_X_P": "2", "QT_X_L": "2"}),
         ("x P=2 L=2 S=3", {"QT_X_P": "2", "QT_X_L": "2", "QT_X_S": "3"}),
         ("x P=1 L=2", {"QT_X_P": "1", "QT_X_L": "2"}), ("x P=4 L=2", {"QT_X_P": "4", "QT_X_L": "2"}),
         ("fast P=4", {"QT_FAST_PATH": "1", "QT_FAST_P": "4"}),
         ("fast P=2", {"QT_FAST_PATH": "1", "QT_FAST_P": "2"}))
if os.environ.get("QT_PROBE_SHORT"):
    cases = (cases[0], cases[3], cases[-2], cases[-1])
for name, env in cases:
    for k in ("QT_XKERNEL", "QT_X_P", "QT_X_L", "QT_X_S", "QT_FAST_PATH", "QT_FAST_P"):
        os.environ.pop(k, None)
    os.environ.update(env)
    if "QT_FAST_PATH" in env:  # fast tables are built by plans created with the path on
        q.set_fast_path(True)
        plan = Plan(ch, grids, 0)
    joint = plan.zeros_joint()
    plan.count(1, 1, 12345, 0, M, 10**9, joint)
    torch.cuda.synchronize()
    j = joint.cpu().numpy().copy()
    same = ref is None or np.array_equal(j, ref)
    ref = j if ref is None else ref
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(reps):
        plan.count(1, 1, 12345, r * M, M, 10**9, joint)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: {ms:.2f} ms per {M} paths -> {M * 50 / ms * 1e3:.3e} transitions/s, same={same}")
