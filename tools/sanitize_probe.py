"""Small estimates through every path kernel, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
    compute-sanitizer --tool racecheck python tools/sanitize_probe.py

Covers the default kernels (certified 1-D paths and Alg III + replays, the cell-list
d >= 2 search and its device-built index, the Alg III samplers), the
selectable alternatives (exact k_paths_x, the FP32 scan), the estimate ->
price path on the device tree, and the GPU Lloyd.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1101_3228_b200 import qtree as Q  # noqa: E402


def run_all():
    ch = Q.BrownianChain1d(10)
    g = Q.build_brownian_grids(ch, 100)                     # GPU Lloyd (k_serial_normals, ...)
    Q.estimate_alg2(ch, g, 20000)                           # 1-D path kernel (resident tables)
    ch50 = Q.BrownianChain1d(50)
    g50 = Q.build_brownian_grids(ch50, 500)
    Q.estimate_alg2(ch50, g50, 20000)                       # 1-D path kernel (staged), permute-add
    ou = Q.OuChain1d(Q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=12))
    go = Q.build_ou_grids(ou, 50)
    Q.estimate_alg3(ou, go, 4000)                           # k_alg3_x
    tf = Q.TwoFactorChain(Q.TwoFactorParams(steps=6))
    gt = Q.build_two_factor_grids(tf, 200)
    Q.estimate_alg2(tf, gt, 4000)                           # k_cell_count/fill + k_paths_cell
    Q.estimate_alg3(tf, gt, 2000)                           # k_alg3_cell
    gb = Q.GbmChain3d(3)
    gg = Q.build_gbm_grids(gb, 300)
    Q.estimate_alg2(gb, gg, 3000)                           # k_paths_cell, d = 3
    with Q.estimate_device(1, tf, gt, 4000) as dt:          # device tree + K5 in place
        Q.solve_swing(dt, Q.make_swing_payoff(Q.TwoFactorParams(steps=6), 2), 0, 3)
        Q.solve_stopping(dt, Q.make_put_payoff(Q.TwoFactorParams(steps=6), 2))


run_all()                                                   # certified k_paths_x / k_alg3_x + replays
Q.set_fast_path(1)
run_all()                                                   # FP32 k_paths_fast + k_replay
Q.set_fast_path(0)
os.environ["QT_NN"] = "scan"
run_all()                                                   # exact k_paths_x / k_alg3_x, FP32 scans
print("sanitize probe ok")
