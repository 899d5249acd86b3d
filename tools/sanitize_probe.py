"""Small estimates through every path kernel, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
    compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1101_3228_b200 import qtree as Q  # noqa: E402

ch = Q.BrownianChain1d(10)
g = Q.build_brownian_grids(ch, 100)
t = Q.estimate_alg2(ch, g, 20000)                       # k_paths_x (resident tables)
ch50 = Q.BrownianChain1d(50)
g50 = Q.build_brownian_grids(ch50, 500)
t = Q.estimate_alg2(ch50, g50, 20000)                   # k_paths_x (staged two-layer ring)
ou = Q.OuChain1d(Q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=12))
go = Q.build_ou_grids(ou, 50)
t = Q.estimate_alg3(ou, go, 4000)                       # k_alg3_x
tf = Q.TwoFactorChain(Q.TwoFactorParams(steps=6))
gt = Q.build_two_factor_grids(tf, 200)
t = Q.estimate_alg2(tf, gt, 4000)                       # k_paths_scan
t = Q.estimate_alg3(tf, gt, 2000)                       # k_alg3_scan
print("sanitize probe ok")
