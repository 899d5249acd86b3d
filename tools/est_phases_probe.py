import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1101_3228_b200 import qtree as q
tf = q.TwoFactorChain(q.TwoFactorParams())
g = q.build_two_factor_grids(tf, 1000)
for rep in range(3):
    t0 = time.perf_counter()
    t = q.estimate_alg2(tf, g, 10**6)
    print(f"estimate call {rep}: {time.perf_counter() - t0:.2f} s", flush=True)
