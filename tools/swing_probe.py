"""C4 swing pricing on the device: 2-factor tree (n = 365, N = 1000, M paths),
swing payoff, Q in [0, 100]; times solve_swing vs the reference's (oracle/_ref)
on the same tree when available. python tools/swing_probe.py [M]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
from paper_1101_3228_b200 import qtree as q
from pyoracle import CHAIN_TWO_FACTOR, PAYOFF_SWING, ChainSpec, Oracle, LIBS

M = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**6
tf = q.TwoFactorChain(q.TwoFactorParams())
g = q.build_two_factor_grids(tf, 1000)
t0 = time.perf_counter()
t = q.estimate_alg2(tf, g, M)
print(f"estimate M={M}: {time.perf_counter() - t0:.2f} s")
orc = Oracle("reference" if os.path.exists(LIBS["reference"]) else "restatement")
spec = ChainSpec(CHAIN_TWO_FACTOR, 365)
pts_all = np.concatenate([np.zeros(2)] + [x.data() for x in g])
phi = orc.payoff_table(spec, PAYOFF_SWING, t.sizes, pts_all)
for qmax in (10, 100):
    q.solve_swing(t, phi, 0, qmax)
    t0 = time.perf_counter()
    r = q.solve_swing(t, phi, 0, qmax)
    dt = time.perf_counter() - t0
    print(f"swing Q=[0,{qmax}]: price {r.price:.10g}, {dt*1e3:.1f} ms")
    if qmax == 10:
        t0 = time.perf_counter()
        rp = orc.solve_swing(t.sizes, t.flat_visits, t.flat_pi, phi, 0, qmax)
        print(f"  reference: price {rp:.10g}, {time.perf_counter() - t0:.2f} s, equal={rp == r.price}")
for rep in range(2):
    t0 = time.perf_counter()
    s = q.solve_stopping(t, phi)
    print(f"stopping (call {rep}): price {s.price:.10g}, {(time.perf_counter() - t0)*1e3:.1f} ms")
