import sys, time
sys.path.insert(0, ".")
import torch
from paper_1101_3228_b200 import qtree as q
from paper_1101_3228_b200.device import Plan
ch = q.BrownianChain1d(50); g = q.build_brownian_grids(ch, 500)
M = 10**9
plan = Plan(ch, g, 0)
joint = plan.zeros_joint()
for i in range(3):
    joint.zero_(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); plan.count(1, 1, 12345, 0, M, M, joint); e1.record(); torch.cuda.synchronize()
    print("plan.count", e0.elapsed_time(e1), flush=True)
q.estimate_alg2(ch, g, M)
for i in range(2):
    t = time.perf_counter(); r = q.estimate_alg2(ch, g, M); print("one-call", time.perf_counter() - t, flush=True)
