import sys, time
sys.path.insert(0, ".")
import torch
from paper_1101_3228_b200 import qtree as q
from paper_1101_3228_b200.device import Plan
ch = q.GbmChain3d(20, 1.0, (0.0, 0.0, 0.0)); g = q.build_gbm_grids(ch, 4000)
plan = Plan(ch, g, 0)
joint = plan.zeros_joint()
for M in [1000, 10**5, 2 * 10**5, 5 * 10**5, 10**6]:
    for rep in range(2):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); plan.count(1, 1, 12345, 0, M, 4 * 10**9, joint); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(M, rep, "%.3f ms" % ms, "%.3g transitions/s" % (M * 20 / ms * 1e3), flush=True)
