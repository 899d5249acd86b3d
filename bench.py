#!/usr/bin/env python
"""bench.py -- MC path-transitions/s of the quantization-tree estimator on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5] [--paths M]

Default workload = BASELINE.json configs[1] (C2): 1-D Black-Scholes American
put, n = 50 layers, N = 500 points per layer, M = 1e9 paths (Algorithm II,
MRG32k3a seed 12345 on the reference's Lloyd grids), strong scaling: the same
1e9 paths are sharded over the N GPUs. One step = zero the joint counts, the
fused path kernel over this rank's paths, one NCCL reduce of the int64
counts to rank 0, visits + row normalisation on rank 0. Under torchrun each
rank drives one GPU; the time is the max over ranks of CUDA-event time.

value  = M n / step time (inputs resident in HBM).
e2e    = the same metric through the public API with host buffers (grids H2D,
         counts + pi D2H every step).
--impl reference times the reference's own CPU implementation (oracle/_ref,
the unmodified reference headers) on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MC path-transitions/sec (M*n) for QTree weights at 1/2/4/8 B200; price err"
UNIT = "transitions/s"

CONFIGS = {
    # name: (workload text, chain kind, n, N, M, estimator)
    "c1": ("C1: 1-D Black-Scholes American put, n=10, N=100, M=1e6 paths", "bm", 10, 100, 10**6, 1),
    "c2": ("C2: 1-D Black-Scholes American put, n=50, N=500, M=1e9 paths", "bm", 50, 500, 10**9, 1),
    "c3": ("C3: 1-D OU swing, Alg III pair sampling, n=365, N=200, M=1e7 per layer", "ou", 365, 200,
           10**7, 2),
    "c4": ("C4: 2-factor AR(1) gas swing, n=365, N=1000, M=1e7 paths", "tf", 365, 1000, 10**7, 1),
    "c5": ("C5: 3-D GBM max-call, n=20, N=4000, M=1e6 paths", "gbm", 20, 4000, 10**6, 1),
}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def profiled_traffic(config: str, transitions: int):
    """dram__bytes_read + dram__bytes_write of one path-kernel launch, scaled
    from the committed ncu --set full capture (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f).get(config)
        if d:
            return d["bytes_per_transition"] * transitions / 1e9  # GB per launch
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def crr_bermudan_put(s0, strike, r, sigma, horizon, exercise_dates, stride=200):
    """Independent CRR binomial value of the Bermudan put (price sanity check)."""
    steps = exercise_dates * stride
    dt = horizon / steps
    up = math.exp(sigma * math.sqrt(dt))
    down = 1.0 / up
    p = (math.exp(r * dt) - down) / (up - down)
    disc = math.exp(-r * dt)
    j = np.arange(steps + 1)
    s = s0 * up ** (2 * j - steps)
    v = np.maximum(strike - s, 0.0)
    for k in range(steps - 1, -1, -1):
        v = disc * (p * v[1:k + 2] + (1 - p) * v[:k + 1])
        if k % stride == 0:
            sk = s0 * up ** (2 * np.arange(k + 1) - k)
            v = np.maximum(v, strike - sk)
    return float(v[0])


def make_inputs(cfg):
    from paper_1101_3228_b200 import qtree as Q
    _, kind, n, N, M, est = CONFIGS[cfg]
    if kind == "bm":
        ch = Q.BrownianChain1d(n)
        grids = Q.build_brownian_grids(ch, N)
    elif kind == "ou":
        ch = Q.OuChain1d(Q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=n))
        grids = Q.build_ou_grids(ch, N)
    elif kind == "tf":
        ch = Q.TwoFactorChain(Q.TwoFactorParams(steps=n))
        grids = Q.build_two_factor_grids(ch, N)
    else:
        ch = Q.GbmChain3d(n)
        grids = Q.build_gbm_grids(ch, N)
    return ch, grids


def put_phi(tree, s0=100.0, strike=100.0, r=0.05, sigma=0.2):
    """make_put_payoff(cfg, 1) (pipeline.hpp:124-137) tabulated on the nodes."""
    n = tree.layers()
    dt = 1.0 / n
    out = []
    for k in range(n + 1):
        t = k * dt
        x = tree.grids[k].data()
        s = s0 * np.exp((r - 0.5 * sigma * sigma) * t + sigma * x)
        out.append(math.exp(-r * t) * np.maximum(strike - s, 0.0))
    return np.concatenate(out)


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation
# ---------------------------------------------------------------------------
def run_reference(args, rank):
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, ChainSpec, Oracle
    which = "reference" if os.path.exists(LIBS["reference"]) else "restatement"
    orc = Oracle(which)
    text, kind, n, N, M, est = CONFIGS[args.config]
    ch, grids = make_inputs(args.config)
    spec = {"bm": lambda: ChainSpec(0, n, sigma1=0.2, r=0.05),
            "ou": lambda: ChainSpec(2, n, sigma1=0.5, alpha1=1.0, sigma2=0.0),
            "tf": lambda: ChainSpec(1, n),
            "gbm": lambda: ChainSpec(3, n)}[kind]()
    sizes = np.array([1] + [g.size() for g in grids], np.uint64)
    pts = np.concatenate([g.data() for g in grids])
    cores = os.cpu_count() or 1
    # bounded sample: ~10-20 s of CPU work per step on this host
    per_core_rate = {"c1": 8e5, "c2": 6e5, "c3": 7e5, "c4": 1.4e5, "c5": 2.5e4}[args.config]
    units = max(1000, int(per_core_rate * cores * args.ref_seconds / n))
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        c = orc.estimate(est, spec, sizes, pts, units, engine=1, seed=12345, workers=cores)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
        assert int(c.joint.sum()) == units * n
    t = statistics.mean(times)
    val = units * n / t
    sample = f"{units} {'samples/layer' if est == 2 else 'paths'} of {text} (estimate_alg{est + 1}, {cores} threads)"
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64+u64",
            "data": "synthetic: MRG32k3a seed 12345 on the reference's Lloyd grids",
            "config": {"workload": text, "n": n, "N": N, "M": M, "sampled_units": units},
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores,
                             "kind": "reference" if which == "reference" else "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, seconds):
    """The reference CPU path timed on this host (rank 0, N = 1 only)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, ChainSpec, Oracle
    which = "reference" if os.path.exists(LIBS["reference"]) else "restatement"
    orc = Oracle(which)
    text, kind, n, N, M, est = CONFIGS[cfg]
    ch, grids = make_inputs(cfg)
    spec = {"bm": lambda: ChainSpec(0, n, sigma1=0.2, r=0.05),
            "ou": lambda: ChainSpec(2, n, sigma1=0.5, alpha1=1.0, sigma2=0.0),
            "tf": lambda: ChainSpec(1, n), "gbm": lambda: ChainSpec(3, n)}[kind]()
    sizes = np.array([1] + [g.size() for g in grids], np.uint64)
    pts = np.concatenate([g.data() for g in grids])
    cores = os.cpu_count() or 1
    per_core_rate = {"c1": 8e5, "c2": 6e5, "c3": 7e5, "c4": 1.4e5, "c5": 2.5e4}[cfg]
    units = max(1000, int(per_core_rate * cores * seconds / n))
    t0 = time.perf_counter()
    orc.estimate(est, spec, sizes, pts, units, engine=1, seed=12345, workers=cores)
    dt = time.perf_counter() - t0
    return {"value": units * n / dt, "unit": UNIT, "cores": cores,
            "kind": "reference" if which == "reference" else "port",
            "sample": f"{units} paths of {text} via estimate_alg{est + 1} with {cores} worker "
                      f"threads ({dt:.1f} s)"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1101_3228_b200 import build as B
    B.build()
    from paper_1101_3228_b200 import _lib
    from paper_1101_3228_b200 import qtree as Q
    from paper_1101_3228_b200.device import Plan
    from paper_1101_3228_b200.dist import estimate_distributed, shard

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    text, kind, n, N, M, est = CONFIGS[args.config]
    if args.paths:
        M = int(args.paths)
        text = f"{text} [--paths override: M={M:.3g}]"
    ch, grids = make_inputs(args.config)
    plan = Plan(ch, grids, local_rank)
    units = M * n if est == 2 else M
    first, count = shard(units, rank, world)
    st = torch.cuda.current_stream()
    joint = plan.zeros_joint()
    visits = torch.empty(plan.n_visits, dtype=torch.int64, device=dev)
    pi = torch.empty(plan.n_joint, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def one_step(ev):
        ev[0].record(st)
        joint.zero_()
        ev[1].record(st)
        plan.count(est, 1, 12345, first, count, units, joint)
        ev[2].record(st)
        if world > 1:  # the one exchange step: an all-reduce of the int64 counts
            dist.all_reduce(joint, op=dist.ReduceOp.SUM)
        if rank == 0:
            plan.finalize(est, M, joint, visits, pi)
        ev[3].record(st)

    for _ in range(args.warmup):
        one_step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
    torch.cuda.synchronize()
    launches0 = plan.launches
    sampler = ClockSampler(local_rank)
    sampler.start()
    step_ms, kern_ms = [], []
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed steps (256 MiB > 126 MB L2)
        torch.cuda.synchronize()
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        one_step(ev)
        torch.cuda.synchronize()
        barrier()
        step_ms.append(ev[0].elapsed_time(ev[3]))
        kern_ms.append(ev[1].elapsed_time(ev[2]))
    clocks = sampler.stop()
    my_launches = plan.launches - launches0
    t_step = statistics.mean(step_ms)
    t_kern = statistics.mean(kern_ms)
    if world > 1:
        tt = torch.tensor([t_step, t_kern], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_kern = float(tt[0]), float(tt[1])
        ln = torch.tensor([my_launches], dtype=torch.int64, device=dev)
        dist.all_reduce(ln, op=dist.ReduceOp.SUM)
        my_launches = int(ln[0])

    # correctness guard on the measured tree: conservation per transition
    ok = None
    price = None
    if rank == 0:
        j = joint.cpu().numpy().view(np.uint64)
        sizes = [int(s) for s in plan.sizes]
        off, ok = 0, True
        for k in range(1, len(sizes)):
            blk = j[off:off + sizes[k - 1] * sizes[k]]
            ok &= int(blk.sum()) == M
            off += sizes[k - 1] * sizes[k]
        if kind == "bm":
            tree = Q.QuantTree([Q.QuantGrid(1, [0.0])] + list(grids), plan.sizes,
                               visits.cpu().numpy().view(np.uint64), j, pi.cpu().numpy(), M)
            price = Q.solve_stopping(tree, put_phi(tree)).price

    # e2e through the public API with host buffers
    barrier()
    e2e_ms = []
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    d2h = (plan.n_visits + 2 * plan.n_joint) * 8
    h2d = int(sum(g.data().nbytes for g in grids) + plan.sizes.nbytes + ch.step_coef.nbytes +
              ch.marg_coef.nbytes)
    # one untimed full-size call: process-level one-time costs (pinned staging
    # buffers, module load, first use of the host copy threads)
    if world == 1:
        Q.estimate(est, ch, grids, M)
    else:
        estimate_distributed(est, ch, grids, M, plan=plan)
    for _ in range(e2e_steps):
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        if world == 1:
            res = Q.estimate(est, ch, grids, M)
        else:
            res = estimate_distributed(est, ch, grids, M, plan=plan)
        torch.cuda.synchronize()
        barrier()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        del res  # the caller's result buffers are released outside the timed call
        if os.environ.get("QT_DEBUG"):
            print(f"bench: e2e call {e2e_ms[-1]:.2f} ms", file=sys.stderr, flush=True)
    t_e2e = statistics.mean(e2e_ms)
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt[0])

    if rank != 0:
        return
    transitions = M * n
    value = transitions / (t_step / 1e3)
    peak, peak_src = measured_peaks()
    # algorithmic bytes of the path kernel: 16 B per transition (one u64 RMW)
    kern_units = count * n if est != 2 else count
    achieved = 16.0 * kern_units / (t_kern / 1e3) / 1e9
    kernel_name = {"bm": "k_paths_x (exact 1-D path kernel: MRG32k3a + FP64 Box-Muller + step + "
                         "threshold projection + RED count)",
                   "ou": "k_alg3_x (layer-parallel pair sampler)" if est == 2 else "k_paths_x",
                   "tf": "k_paths_scan (FP64 path + FP32 FFMA2 brute-force scan, exact decision)",
                   "gbm": "k_paths_scan (FP64 path + FP32 FFMA2 brute-force scan, exact decision)"}[kind]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64+u64",
        "data": "synthetic: MRG32k3a seed 12345 paths on the reference's Lloyd grids",
        "config": {"workload": text, "n": n, "N": N, "M": M,
                   "estimator": ["AlgI", "AlgII", "AlgIII"][est], "engine": "mrg32k3a",
                   "parallelism": f"paths sharded over {world} GPU(s), one NCCL all-reduce",
                   "l2": "flushed between timed steps (256 MiB write)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": profiled_traffic(args.config, kern_units),
                     "traffic_unit": "GB per launch (ncu dram read+write)",
                     "algorithmic_gb_per_launch": 16.0 * kern_units / 1e9,
                     "kernel": kernel_name,
                     "kernel_ms": t_kern, "peak_source": peak_src,
                     "algorithmic_bytes": "16 B per transition (u64 counter read-modify-write)",
                     "binding_unit": ("instruction issue (FP64 Box-Muller, MRG32k3a, exact projection; "
                                      "~60% issue-active) with the L1 data pipe (count REDs + "
                                      "shared loads) at ~75%; see DESIGN.md section 4")},
        "e2e": {"value": transitions / (t_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e, "steps": e2e_steps},
        "gpu_launches": int(my_launches),
        "clocks": clocks,
        "conservation_ok": bool(ok),
        "library": os.path.relpath(B.LIB, ROOT),
    }
    if price is not None:
        crr = crr_bermudan_put(100.0, 100.0, 0.05, 0.2, 1.0, n)
        line["price"] = {"put": price, "crr_bermudan": crr, "rel_err_vs_crr": abs(price - crr) / crr}
    if kind in ("tf", "gbm"):  # FP32-bound configs: 3 d N flop per transition
        fp32_peak = 72.24  # profiles/r01_peaks_fp.json (FFMA microbenchmark, this pool)
        flops = 3.0 * (2 if kind == "tf" else 3) * N * kern_units
        line["roofline_fp32"] = {"bound": "fp32", "achieved": flops / (t_kern / 1e3) / 1e12,
                                 "peak": fp32_peak, "unit": "TFLOP/s",
                                 "frac": flops / (t_kern / 1e3) / 1e12 / fp32_peak,
                                 "algorithmic_flops": "3 d N per transition (brute-force "
                                                      "convention, PAPER.md:540-543)",
                                 "peak_source": "profiles/r01_peaks_fp.json"}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, args.ref_seconds)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--paths", type=float, default=0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and os.environ.get("QT_BENCH_SHARE_GPU"):  # test hook: all ranks on one GPU
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("QT_BENCH_DIST_BACKEND", "nccl")  # gloo: test hook only
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
