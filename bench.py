#!/usr/bin/env python
"""bench.py -- MC path-transitions/s of the quantization-tree estimator on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5] [--paths M]

Default workload = BASELINE.json configs[1] (C2): 1-D Black-Scholes American
put, n = 50 layers, N = 500 points per layer, M = 1e9 paths (Algorithm II,
MRG32k3a seed 12345 on the Lloyd grids, built on the GPU bit-identical to the
reference's), strong scaling: the same 1e9 paths are sharded over the N GPUs.
One step = zero the joint counts, the fused path kernel(s) over this rank's
paths, one NCCL all-reduce of the int64 counts, visits + row normalisation on
rank 0. Under torchrun each rank drives one GPU; the time is the max over
ranks of CUDA-event time.

value  = M n / step time (inputs resident in HBM).
e2e    = the same metric through the public API (qtree.estimate) with host
         buffers, COLD: the library's plan cache is cleared before each call,
         so every call builds + uploads the tables (grids H2D) and copies the
         counts and pi back (D2H). e2e_warm: the same call repeated on cached
         inputs. price: estimate_device + the config's BDP on the device.
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
    # C3 / C4: BASELINE gives no M; SURVEY.md 8(d) proposes 1e8 (per layer) on the GPU.
    # C5: BASELINE's M = 4e9 (8e10 transitions, ~6 s per step on one B200).
    "c3": ("C3: 1-D OU swing, Alg III pair sampling, n=365, N=200, M=1e8 per layer", "ou", 365, 200,
           10**8, 2),
    "c4": ("C4: 2-factor AR(1) gas swing, n=365, N=1000, M=1e8 paths", "tf", 365, 1000, 10**8, 1),
    "c5": ("C5: 3-D GBM max-call, n=20, N=4000, M=4e9 paths", "gbm", 20, 4000, 4 * 10**9, 1),
}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp32_peak_tflops():
    """Non-tensor FP32 peak: MEASURED_PEAKS.json when it carries one, else the
    FFMA microbenchmark committed under profiles/ (tools/peaks_fp.cu, this pool)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        if "fp32_tflops" in d:
            return float(d["fp32_tflops"]), "MEASURED_PEAKS.json"
    with open(os.path.join(ROOT, "profiles", "r01_peaks_fp.json")) as f:
        return float(json.load(f)["fp32_tflops"]), "profiles/r01_peaks_fp.json (tools/peaks_fp.cu)"


def price_problem(Q, cfg):
    """The BDP problem of each config: payoff factory and
    swing window (None: American stopping)."""
    if cfg in ("c1", "c2"):
        p = Q.TwoFactorParams(steps=CONFIGS[cfg][2], sigma1=0.2, r=0.05)
        return Q.make_put_payoff(p, 1), None
    if cfg == "c3":
        p = Q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=365)
        return Q.make_ou_swing_payoff(p), (0, 100)
    if cfg == "c4":
        return Q.make_swing_payoff(Q.TwoFactorParams(steps=365), 2), (0, 100)
    return Q.make_max_call_payoff(Q.TwoFactorParams(steps=20, r=0.05)), None


def reference_price(cfg, M):
    """The reference's own price for this config at this M, when a committed
    golden holds it (tests/golden: c2_full.npz at M = 1e9, configs.npz C1)."""
    g = os.path.join(ROOT, "tests", "golden")
    try:
        if cfg == "c2" and os.path.exists(os.path.join(g, "c2_full.npz")):
            with np.load(os.path.join(g, "c2_full.npz")) as z:
                if int(z["M"]) == M:
                    return float(z["put_price"])
        if cfg == "c1" and M == 10**6:
            with np.load(os.path.join(g, "configs.npz")) as z:
                return float(z["c1_put_price"])
        if cfg in ("c3", "c4", "c5"):
            with np.load(os.path.join(g, "prices.npz")) as z:
                if int(z[f"{cfg}_M"]) == M:
                    return float(z[f"{cfg}_price"])
    except (OSError, KeyError):
        return None
    return None


def golden_price_m(cfg):
    """M of the reference's committed price for a config (tests/golden), or None."""
    g = os.path.join(ROOT, "tests", "golden", "prices.npz")
    if cfg in ("c3", "c4", "c5") and os.path.exists(g):
        with np.load(g) as z:
            if f"{cfg}_M" in z.files:
                return int(z[f"{cfg}_M"])
    return None


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
        t0 = time.perf_counter()  # nvidia-smi takes a while to start: sample from the first step
        while not self.lines and time.perf_counter() - t0 < 3.0:
            time.sleep(0.01)

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


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation
# ---------------------------------------------------------------------------
def _ref_spec(kind, n):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import ChainSpec
    return {"bm": lambda: ChainSpec(0, n, sigma1=0.2, r=0.05),
            "ou": lambda: ChainSpec(2, n, sigma1=0.5, alpha1=1.0, sigma2=0.0),
            "tf": lambda: ChainSpec(1, n), "gbm": lambda: ChainSpec(3, n, r=0.05)}[kind]()


# bounded CPU sample per step: ~seconds x cores x this rate / n units
REF_RATE = {"c1": 8e5, "c2": 6e5, "c3": 7e5, "c4": 1.4e5, "c5": 2.5e4}


def run_reference(args, rank):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference headers) on this host's cores, end to end through its own
    code: grids from its build_*_grids (pipeline.hpp:27-77), counts from
    estimate_alg2 / estimate_alg3 with workers = all host threads. Nothing of
    the product is imported or loaded here."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, Oracle
    which = "reference" if os.path.exists(LIBS["reference"]) else "restatement"
    orc = Oracle(which)
    text, kind, n, N, M, est = CONFIGS[args.config]
    spec = _ref_spec(kind, n)
    t0 = time.perf_counter()
    pts = orc.build_grids(spec, N)  # the reference's own Lloyd grids
    grid_s = time.perf_counter() - t0
    sizes = np.array([1] + [N] * n, np.uint64)
    cores = os.cpu_count() or 1
    units = max(1000, int(REF_RATE[args.config] * cores * args.ref_seconds / n))
    units = min(units, M)
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
    what = "samples/layer" if est == 2 else "paths"
    sample = (f"{units} {what} of {text} per step (estimate_alg{est + 1}, {cores} threads); "
              f"the rate is the metric's (transitions/s), measured on that sample")
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64+u64",
            "data": "synthetic: MRG32k3a seed 12345 on the reference's own Lloyd grids",
            "config": {"workload": text, "n": n, "N": N, "M": M, "sampled_units": units,
                       "extrapolated": units < M,
                       "note": "each step estimates a bounded sample of the workload's units; "
                               "the rate (units x n / time) is what is compared"},
            "impl": "reference",
            "reference_grid_build_s": grid_s,
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores,
                             "kind": "reference" if which == "reference" else "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, seconds, grids):
    """The reference CPU path timed on this host (rank 0, N = 1 only), on the
    same grids as the GPU arm (bit-identical to the reference's own)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, Oracle
    which = "reference" if os.path.exists(LIBS["reference"]) else "restatement"
    orc = Oracle(which)
    text, kind, n, N, M, est = CONFIGS[cfg]
    spec = _ref_spec(kind, n)
    sizes = np.array([1] + [g.size() for g in grids], np.uint64)
    pts = np.concatenate([g.data() for g in grids])
    cores = os.cpu_count() or 1
    units = min(M, max(1000, int(REF_RATE[cfg] * cores * seconds / n)))
    t0 = time.perf_counter()
    orc.estimate(est, spec, sizes, pts, units, engine=1, seed=12345, workers=cores)
    dt = time.perf_counter() - t0
    return {"value": units * n / dt, "unit": UNIT, "cores": cores,
            "kind": "reference" if which == "reference" else "port",
            "sample": f"{units} {'samples/layer' if est == 2 else 'paths'} of {text} via "
                      f"estimate_alg{est + 1} with {cores} worker threads ({dt:.1f} s)"}


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

    reps = 1  # passes of the whole workload per step (short configs only, below)

    def one_step(ev):
        ev[0].record(st)
        joint.zero_()
        ev[1].record(st)
        for _ in range(reps):
            plan.count(est, 1, 12345, first, count, units, joint)
        ev[2].record(st)
        if world > 1:  # the one exchange step: an all-reduce of the int64 counts
            dist.all_reduce(joint, op=dist.ReduceOp.SUM)
        if rank == 0:
            plan.finalize(est, M * reps, joint, visits, pi)
        ev[3].record(st)

    for w in range(args.warmup):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        one_step(ev)
        torch.cuda.synchronize()
        if w == args.warmup - 2 and args.min_step_ms > 0:
            # a workload much shorter than the clock sampler's 200 ms period is
            # repeated within a step (same units, counts accumulate, value
            # counts every pass) so the timed region carries clock evidence;
            # calibrated on a warm step, the last warm-up step runs with it
            t1 = torch.tensor([ev[1].elapsed_time(ev[2])], dtype=torch.float64, device=dev)  # one pass
            if world > 1:
                dist.all_reduce(t1, op=dist.ReduceOp.MAX)
            reps = max(1, math.ceil(args.min_step_ms / max(float(t1[0]), 1e-3)))
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
    if rank == 0:
        j = joint.cpu().numpy().view(np.uint64)
        sizes = [int(s) for s in plan.sizes]
        off, ok = 0, True
        for k in range(1, len(sizes)):
            blk = j[off:off + sizes[k - 1] * sizes[k]]
            ok &= int(blk.sum()) == M * reps
            off += sizes[k - 1] * sizes[k]

    # e2e through the public API with host buffers. COLD: the library's plan
    # cache is cleared before every timed call, so each call builds the device
    # tables, uploads the grids, allocates, counts, finalizes and copies the
    # counts and pi back (exactly the bytes declared below). WARM (reported
    # beside it): a repeated call on the same inputs reuses the cached plan.
    barrier()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    d2h = (plan.n_visits + 2 * plan.n_joint) * 8
    h2d = int(sum(g.data().nbytes for g in grids) + plan.sizes.nbytes + ch.step_coef.nbytes +
              ch.marg_coef.nbytes)

    def e2e_call():
        if world == 1:
            return Q.estimate(est, ch, grids, M)
        return estimate_distributed(est, ch, grids, M, plan=plan)

    e2e_call()  # process-level one-time costs (pinned staging buffers, host copy threads)

    def timed(cold):
        out = []
        for _ in range(e2e_steps):
            if cold:
                Q.plan_cache_clear()
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            res = e2e_call()
            torch.cuda.synchronize()
            barrier()
            out.append((time.perf_counter() - t0) * 1e3)
            del res  # the caller's result buffers are released outside the timed call
        t = statistics.mean(out)
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt[0])
        return t

    t_e2e = timed(cold=True)
    t_e2e_warm = timed(cold=False)

    # estimate -> price on the device (estimate_device + solve_* in place, no pi
    # round trip): the reference's run_pipeline (pipeline.hpp:190-215)
    price_line = None
    if world == 1:
        payoff, q = price_problem(Q, args.config)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with Q.estimate_device(est, ch, grids, M) as dtree:
            t1 = time.perf_counter()
            res = (Q.solve_swing(dtree, payoff, q[0], q[1]) if q
                   else Q.solve_stopping(dtree, payoff))
        t2 = time.perf_counter()
        price_line = {"problem": (f"swing Q in [{q[0]}, {q[1]}]" if q else "American stopping"),
                      "price": res.price, "estimate_s": t1 - t0, "bdp_s": t2 - t1,
                      "estimate_and_price_s": t2 - t0,
                      "path": "estimate_device + solve_* on the device tree (no pi round trip)"}
        ref = reference_price(args.config, M)
        if ref is not None:
            price_line["reference_price"] = ref
            price_line["rel_err_vs_reference"] = abs(res.price - ref) / abs(ref)
        mg = golden_price_m(args.config)
        if ref is None and mg is not None:
            # the config's M has no reference price (the CPU reference would take
            # hours): price the same chain and grids at the golden's M instead,
            # against the reference's own price there
            with Q.estimate_device(est, ch, grids, mg) as dtree:
                rg = (Q.solve_swing(dtree, payoff, q[0], q[1]) if q
                      else Q.solve_stopping(dtree, payoff))
            refg = reference_price(args.config, mg)
            price_line["parity_at_golden_M"] = {
                "M": mg, "price": rg.price, "reference_price": refg,
                "rel_err_vs_reference": abs(rg.price - refg) / abs(refg)}
        if kind == "bm":
            crr = crr_bermudan_put(100.0, 100.0, 0.05, 0.2, 1.0, n)
            price_line["crr_bermudan"] = crr
            price_line["rel_err_vs_crr"] = abs(res.price - crr) / crr

    if rank != 0:
        return
    transitions = M * n
    value = reps * transitions / (t_step / 1e3)
    peak, peak_src = measured_peaks()
    # algorithmic bytes of the path kernel: 16 B per transition (one u64 RMW)
    kern_units = reps * (count * n if est != 2 else count)  # every pass of the timed kernel
    achieved = 16.0 * kern_units / (t_kern / 1e3) / 1e9
    kernel_name = {"bm": "k_paths_x<CERT> + k_replay (certified 1-D path: MRG32k3a, approximate "
                         "FP64 Box-Muller within an exhaustively verified bound of glibc's, "
                         "state error bound, FP64 threshold-pair certificate, sorted-cell RED; "
                         "uncertified paths (~0) replayed with the glibc-exact arithmetic) + "
                         "k_permute_add",
                   "ou": "k_alg3_x (layer-parallel pair sampler)" if est == 2 else "k_paths_x",
                   "tf": "k_paths_cell (FP64 path + exact cell-list nearest-point search: "
                         "FP64 reference d2 over the bucket's candidate list)",
                   "gbm": "k_paths_cell (FP64 path + exact cell-list nearest-point search: "
                          "FP64 reference d2 over the bucket's candidate list)"}[kind]
    if kind in ("tf", "gbm") and os.environ.get("QT_NN") == "scan":
        kernel_name = "k_paths_scan (FP64 path + FP32 FFMA2 brute-force scan, exact decision)"
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
                     "traffic_unit": ("GB per launch (ncu dram read+write)" if reps == 1 else
                                      f"GB per step of {reps} launches (ncu dram read+write)"),
                     "algorithmic_gb_per_launch": 16.0 * kern_units / 1e9,
                     "kernel": kernel_name,
                     "kernel_ms": t_kern, "peak_source": peak_src,
                     "algorithmic_bytes": "16 B per transition (u64 counter read-modify-write)",
                     "binding_unit": (
                         "d = 1: instruction issue (see roofline_issue; 1.565e11/s with the count "
                         "REDs removed) with the count scatter's L2 atomic ceiling close behind "
                         "(one 64-bit RED per transition; tools/red_probe.cu measures 1.3-1.9e11 "
                         "REDs/s on this B200 for such patterns, profiles/r02_red_probe_*.txt)"
                         if kind in ("bm", "ou")
                         else "d >= 2: load latency of the candidate-list gathers (ncu: "
                              "long-scoreboard stalls ~58 %, profiles/r02_ncu_kernels.md)") +
                         "; see DESIGN.md section 4"},
        "e2e": {"value": transitions / (t_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e, "steps": e2e_steps,
                "plan": "cold: plan cache cleared before every call (tables built + uploaded)"},
        "e2e_warm": {"value": transitions / (t_e2e_warm / 1e3), "unit": UNIT,
                     "ms_per_step": t_e2e_warm,
                     "plan": "warm: repeated call on the same inputs (cached device plan; "
                             "counts / pi still copied back)"},
        "gpu_launches": int(my_launches),
        "clocks": clocks,
        "conservation_ok": bool(ok),
        "library": os.path.relpath(B.LIB, ROOT),
    }
    if kind in ("bm", "ou") and est != 2:
        # the kernel's own bound: instruction issue. Warp
        # instructions per transition from the committed ncu capture of this kernel
        # (profiles/r02_ncu_kernels.md section 0, r02bj_cert: 4.71); ceiling = SMs x 4
        # schedulers x the measured SM clock / that count.
        wipt = 4.71
        sm_mhz = (clocks.get("sm_mhz") or 1965.0) if isinstance(clocks, dict) else 1965.0
        ceil = torch.cuda.get_device_properties(dev).multi_processor_count * 4 * sm_mhz * 1e6 / wipt
        kern_rate = kern_units / (t_kern / 1e3)
        line["roofline_issue"] = {"bound": "issue", "achieved": kern_rate, "peak": ceil,
                                  "unit": "transitions/s", "frac": kern_rate / ceil,
                                  "warp_instructions_per_transition": wipt,
                                  "source": "profiles/r02_ncu_kernels.md (ncu r02bj_cert)"}
    if world > 1:
        line["comm"] = {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                        "collective": "all_reduce(int64 joint counts, SUM), once per step"}
    if reps > 1:
        line["config"]["passes_per_step"] = reps
        line["config"]["note"] = ("the workload runs `passes_per_step` times per timed step (counts "
                                  "accumulate) so the step outlasts the 200 ms clock sampler")
    if price_line is not None:
        line["price"] = price_line
    if kind in ("tf", "gbm"):
        # SURVEY 8(d) models d >= 2 as the brute-force scan, FP32-bound at 3 d N flop per
        # transition. The default projection (cell lists) evaluates ~10-40 points, not N:
        # this line states the brute-force-equivalent rate against that FP32 bound (a frac
        # above 1 is work the cell lists do not need to do); the FP32 scan itself
        # (QT_NN=scan) is measured against it in profiles/.
        fp32_peak, fp32_src = fp32_peak_tflops()
        flops = 3.0 * (2 if kind == "tf" else 3) * N * kern_units
        line["roofline_fp32"] = {"bound": "fp32", "achieved": flops / (t_kern / 1e3) / 1e12,
                                 "peak": fp32_peak, "unit": "TFLOP/s",
                                 "frac": flops / (t_kern / 1e3) / 1e12 / fp32_peak,
                                 "algorithmic_flops": "3 d N per transition (brute-force "
                                                      "convention, PAPER.md:540-543)",
                                 "meaning": ("brute-force-equivalent rate of the cell-list "
                                             "search" if os.environ.get("QT_NN") != "scan"
                                             else "FP32 scan"),
                                 "peak_source": fp32_src}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, args.ref_seconds, grids)
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
    ap.add_argument("--min-step-ms", type=float, default=500.0,
                    help="repeat a shorter workload within each step up to this length")
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
            # the communicator's init lines (rank count, NVLS / ring choice) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
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
