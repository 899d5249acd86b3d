"""Paper tables 2-3 style micro-benchmarks on B200 vs the reference CPU code.
    python tools/microbench.py"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1101_3228_b200 import qtree as q
from pyoracle import Oracle, LIBS

ref = Oracle("reference") if os.path.exists(LIBS["reference"]) else None
for engine, name in ((0, "lcg48"), (1, "mrg32k3a"), (2, "xorwow")):
    for streams, skip in ((1, False), (148 * 256, name != "xorwow")):
        # one XORWOW stream cannot be split (no jump-ahead): keep that serial case small
        total = 10**8 if (name == "xorwow" and streams == 1) else 10**10
        samples = 2 * streams * (total // (2 * streams))
        q.bench_pi(engine, 12345, 2 * streams * 64, streams, skip)  # warm-up
        r = q.bench_pi(engine, 12345, samples, streams, skip)
        line = {"bench": "bench-rng", "engine": name, "mode": "skip" if skip else "block",
                "streams": streams, "samples": samples, "estimate": r.estimate,
                "gpu_ms": r.ms, "gpu_draws_per_s": samples / (r.ms / 1e3)}
        if ref is not None:
            small = 2 * streams * max(1, 2 * 10**7 // (2 * streams))
            t0 = time.perf_counter()
            ref.bench_pi(engine, 12345, small, streams, skip)
            dt = time.perf_counter() - t0
            line["ref_draws_per_s"] = small / dt
            line["ref_cores"] = os.cpu_count()
        print(json.dumps(line), flush=True)
for n in (100, 250, 500):
    Q = 36_500_000
    q.bench_nn(n, 1000)
    sink, ms = q.bench_nn(n, Q)
    line = {"bench": "bench-nn", "n": n, "queries": Q, "sink_mod7": sink % 7, "gpu_ms": ms,
            "gpu_queries_per_s": Q / (ms / 1e3)}
    if ref is not None:
        t0 = time.perf_counter()
        ref.bench_nn(n, 365_000, 12345)
        dt = time.perf_counter() - t0
        line["ref_queries_per_s"] = 365_000 / dt
    print(json.dumps(line), flush=True)
