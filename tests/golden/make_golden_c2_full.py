"""Generate tests/golden/c2_full.npz: config 2 at its FULL size, by the REFERENCE.

Config 2 (BASELINE.json configs[1]): BrownianChain1d n = 50, N = 500 (grids from
the reference's build_brownian_grids(chain, 500, 12345), pipeline.hpp:27-53),
M = 1e9 paths, MRG32k3a, seed 12345. The counts are the reference's own
detail::accumulate_paths (estimate.hpp:88-126, through oracle/_ref) summed over
path windows; path m's stream does not depend on the partition
(stream.hpp:190-199), so the sum over windows IS the Alg I / Alg II tree
(test_tree.cpp:128-152). The American put is priced with the reference's own
make_put_payoff + solve_stopping (pipeline.hpp:124-150, bdp.hpp:58-96).

About 3 h on 8 cores. Resumable: each worker thread keeps a running sum of its
windows in WORK/ (git- and gpurun-ignored) and a done-count, so an interrupted
run restarts where it stopped.

    python tests/golden/make_golden_c2_full.py [--workers 8] [--window 5000000]

Writes tests/golden/c2_full.npz: sha256 of joint / visits / pi (the reference's
row-major layouts), the full visits vector, the put price, and the run shape.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import CHAIN_BROWNIAN1D, PAYOFF_PUT, ChainSpec, Oracle  # noqa: E402

WORK = os.path.join(ROOT, ".golden_work", "c2_full")
OUT = os.path.join(ROOT, "tests", "golden", "c2_full.npz")
M = 10**9
SEED = 12345


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--window", type=int, default=5_000_000)
    args = ap.parse_args()
    os.makedirs(WORK, exist_ok=True)
    R = Oracle("reference")
    chain = ChainSpec(CHAIN_BROWNIAN1D, 50, sigma1=0.2, r=0.05)
    gpath = os.path.join(WORK, "grids.npy")
    if os.path.exists(gpath):
        grids = np.load(gpath)
    else:
        grids = R.build_grids(chain, 500)
        np.save(gpath, grids)
    sizes = np.array([1] + [500] * 50, np.uint64)
    W, win = args.workers, args.window
    nwin = (M + win - 1) // win
    t0 = time.time()
    lock = threading.Lock()

    def worker(w: int) -> None:
        state = os.path.join(WORK, f"w{w}_of{W}_win{win}.json")
        vfile = os.path.join(WORK, f"w{w}_of{W}_win{win}_visits.npy")
        jfile = os.path.join(WORK, f"w{w}_of{W}_win{win}_joint.npy")
        done = 0
        vis = jnt = None
        if os.path.exists(state):
            done = json.load(open(state))["done"]
            vis, jnt = np.load(vfile), np.load(jfile)
        mine = list(range(w, nwin, W))
        for idx in mine[done:]:
            first = idx * win
            cnt = min(win, M - first)
            v, j = R.accumulate_paths(chain, sizes, grids, 1, SEED, first, cnt, M)
            if vis is None:
                vis, jnt = v, j
            else:
                vis += v
                jnt += j
            done += 1
            np.save(vfile + ".tmp.npy", vis)
            np.save(jfile + ".tmp.npy", jnt)
            os.replace(vfile + ".tmp.npy", vfile)
            os.replace(jfile + ".tmp.npy", jfile)
            with open(state + ".tmp", "w") as f:
                json.dump({"done": done}, f)
            os.replace(state + ".tmp", state)
            with lock:
                print(f"[{time.time() - t0:8.0f}s] worker {w}: window {idx} ({done}/{len(mine)})",
                      flush=True)

    th = [threading.Thread(target=worker, args=(w,)) for w in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join()

    visits = joint = None
    for w in range(W):
        v = np.load(os.path.join(WORK, f"w{w}_of{W}_win{win}_visits.npy"))
        j = np.load(os.path.join(WORK, f"w{w}_of{W}_win{win}_joint.npy"))
        visits = v if visits is None else visits + v
        joint = j if joint is None else joint + j
    assert int(visits[0]) == M
    pi = R.normalize(sizes, visits, joint)
    pts_all = np.concatenate([[0.0], grids])
    phi = R.payoff_table(chain, PAYOFF_PUT, sizes, pts_all)
    price = R.solve_stopping(sizes, visits, pi, phi)[0]
    np.savez_compressed(
        OUT, M=np.array(M, np.uint64), seed=np.array(SEED, np.uint64), grid_sha=np.array(sha(grids)),
        visits=visits, joint_sha=np.array(sha(joint)), pi_sha=np.array(sha(pi)),
        joint_sum=np.array(int(joint.sum()), np.uint64), put_price=np.array(price),
        seconds=np.array(time.time() - t0))
    print(f"wrote {OUT}: put price {price!r}, {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
