"""Generate tests/golden/prices.npz: configs 3, 4 and 5 at their BASELINE sizes
(or the proposal sizes of SURVEY.md §8(d) where BASELINE gives none), counted
AND priced by the REFERENCE (oracle/_ref: the unmodified reference headers).

  C3  OuChain1d (alpha1 = 1, sigma1 = 0.5, sigma2 = 0), n = 365, N = 200,
      Alg III with 1e6 samples per layer; swing Q in [0, 100] on the OU obstacle
      e^{-rt}(spot(p, t, x, 0) - K) (two_factor.hpp:150-152,172-176).
  C4  TwoFactorChain (TwoFactorParams defaults), n = 365, N = 1000, Alg II with
      M = 1e5 paths (the paper's scenario); swing Q in [0, 100] on
      make_swing_payoff(cfg, 2) (pipeline.hpp:156-170).
  C5  GbmChain3d (rho = 0), n = 20, N = 4000, Alg II with M = 1e6; American
      max-call (s0 = K = 100, sigma_a = 0.2, r = 0.05) by solve_stopping.

Grids are the reference's own builders (pipeline.hpp:27-77 and the C5
analogue); seeds 12345, MRG32k3a. Stored: sha256 of grids / joint / pi, the
visits vectors, the prices. About 10 minutes on 8 cores, 15 GB of RAM.

    python tests/golden/make_golden_prices.py [c3] [c4] [c5]
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import (ALG_II, ALG_III, CHAIN_GBM3D, CHAIN_OU1D, CHAIN_TWO_FACTOR,  # noqa: E402
                      PAYOFF_MAXCALL, PAYOFF_SWING, ChainSpec, Oracle)

OUT = os.path.join(ROOT, "tests", "golden", "prices.npz")

SPECS = {
    "c3": (ChainSpec(CHAIN_OU1D, 365, sigma1=0.5, alpha1=1.0, sigma2=0.0), 200, ALG_III, 10**6,
           PAYOFF_SWING, (0, 100)),
    "c4": (ChainSpec(CHAIN_TWO_FACTOR, 365), 1000, ALG_II, 10**5, PAYOFF_SWING, (0, 100)),
    "c5": (ChainSpec(CHAIN_GBM3D, 20, r=0.05), 4000, ALG_II, 10**6, PAYOFF_MAXCALL, None),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    which = [a for a in sys.argv[1:] if a in SPECS] or list(SPECS)
    R = Oracle("reference")
    out = {}
    if os.path.exists(OUT):
        with np.load(OUT) as z:
            out = {k: z[k] for k in z.files}
    for tag in which:
        spec, N, alg, M, payoff, q = SPECS[tag]
        t0 = time.time()
        grids = R.build_grids(spec, N)
        sizes = np.array([1] + [N] * spec.steps, np.uint64)
        cnt = R.estimate(alg, spec, sizes, grids, M, workers=4)
        t_est = time.time() - t0
        pts_all = np.concatenate([np.zeros(spec.dim), grids])
        phi = R.payoff_table(spec, payoff, sizes, pts_all)
        t1 = time.time()
        if q is None:
            price = R.solve_stopping(sizes, cnt.visits, cnt.pi, phi)[0]
        else:
            price = R.solve_swing(sizes, cnt.visits, cnt.pi, phi, q[0], q[1])
        t_price = time.time() - t1
        out.update({
            f"{tag}_M": np.array(M, np.uint64), f"{tag}_grid_sha": np.array(sha(grids)),
            f"{tag}_visits": cnt.visits, f"{tag}_joint_sha": np.array(sha(cnt.joint)),
            f"{tag}_pi_sha": np.array(sha(cnt.pi)), f"{tag}_phi_sha": np.array(sha(phi)),
            f"{tag}_price": np.array(price),
            f"{tag}_seconds": np.array([t_est, t_price]),
        })
        if q is not None:
            out[f"{tag}_q"] = np.array(q)
        np.savez_compressed(OUT, **out)
        print(f"{tag}: price {price!r}; estimate {t_est:.1f}s, price {t_price:.1f}s", flush=True)
        del cnt


if __name__ == "__main__":
    main()
