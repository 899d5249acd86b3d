"""Micro-benchmarks on the GPU: bench-rng's partitioned
Monte Carlo pi (monte_carlo.hpp:51-77) must return the reference's estimate
exactly (integer inside-count over bit-exact uniforms) for every engine and
partition; bench-nn's index checksum must equal the reference's."""
from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def Q():
    from paper_1101_3228_b200 import qtree
    return qtree


@pytest.mark.parametrize("engine", [0, 1, 2])
@pytest.mark.parametrize("streams,skip", [(1, False), (8, False), (7, True), (4096, True),
                                          (3000, False)])
def test_bench_pi_equals_reference(gpu, reference, engine, streams, skip):
    if engine == 2 and skip and streams > 1:
        with pytest.raises(ValueError):
            Q().bench_pi(engine, 12345, 2 * streams * 100, streams, skip)
        return
    samples = 2 * streams * (1_000_000 // streams + 1)
    got = Q().bench_pi(engine, 12345, samples, streams, skip)
    est, se = reference.bench_pi(engine, 12345, samples, streams, skip)
    assert got.estimate == est and got.std_error == se


def test_bench_nn_checksum_equals_reference(gpu, reference):
    for n in (100, 250, 500):
        sink, ms = Q().bench_nn(n, 200_000, 12345)
        assert sink == reference.bench_nn(n, 200_000, 12345), n
