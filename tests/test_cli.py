"""The reference's own CLI (tools/qtree_main.cpp, unmodified, CLI11 shimmed)
built twice by tests/cpp/Makefile: qtree_cli on the drop-in headers +
libqtree_cuda.so (estimation, pricing and bench-rng on the GPU) and
qtree_cli_ref on the reference headers alone. Same commands, same outputs:
byte-identical tree files, identical prices and pi estimates, the exit-code
contract 1 / 2 / 3 (qtree_main.cpp:291-303)."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin")


def cli(name, *args, cwd):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
        else:
            pytest.fail(f"{path} missing: run __graft_entry__.build() where /root/reference exists")
    return subprocess.run([path, *map(str, args)], capture_output=True, text=True, cwd=cwd,
                          timeout=600)


def test_cli_exit_codes_without_device(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("checks the no-device path")
    r = cli("qtree_cli", "build-tree", "--n", 4, "--N", 10, "--M", 100, "--tree",
            tmp_path / "t.qtre", cwd=tmp_path)
    assert r.returncode == 3 and "cuda: no CUDA device" in r.stderr
    r = cli("qtree_cli", "build-tree", "--bogus", 1, cwd=tmp_path)
    assert r.returncode == 1
    r = cli("qtree_cli", "price-american", "--tree", tmp_path / "missing", "--n", 4, cwd=tmp_path)
    assert r.returncode == 2 and "load_tree: cannot open" in r.stderr
    r = cli("qtree_cli", "build-tree", "--n", 4, "--N", 0, "--tree", "x", cwd=tmp_path)
    assert r.returncode == 1 and "parameter 'N' must be >= 1" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("algorithm", [1, 2, 3])
def test_cli_build_and_price_match_reference(gpu, tmp_path, algorithm):
    common = ["--n", 12, "--N", 50, "--M", 20000, "--algorithm", algorithm, "--seed", 777]
    ref = cli("qtree_cli_ref", "build-tree", *common, "--tree", tmp_path / "ref.qtre", cwd=tmp_path)
    ours = cli("qtree_cli", "build-tree", *common, "--tree", tmp_path / "ours.qtre", cwd=tmp_path)
    assert ref.returncode == 0, ref.stderr
    assert ours.returncode == 0, ours.stderr
    assert (tmp_path / "ours.qtre").read_bytes() == (tmp_path / "ref.qtre").read_bytes()
    for cmd, extra in (("price-american", []), ("price-american", ["--payoff", "call"]),
                       ("price-swing", ["--qmin", 2, "--qmax", 6])):
        a = cli("qtree_cli_ref", cmd, "--tree", tmp_path / "ref.qtre", "--n", 12, *extra,
                cwd=tmp_path)
        b = cli("qtree_cli", cmd, "--tree", tmp_path / "ours.qtre", "--n", 12, *extra,
                cwd=tmp_path)
        assert a.returncode == 0 and b.returncode == 0, (a.stderr, b.stderr)
        # price and std hint identical; the last field is wall time
        assert a.stdout.split(",")[:2] == b.stdout.split(",")[:2], (cmd, a.stdout, b.stdout)


@pytest.mark.gpu
def test_cli_bench_rng_matches_reference(gpu, tmp_path):
    for engine, mode, streams in (("mrg32k3a", "block", 1), ("mrg32k3a", "skip", 16),
                                  ("lcg48", "skip", 5), ("xorwow", "block", 64)):
        args = ["bench-rng", "--engine", engine, "--mode", mode, "--streams", streams,
                "--samples", 2_000_000]
        a = cli("qtree_cli_ref", *args, cwd=tmp_path)
        b = cli("qtree_cli", *args, cwd=tmp_path)
        assert a.returncode == 0 and b.returncode == 0, (a.stderr, b.stderr)
        assert a.stdout.split(",")[:6] == b.stdout.split(",")[:6], (a.stdout, b.stdout)
