"""bench.py's contract pieces that run without a GPU: the seed cycle is
covered by the reference fixtures, the oracle reproduces those fixtures, and
a launch whose world size disagrees with --gpus fails loudly instead of
silently timing one rank."""

import os
import subprocess
import sys

import numpy as np

import bench
from conftest import chain_bundle, golden
from oracle import admm_ref


def test_every_timed_seed_has_a_reference_fixture():
    g = golden("c2_loops_seeds1_20")
    for rank in range(8):
        for k in range(64):
            s = bench.seed_for(k, rank)
            assert 1 <= s <= bench.N_SEEDS
            assert len(g[f"s{s}_iters"]) == bench.T_SIM


def test_oracle_reproduces_bench_seed_fixtures():
    """The checker the reference arm and cpu_baseline time is the reference:
    two more of the bench's seeds, bit for bit (seed 1 is pinned in
    test_oracle_golden.py)."""
    g = golden("c2_loops_seeds1_20")
    b = chain_bundle(100, 10, 3)
    for seed in (7, 20):
        res = admm_ref.simulate(b["system"], b["spec"], b["tables"], b["col_solvers"], g[f"s{seed}_x0"], 20,
                                workers=os.cpu_count() or 1)
        assert res["step_iterations"] == [int(v) for v in g[f"s{seed}_iters"]]
        assert np.array_equal(res["states"], g[f"s{seed}_states"])
        assert np.array_equal(res["inputs"], g[f"s{seed}_inputs"])


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, bench.__file__, "--gpus", "2", "--steps", "1", "--warmup", "3"],
                         env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode != 0
    assert "--gpus 2 but WORLD_SIZE=1" in (res.stdout + res.stderr)
