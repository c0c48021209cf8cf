"""The chain benchmark scenario (synthetic inputs of every measurement).

Same names and semantics as `/root/reference/pkg/src/locality_mpc/bench.py`
`make_benchmark_spec` (36-60), `sample_initial_state` (63-70), `Scenario`
(77-93) and `run_scenario` (96-110). Sweeps, CSV and SVG output of that
module are harness UX and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sls_core import ProblemSpec
from .system_model import SubsystemPartition, build_chain_network, build_locality_mask

STATE_BAND = (-0.2, 1.2)


def make_benchmark_spec(system_or_partition, horizon: int, rho: float = 1.0,
                        eps: float = 1e-4, max_iters: int = 5000,
                        bounded: bool = True) -> ProblemSpec:
    """Unit costs on blocks 1..T-2 plus the terminal block and every input
    block; the first state of every subsystem banded to [-0.2, 1.2] on blocks
    1..T-1 (reference bench.py:36-60)."""
    part = getattr(system_or_partition, "partition", system_or_partition)
    n_x, n_u, t = part.n_states, part.n_inputs, int(horizon)
    state_weights = np.zeros((n_x, t))
    state_weights[:, 1:t - 1] = 1.0
    state_lo = np.full((n_x, t), -np.inf)
    state_hi = np.full((n_x, t), np.inf)
    if bounded:
        firsts = np.asarray([a for a, _ in part.state_ranges], dtype=np.int64)
        state_lo[firsts, 1:] = STATE_BAND[0]
        state_hi[firsts, 1:] = STATE_BAND[1]
    return ProblemSpec(t, state_weights, np.ones((n_u, t - 1)), np.ones(n_x),
                       state_lo, state_hi, np.full((n_u, t - 1), -np.inf),
                       np.full((n_u, t - 1), np.inf), rho=rho, eps_pri=eps,
                       eps_dual=eps, max_iters=max_iters)


def sample_initial_state(partition: SubsystemPartition, rng) -> np.ndarray:
    """First state of each subsystem U[0,1], the others U[-0.5,0.5], drawn in
    global index order (reference bench.py:63-70). One vectorised draw gives
    the same numbers as the reference's per-state `rng.uniform` calls:
    uniform(lo, hi) is lo + (hi-lo)*next_double."""
    n = partition.n_states
    u = rng.random(n)
    first = np.zeros(n, dtype=bool)
    first[np.asarray([a for a, _ in partition.state_ranges], dtype=np.int64)] = True
    return np.where(first, 0.0 + 1.0 * u, -0.5 + 1.0 * u)


@dataclass(frozen=True)
class Scenario:
    """One benchmark run (reference bench.py:77-93); strategy defaults to the device."""

    n: int = 10
    horizon: int = 5
    d: int = 2
    t_sim: int = 20
    seed: int = 1
    strategy: str = "b200"
    workers: int | None = None
    rho: float = 1.0
    eps: float = 1e-4
    max_iters: int = 5000
    coupling_radius: int = 1
    bounded: bool = True
    warm_start: bool = True


def scenario_problem(scn: Scenario):
    """(system, spec, mask, x0) of a scenario."""
    system = build_chain_network(scn.n, scn.coupling_radius)
    spec = make_benchmark_spec(system, scn.horizon, rho=scn.rho, eps=scn.eps,
                               max_iters=scn.max_iters, bounded=scn.bounded)
    mask = build_locality_mask(system, scn.d, scn.horizon)
    x0 = sample_initial_state(system.partition, np.random.default_rng(scn.seed))
    return system, spec, mask, x0


def run_scenario(scn: Scenario, audit: bool = False):
    """Build the chain benchmark and run the closed loop (reference bench.py:96-110)."""
    from .admm import dlmpc_simulate
    from .strategies import ExecStrategy

    system, spec, mask, x0 = scenario_problem(scn)
    traj, report = dlmpc_simulate(system, spec, mask, x0, scn.t_sim,
                                  ExecStrategy(scn.strategy, scn.workers),
                                  warm_start=scn.warm_start, audit=audit)
    report.scenario.update({"N": scn.n, "T": scn.horizon, "d": scn.d, "seed": scn.seed,
                            "coupling_radius": scn.coupling_radius,
                            "max_iters": scn.max_iters})
    return traj, report
