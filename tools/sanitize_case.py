"""Small persistent-kernel runs for compute-sanitizer (memcheck / racecheck /
synccheck), one case per process:

  c1        chain N=10, d=2, T=5: exact and fast kernels, 2-step closed loop
  c2        chain N=100, d=3, T=10: the bench's patch kernel (GEMV pair), 2 steps
  stream    chain N=2500 forced onto the stream kernel (TMA bulk copies,
            mbarriers, warp split), 2 steps
  twophase  N=300 on the generic two-phase kernel, 2 steps
  sched     the reference-layout device schedules (naive, fused, patch-local), 3 iterations each

Iteration caps keep the instrumented runs short; NotConverged is expected
and ignored (the point is the memory / race / sync checking).
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2103_14990_b200 as pb  # noqa: E402


def loop(n, d, t, variants, max_iters, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t, max_iters=max_iters)
    mask = pb.build_locality_mask(system, d, t)
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(1))
    for v in variants:
        sess = pb.DlmpcSession(system, spec, mask, v)
        print(v, sess.device.info(), flush=True)
        try:
            traj, _ = sess.simulate(x0, 2)
            print("  iterations", traj.step_iterations, flush=True)
        except pb.NotConverged as err:
            print("  NotConverged (expected under the cap) at step", err.step, flush=True)
        sess.close()
    for k in (env or {}):
        os.environ.pop(k)


def sched():
    system = pb.build_chain_network(8)
    spec = pb.make_benchmark_spec(system, 4, max_iters=3)
    mask = pb.build_locality_mask(system, 2, 4)
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(1))
    for v in ("naive", "fused", "patch-local"):
        try:
            pb.dlmpc_simulate(system, spec, mask, x0, 1, v)
        except pb.NotConverged:
            print(v, "ran 3 iterations", flush=True)


CASES = {
    "c1": lambda: loop(10, 2, 5, ("b200-exact", "b200"), 40),
    "c2": lambda: loop(100, 3, 10, ("b200",), 12),
    "stream": lambda: loop(2500, 3, 10, ("b200",), 4, {"DLMPC_FORCE_STREAM": "1"}),
    "twophase": lambda: loop(300, 3, 10, ("b200",), 6, {"DLMPC_FORCE_TWOPHASE": "1"}),
    "sched": sched,
}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        print("== case", name, flush=True)
        CASES[name]()
