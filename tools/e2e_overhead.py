"""Host overhead of the public closed-loop API on C2: wall time of
dlmpc_simulate vs the device time of its launch, and a cProfile of 50 calls."""
import cProfile, pstats, sys, time, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2103_14990_b200 as pb
system = pb.build_chain_network(100)
spec = pb.make_benchmark_spec(system, 10)
mask = pb.build_locality_mask(system, 3, 10)
strat = pb.ExecStrategy("b200")
x0 = pb.sample_initial_state(system.partition, np.random.default_rng(1))
for _ in range(5):
    pb.dlmpc_simulate(system, spec, mask, x0, 20, strat)
wall, dev = [], []
for _ in range(50):
    t0 = time.perf_counter()
    traj, rep = pb.dlmpc_simulate(system, spec, mask, x0, 20, strat)
    wall.append(time.perf_counter() - t0)
    dev.append(rep.scenario["device_ms"])
print(f"wall {1e3 * np.median(wall):.3f} ms  device {np.median(dev):.3f} ms  overhead {1e3 * np.median(wall) - np.median(dev):.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    pb.dlmpc_simulate(system, spec, mask, x0, 20, strat)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
