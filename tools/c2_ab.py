"""C2 closed loop (bench workload, seed 1..4) device time per launch, best of 10, for A/B of library
builds: DLMPC_LIB=... python tools/c2_ab.py"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
system = pb.build_chain_network(100)
spec = pb.make_benchmark_spec(system, 10)
mask = pb.build_locality_mask(system, 3, 10)
sess = pb.DlmpcSession(system, spec, mask, "b200")
tot_it, tot_ms = 0, 0.0
for seed in (1, 2, 3, 4):
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(seed))
    traj, _ = sess.simulate(x0, 20)
    best = min(sess.simulate(x0, 20)[1] for _ in range(10))
    tot_it += sum(traj.step_iterations); tot_ms += best
print(f"C2 closed loops: {1e3 * tot_ms / tot_it:.3f} us/iter  {100 * tot_it / (tot_ms * 1e-3) / 1e6:.3f} M subsystem-iters/s")
