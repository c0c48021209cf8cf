"""Host overhead of the closed-loop API on C2: device.simulate vs
DlmpcSession.simulate vs dlmpc_simulate wall time per call, and a cProfile
of dlmpc_simulate."""
import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
system = pb.build_chain_network(100); spec = pb.make_benchmark_spec(system, 10); mask = pb.build_locality_mask(system, 3, 10)
x0 = pb.sample_initial_state(system.partition, np.random.default_rng(1))
st = pb.ExecStrategy("b200")
pb.dlmpc_simulate(system, spec, mask, x0, 20, st)
from paper_2103_14990_b200.admm import _cached_session
sess, _ = _cached_session(system, spec, mask, st)
for name, fn in [("device.simulate", lambda: sess.device.simulate(x0, 20, spec.max_iters, spec.eps_pri, spec.eps_dual)),
                 ("DlmpcSession.simulate", lambda: sess.simulate(x0, 20)),
                 ("dlmpc_simulate", lambda: pb.dlmpc_simulate(system, spec, mask, x0, 20, st))]:
    for _ in range(5): fn()
    t0 = time.perf_counter()
    for _ in range(200): fn()
    wall = (time.perf_counter() - t0) / 200 * 1e3
    print(f"{name:24s} {wall:.3f} ms/call  (device {sess.device.last_timing()[0]:.3f} ms)")
pr = cProfile.Profile(); pr.enable()
for _ in range(200): pb.dlmpc_simulate(system, spec, mask, x0, 20, st)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
