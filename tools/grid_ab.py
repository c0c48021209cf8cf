"""C2 closed loops (seeds 1..4, best of 10) at several grid sizes (DeviceSession
grid_ctas): python tools/grid_ab.py 148 100 ..."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2103_14990_b200 as pb
from paper_2103_14990_b200.device import DeviceSession
system = pb.build_chain_network(100)
spec = pb.make_benchmark_spec(system, 10)
mask = pb.build_locality_mask(system, 3, 10)
base = pb.DlmpcSession(system, spec, mask, "b200")
ref = {}
for g in [int(a) for a in sys.argv[1:]] or [148, 100]:
    sess = pb.DlmpcSession(system, spec, mask, "b200")
    sess.device.close()
    sess.device = DeviceSession(sess.layout, 0, g)
    tot_it, tot_ms, same = 0, 0.0, True
    for seed in (1, 2, 3, 4):
        x0 = pb.sample_initial_state(system.partition, np.random.default_rng(seed))
        traj, _ = sess.simulate(x0, 20)
        r = ref.setdefault(seed, traj)
        same = same and np.array_equal(r.states, traj.states)
        tot_ms += min(sess.simulate(x0, 20)[1] for _ in range(10))
        tot_it += sum(traj.step_iterations)
    print(f"grid {g}: {sess.device.info()['grid']} CTAs, units {sess.device.info()['units']}, "
          f"{1e3 * tot_ms / tot_it:.3f} us/iter, {100 * tot_it / (tot_ms * 1e-3) / 1e6:.3f} M/s, bitwise as first: {same}", flush=True)
    sess.close()
