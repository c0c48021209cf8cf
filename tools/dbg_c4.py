import sys, numpy as np
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
d, t, v = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
system = pb.build_chain_network(1000); spec = pb.make_benchmark_spec(system, t); mask = pb.build_locality_mask(system, d, t)
sess = pb.DlmpcSession(system, spec, mask, v)
print(sess.device.info(), 'm_pad', sess.layout.m_pad if hasattr(sess.layout,'m_pad') else None, flush=True)
x0 = pb.sample_initial_state(system.partition, np.random.default_rng(1))
traj, ms = sess.simulate(x0, 1)
print('ok', traj.step_iterations, ms, flush=True)
