"""Stream kernel: patch-row capacity per unit (DLMPC_STREAM_CAP) vs speed,
step-0 solve, best of 3: python tools/stream_cap_ab.py N cap [cap ...]"""
import os, sys
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
n = int(sys.argv[1])
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=1, seed=1))
for rep in range(2):
    for cap in sys.argv[2:]:
        os.environ["DLMPC_STREAM_CAP"] = cap
        sess = pb.DlmpcSession(system, spec, mask, "b200")
        ms = min(sess.simulate(x0, 1)[1] for _ in range(3))
        traj, _ = sess.simulate(x0, 1)
        it = sum(traj.step_iterations)
        i = sess.device.info()
        print(f"N={n} cap={cap} {i['mode']} units={i['units']} smem={i['smem_bytes']} {1e3 * ms / it:.2f} us/iter", flush=True)
        sess.close()
