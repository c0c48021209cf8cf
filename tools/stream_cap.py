"""Stream kernel: row cap x copy mode sweep, repeated (noise check).
usage: python tools/stream_cap.py N cap1 cap2 ..."""
import os, sys
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
n = int(sys.argv[1]); caps = sys.argv[2:] or ["4096"]
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=1, seed=1))
for rep in range(2):
    for cap in caps:
        for bulk in ("1",):
            os.environ["DLMPC_STREAM_CAP"] = cap
            sess = pb.DlmpcSession(system, spec, mask, "b200")
            best = min(sess.simulate(x0, 1)[1] for _ in range(3))
            it = 0
            traj, _ = sess.simulate(x0, 1)
            it = sum(traj.step_iterations)
            info = sess.device.info()
            print(f"N={n} cap={cap:5s} bulk={bulk} units={info['units']} smem={info['smem_bytes']} "
                  f"{1e3 * best / it:.2f} us/iter", flush=True)
            sess.close()
