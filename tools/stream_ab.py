"""A/B of the stream and patch kernels on chain cases (step 0 solve).
usage: python tools/stream_ab.py N [N ...]"""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2103_14990_b200 as pb
for n in [int(a) for a in sys.argv[1:]] or [100, 1000, 10000]:
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=1, seed=1))
    res = {}
    for tag, env, ws in (("patch", "1", "1"), ("stream", "0", "0"), ("stream-ws", "0", "1")):
        os.environ["DLMPC_NO_STREAM"] = env
        os.environ["DLMPC_WARP_SPEC"] = ws
        sess = pb.DlmpcSession(system, spec, mask, "b200")
        best = None
        for _ in range(3):
            traj, ms = sess.simulate(x0, 1)
            it = sum(traj.step_iterations)
            best = ms if best is None else min(best, ms)
        info = sess.device.info()
        res[tag] = (traj.states[-1], it)
        print(f"N={n} {tag:10s} mode={info['mode']} units={info['units']} smem={info['smem_bytes']} "
              f"iters {it} {best:.3f} ms {1e3 * best / it:.2f} us/iter", flush=True)
        del sess
    a, b = res["patch"][0], res["stream"][0]
    print(f"N={n} iters equal {res['patch'][1] == res['stream'][1] == res['stream-ws'][1]}  max rel diff "
          f"{float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(a)))):.2e}  ws vs lockstep bitwise "
          f"{bool(np.array_equal(res['stream'][0], res['stream-ws'][0]))}", flush=True)
