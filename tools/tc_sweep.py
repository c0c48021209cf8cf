"""Tile-width / staging experiment: device us/iter at several N for TC=8 and 16."""
import os, sys
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
for n in [int(v) for v in sys.argv[1:]] or [1000, 10000, 100000]:
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=1, seed=1))
    for tc in ("8", "16"):
        os.environ["DLMPC_TILE_COLS"] = tc
        sess = pb.DlmpcSession(system, spec, mask, "b200")
        sess.simulate(x0, 1)
        traj, ms = sess.simulate(x0, 1)
        it = traj.step_iterations[0]
        print(f"N={n} TC={tc} {sess.device.info()} iters {it} {1e3*ms/it:.2f} us/iter", flush=True)
        sess.close()
