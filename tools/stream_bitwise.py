"""Stream-kernel trajectories of two library builds must be bit-identical:
python tools/stream_bitwise.py lib_a.so lib_b.so [N ...] (runs each in a subprocess)."""
import os, subprocess, sys
import numpy as np
libs, ns = sys.argv[1:3], [int(a) for a in sys.argv[3:]] or [3000, 10000]
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2103_14990_b200 as pb
n = int(sys.argv[1])
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=3, seed=1))
sess = pb.DlmpcSession(system, spec, mask, "b200")
traj, _ = sess.simulate(x0, 3)
np.save(sys.argv[2], np.concatenate([traj.states.ravel(), np.array(traj.step_iterations, dtype=float)]))
print(sess.device.info()["mode"])
'''
for n in ns:
    outs = []
    for k, lib in enumerate(libs):
        f = f"/tmp/stream_bitwise_{k}.npy"
        r = subprocess.run([sys.executable, "-c", code, str(n), f], env=dict(os.environ, DLMPC_LIB=lib),
                           capture_output=True, text=True)
        outs.append(np.load(f))
        mode = r.stdout.strip()
    print(f"N={n} mode={mode} bitwise equal: {np.array_equal(outs[0], outs[1])}", flush=True)
