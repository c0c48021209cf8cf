"""Parity beyond the pinned fixtures: C2 closed loops (20 steps) for seeds
FIRST..LAST, device fast path and exact path against the CPU oracle
(oracle/admm_ref.py, test infrastructure): per-step iteration lists equal,
exact states bitwise, fast states within 1e-9 relative.
usage: python tools/c2_oracle_sweep.py [first] [last]"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2103_14990_b200 as pb
from oracle import admm_ref
first = int(sys.argv[1]) if len(sys.argv) > 1 else 21
last = int(sys.argv[2]) if len(sys.argv) > 2 else 40
system = pb.build_chain_network(100)
spec = pb.make_benchmark_spec(system, 10)
mask = pb.build_locality_mask(system, 3, 10)
tables = pb.LayoutTables(mask)
cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, 10), mask)
fast = pb.DlmpcSession(system, spec, mask, "b200")
exact = pb.DlmpcSession(system, spec, mask, "b200-exact")
ok_all, worst = True, 0.0
t0 = time.time()
for seed in range(first, last + 1):
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(seed))
    ref = admm_ref.simulate(system, spec, tables, cs, x0, 20, workers=os.cpu_count() or 1)
    tf, _ = fast.simulate(x0, 20)
    te, _ = exact.simulate(x0, 20)
    it_ok = list(tf.step_iterations) == ref["step_iterations"] == list(te.step_iterations)
    ex_ok = np.array_equal(te.states, ref["states"])
    rel = float(np.max(np.abs(tf.states - ref["states"])) / max(1.0, np.max(np.abs(ref["states"]))))
    worst = max(worst, rel)
    ok = it_ok and ex_ok and rel <= 1e-9
    ok_all = ok_all and ok
    print(f"seed {seed}: iterations equal {it_ok} ({sum(ref['step_iterations'])}), exact bitwise {ex_ok}, "
          f"fast rel err {rel:.2e}", flush=True)
print(f"seeds {first}..{last}: all ok {ok_all}, worst fast rel err {worst:.2e} ({time.time() - t0:.0f} s)")
