"""Generate the large-N golden fixtures with the ORACLE (oracle/admm_ref.py).

The reference cannot run these sizes here: its per-column operator storage
is 0.5 MB per column at d=3, T=10 (10 GB at N=10^4) and up to 15 MB per
column at d=6, T=30 (31 GB at N=1000), and its session precompute takes
minutes per thousand columns. The oracle is the reference's iteration
restated in the same operation order and is pinned BIT FOR BIT against the
reference's own outputs (tests/test_oracle_golden.py: C1, C2 seeds 1..20,
N=1000 and N=3000 step 0, d=1/d=4 loops, traces); the setup objects it
consumes (LayoutTables, per-column g / projector / rhs) are pinned bit for
bit against the reference's objects (tests/test_setup_parity.py). So these
fixtures are the reference's results at sizes the reference cannot reach
in this container.

    python tests/golden/make_oracle_golden.py --c3 10000     # ~10 min
    python tests/golden/make_oracle_golden.py --c4           # all 24 cells at N=1000

Each fixture holds the step-0 solve of the seed-1 chain problem (cold
start, the reference's benchmark spec): iteration count, convergence flag,
the residual history (its tail for non-converged cells), the control u0 and
the next state x1 = A x0 + B u0.
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

C4_D = (1, 2, 3, 4, 5, 6)
C4_T = (5, 10, 20, 30)


def step0(n, d, t, seed=1, workers=8):
    import paper_2103_14990_b200 as pb
    from oracle import admm_ref
    t0 = time.perf_counter()
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t)
    mask = pb.build_locality_mask(system, d, t)
    tables = pb.LayoutTables(mask)
    op = pb.build_dynamics_operator(system, t)
    classes = pb.build_column_classes(op, mask)
    cs = pb.precompute_column_solvers(op, mask, classes)
    x0 = pb.sample_initial_state(system.partition, np.random.default_rng(seed))
    t1 = time.perf_counter()
    res = admm_ref.simulate(system, spec, tables, cs, x0, 1, workers=workers)
    hist = np.array(res["histories"][0])
    out = dict(config=np.array([n, d, t, seed]), x0=x0, history_len=np.array(len(hist)),
               converged=np.array(res["status"] == "ok"),
               history_tail=hist[-16:], history_head=hist[:16])
    if res["status"] == "ok":
        out["iterations"] = np.array(res["step_iterations"][0])
        out["u0"] = res["inputs"][0]
        out["x1"] = res["states"][1]
        if len(hist) <= 400:
            out["history"] = hist
    print(f"N={n} d={d} T={t}: {res['status']} after {len(hist)} iterations "
          f"(setup {t1 - t0:.1f}s, solve {time.perf_counter() - t1:.1f}s)", flush=True)
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3", type=int, default=0)
    ap.add_argument("--c4", action="store_true")
    ap.add_argument("--cells", default="", help="subset 'd:T,d:T' of the C4 grid")
    ap.add_argument("--workers", type=int, default=8)
    args = ap.parse_args()
    if args.c3:
        save(f"c3_n{args.c3}_step0_oracle", **step0(args.c3, 3, 10, workers=args.workers))
    if args.c4:
        cells = [(d, t) for t in C4_T for d in C4_D]
        if args.cells:
            cells = [tuple(int(v) for v in c.split(":")) for c in args.cells.split(",")]
        path = os.path.join(HERE, "c4_n1000_step0_oracle.npz")
        out = {}
        if os.path.exists(path):
            with np.load(path) as z:
                out = {k: z[k] for k in z.files}
        for d, t in cells:
            r = step0(1000, d, t, workers=args.workers)
            for k, v in r.items():
                out[f"d{d}t{t}_{k}"] = v
            save("c4_n1000_step0_oracle", **out)    # after every cell: resumable


if __name__ == "__main__":
    main()
