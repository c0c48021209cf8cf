"""Fused MPC-step transitions (patch mode, P.fuse_steps) against the
grid-barrier transition: trajectories and iteration counts must be
bit-identical (C2, seeds 1..20, plus N=1000 d=3 T=10); device time per
iteration best of 10 for each. DLMPC_FUSE_STEPS=0 disables the fused path at
session creation, =1 forces it (the default enables it for the register-blocked
GEMV plans only)."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2103_14990_b200 as pb


def session(n, d, t, fuse):
    os.environ["DLMPC_FUSE_STEPS"] = "1" if fuse else "0"
    system = pb.build_chain_network(n)
    spec = pb.make_benchmark_spec(system, t)
    mask = pb.build_locality_mask(system, d, t)
    s = pb.DlmpcSession(system, spec, mask, "b200")
    os.environ.pop("DLMPC_FUSE_STEPS", None)
    return system, s


for (n, d, t, seeds) in ((100, 3, 10, range(1, 21)), (1000, 3, 10, range(1, 4)), (300, 2, 5, range(1, 4))):
    system, a = session(n, d, t, False)
    _, b = session(n, d, t, True)
    print(f"N={n} d={d} T={t}: grid-barrier plan {a.device.info()} | fused plan fuse_steps={b.device.info()['fuse_steps']}")
    ok = True
    it_a = it_b = 0
    ms_a = ms_b = 0.0
    for seed in seeds:
        x0 = pb.sample_initial_state(system.partition, np.random.default_rng(seed))
        ta, _ = a.simulate(x0, 20)
        tb, _ = b.simulate(x0, 20)
        same = (np.array_equal(ta.states, tb.states) and np.array_equal(ta.inputs, tb.inputs)
                and list(ta.step_iterations) == list(tb.step_iterations))
        ok = ok and same
        if not same:
            print(f"  seed {seed}: MISMATCH iters {list(ta.step_iterations)} vs {list(tb.step_iterations)}")
        if seed <= 4:
            ms_a += min(a.simulate(x0, 20)[1] for _ in range(10))
            ms_b += min(b.simulate(x0, 20)[1] for _ in range(10))
            it_a += sum(ta.step_iterations)
            it_b += sum(tb.step_iterations)
    print(f"  bitwise identical over seeds {list(seeds)[0]}..{list(seeds)[-1]}: {ok}")
    print(f"  grid-barrier transition: {1e3 * ms_a / it_a:.3f} us/iter ({n * it_a / (ms_a * 1e-3) / 1e6:.3f} M subsystem-iters/s)")
    print(f"  fused transition:        {1e3 * ms_b / it_b:.3f} us/iter ({n * it_b / (ms_b * 1e-3) / 1e6:.3f} M subsystem-iters/s)")
    a.close(); b.close()
