"""Device time per ADMM iteration for a fixed iteration count (no stop test:
one host-driven launch of n iterations after set_x), best of 5:
python tools/iter_time.py [N] [iters]"""
import sys
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, t_sim=1, seed=1))
sess = pb.DlmpcSession(system, spec, mask, "b200")
dev = sess.device
best = 1e9
for _ in range(5):
    dev.zero()
    dev.set_x(x0)
    dev.iterate(iters)
    best = min(best, dev.last_timing()[0])
print(f"N={n} {iters} iterations (fixed) {1e3 * best / iters:.2f} us/iter mode={dev.info()['mode']}")
