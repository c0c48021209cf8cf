"""Benchmark of the DLMPC ADMM hot path on B200 (driver contract: one JSON line).

Workload (BASELINE.json configs[1], the metric's config): chain of N=100
coupled 2-state/1-input subsystems, locality d=3, horizon T=10, a 20-step
closed loop (warm-started MPC), synthetic x0 = the reference's seeded
sampler. One bench *step* = one whole 20-step closed loop (one persistent
kernel launch: per MPC step row data, ADMM to convergence, control, plant
step), seeds cycled 1..R so every step does real, different work.

  value  device-timed subsystem-ADMM-iterations/s with x0 resident in HBM
         (CUDA events on the library's stream, L2 flushed between steps)
  e2e    the same metric through the public API `dlmpc_simulate` with host
         buffers (H2D x0, D2H trajectory inside the timed region)

Multi-GPU: `--gpus N` runs N ranks (launched under torch.distributed.run by
the driver, or re-launched that way by this script when WORLD_SIZE is unset).
Independent replicas per rank (weak scaling), no data-path collective; value =
all ranks' subsystem-iterations / max-over-ranks time. At N > 1 the line also
carries `partitioned`: the C5 network (N=10^6) graph-partitioned across the
ranks (strong scaling) beside a same-run single-GPU solve of the same problem.

`--impl reference` times the reference's CPU path on the host cores on the
SAME workload: the oracle port (numpy restatement of the reference's fused
schedule, bit-identical iterates) runs one whole 20-step closed loop per
step over the same seeds, with every host thread.

Parity guard: every timed closed loop's per-step iteration list is compared
with the reference's (tests/golden/c2_loops_seeds1_20.npz, produced by the
reference's own run_scenario), and the last loop's trajectory within 1e-9.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SUB, D, T, T_SIM = 100, 3, 10, 20
WORKLOAD = "chain N=100 d=3 T=10, 20-step closed loop (BASELINE configs[1], C2)"
METRIC = "subsystem-ADMM-iterations/sec"
UNIT = "subsystem-iters/s"
N_SEEDS = 20          # seeds 1..20: the reference fixtures of every timed loop
GOLDEN_C2 = os.path.join(ROOT, "tests", "golden", "c2_loops_seeds1_20.npz")
FP64_FALLBACK_TFLOPS = 37.1   # tools/microbench/fp64_probe.cu, used only if the live probe fails


def golden_c2():
    with np.load(GOLDEN_C2) as z:
        return {k: z[k] for k in z.files}


def seed_for(k, rank=0):
    """Seed of bench step k on `rank`: cycles the 20 pinned seeds."""
    return 1 + (k + 7 * rank) % N_SEEDS


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def reduce_over_ranks(vals, dist, device=None):
    """[iterations, ms, e2e_iterations, e2e_ms] -> work summed over ranks,
    times maxed over ranks (replicas: whole-job throughput = all ranks' work
    / the slowest rank's time)."""
    import torch
    t = torch.tensor([vals[1], vals[3]], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    w = torch.tensor([vals[0], vals[2]], dtype=torch.float64, device=device)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return np.array([w[0].item(), t[0].item(), w[1].item(), t[1].item()])


def problem():
    import paper_2103_14990_b200 as pb
    system = pb.build_chain_network(N_SUB)
    spec = pb.make_benchmark_spec(system, T)
    mask = pb.build_locality_mask(system, D, T)
    return pb, system, spec, mask


def x0_for(pb, system, seed):
    return pb.sample_initial_state(system.partition, np.random.default_rng(seed))


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: an NVML
    polling thread (every 2 ms, so even a 50 ms region yields samples), with
    nvidia-smi as the fallback when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index):
        import threading
        self.samples, self.max_mhz, self.reasons = [], None, set()
        self._stop = threading.Event()
        self._thread = None
        self._smi = None
        try:
            import pynvml
            pynvml.nvmlInit()
            visible = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(visible.split(",")[gpu_index]) if visible and visible.split(",")[0].isdigit() else gpu_index
            self._nv, self._h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self._sample()
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        except Exception:   # noqa: BLE001 -- fall back to nvidia-smi
            self._start_smi(gpu_index)

    def _sample(self):
        nv = self._nv
        self.samples.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except AttributeError:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        for name, mask in self.REASONS.items():
            if bits & mask:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.wait(0.002):
            self._sample()

    def _start_smi(self, gpu_index):
        self._path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        try:
            self._smi = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self._path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self._smi = None

    def stop(self):
        if self._thread is not None:
            self._stop.set()
            self._thread.join()
            self._sample()
            src = "nvml (2 ms polling thread)"
        elif self._smi is not None:
            self._smi.terminate()
            self._smi.wait()
            names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
            for line in open(self._path):
                parts = [p.strip() for p in line.split(",")]
                try:
                    self.samples.append(float(parts[0])); self.max_mhz = float(parts[1])
                except (ValueError, IndexError):
                    continue
                for name, flag in zip(names, parts[2:6]):
                    if flag.lower() == "active":
                        self.reasons.add(name)
            os.unlink(self._path)
            src = "nvidia-smi -lms 20"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": ["no clock source"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples), "reasons": sorted(self.reasons), "source": src}


def algorithmic_work(sess):
    """FLOPs and bytes of ONE ADMM iteration over the whole network for the
    formulation the kernel runs: Ψ = q + N(Nᵀk) costs
    4·s·n0 FLOP per column; the canonical minimum traffic is one read and one
    write of ψ and λ per support entry, 32 B per nnz."""
    L = sess.layout
    s = L.class_s[L.col_class].astype(np.int64)
    n0 = L.class_n0[L.col_class].astype(np.int64)
    flops = int(np.sum(4 * s * n0))
    nnz = int(np.sum(L.col_len))
    return flops, 32 * nnz, nnz


def ncu_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_c2_summary_r02.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def oracle_setup(pb, system, spec, mask):
    tables = pb.LayoutTables(mask)
    cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, T), mask)
    return tables, cs


def oracle_loop(pb, admm_ref, system, spec, tables, solver, x0, sequential=False, budget=None):
    """One closed loop of the oracle (reference recurring phases): per MPC step
    row data, ADMM to convergence, control, plant step. Returns (ADMM
    iterations, MPC steps, per-step iteration list) -- stops early at
    `budget` seconds (bounded sample)."""
    w, lo, hi = spec.row_arrays()
    n_x = system.n_states
    solver.zero_()
    x = np.asarray(x0, dtype=np.float64)
    iters, its = 0, []
    t0 = time.perf_counter()
    for step in range(T_SIM):
        if budget is not None and step > 0 and time.perf_counter() - t0 > budget:
            break
        rd, _ = admm_ref.row_data_for(x, tables, w, lo, hi)
        n, _, ok = solver.solve(rd, spec.max_iters, spec.eps_pri, spec.eps_dual, sequential)
        if not ok:
            raise RuntimeError("oracle did not converge")
        u = admm_ref.extract_control(solver.phi_r, tables, x, [n_x * T + k for k in range(system.n_inputs)])
        x = admm_ref.step_dynamics(system.a, system.b, x, u)
        iters += n
        its.append(n)
    return iters, len(its), its


def cpu_baseline(pb, system, spec, mask, seconds_budget=12.0):
    """The reference's CPU path on this host (oracle port, kind 'port'),
    bounded samples of the same workload:
      value             the fused schedule (the reference's fastest CPU
                        schedule) on every host thread: whole C2 closed loops
                        over the pinned seeds until the budget is spent;
      sequential_1core  the `sequential` schedule (the paper's single-thread
                        "CPU ADMM", one row / column per stage call) on one
                        core: the first MPC steps of the seed-1 loop."""
    from oracle import admm_ref
    tables, cs = oracle_setup(pb, system, spec, mask)
    workers = os.cpu_count() or 1
    solver = admm_ref.OracleSolver(tables, cs, spec.rho, workers)
    oracle_loop(pb, admm_ref, system, spec, tables, solver, x0_for(pb, system, 1), budget=0.0)   # warm-up
    iters, loops, k = 0, 0, 0
    t0 = time.perf_counter()
    while loops == 0 or time.perf_counter() - t0 < seconds_budget:
        n, _, _ = oracle_loop(pb, admm_ref, system, spec, tables, solver, x0_for(pb, system, seed_for(k)))
        iters += n; loops += 1; k += 1
    dt = time.perf_counter() - t0
    solver.close()
    seq = admm_ref.OracleSolver(tables, cs, spec.rho, 1)
    t1 = time.perf_counter()
    s_iters, s_steps, _ = oracle_loop(pb, admm_ref, system, spec, tables, seq, x0_for(pb, system, 1),
                                      sequential=True, budget=seconds_budget)
    sdt = time.perf_counter() - t1
    return {"value": N_SUB * iters / dt, "unit": UNIT, "cores": workers, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{loops} whole C2 closed loops ({iters} ADMM iterations, seeds 1..{loops}) of "
                      f"oracle/admm_ref.py, fused schedule on {workers} threads",
            "ms_per_mpc_step": 1e3 * dt / (loops * T_SIM),
            "sequential_1core": {"value": N_SUB * s_iters / sdt, "unit": UNIT, "cores": 1,
                                 "sample": f"first {s_steps} MPC steps ({s_iters} ADMM iterations) of the seed-1 "
                                           f"C2 loop, reference `sequential` schedule restated "
                                           f"(oracle iterate_sequential)",
                                 "ms_per_mpc_step": 1e3 * sdt / s_steps}}


SWEEP_NS = (100, 300, 1000, 3000, 10000, 100000, 1000000)
# step-0 fixtures of the sweep points (reference or pinned oracle), else the audit
SWEEP_FIXTURES = {100: ("c2_loops_seeds1_20", "reference"), 1000: ("c3_n1000_step0", "reference"),
                  3000: ("c3_n3000_step0", "reference"), 10000: ("c3_n10000_step0_oracle", "oracle")}


def sweep_parity(n, traj, sess, spec):
    """Per-point parity flag: step-0 iterations and x1 against the fixture
    where one exists; beyond the oracle's reach the on-device fixed-point
    audit (reference verify_fixed_point, admm.py:417-434) against 10 eps."""
    fx = SWEEP_FIXTURES.get(n)
    path = os.path.join(ROOT, "tests", "golden", f"{fx[0]}.npz") if fx else None
    if path and os.path.exists(path):
        with np.load(path) as z:
            if fx[0].startswith("c2_"):
                it, x1 = int(z["s1_iters"][0]), z["s1_states"][1]
            elif fx[1] == "reference":
                it, x1 = int(z["step_iters"][0]), z["states"][1]
            else:
                it, x1 = int(z["iterations"]), z["x1"]
        err = float(np.max(np.abs(traj.states[1] - x1)) / max(1.0, float(np.max(np.abs(x1)))))
        return {"kind": f"{fx[1]} fixture {fx[0]}", "iterations_equal": traj.step_iterations[0] == it,
                "x1_rel_err": err, "ok": traj.step_iterations[0] == it and err <= 1e-9}
    dyn, res, gap = sess.device.audit()
    thr = 10.0 * spec.eps_pri
    return {"kind": "on-device fixed-point audit (verify_fixed_point)", "dynamics_residual": dyn,
            "resolve_residual": res, "consensus_gap": gap, "threshold": thr,
            "ok": max(dyn, res, gap) <= thr}


def sweep(pb, hbm_peak, fp64_peak, cpu_seconds=6.0):
    """SURVEY §8(d) C3/C5 on one GPU: the step-0 solve of the chain at
    N = 10^2..10^6 (d=3, T=10), device-timed (CUDA events around the one
    persistent launch, best of 3 after a warm-up), with the per-point
    roofline fractions and a parity flag; plus, for N <= 10^4,
    the rate of the reference's fused CPU schedule (oracle port) on every host
    thread (bounded sample) for the >=50x target of the north star."""
    out = []
    for n in SWEEP_NS:
        t0 = time.perf_counter()
        system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=D, horizon=T, t_sim=1, seed=1))
        sess = pb.DlmpcSession(system, spec, mask, "b200")
        setup_s = time.perf_counter() - t0
        traj, _ = sess.simulate(x0, 1)
        best = min(sess.simulate(x0, 1)[1] for _ in range(3))
        it = int(sum(traj.step_iterations))
        flops_it, bytes_it, nnz = algorithmic_work(sess)
        s_it = best * 1e-3 / it
        entry = {"n_subsystems": n, "iterations": it, "ms_per_mpc_step": best, "us_per_iteration": 1e6 * s_it,
                 "value": n / s_it, "unit": UNIT, "kernel": sess.device.info()["mode"],
                 "setup_s": round(setup_s, 2),
                 "fp64_tflops": flops_it / s_it / 1e12, "fp64_frac": flops_it / s_it / 1e12 / fp64_peak,
                 "hbm_gbs": bytes_it / s_it / 1e9, "hbm_frac": bytes_it / s_it / 1e9 / hbm_peak,
                 "flops_per_iteration": flops_it, "bytes_per_iteration": bytes_it,
                 "parity": sweep_parity(n, traj, sess, spec)}
        summ = os.path.join(ROOT, "profiles", f"ncu_stream_n1e{len(str(n)) - 1}_summary_r02.json")
        if os.path.exists(summ):   # ncu evidence for this size (one capture, committed)
            try:
                with open(summ) as fh:
                    d = json.load(fh)
                its = d.get("admm_iterations_in_launch") or 1
                entry["traffic_per_iteration"] = d["dram_bytes_per_launch"] / its
                entry["traffic_source"] = os.path.relpath(summ, ROOT)
            except (OSError, ValueError, KeyError):
                pass
        if n <= 10000 and cpu_seconds > 0:   # the fused CPU schedule to N = 10^4
            from oracle import admm_ref
            tables, cs = oracle_setup(pb, system, spec, mask)
            workers = os.cpu_count() or 1
            solver = admm_ref.OracleSolver(tables, cs, spec.rho, workers)
            w, lo, hi = spec.row_arrays()
            solver.row_data, _ = admm_ref.row_data_for(x0, tables, w, lo, hi)
            solver.iterate()
            k, t1 = 0, time.perf_counter()
            budget = cpu_seconds if n == 1000 else cpu_seconds / 2
            while k == 0 or time.perf_counter() - t1 < budget:
                solver.iterate()
                k += 1
            cpu_rate = n * k / (time.perf_counter() - t1)
            solver.close()
            entry["cpu_baseline"] = {"value": cpu_rate, "unit": UNIT, "cores": workers, "kind": "port",
                                     "sample": f"{k} ADMM iterations of the N={n} step-0 solve, fused schedule"}
            entry["speedup_vs_cpu"] = entry["value"] / cpu_rate
        out.append(entry)
        sess.close()
        del sess
    return out


C5_N = 1000000


def partitioned_c5(pb, dist, local, solves=2):
    """SURVEY §8(e) C5 on all ranks: the chain N=10^6, d=3, T=10 step-0 solve,
    graph-partitioned across the world with the exchange ON THE DEVICE
    (partition.DeviceExchangeRank: each rank's persistent kernel stores the
    halo into its neighbours' buffers over NVLink and agrees on the global
    stop test through residual slots -- one launch per solve, no host step
    per ADMM iteration). Strong scaling (total work fixed). Beside it, in
    the same run, every rank solves the WHOLE problem alone on its own GPU
    (the world-1 baseline; max over ranks), so the efficiency is
    t_1 / (world * t_world) from one run. Device time of each rank's launch
    (CUDA events on its stream), max over ranks."""
    import torch
    from paper_2103_14990_b200.partition import DeviceExchangeRank, halo_bytes_per_iteration, plan_partition
    rank, world = dist.get_rank(), dist.get_world_size()
    t0 = time.perf_counter()
    ex, err = None, None
    try:
        system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=C5_N, d=D, horizon=T, t_sim=1, seed=1))
        # same-run single-GPU baseline of the same problem
        one = pb.DlmpcSession(system, spec, mask, pb.ExecStrategy("b200", device=local))
        tr, _ = one.simulate(x0, 1)
        one_ms = min(one.simulate(x0, 1)[1] for _ in range(solves))
        one_its = int(tr.step_iterations[0])
        one.close()
        del one
    except Exception as exc:
        err = repr(exc)[:300]
        one_ms, one_its = 0.0, 0
    ok = torch.tensor([0.0 if err else 1.0], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() < 1.0:
        return {"error": err or "setup failed on another rank"}
    try:
        plans = plan_partition(mask, world)
        ex = DeviceExchangeRank(system, spec, mask, "b200", plans=plans)   # raises on every rank on failure
        setup_s = time.perf_counter() - t0
        def solve_agreed():
            # every rank reaches the agreement even if its own solve failed
            # (the kernel's exchange waits are bounded, so no rank hangs)
            try:
                n, _, conv = ex.solve(x0, True)
                ok = True
            except Exception as exc:   # noqa: BLE001 -- reported in the line
                n, conv, ok = 0, False, False
                ex.err = repr(exc)[:300]
            if not ex.agree(ok):
                raise RuntimeError(getattr(ex, "err", None) or "partitioned solve failed on another rank")
            return n, conv

        solve_agreed()                                        # warm-up solve
        ms, its, conv = 0.0, 0, True
        for _ in range(solves):
            n, c = solve_agreed()
            conv = conv and c
            ms += ex.rk.session.last_timing()[0]
            its += n
        t = torch.tensor([its, ms, setup_s, one_ms, one_its, 0.0 if conv else 1.0], dtype=torch.float64,
                         device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        its_m, ms_m, setup_m, one_ms_m, one_its_m, bad = (float(v) for v in t.cpu())
        hb = max(halo_bytes_per_iteration(plans, mask, ex.rk.layout.s_pad))
        ms_it = ms_m / its_m
        one_ms_it = one_ms_m / max(1.0, one_its_m)
        return {"workload": "chain N=1e6 d=3 T=10 step-0 solve (C5), graph-partitioned, cold start",
                "n_gpus": world, "scaling": "strong",
                "exchange": "on the device: halo stores into peer buffers over NVLink (CUDA IPC), arrival "
                            "counters and residual slots inside the persistent kernel, one launch per solve",
                "value": C5_N * its_m / (ms_m * 1e-3), "unit": UNIT,
                "ms_per_iteration": ms_it, "iterations_per_solve": its_m / solves,
                "converged": bad == 0.0,
                "single_gpu_same_run": {"ms_per_iteration": one_ms_it, "iterations": one_its_m,
                                        "value": C5_N / (one_ms_it * 1e-3),
                                        "timing": "whole problem on each rank's own GPU, best of "
                                                  f"{solves}, max over ranks"},
                "speedup_vs_single_gpu": one_ms_it / ms_it,
                "parallel_efficiency": one_ms_it / ms_it / world,
                "iterations_equal_single_gpu": abs(its_m / solves - one_its_m) < 0.5,
                "solves_timed": solves, "per_rank_kernel": ex.rk.session.info()["mode"],
                "halo_bytes_per_iteration_max_rank": hb, "setup_s_max_rank": setup_m,
                "timing": "CUDA events around each rank's persistent launch, max over ranks"}
    finally:
        if ex is not None:
            ex.close()


def run_reference_arm(args):
    """`--impl reference`: the reference's CPU path on the host on the device
    arm's workload -- one bench step = one whole C2 closed loop (20 MPC steps,
    warm-started, cold at step 0) of the seed the device arm times at that
    step, by the oracle port (the reference's fused schedule restated,
    bit-identical iterates) on every host thread. Rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    pb, system, spec, mask = problem()
    from oracle import admm_ref
    tables, cs = oracle_setup(pb, system, spec, mask)
    workers = os.cpu_count() or 1
    solver = admm_ref.OracleSolver(tables, cs, spec.rho, workers)
    gold = golden_c2() if os.path.exists(GOLDEN_C2) else None
    parity = True
    for k in range(args.warmup):
        oracle_loop(pb, admm_ref, system, spec, tables, solver, x0_for(pb, system, seed_for(k)))
    iters = 0
    t0 = time.perf_counter()
    for k in range(args.warmup, args.warmup + args.steps):
        n, _, its = oracle_loop(pb, admm_ref, system, spec, tables, solver, x0_for(pb, system, seed_for(k)))
        iters += n
        if gold is not None:
            parity = parity and its == [int(v) for v in gold[f"s{seed_for(k)}_iters"]]
    dt = time.perf_counter() - t0
    solver.close()
    value = N_SUB * iters / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "ms_per_mpc_step": 1e3 * dt / args.steps / T_SIM, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "n_subsystems": N_SUB, "d": D, "T": T, "t_sim": T_SIM,
                       "admm_iters_per_step": iters / args.steps,
                       "seeds": f"cycled over {N_SEEDS} (the device arm's seeds, step for step)",
                       "step": "one whole 20-step closed loop (the device arm's bench step)",
                       "parity_iterations_equal_reference": parity},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                             "cpu_model": cpu_model(),
                             "sample": f"{args.steps} whole C2 closed loops ({iters} ADMM iterations), "
                                       f"oracle/admm_ref.py fused schedule on {workers} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_device_arm(args):
    import torch
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch with "
                         f"torch.distributed.run --nproc-per-node {args.gpus} (or unset WORLD_SIZE "
                         f"and let bench.py launch the ranks itself)")
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    pb, system, spec, mask = problem()
    sess = pb.DlmpcSession(system, spec, mask, pb.ExecStrategy("b200", device=local))
    dev = sess.device
    seeds = [seed_for(k, rank) for k in range(args.warmup + args.steps)]
    xs = {s: torch.tensor(x0_for(pb, system, s), dtype=torch.float64, device=f"cuda:{local}") for s in set(seeds)}
    nx, nu = system.n_states, system.n_inputs
    states = torch.zeros((T_SIM + 1) * nx, dtype=torch.float64, device=f"cuda:{local}")
    inputs = torch.zeros(T_SIM * nu, dtype=torch.float64, device=f"cuda:{local}")
    iters = torch.zeros((len(seeds), T_SIM), dtype=torch.int32, device=f"cuda:{local}")
    status = torch.zeros((len(seeds), 8), dtype=torch.int32, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")   # > 126 MB L2
    ext = torch.cuda.ExternalStream(dev.stream, device=f"cuda:{local}")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in seeds]

    def one(k, timed):
        flush.zero_()
        torch.cuda.synchronize()
        if timed:
            ev[k][0].record(ext)
        sess.device.simulate_device(xs[seeds[k]].data_ptr(), T_SIM, spec.max_iters, spec.eps_pri, spec.eps_dual,
                                    states.data_ptr(), inputs.data_ptr(), iters[k].data_ptr(),
                                    status[k].data_ptr())
        if timed:
            ev[k][1].record(ext)

    for k in range(args.warmup):
        one(k, False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    for k in range(args.warmup, args.warmup + args.steps):
        one(k, True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    dev_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.warmup, args.warmup + args.steps)]
    st = status.cpu().numpy()
    if np.any(st[:, 0] != 0):
        raise RuntimeError(f"device solve failed: status {st[st[:, 0] != 0][0]}")
    it_np = iters.cpu().numpy()
    timed_iters = int(it_np[args.warmup:].sum())
    total_ms = float(sum(dev_ms))
    # parity guard: every timed loop's per-step iterations against the
    # reference's; the last timed loop's trajectory (still in `states`)
    parity = {"timed_loops_checked": 0, "iterations_equal_reference": None}
    if os.path.exists(GOLDEN_C2):
        gold = golden_c2()
        eq = all(list(it_np[k]) == [int(v) for v in gold[f"s{seeds[k]}_iters"]]
                 for k in range(args.warmup, args.warmup + args.steps))
        last = gold[f"s{seeds[-1]}_states"]
        err = float(np.max(np.abs(states.cpu().numpy().reshape(T_SIM + 1, nx) - last)) /
                    max(1.0, float(np.max(np.abs(last)))))
        parity = {"timed_loops_checked": args.steps, "iterations_equal_reference": bool(eq),
                  "last_loop_states_rel_err": err, "tolerance": 1e-9,
                  "fixture": "tests/golden/c2_loops_seeds1_20.npz (reference run_scenario)"}

    # e2e through the public API with host buffers (session cached by dlmpc_simulate)
    e2e_iters, e2e_s = 0, 0.0
    pb.dlmpc_simulate(system, spec, mask, x0_for(pb, system, 1), T_SIM, pb.ExecStrategy("b200", device=local))
    for k in range(args.warmup, args.warmup + args.steps):
        x0h = x0_for(pb, system, seeds[k])
        t0 = time.perf_counter()
        traj, _ = pb.dlmpc_simulate(system, spec, mask, x0h, T_SIM, pb.ExecStrategy("b200", device=local))
        e2e_s += time.perf_counter() - t0
        e2e_iters += sum(traj.step_iterations)

    vals = np.array([timed_iters, total_ms, e2e_iters, e2e_s * 1e3], dtype=np.float64)
    if world > 1:
        vals = reduce_over_ranks(vals, dist, device=f"cuda:{local}")
    part = None
    force_part = os.environ.get("DLMPC_BENCH_PARTITIONED") == "1"   # exercise at world size 1
    if (world > 1 or force_part) and not args.no_partitioned:
        if world == 1:
            import torch.distributed as dist
            if not dist.is_initialized():
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29533")
                dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        try:
            part = partitioned_c5(pb, dist, local)
        except Exception as exc:   # reported, never fatal for the replica line
            part = {"error": repr(exc)[:300]}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    flops_it, bytes_it, nnz = algorithmic_work(sess)
    it_per_launch = timed_iters / args.steps
    launch_ms = total_ms / args.steps
    achieved_gbs = bytes_it * it_per_launch / (launch_ms * 1e-3) / 1e9
    achieved_tf = flops_it * it_per_launch / (launch_ms * 1e-3) / 1e12
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except (OSError, ValueError):
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    try:
        from paper_2103_14990_b200.device import fp64_peak_tflops
        fp64_peak, fp64_src = fp64_peak_tflops(local), "measured live: dlmpc_fp64_peak (DMMA m8n8k4 chains, all SMs)"
    except Exception as exc:   # noqa: BLE001 -- reported in the line
        fp64_peak, fp64_src = FP64_FALLBACK_TFLOPS, f"fallback (probe failed: {exc!r:.80})"
    traffic = ncu_traffic()
    line = {
        "metric": METRIC,
        "value": N_SUB * vals[0] / (vals[1] * 1e-3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": vals[1] / args.steps,
        "ms_per_mpc_step": vals[1] / args.steps / T_SIM,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference seeded sampler; chain plant of the reference)",
        "config": {"workload": WORKLOAD, "n_subsystems": N_SUB, "d": D, "T": T, "t_sim": T_SIM,
                   "admm_iters_per_step": it_per_launch, "seeds": f"cycled over {N_SEEDS} per rank",
                   "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "arithmetic": "b200 fast path (null-space Ψ on FP64 DMMA)",
                   "parity": parity},
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback B200_PROFILING.md",
                     "algorithmic_bytes_per_iteration": bytes_it, "nnz": nnz,
                     "fp64": {"achieved_tflops": achieved_tf, "peak_tflops": fp64_peak,
                              "frac": achieved_tf / fp64_peak, "flops_per_iteration": flops_it,
                              "peak_source": fp64_src},
                     "note": "latency-bound at N=100: one grid barrier + dependent L2 round trips per iteration"},
        "e2e": {"value": N_SUB * vals[2] / (vals[3] * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": 8 * system.n_states,
                "d2h_bytes_per_step": 8 * ((T_SIM + 1) * nx + T_SIM * nu) + 4 * T_SIM + 4 * 8},
        "gpu_launches": args.steps,
        "clocks": clk,
    }
    if not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_baseline(pb, system, spec, mask)
    if not args.no_sweep and world == 1:
        sess.close()
        line["sweep"] = sweep(pb, hbm_peak, fp64_peak, 0.0 if args.no_cpu else 6.0)
    if part is not None:
        line["partitioned"] = part
    print(json.dumps(line), flush=True)
    if world > 1 or (part is not None and dist.is_initialized()):
        dist.destroy_process_group()


def relaunch_distributed(args):
    """`python bench.py --gpus N` without a launcher: run the N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-sweep", action="store_true", help="skip the N=1e2..1e6 step-0 sweep")
    ap.add_argument("--no-partitioned", action="store_true",
                    help="N>1: skip the graph-partitioned C5 (N=1e6) measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.impl == "reference":
        run_reference_arm(args)
    elif "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_distributed(args))
    else:
        run_device_arm(args)


if __name__ == "__main__":
    main()
