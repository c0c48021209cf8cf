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

Multi-GPU (torchrun): independent replicas per rank (weak scaling, different
seeds), no data-path collective; value = all ranks' subsystem-iterations /
max-over-ranks time. `--impl reference` times the CPU reference path (the
oracle port of the reference's numpy iteration) on the host cores instead.
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
GOLDEN_SEED1_ITERS = [72, 53, 45, 38, 30, 23, 18, 14, 11, 9, 7, 6, 5, 4, 4, 3, 3, 3, 3, 2]
FP64_DMMA_PEAK_TFLOPS = 37.1   # measured, tools/microbench/fp64_probe.cu (profiles/fp64_probe_r01.txt)


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
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


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
    path = os.path.join(ROOT, "profiles", "ncu_c2_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def cpu_baseline(pb, system, spec, mask, seconds_budget=20.0):
    """The oracle (numpy restatement of the reference iteration, kind 'port')
    on the host cores: complete MPC steps of the same closed loop until the
    budget is spent (bounded sample)."""
    from oracle import admm_ref
    tables = pb.LayoutTables(mask)
    cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, T), mask)
    workers = max(1, min(8, os.cpu_count() or 1))
    solver = admm_ref.OracleSolver(tables, cs, spec.rho, workers)
    w, lo, hi = spec.row_arrays()
    x = x0_for(pb, system, 1)
    n_x = system.n_states
    iters, steps = 0, 0
    t0 = time.perf_counter()
    while steps < T_SIM and time.perf_counter() - t0 < seconds_budget:
        rd, _ = admm_ref.row_data_for(x, tables, w, lo, hi)
        n, _, _ = solver.solve(rd, spec.max_iters, spec.eps_pri, spec.eps_dual)
        u = admm_ref.extract_control(solver.phi_r, tables, x, [n_x * T + k for k in range(system.n_inputs)])
        x = admm_ref.step_dynamics(system.a, system.b, x, u)
        iters += n
        steps += 1
    dt = time.perf_counter() - t0
    solver.close()
    return {"value": N_SUB * iters / dt, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"first {steps} MPC steps ({iters} ADMM iterations) of the seed-1 C2 closed loop, "
                      f"oracle/admm_ref.py (numpy restatement of the reference, fused-style thread pool)",
            "ms_per_mpc_step": 1e3 * dt / steps}


SWEEP_NS = (100, 300, 1000, 3000, 10000, 100000, 1000000)


def sweep(pb, hbm_peak, cpu_seconds=6.0):
    """SURVEY §8(d) C3/C5 on one GPU: the step-0 solve of the chain at
    N = 10^3..10^6 (d=3, T=10), device-timed (CUDA events around the one
    persistent launch, best of 3 after a warm-up), with the per-point
    roofline fractions; plus the oracle's rate at N=1000 on the host cores
    (bounded sample) for the >=50x target of the north star."""
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
                 "fp64_tflops": flops_it / s_it / 1e12, "fp64_frac": flops_it / s_it / 1e12 / FP64_DMMA_PEAK_TFLOPS,
                 "hbm_gbs": bytes_it / s_it / 1e9, "hbm_frac": bytes_it / s_it / 1e9 / hbm_peak,
                 "flops_per_iteration": flops_it, "bytes_per_iteration": bytes_it}
        summ = os.path.join(ROOT, "profiles", f"ncu_stream_n1e{len(str(n)) - 1}_summary.json")
        if os.path.exists(summ):   # ncu evidence for this size (one capture, committed)
            try:
                with open(summ) as fh:
                    d = json.load(fh)
                its = d.get("admm_iterations_in_launch") or 1
                entry["traffic_per_iteration"] = d["dram_bytes_per_launch"] / its
                entry["traffic_source"] = os.path.relpath(summ, ROOT)
            except (OSError, ValueError, KeyError):
                pass
        if n == 1000 and cpu_seconds > 0:
            from oracle import admm_ref
            tables = pb.LayoutTables(mask)
            cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, T), mask)
            workers = max(1, min(8, os.cpu_count() or 1))
            solver = admm_ref.OracleSolver(tables, cs, spec.rho, workers)
            w, lo, hi = spec.row_arrays()
            solver.row_data, _ = admm_ref.row_data_for(x0, tables, w, lo, hi)
            k, t1 = 0, time.perf_counter()
            while time.perf_counter() - t1 < cpu_seconds:
                solver.iterate()
                k += 1
            cpu_rate = n * k / (time.perf_counter() - t1)
            solver.close()
            entry["cpu_baseline"] = {"value": cpu_rate, "unit": UNIT, "cores": workers, "kind": "port",
                                     "sample": f"{k} ADMM iterations of the N=1000 step-0 solve"}
            entry["speedup_vs_cpu"] = entry["value"] / cpu_rate
        out.append(entry)
        sess.close()
        del sess
    return out


C5_N = 1000000


def partitioned_c5(pb, dist, local, solves=2):
    """SURVEY §8(e) C5 on all ranks: the chain N=10^6, d=3, T=10 step-0 solve,
    graph-partitioned across the world (each rank: own subsystem range + 2d
    halo; per iteration an all-reduce(max) of the residuals and one NCCL
    message per neighbour). Strong scaling (total work fixed). Timed with
    CUDA events on each rank's library stream around whole solves, max over
    ranks; the single-GPU number is the sweep's N=10^6 point."""
    import torch
    from paper_2103_14990_b200.partition import DistExchange, RankSolver, halo_bytes_per_iteration, plan_partition
    rank, world = dist.get_rank(), dist.get_world_size()
    t0 = time.perf_counter()
    rk, err = None, None
    try:
        system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=C5_N, d=D, horizon=T, t_sim=1, seed=1))
        plans = plan_partition(mask, world)
        rk = RankSolver(system, spec, mask, plans, rank, "b200", local)
    except Exception as exc:
        err = repr(exc)[:300]
    setup_s = time.perf_counter() - t0
    # no rank enters the per-iteration collectives unless every rank is set up
    ok = torch.tensor([0.0 if err else 1.0], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() < 1.0:
        if rk is not None:
            rk.close()
        return {"error": err or "setup failed on another rank"}
    try:
        ex = DistExchange(rk)
        ext = torch.cuda.ExternalStream(rk.session.stream, device=f"cuda:{local}")
        ex.solve_step(x0, True, spec)                       # warm-up solve
        dist.barrier()
        torch.cuda.synchronize()
        ms, its = 0.0, 0
        for _ in range(solves):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            hist = ex.solve_step(x0, True, spec)
            e1.record(ext)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
            its += len(hist)
        # every rank runs the same (global) iterations: max over ranks for all three
        t = torch.tensor([its, ms, setup_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        its_m, ms_m, setup_m = (float(v) for v in t.cpu())
        hb = max(halo_bytes_per_iteration(plans, mask, rk.layout.s_pad))
        return {"workload": "chain N=1e6 d=3 T=10 step-0 solve (C5), graph-partitioned, cold start",
                "n_gpus": world, "scaling": "strong",
                "value": C5_N * its_m / (ms_m * 1e-3), "unit": UNIT,
                "ms_per_iteration": ms_m / its_m, "iterations_per_solve": its_m / solves,
                "solves_timed": solves, "per_rank_kernel": rk.session.info()["mode"],
                "halo_bytes_per_iteration_max_rank": hb, "setup_s_max_rank": setup_m,
                "timing": "CUDA events on each rank's stream around whole solves, max over ranks"}
    finally:
        rk.close()


def run_reference_arm(args):
    """`--impl reference`: the reference's CPU path (oracle port) on the host."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    pb, system, spec, mask = problem()
    from oracle import admm_ref
    tables = pb.LayoutTables(mask)
    cs = pb.precompute_column_solvers(pb.build_dynamics_operator(system, T), mask)
    workers = max(1, min(8, os.cpu_count() or 1))
    solver = admm_ref.OracleSolver(tables, cs, spec.rho, workers)
    w, lo, hi = spec.row_arrays()
    rd, _ = admm_ref.row_data_for(x0_for(pb, system, 1), tables, w, lo, hi)
    solver.row_data = rd
    per_step = 5   # ADMM iterations per bench step (bounded sample)
    for _ in range(args.warmup):
        for _ in range(per_step):
            solver.iterate()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(per_step):
            solver.iterate()
    dt = time.perf_counter() - t0
    solver.close()
    value = N_SUB * per_step * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "step": f"{per_step} ADMM iterations of the C2 step-0 solve",
                       "n_subsystems": N_SUB, "d": D, "T": T},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                             "sample": f"{args.steps}x{per_step} ADMM iterations, oracle/admm_ref.py"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_device_arm(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    pb, system, spec, mask = problem()
    sess = pb.DlmpcSession(system, spec, mask, pb.ExecStrategy("b200", device=local))
    dev = sess.device
    n_seeds = max(8, args.steps)
    seeds = [1 + rank * 100000 + (k % n_seeds) for k in range(args.warmup + args.steps)]
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
    clk = clocks.stop()
    dev_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.warmup, args.warmup + args.steps)]
    st = status.cpu().numpy()
    if np.any(st[:, 0] != 0):
        raise RuntimeError(f"device solve failed: status {st[st[:, 0] != 0][0]}")
    it_np = iters.cpu().numpy()
    timed_iters = int(it_np[args.warmup:].sum())
    total_ms = float(sum(dev_ms))
    # parity guard: the seed-1 loop must take the reference's per-step iteration counts
    x1 = x0_for(pb, system, 1)
    traj1, _ = sess.simulate(x1, T_SIM)
    parity_ok = list(traj1.step_iterations) == GOLDEN_SEED1_ITERS

    # e2e through the public API with host buffers (session cached by dlmpc_simulate)
    e2e_iters, e2e_s = 0, 0.0
    pb.dlmpc_simulate(system, spec, mask, x1, T_SIM, pb.ExecStrategy("b200", device=local))
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
                   "admm_iters_per_step": it_per_launch, "seeds": f"cycled over {n_seeds} per rank",
                   "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "arithmetic": "b200 fast path (null-space Ψ on FP64 DMMA)",
                   "parity_seed1_iterations_equal_reference": parity_ok},
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback B200_PROFILING.md",
                     "algorithmic_bytes_per_iteration": bytes_it, "nnz": nnz,
                     "fp64": {"achieved_tflops": achieved_tf, "peak_tflops": FP64_DMMA_PEAK_TFLOPS,
                              "frac": achieved_tf / FP64_DMMA_PEAK_TFLOPS, "flops_per_iteration": flops_it,
                              "peak_source": "measured DMMA m8n8k4 f64 microbenchmark (profiles/fp64_probe_r01.txt)"},
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
        line["sweep"] = sweep(pb, hbm_peak, 0.0 if args.no_cpu else 6.0)
    if part is not None:
        line["partitioned"] = part
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-sweep", action="store_true", help="skip the N=1e3..1e6 step-0 sweep")
    ap.add_argument("--no-partitioned", action="store_true",
                    help="N>1: skip the graph-partitioned C5 (N=1e6) measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_device_arm(args)


if __name__ == "__main__":
    main()
