"""Summarise one ncu --set full capture (raw page) into a JSON dict.
usage: python tools/ncu_summary.py report.ncu-rep out.json 'command' 'workload' algorithmic_bytes iterations"""
import csv, io, json, subprocess, sys
rep, out, cmd, workload = sys.argv[1:5]
alg_bytes = float(sys.argv[5]) if len(sys.argv) > 5 else None
iters = int(sys.argv[6]) if len(sys.argv) > 6 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v)); un = dict(zip(h, u))
def f(k, scale=1.0):
    try:
        return float(d[k]) * scale
    except (KeyError, ValueError):
        return None
unit_scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
rd = f("dram__bytes_read.sum", unit_scale.get(un.get("dram__bytes_read.sum"), 1.0))
wr = f("dram__bytes_write.sum", unit_scale.get(un.get("dram__bytes_write.sum"), 1.0))
dur = f("gpu__time_duration.sum", {"ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(un.get("gpu__time_duration.sum"), 1.0))
res = {
    "command": cmd, "workload": workload,
    "kernel": d.get("Kernel Name", "")[:120],
    "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
    "registers_per_thread": d.get("launch__registers_per_thread"),
    "dynamic_smem_kb": d.get("launch__shared_mem_per_block_dynamic"),
    "duration_ms_under_ncu": dur,
    "dram_bytes_read": rd, "dram_bytes_write": wr,
    "dram_bytes_per_launch": (rd or 0) + (wr or 0),
    "algorithmic_bytes_per_launch": alg_bytes,
    "admm_iterations_in_launch": iters,
    "l2_hit_rate_pct": f("lts__t_sector_hit_rate.pct"),
    "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "tensor_pipe_active_pct": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
