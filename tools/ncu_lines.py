"""Summarise an ncu report's per-source-line warp-stall samples.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
hdr = None
lines = []
for ln in out:
    if ln.startswith('"Line No"'):
        hdr = next(csv.reader([ln]))
        continue
    if hdr is None or not ln.startswith('"') or not ln[1:2].isdigit():
        continue
    parts = ln.split('","')
    nmet = len(hdr) - 4
    met = [p.strip('"') for p in parts[-nmet:]]
    src = '","'.join(parts[1:len(parts) - nmet - 2])
    lines.append((int(parts[0].strip('"')), src, met))
names = hdr[4:]
i_all = names.index("Warp Stall Sampling (All Samples)")
i_inst = names.index("Instructions Executed")
tot = sum(float(m[i_all] or 0) for _, _, m in lines)
tot_i = sum(float(m[i_inst] or 0) for _, _, m in lines)
print(f"total stall samples {tot:.0f}, instructions {tot_i:.3g}")
for no, src, m in sorted(lines, key=lambda x: -float(x[2][i_all] or 0))[:top]:
    print(f"{100 * float(m[i_all]) / tot:5.1f}%  inst {100 * float(m[i_inst] or 0) / tot_i:5.1f}%  L{no:<5} {src.strip()[:100]}")
