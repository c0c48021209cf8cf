"""Per-source-line stall-reason breakdown of an ncu report (top lines by samples).
usage: python tools/ncu_stalls.py report.ncu-rep [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
data = [r for r in rows if r and r[0].isdigit() and len(r) == len(hdr)]
ia = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[ia] or 0) for r in data)
tot_r = {hdr[i]: sum(float(r[i] or 0) for r in data) for i in reasons}
print("kernel stall reasons:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(tot_r.items(), key=lambda x: -x[1]) if v / tot > 0.01))
for r in sorted(data, key=lambda r: -float(r[ia] or 0))[:top]:
    s = float(r[ia] or 0)
    br = sorted(((hdr[i][6:], float(r[i] or 0)) for i in reasons), key=lambda x: -x[1])[:3]
    print(f"{100 * s / tot:5.1f}% L{r[0]:<5} {' '.join(f'{n}:{100 * v / s:.0f}%' for n, v in br if s)}  {r[1].strip()[:70]}")
