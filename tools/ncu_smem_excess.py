"""Per-source-line shared-memory wavefronts (total and excessive = bank
conflicts) of an ncu --set full capture with source.
usage: python tools/ncu_smem_excess.py report.ncu-rep [top]"""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
hdr=None; lines=[]
for ln in out:
    if ln.startswith('"Line No"'):
        hdr = next(csv.reader([ln])); continue
    if hdr is None or not ln.startswith('"') or not ln[1:2].isdigit(): continue
    parts = ln.split('","'); nmet = len(hdr) - 4
    met = [p.strip('"') for p in parts[-nmet:]]
    src = '","'.join(parts[1:len(parts) - nmet - 2])
    lines.append((int(parts[0].strip('"')), src, met))
names = hdr[4:]
ix = names.index("L1 Wavefronts Shared Excessive"); iw = names.index("L1 Wavefronts Shared")
tot = sum(float(m[ix] or 0) for _,_,m in lines); totw = sum(float(m[iw] or 0) for _,_,m in lines)
print("excessive shared wavefronts", tot, "of", totw)
for no, src, m in sorted(lines, key=lambda x: -float(x[2][ix] or 0))[:top]:
    print(int(float(m[ix] or 0)), int(float(m[iw] or 0)), no, src.strip()[:110])
