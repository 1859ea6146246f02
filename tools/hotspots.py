"""Per-CUDA-source-line stall samples from an ncu report (cuda,sass source page).
usage: hotspots.py REPORT FUNC_SUBSTRING [TOP]"""
import csv, io, re, subprocess, sys
from collections import defaultdict
rep, func = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg = defaultdict(lambda: [0.0, 0.0, ""])
cur_file = cur_func = None
hdr = None
for line in out:
    if line.startswith('"File Path"'):
        cur_file = next(csv.reader([line]))[1]; hdr = None; continue
    if line.startswith('"Function Name"'):
        cur_func = next(csv.reader([line]))[1]; continue
    if line.startswith('"Line No"'):
        hdr = next(csv.reader([line])); continue
    if hdr is None or func not in (cur_func or ""):
        continue
    r = next(csv.reader([line]))
    if len(r) < 8 or not r[0].strip().isdigit():
        continue
    try:
        s = float(r[4] or 0); ins = float(r[7] or 0)
    except ValueError:
        continue
    key = (cur_file.split("/")[-1], int(r[0]))
    agg[key][0] += s; agg[key][1] += ins; agg[key][2] = r[1]
tot = sum(v[0] for v in agg.values()) or 1; ti = sum(v[1] for v in agg.values()) or 1
print(f"# {func}: total samples {tot:.0f} instr {ti:.0f}")
for (f, ln), (s, ins, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot:5.1f}% ins={100*ins/ti:5.1f}% {f}:{ln}: {src.strip()[:100]}")
