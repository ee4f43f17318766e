"""Warp-stall samples per CUDA source line from an .ncu-rep (dev tool).

python tools/ncu_stalls.py report.ncu-rep [top]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
items, tot, path = [], 0.0, "?"
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) < 5 or r[0] == "Line No" or r[2] != "-":
        continue                                   # cuda rows carry Address "-"
    try:
        v = float(r[4])
    except ValueError:
        continue
    tot += v
    items.append((v, f"{path}:{r[0]}", r[1].strip()[:100]))
items.sort(reverse=True)
for v, loc, src in items[:top]:
    print(f"{100 * v / tot:5.1f}% {loc:>16} {src}")
