"""Top CUDA source lines by warp-stall samples from an ncu report (needs -lineinfo builds).
usage: python tools/ncu_src.py report.ncu-rep [N]"""
import csv, io, os, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
items, file, hdr = [], "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        file = os.path.basename(r[1]); continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 5 or not r[0].isdigit():
        continue
    try:
        v = int(r[4])
    except ValueError:
        continue
    items.append((v, f"{file}:{r[0]}", r[1].strip()[:100]))
tot = sum(v for v, *_ in items)
print("total samples", tot)
for v, loc, src in sorted(items, reverse=True)[:n]:
    print(f"{v:7d} {100 * v / max(tot, 1):5.1f}%  {loc:22s} {src}")
