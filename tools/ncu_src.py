"""Top CUDA source lines by warp-stall samples (with the dominant stall reasons) from an ncu report.
usage: python tools/ncu_src.py report.ncu-rep [N] [line_lo line_hi]"""
import csv, io, os, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
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
    ln = int(r[0])
    if not (lo <= ln <= hi) and file == "kernels_tc.cu":
        continue
    reasons = []
    for ci, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try:
                c = int(r[ci])
            except (ValueError, IndexError):
                continue
            if c:
                reasons.append((c, name[6:]))
    reasons.sort(reverse=True)
    items.append((v, f"{file}:{ln}", r[1].strip()[:80], " ".join(f"{nm}={c}" for c, nm in reasons[:3])))
tot = sum(v for v, *_ in items)
print("total samples", tot)
for v, loc, src, rs in sorted(items, reverse=True)[:n]:
    print(f"{v:6d} {100 * v / max(tot, 1):5.1f}% {loc:20s} {src:80s} | {rs}")
