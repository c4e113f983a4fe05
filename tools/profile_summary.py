"""Summarise ncu artefacts into profiles/ (tracked).

usage:
  python tools/profile_summary.py launches <launches.csv> <out.md>          # per-launch device times
  python tools/profile_summary.py full <report.ncu-rep> <out.md> [key]      # one --set full capture
     (key, e.g. "tnl04b:core_fwd_tc", also records dram bytes/launch into profiles/ncu_traffic.json)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
]


def launches(path, out):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        t = float(r["Metric Value"]) / (1e3 if r["Metric Unit"] == "ns" else 1.0)
        agg.setdefault(name, []).append(t)
    total = sum(sum(v) for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({os.path.basename(path)})\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised launches: "
                "compare shares, not absolutes)\n\n| kernel | launches | mean us | total us | share |\n|---|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {100 * sum(v) / total:.1f}% |\n")
    print(open(out).read())


def full(rep, out, key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    got = {}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            got[m] = (vals[i], units[i])
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    with open(out, "w") as f:
        f.write(f"# ncu --set full: `{kname[:120]}`\n\nreport: `{os.path.basename(rep)}` (gpurun_out/, not tracked)\n\n")
        f.write("| metric | value | unit |\n|---|---|---|\n")
        for m, (v, u) in got.items():
            f.write(f"| {m} | {v} | {u} |\n")
        f.write("\n## Section summary (ncu details page)\n\n")
        want = ("Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
                "Executed Ipc Active", "Registers Per Thread", "Achieved Occupancy", "L2 Hit Rate",
                "Warp Cycles Per Issued Instruction", "No Eligible")
        rows = list(csv.reader(io.StringIO(det)))
        if rows:
            h = rows[0]
            iname, iunit, ival = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
            isec = h.index("Section Name")
            seen = set()
            for r in rows[1:]:
                if len(r) > ival and r[iname] in want and (r[isec], r[iname]) not in seen:
                    seen.add((r[isec], r[iname]))
                    f.write(f"- {r[isec]} / {r[iname]}: {r[ival]} {r[iunit]}\n")
    print(open(out).read())
    if key and "dram__bytes_read.sum" in got:
        def to_bytes(v, u):
            v = float(v)
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic = to_bytes(*got["dram__bytes_read.sum"]) + to_bytes(*got["dram__bytes_write.sum"])
        p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        git = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True,
                             cwd=os.path.dirname(p)).stdout.strip() or None
        d[key] = {"bytes": traffic, "report": os.path.basename(rep), "git": git,
                  "note": "dram__bytes_read.sum + dram__bytes_write.sum of one --set full capture (per launch)"}
        json.dump(d, open(p, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
