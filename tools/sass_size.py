"""Instruction count per kernel in liblasp.so (code size matters: the warp-specialized kernels
must keep their hot loops inside the SM instruction caches)."""
import re, subprocess, sys
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2404_02882_b200/liblasp.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, counts = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1); counts[cur] = 0; continue
    if cur and re.match(r"\s+/\*[0-9a-f]+\*/", line):
        counts[cur] += 1
for k, v in sorted(counts.items(), key=lambda kv: -kv[1]):
    if "tc_kernel" in k or len(sys.argv) > 2:
        print(f"{v:6d} instr ({v * 16 / 1024:6.1f} KB)  {k[:110]}")
