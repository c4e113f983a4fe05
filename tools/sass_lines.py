"""Attribute SASS instructions of one kernel to source lines / role sections (code-size analysis)."""
import re, subprocess, sys, collections, os, tempfile
lib = "paper_2404_02882_b200/liblasp.so"
pat = sys.argv[1] if len(sys.argv) > 1 else "core_tc_kernelILi64ELNS_3DirE0"
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if "kernels_tc" in f][0]
out = subprocess.run(["nvdisasm", "--print-line-info", "--print-code", os.path.join(d, cub)], capture_output=True, text=True).stdout
cur_fn, loc, counts = None, None, collections.Counter()
for line in out.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        cur_fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        loc = (os.path.basename(m.group(1)), int(m.group(2))); continue
    if cur_fn and pat in cur_fn and re.match(r"\s+/\*[0-9a-f]+\*/", line) and loc:
        counts[loc] += 1
src = open("paper_2404_02882_b200/csrc/kernels_tc.cu").read().splitlines()
# role sections by marker comments
marks = [(i + 1, l.strip()) for i, l in enumerate(src) if "// ----------------------------------------------------------------" in l]
def role(ln):
    r = "prologue"
    for mln, txt in marks:
        if ln >= mln: r = txt.split("-----")[-1].strip()
    return r
by_role = collections.Counter()
for (f, ln), c in counts.items():
    by_role[role(ln) if f == "kernels_tc.cu" else f] += c
print("by role/file:", by_role.most_common())
print("top lines:", [(f"{f}:{ln}", c) for (f, ln), c in counts.most_common(25)])
