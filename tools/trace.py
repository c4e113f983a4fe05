"""Timeline of CTA 0 of the tcgen05 core kernel (cycles relative to the first event)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2404_02882_b200 as L
from paper_2404_02882_b200 import _native as N
# usage: python tools/trace.py [n_blocks] [fwd|bwd] [head_dim]   (bwd: the fused dQ/dV/dK launch)
mode = sys.argv[2] if len(sys.argv) > 2 else "fwd"
HD = int(sys.argv[3]) if len(sys.argv) > 3 else 64
p = synth.problem(0, 1, 32768, 16, HD, dtype="bf16")
q, k, v, do = (torch.from_numpy(p[x]).cuda().to(torch.bfloat16) for x in ("q", "k", "v", "do"))
o, _, cache = L.fwd_local(q, k, v, p["lam"]); torch.cuda.synchronize()
buf = torch.zeros(3 * 1024 + 2 * 148, dtype=torch.int64, device="cuda")
N.lib().lasp_debug_trace(ctypes.c_void_p(buf.data_ptr()))
if mode == "bwd":
    L.bwd_local(q, k, v, p["lam"], do, cache)
else:
    L.fwd_local(q, k, v, p["lam"])
torch.cuda.synchronize()
N.lib().lasp_debug_trace(None)
buf = buf[:2 * 16 * 64]
tt = buf.cpu().numpy().reshape(2, 16, 64).astype(np.int64)
t = tt[0]
base = t[t > 0].min()
names = ["tma_issue", "qk_iss", "ds_iss", "out_iss", "mask_beg", "mask_end", "ds_ready", "sbf_next", "o_full", "store", "g_full", "g_pfull", "g_oempty", "st_loaded", "st_iss", "st_done"]
print("J   " + " ".join(f"{n:>9s}" for n in names))
for J in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    print(f"{J:3d} " + " ".join(f"{(t[e, J] - base) if t[e, J] else -1:9d}" for e in range(len(names))))

print("mask warp 3 chunks (c4: before ld, after ld wait, after st), relative to mask_beg")
for J in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    if t[4, J] == 0:
        break
    print(f"{J:3d} " + " ".join(f"{(tt[1, e, J] - t[4, J]) if tt[1, e, J] else -1:6d}" for e in range(12)))
print("state warps: item fetched (absolute, cycles)")
for J in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    if tt[1, 12, J]:
        print(f"{J:3d} {tt[1, 12, J] - base:9d}")
