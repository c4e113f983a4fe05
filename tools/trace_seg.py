"""Per-block role timeline of the segment-state kernel (lasp_debug_trace; build with LASP_TRACE_BUILD)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2404_02882_b200 as L
from paper_2404_02882_b200 import _native as N
p = synth.problem(0, 1, 32768, 16, 64, dtype="bf16", with_do=False)
q, k, v = (torch.from_numpy(p[x]).cuda().to(torch.bfloat16) for x in ("q", "k", "v"))
o, kv, cache = L.fwd_local(q, k, v, p["lam"]); torch.cuda.synchronize()
buf = torch.zeros(2 * 16 * 64, dtype=torch.int64, device="cuda")
N.lib().lasp_debug_trace(ctypes.c_void_p(buf.data_ptr()))
L.fwd_local(q, k, v, p["lam"], o=o, cache=cache); torch.cuda.synchronize()
N.lib().lasp_debug_trace(None)
t = buf.cpu().numpy().reshape(2, 16, 64)[1].astype(np.int64)
# the core kernel overwrote events 0..; seg_state uses 0-3 too, so run seg only: first 4 rows are from the
# last kernel that traced (core). Print rows 0-3.
base = t[t > 0].min()
print("J  " + " ".join(f"{n:>9s}" for n in ["tma_iss", "scl_beg", "scl_end", "mma_iss"]))
for J in range(20):
    print(f"{J:3d} " + " ".join(f"{(t[e, J] - base) if t[e, J] else -1:9d}" for e in range(4)))
