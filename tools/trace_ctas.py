"""Per-CTA start/end (globaltimer) of the core kernel vs the CUDA-event duration of the whole launch."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2404_02882_b200 as L
from paper_2404_02882_b200 import _native as N
p = synth.problem(0, 1, 32768, 16, 64, dtype="bf16", with_do=False)
q, k, v = (torch.from_numpy(p[x]).cuda().to(torch.bfloat16) for x in ("q", "k", "v"))
o, kv, cache = L.fwd_local(q, k, v, p["lam"]); torch.cuda.synchronize()
buf = torch.zeros(2 * 1024 + 2 * 148, dtype=torch.int64, device="cuda")
N.lib().lasp_debug_trace(ctypes.c_void_p(buf.data_ptr()))
L.lib = N.lib()
N.lib().lasp_profile_enable(1)
L.fwd_local(q, k, v, p["lam"], o=o, cache=cache); torch.cuda.synchronize()
N.lib().lasp_profile_enable(0)
b = ctypes.create_string_buffer(4096); N.lib().lasp_profile_read(b, 4096); print(b.value.decode())
N.lib().lasp_debug_trace(None)
t = buf.cpu().numpy()[2048:].reshape(148, 2).astype(np.int64)
t0 = t[:, 0].min()
st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
print("start us: min %.2f med %.2f max %.2f" % (st.min(), np.median(st), st.max()))
print("end   us: min %.2f med %.2f max %.2f" % (en.min(), np.median(en), en.max()))
print("slowest CTAs:", np.argsort(-en)[:8], en[np.argsort(-en)[:8]])
