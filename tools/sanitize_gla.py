"""The NEXT-4 generalised-decay kernels alone (plain global stores, cp.async loads) for compute-sanitizer
initcheck: outputs read back by torch must not be flagged (contrast: TMA-stored outputs of the tcgen05 path are
not tracked by initcheck and are flagged when torch reads them)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2404_02882_b200 as L

for D in (32, 64, 128):
    t = synth.gla_problem(4, 1, 333, 2, D)
    q, k, v, lg, do = (torch.from_numpy(t[n]).cuda() for n in ("q", "k", "v", "lg", "do"))
    o, kv, cache = L.gla_fwd_local(q, k, v, lg)
    dq, dk, dv, dlg, dkv = L.gla_bwd_local(q, k, v, lg, do, cache)
    torch.cuda.synchronize()
    print("ok gla", D, float(o.abs().sum()), float(dlg.abs().sum()), flush=True)
