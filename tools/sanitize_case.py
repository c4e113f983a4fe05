"""Small fwd + bwd through every kernel family (tcgen05 D=64 / D=128, CUDA-core fp32, prefix, combine via
the loopback ring) for compute-sanitizer runs: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2404_02882_b200 as L

for D, dt, tdt in ((64, "bf16", torch.bfloat16), (128, "bf16", torch.bfloat16), (32, "fp32", torch.float32)):
    p = synth.problem(1, 1, 1000, 2, D, dtype=dt)  # ragged: 1000 = 7 blocks + 104
    q, k, v, do = (torch.from_numpy(p[x]).cuda().to(tdt) for x in ("q", "k", "v", "do"))
    kv_in = torch.randn(1, 2, D, D, device="cuda")
    o, kv, cache = L.fwd_local(q, k, v, p["lam"], kv_in=kv_in)
    dq, dk, dv, dkv = L.bwd_local(q, k, v, p["lam"], do, cache, dkv_in=kv_in)
    torch.cuda.synchronize()
    print("ok", D, dt, float(o.float().abs().sum()), float(dq.float().abs().sum()), flush=True)
