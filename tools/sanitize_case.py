"""Small fwd + bwd through every kernel family (tcgen05 D=64 / D=128, grouped queries, the NEXT-3 layer with the
Norm epilogue / Norm-backward B1, CUDA-core fp32, prefix, the NEXT-4 generalised-decay kernels) for
compute-sanitizer runs: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
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

# grouped queries (tcgen05 GQ instantiations)
p = synth.problem(2, 1, 700, 4, 64, dtype="bf16", kv_heads=2)
q, do = (torch.from_numpy(p[x]).cuda().to(torch.bfloat16) for x in ("q", "do"))
k, v = (torch.from_numpy(p[x]).cuda().to(torch.bfloat16) for x in ("k", "v"))
o, kv, cache = L.fwd_local(q, k, v, p["lam"])
g = L.bwd_local(q, k, v, p["lam"], do, cache)
torch.cuda.synchronize()
print("ok gqa", float(o.float().abs().sum()), flush=True)
# NEXT-3 layer (Norm epilogue at D = 64 and D = 128)
for D in (64, 128):
    t = synth.layer_problem(3, 1, 600, 2, 2, D, 2 * D)
    x, wq, wk, wv, dy = (torch.from_numpy(t[n]).cuda().to(torch.bfloat16) for n in ("x", "w_q", "w_k", "w_v", "dy"))
    fw = L.layer_fwd(x, wq, wk, wv, t["lam"], 2)
    gb = L.layer_bwd(x, wq, wk, wv, t["lam"], fw, dy)
    torch.cuda.synchronize()
    print("ok layer", D, float(gb["dx"].float().abs().sum()), flush=True)
# NEXT-4 generalised decay (all modes, D = 32 / 64 / 128, ragged)
for D in (32, 64, 128):
    t = synth.gla_problem(4, 1, 333, 2, D)
    q, k, v, lg, do = (torch.from_numpy(t[n]).cuda() for n in ("q", "k", "v", "lg", "do"))
    o, kv, cache = L.gla_fwd_local(q, k, v, lg)
    dq, dk, dv, dlg, dkv = L.gla_bwd_local(q, k, v, lg, do, cache)
    torch.cuda.synchronize()
    print("ok gla", D, float(dlg.abs().sum()), flush=True)
