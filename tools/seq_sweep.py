"""Sequence-length sweep on one GPU (BASELINE configs[4]: 2K - 2048K tokens, TNL-1B shape 16 x 128 and the
TNL-0.4B shape 16 x 64): device time of one fwd+bwd step replayed from a CUDA graph, inputs resident, L2
flushed between steps. Prints a markdown table (profiles/<tag>_seq_sweep.md).
usage: python tools/seq_sweep.py [steps]   (SWEEP_HD="64,128", SWEEP_N="2048,...": subsets)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2404_02882_b200 as L

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
flush = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
sink = torch.zeros((), dtype=torch.int64, device="cuda")
print("| shape | tokens | us / step | M tokens/s | GB/s (22D algorithmic bytes) |")
print("|---|---|---|---|---|")
hds = [int(x) for x in os.environ.get("SWEEP_HD", "64,128").split(",")]
ns = [int(x) for x in os.environ.get("SWEEP_N", "2048,8192,32768,131072,524288,2097152").split(",")]
for H, D, name in ((16, 64, "16 x 64"), (16, 128, "16 x 128")):
    if D not in hds:
        continue
    for N in ns:
        lam = synth.head_lambdas(H, None)
        g = torch.Generator(device="cuda").manual_seed(N)
        q, k, v, do = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.3).to(torch.bfloat16) for _ in range(4))
        o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))
        cache, ws = L.alloc_cache(q), L.alloc_workspace(q)

        def step():
            L.fwd_local(q, k, v, lam, o=o, kv_out=False, cache=cache, workspace=ws)
            L.bwd_local(q, k, v, lam, do, cache, dq=dq, dk=dk, dv=dv, dkv_out=False, workspace=ws)

        for _ in range(2):
            step()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            step()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(steps):
            torch.sum(flush, dim=0, dtype=torch.int64, out=sink)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gr.replay(); b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        us = tot / steps * 1e3
        print(f"| {name} | {N} | {us:.1f} | {N / us:.1f} | {22 * D * H * N / us / 1e3:.0f} |", flush=True)
        del q, k, v, do, o, dq, dk, dv, cache, ws, gr
        torch.cuda.empty_cache()
