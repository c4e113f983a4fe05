"""Quick GPU check of the bf16 path on small shapes: prints normwise errors vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2404_02882_b200 as L

def run(N, H, D, seed=0, lam=None, B=1):
    p = synth.problem(seed, B, N, H, D, dtype="bf16", lam=lam)
    dev = {k: torch.from_numpy(p[k]).cuda().to(torch.bfloat16) for k in ("q", "k", "v", "do")}
    o, kv, cache = L.fwd_local(dev["q"], dev["k"], dev["v"], p["lam"])
    torch.cuda.synchronize()
    ref = oracle.fwd(p["q"], p["k"], p["v"], p["lam"])
    e = oracle.normwise_err(o.float().cpu().numpy(), ref)
    print(f"N={N} H={H} D={D} lam={lam} fwd o err {e:.3e}", flush=True)
    if e > 2e-2:
        oo = o.float().cpu().numpy()
        bad = np.abs(oo - ref).max(axis=(0, 2, 3))
        rows = np.nonzero(bad > 1e-2 * np.abs(ref).max())[0]
        print("  bad rows:", rows[:20], "count", len(rows))
        print("  got", oo[0, rows[:2], 0, :4], "ref", ref[0, rows[:2], 0, :4])
    dq, dk, dv, dkv = L.bwd_local(dev["q"], dev["k"], dev["v"], p["lam"], dev["do"], cache)
    torch.cuda.synchronize()
    g = oracle.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])
    for name, x, r in zip(("dq", "dk", "dv"), (dq, dk, dv), g):
        print(f"   {name} err {oracle.normwise_err(x.float().cpu().numpy(), r):.3e}", flush=True)

if __name__ == "__main__":
    for args in [(128, 1, 64, 0, 0.9), (256, 1, 64, 0, 0.9), (1000, 2, 64, 1, None), (4096, 4, 64, 2, None)]:
        run(*args)
