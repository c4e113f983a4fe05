"""Closed-form spot check at long lengths: constant inputs per head (lambda = 0.999 and 1) through fwd_local,
compared with the geometric-series closed form (debug companion of the config-5 closed-form tests)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2404_02882_b200 as L
N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
H, D = 2, 64
lam = np.array([0.999, 1.0], dtype=np.float32)
rng = np.random.default_rng(0)
qv, kv_, vv, dov = (synth.round_bf16(rng.standard_normal((H, D)).astype(np.float32) * 0.3) for _ in range(4))
mk = lambda a: torch.from_numpy(np.broadcast_to(a, (1, N, H, D)).copy()).to(torch.bfloat16).cuda()
o, kvo, cache = L.fwd_local(mk(qv), mk(kv_), mk(vv), lam)
torch.cuda.synchronize()
s = np.arange(1, N + 1, dtype=np.float64)
for h in range(H):
    l = float(lam[h]); geo = (lambda n: n) if l == 1.0 else (lambda n: (1 - l ** n) / (1 - l))
    qk = float(qv[h].astype(np.float64) @ kv_[h])
    idx = np.arange(0, N, max(1, N // 64))
    got = o[0, idx, h].float().cpu().numpy()
    ref = qk * np.outer(geo(s[idx]), vv[h])
    err = np.abs(got - ref).max(axis=1) / np.abs(ref).max(axis=1)
    print("h", h, "rel err by row:", " ".join(f"{i}:{e:.1e}" for i, e in zip(idx[::4], err[::4])))
    kref = geo(N) * np.outer(kv_[h], vv[h])
    print("   kv_out rel err", np.abs(kvo[0, h].cpu().numpy() - kref).max() / np.abs(kref).max())
dov_t = mk(dov)
dq, dk, dv, dkv = L.bwd_local(mk(qv), mk(kv_), mk(vv), lam, dov_t, cache)
torch.cuda.synchronize()
for h in range(H):
    l = float(lam[h]); geo = (lambda n: n) if l == 1.0 else (lambda n: (1 - l ** n) / (1 - l))
    qk = float(qv[h].astype(np.float64) @ kv_[h]); vd = float(vv[h].astype(np.float64) @ dov[h])
    idx = np.arange(0, N, max(1, N // 64))
    for name, t, ref in (("dq", dq, vd * np.outer(geo(s[idx]), kv_[h])), ("dk", dk, vd * np.outer(geo(N - s[idx] + 1), qv[h])),
                         ("dv", dv, qk * np.outer(geo(N - s[idx] + 1), dov[h]))):
        got = t[0, idx, h].float().cpu().numpy()
        err = np.abs(got - ref).max(axis=1) / np.abs(ref).max(axis=1)
        print("h", h, name, " ".join(f"{i}:{e:.1e}" for i, e in zip(idx[::4], err[::4])))
