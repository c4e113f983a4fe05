"""Overlap experiment: does a persistent core launch stretch when another stream holds
k SMs while it runs?  A stand-in kernel (lasp_debug_occupy: k CTAs of 200 KB shared memory, one per SM, no
co-resident 224 KB core CTA) starts on a second stream just before the backward and spins for `hold_us`.
The fused backward launch (core_bwd3_tc: dQ, dV, dK) is timed by the library's per-launch CUDA events.

  static assignment (round 1, LASP_STATIC_ITEMS=1): a CTA owns items blockIdx.x + k*grid; the k CTAs that
      cannot start until the hog ends carry a full 1/grid share each -> the launch ends ~hold_us late.
  dynamic claiming (round 2): resident CTAs claim items from a counter -> ~T0 * 148 / (148 - k).

usage: python tools/overlap_exp.py [--config tnl04b|tnl1b] [--child static|dynamic]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(cfg, ks, hold_us, reps):
    import numpy as np
    import torch
    import synth
    import paper_2404_02882_b200 as L
    from paper_2404_02882_b200 import _native as N
    H, D, C = {"tnl04b": (16, 64, 32768), "tnl1b": (16, 128, 32768)}[cfg]
    p = synth.problem(0, 1, C, H, D, dtype="bf16")
    q, k, v, do = (torch.from_numpy(np.ascontiguousarray(p[x])).cuda().to(torch.bfloat16) for x in ("q", "k", "v", "do"))
    o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))
    cache, ws = L.alloc_cache(q), L.alloc_workspace(q)
    lib = N.lib()
    s2 = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    out = {}
    for kk in ks:
        times = []
        for r in range(reps + 1):
            L.fwd_local(q, k, v, p["lam"], o=o, kv_out=False, cache=cache, workspace=ws)
            torch.cuda.synchronize()
            if kk > 0:
                N.check(lib.lasp_debug_occupy(kk, 200 * 1024, float(hold_us), ctypes.c_void_p(s2.cuda_stream)))
            lib.lasp_profile_enable(1)
            L.bwd_local(q, k, v, p["lam"], do, cache, dq=dq, dk=dk, dv=dv, dkv_out=False, workspace=ws)
            lib.lasp_profile_enable(0)
            torch.cuda.synchronize()
            buf = ctypes.create_string_buffer(1 << 14)
            lib.lasp_profile_read(buf, len(buf))
            st = json.loads(buf.value.decode())
            if r > 0:
                times.append(st["core_bwd3_tc"][1] * 1e3)
        out[kk] = sorted(times)[len(times) // 2]
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tnl04b")
    ap.add_argument("--child", default="")
    ap.add_argument("--hold-us", type=float, default=400.0)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    ks = [0, 4, 16, 37]
    if a.child:
        return child(a.config, ks, a.hold_us, a.reps)
    res = {}
    for mode in ("static", "dynamic"):
        env = dict(os.environ, LASP_STATIC_ITEMS="1" if mode == "static" else "0")
        r = subprocess.run([sys.executable, __file__, "--config", a.config, "--child", mode, "--hold-us",
                            str(a.hold_us), "--reps", str(a.reps)], env=env, capture_output=True, text=True, timeout=600)
        if r.returncode:
            print(r.stderr[-3000:])
            return 1
        res[mode] = {int(kk): vv for kk, vv in json.loads(r.stdout.strip().splitlines()[-1]).items()}
    print(f"# {a.config}: fused backward launch (us, median of {a.reps}); hog holds k SMs for {a.hold_us:.0f} us")
    print("| k SMs held | static (r1) | dynamic (r2) | ideal T0*148/(148-k) |")
    print("|---|---|---|---|")
    t0 = res["dynamic"][0]
    for kk in ks:
        print(f"| {kk} | {res['static'][kk]:.1f} | {res['dynamic'][kk]:.1f} | {t0 * 148 / (148 - kk):.1f} |")


if __name__ == "__main__":
    sys.exit(main())
