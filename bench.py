#!/usr/bin/env python
"""bench.py -- LASP forward+backward tokens/s per layer on B200 (BASELINE.json metric).

One step = one pass of the whole hot path over one batch: lasp forward (F1 seg states, F2 prefix /
ring hop, F3 fused intra+inter core) and lasp backward (B3 dQ core, B1 seg states, B2 prefix / ring
hop, B3 dV and dK cores) for one attention layer, inputs resident in HBM.

Workload (N=1: BASELINE configs[1], the TNL-0.4B layer): 16 heads x 64, batch 1, 32K tokens per GPU,
bf16, per-head lambda_h = 1 - 2^-(1 + 14h/15). N>1 keeps 32K tokens per GPU (weak scaling) and runs the
NCCL KV/dKV ring (one process per GPU, launched by torchrun). Synthetic inputs from synth/ (seeded).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lasp|reference] [--config tnl04b|tnl1b|tnl7b]
       [--exchange all|both|ring|allgather|p2p] [--sp-size T] [--loopback N] [--tokens C] [--no-graph] [--no-e2e]
       [--no-cpu-baseline]

Before timing, every rank runs one fwd+bwd of constant per-head inputs through the same code path (ring /
all-gather / local) and checks the closed forms of SURVEY §8(c) pin 5 at sampled global positions; the worst
error (max over ranks) is printed as parity_max_err / parity_ok.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (heads, head_dim, tokens per GPU, description)
    "tnl04b": (16, 64, 32768, "TNL-0.4B layer (BASELINE configs[1]): 16 heads x 64, batch 1, 32K tokens/GPU"),
    "tnl1b": (16, 128, 32768, "TNL-1B layer (BASELINE configs[2] per-GPU shard): 16 heads x 128, 32K tokens/GPU"),
    "tnl7b": (32, 128, 131072, "TNL-7B layer (BASELINE configs[3] per-GPU shard): 32 heads x 128, 128K tokens/GPU"),
}
METRIC = "LASP fwd+bwd tokens/sec per layer"
FLOP_BLOCK = 64  # algorithmic flops fixed at b = 64


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", 0)), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def alg_flops_per_token_head(D):
    return 7 * (FLOP_BLOCK + 1) * D + 12 * D * D


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        if self.index is None or self.index < 0:
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "hw_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                "sw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "hw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_power_cap": getattr(pynvml, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for n, bit in names.items():
                            if r & bit:
                                self.reasons.add(n)
                    except Exception:
                        pass
                    self._stop.wait(0.02)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML unavailable: report it instead of inventing clocks
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------------------------------
def run_reference(args):
    """The oracle as it stands (fp64 C, host cores) on a bounded token sample of the same workload."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    import synth
    H, D, C, desc = CONFIGS[args.config]
    oracle.build()
    threads = os.cpu_count() or 1
    cores = min(threads, H)  # one work item per (batch, head)

    def step(p):
        oracle.fwd(p["q"], p["k"], p["v"], p["lam"], nthreads=threads)
        oracle.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"], nthreads=threads)

    cal = synth.problem(0, 1, 256, H, D, dtype="bf16", token_hi=256)
    t = time.perf_counter()
    step(cal)
    per_tok = (time.perf_counter() - t) / 256
    budget = float(os.environ.get("LASP_REF_BUDGET_S", "90"))
    S = int(max(128, min(C, budget / max(1, args.steps + args.warmup) / max(per_tok, 1e-9))))
    p = synth.problem(0, 1, C * world, H, D, dtype="bf16", token_lo=0, token_hi=S)
    for _ in range(args.warmup):
        step(p)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(p)
    el = time.perf_counter() - t0
    value = S * args.steps / el
    sample = f"first {S} tokens of the {desc} sequence, fwd+bwd, fp64 oracle, {args.steps} steps"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (synth/, seed 0)",
            "config": {"workload": desc, "global_batch": 1, "seq_len": C * world, "n_local": C, "heads": H,
                       "head_dim": D, "parallelism": f"sp{world}"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "nproc": cpu_info()[0],
                             "cpu_model": cpu_info()[1], "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(H, D, C, desc):
    import oracle
    import synth
    oracle.build()
    threads = os.cpu_count() or 1
    p = synth.problem(0, 1, C, H, D, dtype="bf16")
    reps, el = 0, 0.0
    t0 = time.perf_counter()
    while reps < 3 and (el < 10.0 or reps == 0):
        oracle.fwd(p["q"], p["k"], p["v"], p["lam"], nthreads=threads)
        oracle.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"], nthreads=threads)
        reps += 1
        el = time.perf_counter() - t0
    nproc, model = cpu_info()
    return {"value": C * reps / el, "unit": "tokens/s", "cores": min(threads, H), "nproc": nproc, "cpu_model": model,
            "kind": "oracle",
            "sample": f"full {desc} layer, fwd+bwd in fp64, {reps} rep(s), {el:.1f} s on {min(threads, H)} threads "
                      f"(one per (batch, head) work item; host has {nproc})"}


# ----------------------------------------------------------------------------------------------------
class TorchComm:
    """Barrier / max-over-ranks for one process per GPU (torch.distributed over NCCL; gloo with --transport p2p)."""

    def __init__(self, world, dev, gloo=False):
        self.world, self.dev, self.gloo = world, dev, gloo

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            if self.gloo:
                dist.barrier()
            else:
                dist.barrier(device_ids=[self.dev.index])

    def max(self, x):
        if self.world == 1:
            return float(x)
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(x)], dtype=torch.float64, device="cpu" if self.gloo else self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())


class ThreadComm:
    """The same for --loopback: ranks are threads of this process on one GPU."""

    def __init__(self, world):
        self.world = world
        self._bar = threading.Barrier(world)
        self._vals = [0.0] * world
        self._lock = threading.Lock()

    def barrier(self):
        self._bar.wait(timeout=600)

    def max(self, x, rank=None):
        self.barrier()
        with self._lock:
            self._vals[rank] = float(x)
        self.barrier()
        m = max(self._vals)
        self.barrier()
        return m


def closed_form_check(lasp, dev, B, C, H, D, lam, rank, T, run, Hk=None, sync=None):
    """Self-check of the timed configuration before timing (every rank, every exchange): constant inputs
    q_s = q, k_s = k, v_s = v, do_s = do per head have closed forms derived from Eq. 4 (SURVEY §8(c) pin 5,
    the same forms tests/test_gpu_parity.py checks): with s the GLOBAL 1-based position and N = T*C,
      o_s = (q.k) v g(s),  dq_s = (v.do) k g(s),  dk_s = (v.do) q g(N-s+1),  dv_s = (q.k) do g(N-s+1),
    g(n) = (1 - lam^n) / (1 - lam) (n for lam = 1). Grouped queries (Hk < H): query head h uses kv-head
    h // (H/Hk) and its lambda; dk, dv of a kv-head sum the terms of its query heads.
    Returns the worst normwise error at sampled positions."""
    import numpy as np
    import torch
    Hk = Hk or H
    G = H // Hk
    rng = np.random.default_rng(123)
    shapes = [(H, D), (Hk, D), (Hk, D), (H, D)]
    vecs = [rng.standard_normal(sh).astype(np.float32) * 0.3 for sh in shapes]
    vecs = [torch.from_numpy(v).to(torch.bfloat16).float().numpy().astype(np.float64) for v in vecs]
    qv, kv_, vv, dov = vecs
    mk = lambda a: torch.from_numpy(np.broadcast_to(a.astype(np.float32), (B, C) + a.shape).copy()).to(
        device=dev, dtype=torch.bfloat16)
    o, dq, dk, dv = run(mk(qv), mk(kv_), mk(vv), mk(dov))
    (sync or (lambda: torch.cuda.synchronize(dev)))()
    N = T * C
    idx = np.unique(np.clip(np.array([0, 1, 2, 127, 128, 1000, C // 2, C - 2, C - 1]), 0, C - 1))
    s = (rank * C + idx + 1).astype(np.float64)
    worst = 0.0

    def geo(l):
        return (lambda n: n) if l == 1.0 else (lambda n: (1 - l ** n) / (1 - l))

    def err(got, h, ref):
        x = got[0, idx, h].float().cpu().numpy().astype(np.float64)
        return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-30))

    for h in range(H):
        hk = h // G
        g = geo(float(np.float64(np.float32(lam[hk]))))
        qk, vd = float(qv[h] @ kv_[hk]), float(vv[hk] @ dov[h])
        worst = max(worst, err(o, h, qk * np.outer(g(s), vv[hk])), err(dq, h, vd * np.outer(g(s), kv_[hk])))
    for hk in range(Hk):
        g = geo(float(np.float64(np.float32(lam[hk]))))
        rk = sum(float(vv[hk] @ dov[h]) * qv[h] for h in range(hk * G, (hk + 1) * G))
        rv = sum(float(qv[h] @ kv_[hk]) * dov[h] for h in range(hk * G, (hk + 1) * G))
        worst = max(worst, err(dk, hk, np.outer(g(N - s + 1), rk)), err(dv, hk, np.outer(g(N - s + 1), rv)))
    return worst


def layer_bench(args, lasp, dev, stream, B, C, H, Hk, D, l2_flush):
    """one whole attention layer, Y = Norm(LASP(X W_Q, X W_K, X W_V)) forward and its
    backward (dX, dW_Q, dW_K, dW_V) through lasp_layer_fwd / lasp_layer_bwd (cuBLAS projections, Norm fused
    into the core epilogue / the B1 kernel), d_model = H * D, graph-replayed like the main line, L2 flushed
    between steps. Reported next to the attention-only number, not instead of it."""
    import torch

    import synth
    d = H * D
    t = synth.layer_problem(0, B, C, H, Hk, D, d)
    x, wq, wk, wv, dy = (torch.from_numpy(t[n]).to(dev, torch.bfloat16) for n in ("x", "w_q", "w_k", "w_v", "dy"))
    fw = lasp.layer_fwd(x, wq, wk, wv, t["lam"], H)
    g = lasp.layer_bwd(x, wq, wk, wv, t["lam"], fw, dy)
    outs_f = {n: fw[n] for n in ("q", "k", "v", "y", "rnorm", "cache")}
    outs_b = dict(g)

    def step():
        lasp.layer_fwd(x, wq, wk, wv, t["lam"], H, out=outs_f, workspace=fw["workspace"])
        lasp.layer_bwd(x, wq, wk, wv, t["lam"], fw, dy, out=outs_b)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    graph = None
    if args.graph:
        try:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                step()
            gr.replay()
            torch.cuda.synchronize(dev)
            graph = gr
        except Exception:  # noqa: BLE001 - eager fallback, reported
            torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        l2_flush()
        ev[i][0].record(stream)
        graph.replay() if graph is not None else step()
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    flops = 2 * 3 * B * C * d * (H + 2 * Hk) * D  # projection GEMMs: fwd X W, bwd dX and dW; 2 flop per MAC
    return {"metric": "layer fwd+bwd tokens/sec (projections + LASP + Norm)", "value": B * C / (ms / 1e3),
            "unit": "tokens/s", "ms_per_step": ms, "d_model": d, "launch": "cuda-graph replay" if graph else "eager",
            "projection_gflop_per_step": flops / 1e9}


def gla_bench(args, lasp, lib, dev, stream, B, C, H, D, l2_flush):
    """the generalised-decay path (GLA / GateLoop row of Table 3) at the same shape, fp32
    inputs (q, k, v, do, log decay), fwd + bwd (dQ, dK, dV, dlog_g) through lasp_gla_fwd_local / _bwd_local,
    graph-replayed, L2 flushed between steps. Roofline: CUDA-core ALU issue (the kernels are FP32-pipe
    recurrences): 16 D^2 FP32 lane-instructions per token-head (F1 2, F3 3, B1 2, dQ 3, dV 3, dK 3) against
    148 SMs x 128 FP32 lanes x the max SM clock."""
    import ctypes
    import json as _json

    import torch

    import synth
    t = synth.gla_problem(0, B, C, H, D)
    q, k, v, do, lg = (torch.from_numpy(t[n]).to(dev) for n in ("q", "k", "v", "do", "lg"))
    cache, ws = lasp.gla_alloc(q)
    o, dq, dk, dv, dlg = (torch.empty_like(q) for _ in range(5))

    def step():
        lasp.gla_fwd_local(q, k, v, lg, o=o, kv_out=False, cache=cache, workspace=ws)
        lasp.gla_bwd_local(q, k, v, lg, do, cache, dq=dq, dk=dk, dv=dv, dlog_g=dlg, dkv_out=False, workspace=ws)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    graph = None
    if args.graph:
        try:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                step()
            gr.replay()
            torch.cuda.synchronize(dev)
            graph = gr
        except Exception:  # noqa: BLE001 - eager, reported
            torch.cuda.synchronize(dev)
    n = max(3, min(args.steps, 10))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for i in range(n):
        l2_flush()
        ev[i][0].record(stream)
        graph.replay() if graph is not None else step()
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = sum(a.elapsed_time(b) for a, b in ev) / n
    # per-kernel times (profiled eager pass)
    lib.lasp_profile_enable(1)
    for _ in range(n):
        step()
    torch.cuda.synchronize(dev)
    lib.lasp_profile_enable(0)
    buf = ctypes.create_string_buffer(1 << 16)
    lib.lasp_profile_read(buf, len(buf))
    stages = {kk: vv[1] / n for kk, vv in _json.loads(buf.value.decode() or "{}").items()}
    ops = 16 * D * D * B * C * H
    clk = peaks_clock()
    peak = 148 * 128 * clk * 1e6 / 1e9  # G lane-ops / s
    return {"metric": "generalised-decay (GLA) fwd+bwd tokens/sec", "value": B * C / (ms / 1e3), "unit": "tokens/s",
            "ms_per_step": ms, "dtype": "fp32", "launch": "cuda-graph replay" if graph else "eager",
            "stages_ms_per_step": stages,
            "roofline": {"bound": "alu", "achieved": ops / (ms / 1e3) / 1e9, "peak": peak, "unit": "G FP32 lane-ops/s",
                         "frac": ops / (ms / 1e3) / 1e9 / peak, "ops_rule": "16 D^2 FP32 lane-instructions per token-head",
                         "peak_rule": "148 SMs x 128 FP32 lanes x sm_max_mhz"}}


def peaks_clock():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0))
    except Exception:  # noqa: BLE001
        return 1965.0


def cpu_info():
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def rank_bench(args, rank, world, dev, comm, make_ring, loopback=False, shared_device=False):
    """One rank's measurement (returns the JSON line on rank 0, None elsewhere)."""
    import ctypes

    import torch

    import synth
    import paper_2404_02882_b200 as lasp
    from paper_2404_02882_b200 import _native as N

    H, D, C, desc = CONFIGS[args.config]
    if args.tokens:
        C = args.tokens
    Hk = args.kv_heads or H
    if Hk != H:
        desc = f"{desc} [grouped-query: {Hk} kv-heads]"
    B = 1
    lib = N.lib()
    T = args.sp_size or world
    grp_id, grank, _ = lasp.topology(rank, world, T)
    G = world // T
    stream = torch.cuda.current_stream(dev)

    def sync():
        # loopback ranks are threads sharing one device: a device-wide synchronize from one rank's thread would also
        # wait for the other ranks' streams, which the P2P exchange's device-side waits make mutually dependent
        if loopback or shared_device:
            stream.synchronize()
        else:
            torch.cuda.synchronize(dev)
    # inputs: this rank's shard [t*C, (t+1)*C) of its group's sequence (seed = group id)
    p = synth.problem(grp_id, B, C * T, H, D, dtype="bf16", token_lo=grank * C, token_hi=(grank + 1) * C,
                      kv_heads=Hk)
    lam = p["lam"]
    host = {k: torch.from_numpy(p[k]) for k in ("q", "k", "v", "do")}
    d_in = {k: v.to(dev, torch.bfloat16) for k, v in host.items()}
    q, k, v, do = d_in["q"], d_in["k"], d_in["v"], d_in["do"]
    o, dq = torch.empty_like(q), torch.empty_like(q)
    dk, dv = torch.empty_like(k), torch.empty_like(v)
    cache, ws = lasp.alloc_cache(q, k), lasp.alloc_workspace(q, k)
    p2p_skipped = None
    # N > 1: time the paper's ring and the all-gather exchange (NEXT-2) in the same run; `value` is the ring
    if T > 1:
        exchanges = {"all": ["ring", "allgather", "p2p", "p2p_allgather"], "both": ["ring", "allgather"]}.get(args.exchange,
                                                                                            [args.exchange])
        ring = make_ring()
        if any(x.startswith("p2p") for x in exchanges) and not getattr(ring, "_p2p", False):  # peer-memory exchanges
            ok, p2p_note = 1.0, "a peer rank failed to set up"
            try:
                ring.enable_p2p(B * Hk * D * D)
            except Exception as e:  # noqa: BLE001 - e.g. no CUDA IPC between these processes: reported, not fatal
                ok = 0.0
                p2p_note = f"{type(e).__name__}: {e}"
            ok = -(comm.max(-ok, rank) if loopback else comm.max(-ok))  # every rank must have connected
            if ok < 1.0:
                exchanges = [x for x in exchanges if not x.startswith("p2p")]
                ring.set_exchange("ring")
                p2p_skipped = p2p_note
    else:
        exchanges, ring = ["none"], None

    def step_fn(ex):
        def step():
            if ring is None:
                lasp.fwd_local(q, k, v, lam, o=o, kv_out=False, cache=cache, workspace=ws)
                lasp.bwd_local(q, k, v, lam, do, cache, dq=dq, dk=dk, dv=dv, dkv_out=False, workspace=ws)
            else:
                ring.fwd(q, k, v, lam, o=o, cache=cache, workspace=ws)
                ring.bwd(q, k, v, lam, do, cache, dq=dq, dk=dk, dv=dv, workspace=ws)
        return step

    if loopback and exchanges and exchanges[0].startswith("p2p"):
        # thread-ranks share one context: load every kernel over the host transport first, since a first launch
        # (lazy module loading) synchronizes the context and must not meet a peer's spinning hop kernel
        ring.set_exchange("ring")
        step_fn("ring")()
        sync()

    # L2 flush between timed steps: READ a 256 MiB buffer (> 126 MB L2), so L2 holds clean lines and no
    # write-back of the flush lands inside the next step (a write-based flush would)
    flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)
    flush_sink = torch.zeros((), dtype=torch.int64, device=dev)

    def l2_flush():
        torch.sum(flush, dim=0, dtype=torch.int64, out=flush_sink)

    results = {}
    clk_summary = None
    for ex in exchanges:
        if ring is not None:
            ring.set_exchange(ex)
        # (0) parity gate through this exact code path (closed forms, every rank), before any timing
        cws, ccache = lasp.alloc_workspace(q, k), lasp.alloc_cache(q, k)

        def run_const(a, b, c, d):
            oo, dd = torch.empty_like(a), [torch.empty_like(a), torch.empty_like(b), torch.empty_like(c)]
            if ring is None:
                lasp.fwd_local(a, b, c, lam, o=oo, kv_out=False, cache=ccache, workspace=cws)
                lasp.bwd_local(a, b, c, lam, d, ccache, dq=dd[0], dk=dd[1], dv=dd[2], dkv_out=False, workspace=cws)
            else:
                ring.fwd(a, b, c, lam, o=oo, cache=ccache, workspace=cws)
                ring.bwd(a, b, c, lam, d, ccache, dq=dd[0], dk=dd[1], dv=dd[2], workspace=cws)
            return [oo] + dd
        err = closed_form_check(lasp, dev, B, C, H, D, lam, grank, T, run_const, Hk, sync)
        err = comm.max(err, rank) if loopback else comm.max(err)
        del cws, ccache
        step = step_fn(ex)
        for _ in range(args.warmup):
            step()
        sync()
        # the step's launches captured once into a CUDA graph (programmatic-dependent-launch edges and the
        # NCCL ring kept), replayed in the timed region: same kernels, no per-launch host work
        graph, graph_launches, graph_note = None, 0, None
        if args.graph and not loopback:
            try:
                comm.barrier()
                g = torch.cuda.CUDAGraph()
                l0 = lib.lasp_launch_count()
                with torch.cuda.graph(g):
                    step()
                graph_launches = lib.lasp_launch_count() - l0
                g.replay()
                sync()
                graph = g
            except Exception as e:  # noqa: BLE001 - reported in the line
                graph_note = f"capture failed ({type(e).__name__}: {e}); eager"
                sync()

        def timed_loop(n, profile):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
            if not loopback or rank == 0:
                lib.lasp_profile_enable(1 if profile else 0)
            comm.barrier()
            sync()
            comm.barrier()
            for i in range(n):
                l2_flush()                       # outside the step events
                ev[i][0].record(stream)
                if graph is not None and not profile:
                    graph.replay()
                else:
                    step()
                ev[i][1].record(stream)
            sync()
            comm.barrier()
            if not loopback or rank == 0:
                lib.lasp_profile_enable(0)
            return sum(a.elapsed_time(b) for a, b in ev)

        # (1) the measured region: K steps, no per-stage events (they would break programmatic dependent
        # launch between the library's kernels)
        launches0 = lib.lasp_launch_count()
        with ClockSampler(dev.index if rank == 0 else -1) as clk:
            total_ms = timed_loop(args.steps, False)
        launches = (lib.lasp_launch_count() - launches0) // (world if loopback else 1) + graph_launches * args.steps
        if rank == 0:
            clk_summary = clk.summary()
        # (2) the same K steps again with CUDA events recorded by the library around every kernel launch and
        # around the ring hop (on the launching stream): per-kernel durations for the roofline of the dominant
        # kernel, and the exchange time per step (in --loopback only rank 0's launches are recorded)
        prof_ms = timed_loop(args.steps, True)
        stages = {}
        if not loopback or rank == 0:
            buf = ctypes.create_string_buffer(1 << 16)
            lib.lasp_profile_read(buf, len(buf))
            stages = json.loads(buf.value.decode() or "{}")
        hop = {kk: vv[1] / args.steps * 1e3 for kk, vv in stages.items() if kk.startswith("exchange")}
        hop = {kk: (comm.max(vv, rank) if loopback else comm.max(vv)) for kk, vv in sorted(hop.items())} \
            if (T > 1 and not loopback) else hop
        total_ms = comm.max(total_ms, rank) if loopback else comm.max(total_ms)
        results[ex] = {"total_ms": total_ms, "prof_ms": prof_ms, "stages": stages, "launches": launches,
                       "graph": graph is not None, "graph_note": graph_note, "parity_err": err,
                       "hop_us_per_step": hop}
        del graph

    # `value`: the paper's ring protocol (Alg. 2 / 3 hops), over NCCL or as fused P2P hop kernels -- whichever ran
    # faster on this box (both are parity-gated; the all-gather exchange, NEXT-2, is reported beside them)
    ring_like = [x for x in ("p2p", "ring") if x in results]
    main_ex = min(ring_like, key=lambda x: results[x]["total_ms"]) if ring_like else exchanges[0]
    R = results[main_ex]
    ms_step = R["total_ms"] / args.steps
    value = world * B * C * args.steps / (R["total_ms"] / 1e3)

    # e2e through the public API with pinned host buffers: every step copies its inputs H2D, runs fwd + bwd
    # and copies its outputs D2H. Streamed the way a training loop feeds a layer: two device buffer sets and
    # three streams (H2D copy engine, compute, D2H copy engine), so step i+1's upload and step i-1's
    # download overlap step i's compute (PCIe is full duplex; the copies dominate at these sizes).
    e2e = None
    if not args.no_e2e and not loopback:
        if ring is not None:
            ring.set_exchange(main_ex)
        pin = {kk: vv.to(torch.bfloat16).pin_memory() for kk, vv in host.items()}
        outs_h = [torch.empty(t.shape, dtype=torch.bfloat16).pin_memory() for t in (q, q, k, v)]
        n_e2e = max(3, min(args.steps, 20))
        h2d = sum(int(x.numel()) * 2 for x in pin.values())
        d2h = sum(int(x.numel()) * 2 for x in outs_h)
        bufs = [({kk: torch.empty_like(d_in[kk]) for kk in d_in}, [torch.empty_like(t) for t in (q, q, k, v)])
                for _ in range(2)]
        s_up, s_dn = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def e2e_run(n):
            for i in range(n):
                b = i & 1
                ins, outs = bufs[b]
                with torch.cuda.stream(s_up):
                    if i >= 2:
                        s_up.wait_event(ev_done[b])       # compute of step i-2 has consumed buffer b
                    for kk in ("q", "k", "v", "do"):
                        ins[kk].copy_(pin[kk], non_blocking=True)
                    ev_in[b].record(s_up)
                stream.wait_event(ev_in[b])
                if i >= 2:
                    stream.wait_event(ev_out[b])          # outputs of step i-2 are on the host
                if ring is None:
                    lasp.fwd_local(ins["q"], ins["k"], ins["v"], lam, o=outs[0], kv_out=False, cache=cache,
                                   workspace=ws)
                    lasp.bwd_local(ins["q"], ins["k"], ins["v"], lam, ins["do"], cache, dq=outs[1], dk=outs[2],
                                   dv=outs[3], dkv_out=False, workspace=ws)
                else:
                    ring.fwd(ins["q"], ins["k"], ins["v"], lam, o=outs[0], cache=cache, workspace=ws)
                    ring.bwd(ins["q"], ins["k"], ins["v"], lam, ins["do"], cache, dq=outs[1], dk=outs[2],
                             dv=outs[3], workspace=ws)
                ev_done[b].record(stream)
                with torch.cuda.stream(s_dn):
                    s_dn.wait_event(ev_done[b])
                    for hbuf, dbuf in zip(outs_h, outs):
                        hbuf.copy_(dbuf, non_blocking=True)
                    ev_out[b].record(s_dn)
            stream.wait_stream(s_up)
            stream.wait_stream(s_dn)

        e2e_run(2)
        sync()
        comm.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s_up.wait_event(e0)
        e2e_run(n_e2e)
        e1.record(stream)
        sync()
        et = comm.max(e0.elapsed_time(e1))
        e2e = {"value": world * B * C * n_e2e / (et / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n_e2e,
               "pipelining": "double-buffered: H2D(i+1) and D2H(i-1) overlap compute(i) on separate streams"}

    if ring is not None:
        ring.close()
    if rank != 0:
        return None

    # roofline of the dominant kernel, from the live per-stage CUDA events of the measured exchange
    stages = R["stages"]
    hbm, tflops, tflops_sus, peak_src = peaks()
    fam = {}
    for kk, (n_, ms_) in stages.items():  # one kernel family per template (fwd / rev directions pooled)
        if kk.startswith("exchange") or kk.startswith("tag_"):
            continue
        f_ = kk.replace("_fwd", "").replace("_rev", "")
        a_ = fam.setdefault(f_, [0, 0.0])
        a_[0] += n_
        a_[1] += ms_
    dom_name, (dom_n, dom_ms) = max(fam.items(), key=lambda kv: kv[1][1]) if fam else ("none", (1, 0.0))
    per_launch_ms = dom_ms / max(dom_n, 1)
    seg_len = lasp.segment_len(N.shape(B, C, H, D, N.LASP_BF16, Hk if Hk != H else 0))
    nseg = -(-C // seg_len)
    st_bytes = 4 * B * Hk * D * D                       # one fp32 D x D state per (batch, kv-head)
    hq = (H + Hk) / 2                                   # mean heads per tensor (q-side H, kv-side Hk)
    if dom_name.startswith("core_bwd3"):
        # the B3 row reads Q, K, V, dO and writes dQ, dK, dV once (14D B per token-head) plus
        # 2 states per pass (the cached KV_in and the received dKV_in)
        bytes_per_launch = int(2 * D * B * C * (3 * H + 4 * Hk)) + 2 * st_bytes  # Q, dO, dQ: H heads; K, V, dK, dV: Hk
        unit_note = "14*D bytes per token-head (Q,K,V,dO bf16 reads + dQ,dK,dV bf16 writes; B3 row) + 2*B*H*D^2*4"
        # this design's extra state traffic: the 3 passes read one prefix state per segment, and (fused B2)
        # the fold reads and writes the nseg segment states
        overhead = 3 * nseg * st_bytes - 2 * st_bytes + (2 * nseg * st_bytes if "prefix_rev" not in stages else 0)
    elif dom_name.startswith("core"):
        bytes_per_launch = int(2 * D * B * C * (2 * H + 2 * Hk)) + 2 * st_bytes  # Q, K, V read + O written
        unit_note = "8*D bytes per token-head (3 bf16 reads + 1 bf16 write) + 2*B*H*D^2*4"
        overhead = nseg * st_bytes - 2 * st_bytes + (2 * nseg * st_bytes if "prefix" not in stages else 0)
    elif dom_name.startswith("seg_state"):
        bytes_per_launch = int(2 * 2 * D * B * C * hq)    # reads two bf16 tensors: 4D B/token-head
        unit_note = "4*D bytes per token-head (2 bf16 reads)"
        overhead = nseg * st_bytes
    else:
        bytes_per_launch, unit_note, overhead = 0, "n/a", 0
    achieved = bytes_per_launch / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else 0.0
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            ent = json.load(open(tpath)).get(f"{args.config}:{dom_name}")
            if isinstance(ent, dict):
                traffic, traffic_src = ent.get("bytes"), {kk: ent.get(kk) for kk in ("report", "git", "note")}
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "traffic_source": traffic_src, "kernel": dom_name,
                "launches_per_step": dom_n / args.steps, "bytes_per_launch": bytes_per_launch,
                "overhead_bytes_per_launch": overhead, "overhead_frac": (bytes_per_launch + overhead) / max(
                    per_launch_ms / 1e3, 1e-12) / 1e9 / hbm, "bytes_rule": unit_note, "peak_source": peak_src,
                "duration_us": per_launch_ms * 1e3}
    path_bytes = int(2 * D * B * C * (5 * H + 6 * Hk))  # 22D per token-head at Hk = H
    path = {"bytes_per_step": path_bytes, "achieved_gbs": path_bytes / (ms_step / 1e3) / 1e9,
            "frac_of_hbm": path_bytes / (ms_step / 1e3) / 1e9 / hbm,
            "tc_peak_frac": B * C * H * alg_flops_per_token_head(D) / (ms_step / 1e3) / (tflops * 1e12),
            "stages_ms_per_step": {kk: vv[1] / args.steps for kk, vv in stages.items()},
            "profiled_ms_per_step": R["prof_ms"] / args.steps}

    layer = None
    if world == 1 and not loopback and not args.no_layer:
        layer = layer_bench(args, lasp, dev, stream, B, C, H, Hk, D, l2_flush)
    gla = None
    if world == 1 and not loopback and not args.no_gla and Hk == H:
        gla = gla_bench(args, lasp, lib, dev, stream, B, C, H, D, l2_flush)

    cpu = None
    if world == 1 and not loopback and not args.no_cpu_baseline:
        cpu = cpu_baseline(H, D, C, desc)

    ex_report = {ex: {"value": world * B * C * args.steps / (r["total_ms"] / 1e3), "ms_per_step": r["total_ms"] /
                      args.steps, "parity_max_err": r["parity_err"], "parity_ok": r["parity_err"] <= 2e-2,
                      "exchange_us_per_step": r["hop_us_per_step"],
                      "launch": "cuda-graph replay" if r["graph"] else (r["graph_note"] or "eager (PDL)")}
                 for ex, r in results.items()}
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 1 if loopback else world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (synth/, seed 0; bf16 inputs)",
            "config": {"workload": desc if not args.tokens else f"{desc} [n_local overridden: {C}]",
                       "global_batch": B * G, "seq_len": C * T, "n_local": C, "heads": H,
                       "head_dim": D, "kv_heads": Hk, "lambda": "per-head 1-2^-(1+14h/(H-1))", "segment_len": seg_len,
                       "l2": "flushed between timed steps (256 MiB read outside the step events); inputs 4x"
                             f" {B * C * H * D * 2 >> 20} MiB", "parallelism": f"dp{G}xsp{T}" if G > 1 else f"sp{T}",
                       "launch": ex_report[main_ex]["launch"], "exchange": main_ex},
            "parity_ok": all(r["parity_ok"] for r in ex_report.values()),
            "gpu_launches": int(R["launches"]), "clocks": clk_summary, "e2e": e2e, "roofline": roofline,
            "path": path, "cpu_baseline": cpu, "layer": layer, "gla": gla}
    if T > 1:
        line["exchanges"] = ex_report
        if p2p_skipped:
            line["exchanges_skipped"] = {"p2p, p2p_allgather": p2p_skipped}
    else:
        line["parity_max_err"] = ex_report[main_ex]["parity_max_err"]
    if loopback:
        line["loopback"] = {"ranks": world, "note": "all ranks are threads sharing ONE GPU (in-process transport): "
                            "checks the N>1 code path and its parity; value is not a scaling number"}
    return line


def run_lasp(args):
    import torch
    import torch.distributed as dist

    if args.loopback > 1:
        import paper_2404_02882_b200 as lasp
        world = args.loopback
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        comm = ThreadComm(world)
        out, errs = [None] * world, []

        def worker(r):
            try:
                torch.cuda.set_device(0)
                s = torch.cuda.Stream(dev)
                with torch.cuda.stream(s):
                    out[r] = rank_bench(args, r, world, dev, comm,
                                        lambda: lasp.Ring.loopback(r, world, f"bench-{os.getpid()}"), loopback=True)
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
                comm._bar.abort()

        ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]
        print(json.dumps(out[0]), flush=True)
        return 0

    world, rank, local = dist_env()
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    p2p_only = args.transport == "p2p"
    # --transport p2p: no NCCL (gloo for the host-side barriers, the P2P exchange over CUDA IPC), so several ranks
    # may share one GPU (local rank modulo the visible devices): the multi-process path on a one-GPU lease
    local_dev = local % torch.cuda.device_count() if p2p_only else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if p2p_only:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    import paper_2404_02882_b200 as lasp
    T = args.sp_size or world
    group = None
    if 1 < T < world:
        group = lasp.sp_group(T)
    if p2p_only:
        H_, D_ = CONFIGS[args.config][:2]
        n_state = (args.kv_heads or H_) * D_ * D_
        if args.exchange not in ("p2p", "p2p_allgather"):
            args.exchange = "p2p"
        make_ring = lambda: lasp.Ring.p2p_only(n_state, dev, group=group)  # noqa: E731
    else:
        make_ring = lambda: lasp.Ring(dev, group=group)  # noqa: E731
    line = rank_bench(args, rank, world, dev, TorchComm(world, dev, gloo=p2p_only), make_ring,
                      shared_device=p2p_only and world > torch.cuda.device_count())
    if line is not None and p2p_only:
        line["transport"] = "p2p-only ctx (no NCCL; CUDA IPC), " + (
            f"{world} processes sharing {torch.cuda.device_count()} GPU(s): checks the multi-process path, not a "
            "scaling number" if world > torch.cuda.device_count() else "one process per GPU")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["lasp", "reference"], default="lasp")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="tnl04b")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch every step eagerly instead of replaying it from a CUDA graph captured once "
                         "(same kernels and order; the graph keeps the programmatic-dependent-launch edges)")
    ap.add_argument("--sp-size", type=int, default=0,
                    help="sequence-parallel size T (default: all ranks in one ring); G = N/T data-parallel groups "
                         "(Alg. 1 data-sequence hybrid, NEXT-1)")
    ap.add_argument("--exchange", choices=["all", "both", "ring", "allgather", "p2p", "p2p_allgather"], default="all",
                    help="state exchange at N > 1: the paper's ring over NCCL, one all-gather (NEXT-2), the ring with "
                         "fused P2P hop kernels (p2p), ring + allgather (both), or all three (default: each timed in "
                         "the same run; `value` is the NCCL ring's, every one is reported under `exchanges`)")
    ap.add_argument("--loopback", type=int, default=0,
                    help="run N ranks as threads on ONE GPU with the in-process loopback transport (the whole N>1 "
                         "code path incl. the closed-form parity gate; not a scaling measurement)")
    ap.add_argument("--tokens", type=int, default=0, help="override n_local (tokens per GPU) of --config")
    ap.add_argument("--kv-heads", type=int, default=0,
                    help="grouped-query attention: key/value heads (default: the config's heads, i.e. multi-head)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-layer", action="store_true", help="skip the NEXT-3 whole-layer line")
    ap.add_argument("--transport", choices=["nccl", "p2p"], default="nccl",
                    help="N > 1 ring context: NCCL (default) or a P2P-only context without NCCL (CUDA IPC; ranks may "
                         "share a GPU)")
    ap.add_argument("--no-gla", action="store_true", help="skip the NEXT-4 generalised-decay line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_lasp(args)


if __name__ == "__main__":
    sys.exit(main())
