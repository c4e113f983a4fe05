"""GPU: the NCCL ring entry points (lasp_fwd / lasp_bwd with a ctx) on one rank, against the oracle.

Only one GPU exists in this environment, so the ring runs with world size 1 (the NCCL communicator,
comm stream, events and the ctx code path are exercised; no hop is taken). Multi-rank behaviour is
covered by tests/test_ring_gloo.py (protocol) and the simulated ring of tests/test_gpu_parity.py.
"""
import os
import socket

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ring():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    import paper_2404_02882_b200 as lasp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    r = lasp.Ring(torch.device("cuda", 0))
    yield r
    r.close()
    dist.destroy_process_group()


def test_ring_world1_matches_oracle(ring, oracle_mod):
    p = synth.problem(21, 1, 3000, 4, 64, dtype="bf16")
    q, k, v, do = (torch.from_numpy(p[x]).cuda().to(torch.bfloat16) for x in ("q", "k", "v", "do"))
    o, cache = ring.fwd(q, k, v, p["lam"])
    dq, dk, dv = ring.bwd(q, k, v, p["lam"], do, cache)
    torch.cuda.synchronize()
    refs = [oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])] + \
        list(oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"]))
    for x, r in zip((o, dq, dk, dv), refs):
        assert oracle_mod.normwise_err(x.float().cpu().numpy(), r) <= 2e-2
    assert ring.protocol(q) == (0, 0, 4 * 64 * 64)


def test_ring_world1_fp32(ring, oracle_mod):
    p = synth.problem(22, 1, 512, 1, 32, dtype="fp32", lam=0.99)
    q, k, v, do = (torch.from_numpy(p[x]).cuda() for x in ("q", "k", "v", "do"))
    o, cache = ring.fwd(q, k, v, p["lam"])
    dq, dk, dv = ring.bwd(q, k, v, p["lam"], do, cache)
    torch.cuda.synchronize()
    refs = [oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])] + \
        list(oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"]))
    for x, r in zip((o, dq, dk, dv), refs):
        assert oracle_mod.normwise_err(x.cpu().numpy(), r) <= 1e-5


def test_ring_world1_generalised_decay(ring, oracle_mod):
    """The NEXT-4 generalised-decay ring entry points (lasp_gla_fwd / lasp_gla_bwd) through the NCCL ctx at world
    size 1 against the oracle (fp32: 1e-5, decay gradient 1e-4; reading D3)."""
    t = synth.gla_problem(23, 1, 1500, 2, 64)
    q, k, v, lg, do = (torch.from_numpy(t[x]).cuda() for x in ("q", "k", "v", "lg", "do"))
    o, cache = ring.gla_fwd(q, k, v, lg)
    dq, dk, dv, dlg = ring.gla_bwd(q, k, v, lg, do, cache)
    torch.cuda.synchronize()
    refs = [oracle_mod.gla_fwd(t["q"], t["k"], t["v"], t["lg"])] + \
        list(oracle_mod.gla_bwd(t["q"], t["k"], t["v"], t["lg"], t["do"]))
    for x, r, tol in zip((o, dq, dk, dv, dlg), refs, (1e-5, 1e-5, 1e-5, 1e-5, 1e-4)):
        assert oracle_mod.normwise_err(x.cpu().numpy(), r) <= tol


def test_ring_graph_capture_matches_eager(ring):
    """The NCCL-ctx entry points (comm stream fork/join, events, memsets) captured into a CUDA graph
    reproduce the eager results bit for bit (include/lasp.h "Graphs")."""
    p = synth.problem(21, 1, 2048, 4, 64, dtype="bf16")
    q, k, v, do = (torch.from_numpy(p[x]).cuda().to(torch.bfloat16) for x in ("q", "k", "v", "do"))
    o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))
    import paper_2404_02882_b200 as lasp
    cache, ws = lasp.alloc_cache(q), lasp.alloc_workspace(q)

    def step():
        ring.fwd(q, k, v, p["lam"], o=o, cache=cache, workspace=ws)
        ring.bwd(q, k, v, p["lam"], do, cache, dq=dq, dk=dk, dv=dv, workspace=ws)

    step()
    torch.cuda.synchronize()
    eager = [t.clone() for t in (o, dq, dk, dv)]
    for t in (o, dq, dk, dv):
        t.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, (o, dq, dk, dv)):
        assert torch.equal(a, b)


def test_ring_cache_tag_checks_rank(ring):
    import paper_2404_02882_b200 as lasp
    from paper_2404_02882_b200._native import LaspError
    q = torch.zeros((1, 256, 2, 64), dtype=torch.bfloat16, device="cuda")
    _, _, cache = lasp.fwd_local(q, q, q, [0.9, 0.9])   # local cache: (rank, world) = (-1, -1)
    with pytest.raises(LaspError) as e:
        ring.bwd(q, q, q, [0.9, 0.9], q, cache, check_state=True)
    assert e.value.name == "LASP_ERR_STATE" and "rank" in str(e.value)


# ---- world > 1 on one GPU: the same lasp_fwd / lasp_bwd code with the in-process loopback transport ----
def _run_loopback(p, world, n_global, dtype, group, exchange="ring", bounds=None, steps=1):
    """Each rank is a thread with its own CUDA stream and ring context; returns the gathered outputs.
    ``bounds``: per-rank token ranges (default: equal shares C = N/T). ``steps``: fwd + bwd repeated (the P2P
    exchange's epoch flags and acks advance every step); the outputs of every step must be identical."""
    import threading
    import paper_2404_02882_b200 as lasp
    C = n_global // world
    bounds = bounds or [(r * C, (r + 1) * C) for r in range(world)]
    out, errors = [None] * world, []
    done = threading.Barrier(world)

    def worker(r):
        ring = None
        try:
            torch.cuda.set_device(0)
            ring = lasp.Ring.loopback(r, world, group)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sl = slice(*bounds[r])
                q, k, v, do = (torch.from_numpy(np.ascontiguousarray(p[x][:, sl])).cuda().to(dtype)
                               for x in ("q", "k", "v", "do"))
                if exchange.startswith("p2p"):
                    # warm-up over the host transport: no kernel may load lazily (a context synchronize) while a
                    # peer's hop kernel spins on this GPU (include/lasp.h, LASP_EXCHANGE_P2P)
                    o, cache = ring.fwd(q, k, v, p["lam"])
                    ring.bwd(q, k, v, p["lam"], do, cache)
                    stream.synchronize()
                    kk = p["k"]
                    ring.enable_p2p(kk.shape[0] * kk.shape[2] * kk.shape[3] ** 2).set_exchange(exchange)
                else:
                    ring.set_exchange(exchange)
                first = None
                for _ in range(steps):
                    o, cache = ring.fwd(q, k, v, p["lam"])
                    dq, dk, dv = ring.bwd(q, k, v, p["lam"], do, cache)
                    if first is None:
                        first = [t.clone() for t in (o, dq, dk, dv)]
                    else:
                        for a_, b_ in zip(first, (o, dq, dk, dv)):
                            assert torch.equal(a_, b_), "a later step differs from the first"
            stream.synchronize()
            B, Cr, H, D = k.shape   # states are per kv-head
            seg = lasp.segment_len(lasp.api._shape(q, k))
            nseg = (Cr + seg - 1) // seg
            # cache [B][H][nseg][D][D]; entry 0 of each (b, h) = KV_in(r), the state entering the rank
            kv_in = cache.view(torch.float32)[:B * H * nseg * D * D].view(B, H, nseg, D, D)[:, :, 0]
            out[r] = [t.float().cpu().numpy() for t in (o, dq, dk, dv)] + [kv_in.cpu().numpy()]
        except BaseException as e:  # noqa: BLE001 - re-raised by the test
            errors.append(e)
            done.abort()
            return
        finally:
            try:
                done.wait(timeout=300)  # keep every context alive until all ranks are finished
            except threading.BrokenBarrierError:
                pass
            if ring is not None:
                ring.close()

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errors, errors
    return [np.concatenate([out[r][i] for r in range(world)], axis=1) for i in range(4)], [o[4] for o in out]


@pytest.mark.parametrize("exchange", ["ring", "allgather", "p2p", "p2p_allgather"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_loopback_ring_bf16_matches_oracle(oracle_mod, world, exchange):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    N = 768 * world
    p = synth.problem(40 + world, 1, N, 4, 64, dtype="bf16")
    got, _ = _run_loopback(p, world, N, torch.bfloat16, f"bf16-w{world}-{exchange}", exchange,
                           steps=3 if exchange.startswith("p2p") else 1)
    refs = [oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])] + \
        list(oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"]))
    for x, r in zip(got, refs):
        assert oracle_mod.normwise_err(x, r) <= 2e-2


@pytest.mark.parametrize("exchange", ["ring", "allgather"])
def test_loopback_gqa_ring(oracle_mod, exchange):
    """Grouped-query attention across a 3-rank ring: the messages are the Hk = 2 shared kv-head states."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = synth.problem(48, 1, 3 * 768, 8, 128, dtype="bf16", kv_heads=2)
    got, _ = _run_loopback(p, 3, 3 * 768, torch.bfloat16, f"gqa-{exchange}", exchange)
    refs = [oracle_mod.fwd_gqa(p["q"], p["k"], p["v"], p["lam"])] + \
        list(oracle_mod.bwd_gqa(p["q"], p["k"], p["v"], p["lam"], p["do"]))
    for x, r in zip(got, refs):
        assert oracle_mod.normwise_err(x, r) <= 2e-2


@pytest.mark.parametrize("exchange", ["ring", "allgather"])
def test_loopback_unequal_rank_lengths(oracle_mod, exchange):
    """Ranks holding different token counts (reading R3): the ring combines with each rank's own lam^C, and
    the all-gather exchange carries every rank's n_local with its state, so both match the
    oracle on the whole sequence."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    bounds = [(0, 300), (300, 1324), (1324, 1500), (1500, 2200)]
    p = synth.problem(47, 1, 2200, 4, 64, dtype="bf16")
    got, _ = _run_loopback(p, 4, 2200, torch.bfloat16, f"unequal-{exchange}", exchange, bounds=bounds)
    refs = [oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])] + \
        list(oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"]))
    for x, r in zip(got, refs):
        assert oracle_mod.normwise_err(x, r) <= 2e-2


@pytest.mark.parametrize("exchange", ["ring", "allgather"])
def test_loopback_ring_config1_fp32(oracle_mod, exchange):
    """BASELINE configs[0] on the real ring code: 1 head x 32, N=512, lambda=0.99, 4 ranks, fp32."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = synth.problem(0, 1, 512, 1, 32, dtype="fp32", lam=0.99)
    got, kv_in = _run_loopback(p, 4, 512, torch.float32, f"config1-{exchange}", exchange)
    refs = [oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])] + \
        list(oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"]))
    for x, r in zip(got, refs):
        assert oracle_mod.normwise_err(x, r) <= 1e-5
    # each rank's cache holds the state that entered it (Alg. 2, reading A4)
    _, cache, _, _ = oracle_mod.lasp_fwd_sim(p["q"], p["k"], p["v"], p["lam"], 4)
    for r in range(4):
        ref = np.asarray(cache[r]).reshape(kv_in[r].shape)
        den = max(np.max(np.abs(ref)), 1e-30)
        assert np.max(np.abs(kv_in[r] - ref)) / den <= 1e-5 or (r == 0 and np.max(np.abs(kv_in[r])) == 0)


def test_allgather_protocol_and_domain(ring):
    import paper_2404_02882_b200 as lasp
    from paper_2404_02882_b200._native import LaspError
    q = torch.zeros((1, 256, 2, 64), dtype=torch.bfloat16, device="cuda")
    r = lasp.Ring.loopback(0, 3, "proto").set_exchange("allgather")
    try:
        assert r.protocol(q) == (1, 1, 2 * 64 * 64)
        with pytest.raises(LaspError) as e:
            lasp._native.check(lasp._native.lib().lasp_ctx_set_exchange(r._ctx, 7))
        assert e.value.name == "LASP_ERR_DOMAIN"
    finally:
        r.close()


_RING_FOLD_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import synth, test_gpu_ring as T
out = {{}}
for exchange in ("ring", "allgather"):
    p = synth.problem(61, 1, 3 * 1152, 4, 64, dtype="bf16")
    got, kv = T._run_loopback(p, 3, 3 * 1152, torch.bfloat16, "fold-" + exchange, exchange)
    for n, x in zip(("o", "dq", "dk", "dv"), got):
        out[n + exchange] = x
    out["kv" + exchange] = np.stack(kv)
np.savez({dst!r}, **out)
"""


def test_ring_fused_fold_matches_separate_kernel(tmp_path):
    """The ring entry points fold F2 (after the hop) into the F3 launch and B2 into the dV / dK launch; with
    LASP_NO_FUSED_FOLD=1 they run the prefix kernel. 3 loopback ranks, ring and all-gather exchange: every
    output and every rank's received state must agree bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for off in ("0", "1"):
        dst = str(tmp_path / f"ringfold{off}.npz")
        script = _RING_FOLD_SCRIPT.format(root=root, tests=os.path.join(root, "tests"), dst=dst)
        subprocess.run([sys.executable, "-c", script], env=dict(os.environ, LASP_NO_FUSED_FOLD=off), check=True,
                       timeout=600)
        res[off] = np.load(dst)
    for key in res["0"].files:
        assert np.array_equal(res["0"][key], res["1"][key]), key


# ---- the P2P exchange across PROCESSES (CUDA IPC peer buffers; two processes share GPU 0) -----------------
def _p2p_proc(rank, world, port, N, errq, exchange="p2p"):
    try:
        import torch.distributed as dist
        import paper_2404_02882_b200 as lasp
        import oracle
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        p = synth.problem(77, 1, N, 4, 64, dtype="bf16")
        C = N // world
        sl = slice(rank * C, (rank + 1) * C)
        q, k, v, do = (torch.from_numpy(np.ascontiguousarray(p[x][:, sl])).cuda().to(torch.bfloat16)
                       for x in ("q", "k", "v", "do"))
        ring = lasp.Ring.p2p_only(1 * 4 * 64 * 64).set_exchange(exchange)
        refs = [oracle.fwd(p["q"], p["k"], p["v"], p["lam"])] + list(oracle.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"]))
        for step in range(3):
            o, cache = ring.fwd(q, k, v, p["lam"])
            dq, dk, dv = ring.bwd(q, k, v, p["lam"], do, cache)
            torch.cuda.synchronize()
            for x, r in zip((o, dq, dk, dv), refs):
                err = oracle.normwise_err(x.float().cpu().numpy(), r[:, sl])
                assert err <= 2e-2, (rank, step, err)
        dist.barrier()
        ring.close()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")


@pytest.mark.parametrize("exchange,world", [("p2p", 2), ("p2p_allgather", 3)])
def test_p2p_exchange_processes_one_gpu(exchange, world):
    """lasp_fwd / lasp_bwd with a P2P exchange (ring hops, or the one-step all-gather) between PROCESSES sharing
    GPU 0 through CUDA IPC handles (the code path multi-GPU ranks take; NCCL refuses two ranks on one device, the
    P2P transport does not): three steps (epoch flags and acks advancing) against the oracle on each rank's shard."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    procs = [ctx.Process(target=_p2p_proc, args=(r, world, port, 1024 * world, errq, exchange)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=600)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]


def _p2p_hybrid_proc(rank, world, sp, port, C, errq):
    try:
        import torch.distributed as dist
        import paper_2404_02882_b200 as lasp
        import oracle
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        grp = lasp.sp_group(sp)
        gid, grank, _ = lasp.topology(rank, world, sp)
        p = synth.problem(90 + gid, 1, C * sp, 4, 64, dtype="bf16")   # each group its own sequence (Alg. 1)
        sl = slice(grank * C, (grank + 1) * C)
        q, k, v, do = (torch.from_numpy(np.ascontiguousarray(p[x][:, sl])).cuda().to(torch.bfloat16)
                       for x in ("q", "k", "v", "do"))
        ring = lasp.Ring.p2p_only(4 * 64 * 64, group=grp).set_exchange("p2p_allgather" if gid else "p2p")
        refs = [oracle.fwd(p["q"], p["k"], p["v"], p["lam"])] + list(oracle.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"]))
        for step in range(2):
            o, cache = ring.fwd(q, k, v, p["lam"])
            dq, dk, dv = ring.bwd(q, k, v, p["lam"], do, cache)
            torch.cuda.synchronize()
            for x, r in zip((o, dq, dk, dv), refs):
                err = oracle.normwise_err(x.float().cpu().numpy(), r[:, sl])
                assert err <= 2e-2, (rank, step, err)
        dist.barrier()
        ring.close()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")


def test_p2p_hybrid_groups_processes_one_gpu():
    """Data-sequence hybrid (Alg. 1, NEXT-1) with the P2P exchanges: 4 processes on GPU 0, two sequence-parallel
    groups of 2 (group 0 the P2P ring, group 1 the P2P all-gather), each with its own sequence; every rank's shard
    against the oracle on its group's sequence, two steps."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    procs = [ctx.Process(target=_p2p_hybrid_proc, args=(r, 4, 2, port, 768, errq)) for r in range(4)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=600)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
