"""Data-sequence hybrid parallelism (Alg. 1).

W ranks form G = W/T sequence-parallel groups of T consecutive ranks; each group trains on its own
sequence, its source rank R_src = floor(R/T)*T scatters the T chunks (Alg. 1 lines 6-8), and each group runs
its own LASP ring. Host logic (`lasp_topology`, `sp_group`, `scatter_sequence`) is tested over gloo with
the fp64 oracle's chunk operations as the per-rank arithmetic (test-only stand-in for the GPU kernels);
the GPU test runs two independent loopback rings of the real library on one device.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_topology_examples():
    from paper_2404_02882_b200 import topology
    # Fig. 2 / P:126: W=8, T=4 -> G=2, R_src=[0,4]; ranks 0..3 hold Seq0's chunks, 4..7 Seq1's
    t = [topology(r, 8, 4) for r in range(8)]
    assert sorted({g for g, _, _ in t}) == [0, 1]
    assert sorted({s for _, _, s in t}) == [0, 4]
    assert [c for _, c, _ in t] == [0, 1, 2, 3, 0, 1, 2, 3]
    # W=4, T=2 -> G=2, R_src=[0,2]; W=T=4 -> one group
    assert [topology(r, 4, 2) for r in range(4)] == [(0, 0, 0), (0, 1, 0), (1, 0, 2), (1, 1, 2)]
    assert [topology(r, 4, 4) for r in range(4)] == [(0, r, 0) for r in range(4)]
    # T = 1: pure data parallelism, every rank is its own group
    assert [topology(r, 3, 1) for r in range(3)] == [(r, 0, r) for r in range(3)]


def test_topology_errors():
    from paper_2404_02882_b200 import topology
    from paper_2404_02882_b200._native import LaspError
    for args in [(0, 6, 4), (0, 4, 0), (4, 4, 2), (-1, 4, 2)]:
        with pytest.raises(LaspError) as e:
            topology(*args)
        assert e.value.name == "LASP_ERR_PARTITION"


def _hybrid_worker(rank, world, sp_size, port, N, H, D, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2404_02882_b200 import scatter_sequence, sp_group, topology
        from paper_2404_02882_b200.api import ring_peers
        grp_id, grank, src = topology(rank, world, sp_size)
        grp = sp_group(sp_size)
        T, C = sp_size, N // sp_size
        # Alg. 1: only the group's source rank holds the group's sequence (batch = seed 200 + group id)
        full = synth.problem(200 + grp_id, 1, N, H, D, dtype="fp32") if rank == src else None
        p = {x: scatter_sequence(torch.from_numpy(full[x]) if full else None, grp, T).numpy()
             for x in ("q", "k", "v", "do")}
        lam = synth.head_lambdas(H, None)
        glob = lambda r: dist.get_global_rank(grp, r)  # noqa: E731
        log = []
        parts = [oracle.build_decay(C, lam[h]) for h in range(H)]
        # forward ring inside the group (Alg. 2), local part hoisted before the hop
        L = np.stack([oracle.kv_update(None, p["k"][0, :, h], p["v"][0, :, h], parts[h][2], parts[h][3])
                      for h in range(H)])
        frm, to = ring_peers(grank, T, False)
        kv_in = torch.zeros(H * D * D, dtype=torch.float64)
        if frm >= 0:
            dist.recv(kv_in, src=glob(frm))
        kv_in = kv_in.numpy().reshape(H, D, D)
        if to >= 0:
            out = np.stack([parts[h][3] * kv_in[h] + L[h] for h in range(H)])
            dist.send(torch.from_numpy(np.ascontiguousarray(out).reshape(-1)), dst=glob(to))
            log.append(("fwd", rank, glob(to)))
        o = np.stack([oracle.intra_fwd(p["q"][0, :, h], p["k"][0, :, h], p["v"][0, :, h], parts[h][0]) +
                      oracle.inter_fwd(p["q"][0, :, h], kv_in[h], parts[h][1]) for h in range(H)], axis=1)
        # backward ring inside the group (Alg. 3)
        G = np.stack([oracle.dkv_update(None, p["q"][0, :, h], p["do"][0, :, h], parts[h][1], parts[h][3])
                      for h in range(H)])
        frm, to = ring_peers(grank, T, True)
        dkv_in = torch.zeros(H * D * D, dtype=torch.float64)
        if frm >= 0:
            dist.recv(dkv_in, src=glob(frm))
        dkv_in = dkv_in.numpy().reshape(H, D, D)
        if to >= 0:
            out = np.stack([parts[h][3] * dkv_in[h] + G[h] for h in range(H)])
            dist.send(torch.from_numpy(np.ascontiguousarray(out).reshape(-1)), dst=glob(to))
            log.append(("bwd", rank, glob(to)))
        dq, dk, dv = (np.zeros((C, H, D)) for _ in range(3))
        for h in range(H):
            q, k, v, do = (p[x][0, :, h] for x in ("q", "k", "v", "do"))
            iq, ik, iv = oracle.intra_bwd(q, k, v, do, parts[h][0])
            dq[:, h] = iq + oracle.inter_bwd_q(do, kv_in[h], parts[h][1])
            dk[:, h] = ik + oracle.inter_bwd_k(v, dkv_in[h], parts[h][2])
            dv[:, h] = iv + oracle.inter_bwd_v(k, dkv_in[h], parts[h][2])
        np.savez(os.path.join(out_dir, f"hy{rank}.npz"), o=o, dq=dq, dk=dk, dv=dv, q=p["q"],
                 log=np.array(log, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,sp_size,N", [(4, 2, 64), (6, 3, 96), (4, 1, 32)])
def test_hybrid_groups_over_gloo(tmp_path, oracle_mod, world, sp_size, N):
    H, D = 2, 4
    mp.start_processes(_hybrid_worker, args=(world, sp_size, _free_port(), N, H, D, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    res = [np.load(tmp_path / f"hy{r}.npz", allow_pickle=True) for r in range(world)]
    G = world // sp_size
    for g in range(G):
        ranks = range(g * sp_size, (g + 1) * sp_size)
        p = synth.problem(200 + g, 1, N, H, D, dtype="fp32")
        # scatter: rank with group_rank t holds tokens [tC, (t+1)C) of its group's sequence, bit for bit
        assert np.array_equal(np.concatenate([res[r]["q"] for r in ranks], axis=1), p["q"])
        got = {k: np.concatenate([res[r][k] for r in ranks])[None] for k in ("o", "dq", "dk", "dv")}
        refs = (oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"]),) + \
            tuple(oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"]))
        for name, ref in zip(("o", "dq", "dk", "dv"), refs):
            assert oracle_mod.normwise_err(got[name], ref) <= 1e-12, (g, name)
    # group isolation: every message stays inside its group; T-1 hops per group and direction
    sends = [tuple(m) for r in res for m in r["log"]]
    assert all(src // sp_size == dst // sp_size for _, src, dst in sends)
    for d, step in (("fwd", 1), ("bwd", -1)):
        got = sorted((s, t) for dd, s, t in sends if dd == d)
        want = sorted((g * sp_size + i, g * sp_size + i + step) for g in range(G)
                      for i in (range(sp_size - 1) if step > 0 else range(1, sp_size)))
        assert got == want


@pytest.mark.gpu
def test_hybrid_loopback_groups_matches_oracle(oracle_mod):
    """Two sequence-parallel groups of 2 ranks each (W=4, T=2) on one GPU: each group is its own loopback
    ring over its own sequence; every group's gathered result matches the oracle on that sequence."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import threading
    import paper_2404_02882_b200 as lasp
    W, T, N, H, D = 4, 2, 1536, 4, 64
    C = N // T
    probs = [synth.problem(300 + g, 1, N, H, D, dtype="bf16") for g in range(W // T)]
    out, errors = [None] * W, []
    done = threading.Barrier(W)

    def worker(r):
        ring = None
        try:
            torch.cuda.set_device(0)
            g, t, _ = lasp.topology(r, W, T)
            ring = lasp.Ring.loopback(t, T, f"hybrid-group{g}")
            p = probs[g]
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sl = slice(t * C, (t + 1) * C)
                q, k, v, do = (torch.from_numpy(np.ascontiguousarray(p[x][:, sl])).cuda().to(torch.bfloat16)
                               for x in ("q", "k", "v", "do"))
                o, cache = ring.fwd(q, k, v, p["lam"])
                dq, dk, dv = ring.bwd(q, k, v, p["lam"], do, cache)
            stream.synchronize()
            out[r] = [x.float().cpu().numpy() for x in (o, dq, dk, dv)]
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errors.append(e)
            done.abort()
            return
        finally:
            try:
                done.wait(timeout=300)
            except threading.BrokenBarrierError:
                pass
            if ring is not None:
                ring.close()

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(W)]
    for th in ts:
        th.start()
    for th in ts:
        th.join(timeout=600)
    assert not errors, errors
    for g, p in enumerate(probs):
        got = [np.concatenate([out[r][i] for r in range(g * T, (g + 1) * T)], axis=1) for i in range(4)]
        refs = [oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])] + \
            list(oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"]))
        for x, ref in zip(got, refs):
            assert oracle_mod.normwise_err(x, ref) <= 2e-2
