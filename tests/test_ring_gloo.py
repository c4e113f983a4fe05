"""Multi-process (gloo, CPU) tests of the ring's host-side logic.

The library's ring schedule (`lasp_ring_peers`, used verbatim by lasp_fwd/lasp_bwd) and its hop rule
(the local state is computed before the hop; the hop sends lambda^C * received + local, Alg. 2 P:171 /
Alg. 3) are driven over real processes with torch.distributed P2P on gloo. The per-rank arithmetic
is the fp64 oracle's chunk operations (test-only stand-in for the GPU kernels, which need a B200). The
gathered outputs must equal the oracle's definition-mode results on the whole sequence, and the message
log must follow the protocol: world-1 hops per direction, B*H*D*D elements each, independent of N.
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


def _worker(rank, world, port, N, H, D, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2404_02882_b200.api import ring_peers
        C = N // world
        p = synth.problem(11, 1, N, H, D, dtype="fp32", token_lo=rank * C, token_hi=(rank + 1) * C)
        lam = p["lam"]
        log = []
        # ---- forward (Alg. 2) ----
        L = np.zeros((H, D, D))
        parts = []
        for h in range(H):
            mask, lf, lr, lc = oracle.build_decay(C, lam[h])
            parts.append((mask, lf, lr, lc))
            L[h] = oracle.kv_update(None, p["k"][0, :, h], p["v"][0, :, h], lr, lc)  # local part, hoisted
        frm, to = ring_peers(rank, world, False)
        kv_in = torch.zeros(H * D * D, dtype=torch.float64)
        if frm >= 0:
            dist.recv(kv_in, src=frm)
            log.append(("fwd", "recv", frm, kv_in.numel()))
        kv_in = kv_in.numpy().reshape(H, D, D)
        if to >= 0:
            out = np.stack([parts[h][3] * kv_in[h] + L[h] for h in range(H)])
            dist.send(torch.from_numpy(np.ascontiguousarray(out).reshape(-1)), dst=to)
            log.append(("fwd", "send", to, out.size))
        o = np.zeros((C, H, D))
        for h in range(H):
            mask, lf, lr, lc = parts[h]
            o[:, h] = oracle.intra_fwd(p["q"][0, :, h], p["k"][0, :, h], p["v"][0, :, h], mask) + \
                oracle.inter_fwd(p["q"][0, :, h], kv_in[h], lf)
        cache = kv_in  # state entering the rank (reading A4)
        # ---- backward (Alg. 3) ----
        G = np.stack([oracle.dkv_update(None, p["q"][0, :, h], p["do"][0, :, h], parts[h][1], parts[h][3])
                      for h in range(H)])
        frm, to = ring_peers(rank, world, True)
        dkv_in = torch.zeros(H * D * D, dtype=torch.float64)
        if frm >= 0:
            dist.recv(dkv_in, src=frm)
            log.append(("bwd", "recv", frm, dkv_in.numel()))
        dkv_in = dkv_in.numpy().reshape(H, D, D)
        if to >= 0:
            out = np.stack([parts[h][3] * dkv_in[h] + G[h] for h in range(H)])
            dist.send(torch.from_numpy(np.ascontiguousarray(out).reshape(-1)), dst=to)
            log.append(("bwd", "send", to, out.size))
        dq, dk, dv = (np.zeros((C, H, D)) for _ in range(3))
        for h in range(H):
            mask, lf, lr, lc = parts[h]
            q, k, v, do = (p[x][0, :, h] for x in ("q", "k", "v", "do"))
            iq, ik, iv = oracle.intra_bwd(q, k, v, do, mask)
            dq[:, h] = iq + oracle.inter_bwd_q(do, cache[h], lf)
            dk[:, h] = ik + oracle.inter_bwd_k(v, dkv_in[h], lr)
            dv[:, h] = iv + oracle.inter_bwd_v(k, dkv_in[h], lr)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), o=o, dq=dq, dk=dk, dv=dv,
                 log=np.array(log, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 96), (4, 128), (4, 256)])
def test_ring_protocol_over_gloo(tmp_path, oracle_mod, world, N):
    H, D = 2, 4
    mp.start_processes(_worker, args=(world, _free_port(), N, H, D, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    res = [np.load(tmp_path / f"rank{r}.npz", allow_pickle=True) for r in range(world)]
    got = {k: np.concatenate([r[k] for r in res])[None] for k in ("o", "dq", "dk", "dv")}
    p = synth.problem(11, 1, N, H, D, dtype="fp32")
    o_ref = oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])
    g_ref = oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])
    for name, ref in zip(("o", "dq", "dk", "dv"), (o_ref,) + tuple(g_ref)):
        err = np.max(np.abs(got[name] - ref)) / np.max(np.abs(ref))
        assert err <= 1e-12, (name, err)
    # protocol: world-1 sends per direction, r -> r+1 forward and r+1 -> r backward, H*D*D elements each
    sends = [(d, r, peer, n) for r, x in enumerate(res) for (d, kind, peer, n) in x["log"] if kind == "send"]
    assert sorted((r, peer) for d, r, peer, n in sends if d == "fwd") == [(r, r + 1) for r in range(world - 1)]
    assert sorted((r, peer) for d, r, peer, n in sends if d == "bwd") == [(r + 1, r) for r in range(world - 1)]
    assert {n for *_, n in sends} == {H * D * D}


def test_ring_peers_edges():
    from paper_2404_02882_b200.api import ring_peers
    from paper_2404_02882_b200._native import LaspError
    assert ring_peers(0, 1, False) == (-1, -1) and ring_peers(0, 1, True) == (-1, -1)
    assert [ring_peers(r, 3, False) for r in range(3)] == [(-1, 1), (0, 2), (1, -1)]
    assert [ring_peers(r, 3, True) for r in range(3)] == [(1, -1), (2, 0), (-1, 1)]
    with pytest.raises(LaspError):
        ring_peers(3, 3, False)


def _allgather_worker(rank, world, port, N, H, D, out_dir):
    """SURVEY §8(f) NEXT-2 rule on real processes: all-gather the local states, fold the received ones."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        C = N // world
        p = synth.problem(12, 1, N, H, D, dtype="fp32", token_lo=rank * C, token_hi=(rank + 1) * C)
        lam = p["lam"]
        parts = [oracle.build_decay(C, lam[h]) for h in range(H)]
        L = np.stack([oracle.kv_update(None, p["k"][0, :, h], p["v"][0, :, h], parts[h][2], parts[h][3])
                      for h in range(H)])
        G = np.stack([oracle.dkv_update(None, p["q"][0, :, h], p["do"][0, :, h], parts[h][1], parts[h][3])
                      for h in range(H)])
        gl = [torch.zeros(H * D * D, dtype=torch.float64) for _ in range(world)]
        gg = [torch.zeros(H * D * D, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gl, torch.from_numpy(np.ascontiguousarray(L).reshape(-1)))
        dist.all_gather(gg, torch.from_numpy(np.ascontiguousarray(G).reshape(-1)))
        lc = np.array([parts[h][3] for h in range(H)])[:, None, None]  # lam^C per head
        kv_in = np.zeros((H, D, D))
        for j in range(rank):                      # KV_in(r) = sum_{j<r} lam^(C(r-1-j)) L_j
            kv_in = lc * kv_in + gl[j].numpy().reshape(H, D, D)
        dkv_in = np.zeros((H, D, D))
        for j in range(world - 1, rank, -1):       # dKV_in(r) = sum_{j>r} lam^(C(j-r-1)) G_j
            dkv_in = lc * dkv_in + gg[j].numpy().reshape(H, D, D)
        np.savez(os.path.join(out_dir, f"ag{rank}.npz"), kv_in=kv_in, dkv_in=dkv_in)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 64), (4, 128)])
def test_allgather_exchange_over_gloo(tmp_path, oracle_mod, world, N):
    """The folded all-gather states equal the ring's messages: the oracle's Alg. 2 cache (state entering
    each rank) and, for the backward, the definition of dKV_in(r) evaluated directly."""
    H, D = 2, 4
    mp.start_processes(_allgather_worker, args=(world, _free_port(), N, H, D, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    res = [np.load(tmp_path / f"ag{r}.npz") for r in range(world)]
    p = synth.problem(12, 1, N, H, D, dtype="fp32")
    _, cache, _, _ = oracle_mod.lasp_fwd_sim(p["q"], p["k"], p["v"], p["lam"], world)
    C = N // world
    for r in range(world):
        assert np.max(np.abs(res[r]["kv_in"] - cache[r][0])) <= 1e-12 * max(1.0, np.max(np.abs(cache[r][0])))
        # dKV_in(r) = sum_{g >= (r+1)C} lam^(g-(r+1)C+1) q_g do_g^T  (reading A3)
        ref = np.zeros((H, D, D))
        for h in range(H):
            lam = float(np.float32(p["lam"][h]))
            for g in range((r + 1) * C, N):
                ref[h] += lam ** (g - (r + 1) * C + 1) * np.outer(p["q"][0, g, h].astype(np.float64),
                                                                 p["do"][0, g, h].astype(np.float64))
        assert np.max(np.abs(res[r]["dkv_in"] - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
