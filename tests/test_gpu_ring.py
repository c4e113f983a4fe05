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


def test_ring_cache_tag_checks_rank(ring):
    import paper_2404_02882_b200 as lasp
    from paper_2404_02882_b200._native import LaspError
    q = torch.zeros((1, 256, 2, 64), dtype=torch.bfloat16, device="cuda")
    _, _, cache = lasp.fwd_local(q, q, q, [0.9, 0.9])   # local cache: (rank, world) = (-1, -1)
    with pytest.raises(LaspError) as e:
        ring.bwd(q, q, q, [0.9, 0.9], q, cache)
    assert e.value.name == "LASP_ERR_STATE"
