"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical seeded inputs.

Tolerances (normwise per tensor and head, max|x - ref| / max|ref|, reading A14):
bf16 <= 2e-2, fp32 <= 1e-5 (BASELINE.json north_star). Inputs come from synth/ only.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
FP32_TOL = 1e-5


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_02882_b200 as lasp
    return lasp


def to_dev(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(dtype).contiguous()


def per_head_err(x, ref):
    """max over heads of normwise error; x, ref [B][N][H][D]."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    worst = 0.0
    for h in range(ref.shape[2]):
        den = np.max(np.abs(ref[:, :, h]))
        num = np.max(np.abs(x[:, :, h] - ref[:, :, h]))
        worst = max(worst, num / den if den > 0 else num)
    return worst


def run_sim_ring(L, p, T, dtype, n_global):
    """Alg. 2/3 with T ranks simulated on one GPU by chaining kv_out -> kv_in (and dkv back)."""
    C = n_global // T
    dev = {k: to_dev(p[k], dtype) for k in ("q", "k", "v", "do")}
    lam = p["lam"]
    outs, caches, kvs = [], [], []
    kv = None
    for r in range(T):
        sl = slice(r * C, (r + 1) * C)
        q, k, v = (dev[x][:, sl].contiguous() for x in ("q", "k", "v"))
        o, kv_out, cache = L.fwd_local(q, k, v, lam, kv_in=kv)
        outs.append(o)
        caches.append(cache)
        kvs.append(kv_out)
        kv = kv_out
    grads = [None] * T
    dkv = None
    for r in range(T - 1, -1, -1):
        sl = slice(r * C, (r + 1) * C)
        q, k, v, do = (dev[x][:, sl].contiguous() for x in ("q", "k", "v", "do"))
        dq, dk, dv, dkv_out = L.bwd_local(q, k, v, lam, do, caches[r], dkv_in=dkv)
        grads[r] = (dq, dk, dv)
        dkv = dkv_out
    torch.cuda.synchronize()
    cat = lambda ts: torch.cat(ts, dim=1).float().cpu().numpy()
    return (cat(outs), cat([g[0] for g in grads]), cat([g[1] for g in grads]), cat([g[2] for g in grads]),
            [x.cpu().numpy() for x in kvs], dkv.cpu().numpy())


def check_against_oracle(oracle_mod, p, res, tol):
    o_ref = oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])
    dq_ref, dk_ref, dv_ref = oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])
    errs = {"o": per_head_err(res[0], o_ref), "dq": per_head_err(res[1], dq_ref),
            "dk": per_head_err(res[2], dk_ref), "dv": per_head_err(res[3], dv_ref)}
    assert max(errs.values()) <= tol, errs
    return errs


# ---- config 1 (BASELINE configs[0]): 1 head x 32, N=512, lambda=0.99, 4-rank ring, fp32 ------------
def test_config1_fp32_sim_ring(L, oracle_mod):
    p = synth.problem(0, 1, 512, 1, 32, dtype="fp32", lam=0.99)
    res = run_sim_ring(L, p, 4, torch.float32, 512)
    check_against_oracle(oracle_mod, p, res, FP32_TOL)
    # the states crossing the ring equal the oracle's Alg. 2 cache entries (state entering rank r+1)
    _, cache, _, _ = oracle_mod.lasp_fwd_sim(p["q"], p["k"], p["v"], p["lam"], 4)
    for r in range(3):
        ref = cache[r + 1]
        assert np.max(np.abs(res[4][r] - ref)) / np.max(np.abs(ref)) <= FP32_TOL


@pytest.mark.parametrize("seed", range(5))
def test_config1_fp32_seeds(L, oracle_mod, seed):
    p = synth.problem(seed, 1, 512, 1, 32, dtype="fp32", lam=0.99)
    res = run_sim_ring(L, p, 4, torch.float32, 512)
    check_against_oracle(oracle_mod, p, res, FP32_TOL)


# ---- bf16 across head dims, rank counts, lambdas, ragged tails --------------------------------------
@pytest.mark.parametrize("D", [32, 64, 128])
@pytest.mark.parametrize("T", [1, 2, 4, 8])
def test_bf16_sim_ring_head_dims(L, oracle_mod, D, T):
    N = 2048
    p = synth.problem(1, 1, N, 4, D, dtype="bf16")
    res = run_sim_ring(L, p, T, torch.bfloat16, N)
    check_against_oracle(oracle_mod, p, res, BF16_TOL)


@pytest.mark.parametrize("lam", [1.0, 0.99, 0.9, 0.5, 0.1, 1e-3])
def test_bf16_scalar_lambdas(L, oracle_mod, lam):
    p = synth.problem(2, 2, 1536, 2, 64, dtype="bf16", lam=lam)
    res = run_sim_ring(L, p, 2, torch.bfloat16, 1536)
    check_against_oracle(oracle_mod, p, res, BF16_TOL)


@pytest.mark.parametrize("N", [1, 5, 127, 129, 1000, 3001])
def test_bf16_ragged_lengths(L, oracle_mod, N):
    p = synth.problem(3, 1, N, 3, 64, dtype="bf16")
    res = run_sim_ring(L, p, 1, torch.bfloat16, N)
    check_against_oracle(oracle_mod, p, res, BF16_TOL)


@pytest.mark.parametrize("B,N,H,D,T", [(1, 130, 256, 64, 1),   # the maximum head count (kMaxHeads)
                                       (1, 256, 256, 128, 2),  # max heads at head_dim 128, 2 ranks
                                       (8, 2, 2, 128, 2),      # one token per rank, batch 8
                                       (5, 387, 3, 64, 3)])    # batch 5, ragged 129-token ranks
def test_extreme_shapes(L, oracle_mod, B, N, H, D, T):
    """Edge sizes: 256 heads (per-head lambda of the TNL recipe, every head checked), batch 8 with a single
    token per rank, batch 5 with ragged ranks -- against the oracle, through the simulated ring."""
    p = synth.problem(5, B, N, H, D, dtype="bf16")
    res = run_sim_ring(L, p, T, torch.bfloat16, N)
    check_against_oracle(oracle_mod, p, res, BF16_TOL)


@pytest.mark.parametrize("D", [32, 128])
def test_fp32_path_other_dims(L, oracle_mod, D):
    p = synth.problem(4, 1, 700, 2, D, dtype="fp32")
    res = run_sim_ring(L, p, 1, torch.float32, 700)
    check_against_oracle(oracle_mod, p, res, FP32_TOL)


def test_forced_segment_lengths(L, oracle_mod, monkeypatch):
    """Several segments per head plus a ragged last segment (the in-GPU LASP level)."""
    p = synth.problem(5, 1, 1000, 2, 64, dtype="bf16")
    for seg in ("128", "384"):
        monkeypatch.setenv("LASP_SEG_LEN", seg)
        res = run_sim_ring(L, p, 1, torch.bfloat16, 1000)
        check_against_oracle(oracle_mod, p, res, BF16_TOL)


# ---- edge cases --------------------------------------------------------------------------------------
def test_empty_rank_forwards_state(L):
    q = torch.empty((1, 0, 2, 64), dtype=torch.bfloat16, device="cuda")
    kv_in = torch.randn(1, 2, 64, 64, device="cuda")
    o, kv_out, cache = L.fwd_local(q, q, q, [0.9, 0.5], kv_in=kv_in)
    dkv_in = torch.randn(1, 2, 64, 64, device="cuda")
    dq, dk, dv, dkv_out = L.bwd_local(q, q, q, [0.9, 0.5], q, cache, dkv_in=dkv_in)
    torch.cuda.synchronize()
    assert torch.equal(kv_out, kv_in) and torch.equal(dkv_out, dkv_in)
    assert o.numel() == 0 and dq.numel() == 0


def test_deterministic_bitwise(L):
    p = synth.problem(6, 1, 4096, 4, 64, dtype="bf16")
    a = run_sim_ring(L, p, 2, torch.bfloat16, 4096)
    b = run_sim_ring(L, p, 2, torch.bfloat16, 4096)
    for x, y in zip(a[:4], b[:4]):
        assert np.array_equal(x, y)


def test_state_error_on_mismatched_cache(L):
    """The cache tag is checked on the device: a mismatch makes every output NaN and
    lasp_workspace_status report LASP_ERR_STATE; a matching pair reports OK with finite outputs."""
    from paper_2404_02882_b200._native import LaspError
    q = torch.full((1, 256, 2, 64), 0.25, dtype=torch.bfloat16, device="cuda")
    ws = L.alloc_workspace(q)
    _, _, cache = L.fwd_local(q, q, q, [0.9, 0.9])
    dq, dk, dv, dkv = L.bwd_local(q, q, q, [0.9, 0.9], q, cache, workspace=ws, check_state=True)
    assert all(torch.isfinite(t.float()).all() for t in (dq, dk, dv, dkv))
    with pytest.raises(LaspError) as e:
        L.bwd_local(q, q, q, [0.9, 0.8], q, cache, workspace=ws, check_state=True)   # different lambda
    assert e.value.name == "LASP_ERR_STATE" and "lambda" in str(e.value)
    dq, dk, dv, dkv = L.bwd_local(q, q, q, [0.9, 0.8], q, cache, workspace=ws)
    assert all(torch.isnan(t.float()).all() for t in (dq, dk, dv))      # loud without the check too
    with pytest.raises(LaspError) as e:
        L.bwd_local(q, q, q, [0.9, 0.9], q, torch.zeros_like(cache), workspace=ws, check_state=True)  # never written
    assert e.value.name == "LASP_ERR_STATE" and "magic" in str(e.value)
    q2 = torch.full((1, 128, 2, 64), 0.25, dtype=torch.bfloat16, device="cuda")
    _, _, cache2 = L.fwd_local(q2, q2, q2, [0.9, 0.9], cache=torch.empty_like(cache))
    with pytest.raises(LaspError) as e:   # a cache of another length in a buffer large enough for this one
        L.bwd_local(q, q, q, [0.9, 0.9], q, cache2, workspace=ws, check_state=True)
    assert e.value.name == "LASP_ERR_STATE" and "n_local" in str(e.value)


def test_state_error_on_reused_cache_address(L):
    """A freed cache whose address the caching allocator hands out again is judged by its contents: after a
    forward with another lambda has written the reused block, a backward expecting the first forward's
    lambda fails with LASP_ERR_STATE (the r1 host-side pointer registry accepted it)."""
    from paper_2404_02882_b200._native import LaspError
    q = torch.full((1, 512, 4, 64), 0.5, dtype=torch.bfloat16, device="cuda")
    ws = L.alloc_workspace(q)
    cache = L.alloc_cache(q)
    addr = cache.data_ptr()
    L.fwd_local(q, q, q, [0.9] * 4, cache=cache)
    torch.cuda.synchronize()
    del cache
    reused = L.alloc_cache(q)
    assert reused.data_ptr() == addr              # the allocator reused the block
    L.fwd_local(q, q, q, [0.7] * 4, cache=reused)  # another layer's forward writes it
    with pytest.raises(LaspError) as e:
        L.bwd_local(q, q, q, [0.9] * 4, q, reused, workspace=ws, check_state=True)
    assert e.value.name == "LASP_ERR_STATE"


@pytest.mark.parametrize("D", [64, 128])
def test_many_segments_parity(L, oracle_mod, monkeypatch, D):
    """52 segments of 128 tokens (ragged tail): the prefix fold runs in two load batches of at most 40 segments
    (fused fold and prefix kernel alike), against the fp64 oracle."""
    monkeypatch.setenv("LASP_SEG_LEN", "128")
    p = synth.problem(13 + D, 1, 51 * 128 + 40, 2, D, dtype="bf16")
    res = run_sim_ring(L, p, 1, torch.bfloat16, 51 * 128 + 40)
    check_against_oracle(oracle_mod, p, res, BF16_TOL)


def test_ragged_multi_segment_rev_store_deterministic(L, oracle_mod, monkeypatch):
    """with several segments and a ragged rank length, the REV passes' ragged block starts inside
    the previous segment; only the segment's own rows may be stored (else two CTAs race on those rows with
    differently rounded values). B=1, H=4, D=64, C=1000: 8 segments of 128 tokens with a 104-token tail
    (forced: the plan itself now keeps at least 2 blocks per segment at this length)."""
    monkeypatch.setenv("LASP_SEG_LEN", "128")
    assert L.segment_len(L.api._shape(torch.empty((1, 1000, 4, 64), dtype=torch.bfloat16, device="meta"))) == 128
    p = synth.problem(11, 1, 1000, 4, 64, dtype="bf16")
    runs = [run_sim_ring(L, p, 1, torch.bfloat16, 1000) for _ in range(6)]
    for r in runs[1:]:
        for x, y in zip(runs[0][:4], r[:4]):
            assert np.array_equal(x, y)
    check_against_oracle(oracle_mod, p, runs[0], BF16_TOL)


def test_autograd_function(L, oracle_mod):
    p = synth.problem(7, 1, 640, 2, 64, dtype="bf16")
    q, k, v = (to_dev(p[x], torch.bfloat16).requires_grad_() for x in ("q", "k", "v"))
    o = L.lasp_attention(q, k, v, p["lam"])
    o.backward(to_dev(p["do"], torch.bfloat16))
    res = (o.detach().float().cpu().numpy(), q.grad.float().cpu().numpy(), k.grad.float().cpu().numpy(),
           v.grad.float().cpu().numpy())
    check_against_oracle(oracle_mod, p, res, BF16_TOL)


# ---- config 2 (BASELINE configs[1], the bench workload) at full size --------------------------------
def test_config2_full_size_parity(L, oracle_mod):
    """TNL-0.4B layer: 16 heads x 64, N=32K, bf16, one GPU -- every element against the oracle,
    in the launch configuration bench.py times (fwd_local + bwd_local, default plan)."""
    p = synth.problem(0, 1, 32768, 16, 64, dtype="bf16")
    res = run_sim_ring(L, p, 1, torch.bfloat16, 32768)
    errs = check_against_oracle(oracle_mod, p, res, BF16_TOL)
    # Euler identity (L is linear in each of Q, K, V): <Q,dQ> = <K,dK> = <V,dV> = <O,dO>
    lo = float(np.sum(res[0].astype(np.float64) * p["do"]))
    for x, g in (("q", res[1]), ("k", res[2]), ("v", res[3])):
        assert abs(float(np.sum(p[x].astype(np.float64) * g)) - lo) <= 2e-2 * abs(lo)
    print("config2 errors", errs)


# ---- config 3 (TNL-1B, 16 heads x 128) at the per-rank shape bench.py --config tnl1b times -------
def test_config3_rank_shape_parity(L, oracle_mod):
    """16 heads x 128, n_local = 32K (config 3's per-rank shard), two simulated ranks so that the second
    one runs with a received KV_in / dKV_in; every element against the oracle."""
    p = synth.problem(3, 1, 65536, 16, 128, dtype="bf16")
    res = run_sim_ring(L, p, 2, torch.bfloat16, 65536)
    errs = check_against_oracle(oracle_mod, p, res, BF16_TOL)
    print("config3 errors", errs)


@pytest.mark.parametrize("D", [64, 128])
def test_constant_input_closed_form_long_sequence(L, D):
    """Closed forms for constant inputs (derived from Eq. 4): no oracle needed, N = 256K."""
    N, H = 262144, 2
    lam = np.array([0.999, 1.0], dtype=np.float32)
    rng = np.random.default_rng(0)
    qv, kv_, vv, dov = (synth.round_bf16(rng.standard_normal((H, D)).astype(np.float32) * 0.3) for _ in range(4))
    mk = lambda a: torch.from_numpy(np.broadcast_to(a, (1, N, H, D)).copy()).to(torch.bfloat16).cuda()
    o, _, cache = L.fwd_local(mk(qv), mk(kv_), mk(vv), lam)
    dq, dk, dv, _ = L.bwd_local(mk(qv), mk(kv_), mk(vv), lam, mk(dov), cache)
    torch.cuda.synchronize()
    s = np.arange(1, N + 1, dtype=np.float64)
    for h in range(H):
        l = float(lam[h])
        geo = (lambda n: n) if l == 1.0 else (lambda n: (1 - l ** n) / (1 - l))
        qk = float(qv[h].astype(np.float64) @ kv_[h]); vd = float(vv[h].astype(np.float64) @ dov[h])
        idx = np.array([0, 1, 100, 4095, 65535, N - 1])
        for got, ref in ((o, qk * np.outer(geo(s[idx]), vv[h])), (dq, vd * np.outer(geo(s[idx]), kv_[h])),
                         (dk, vd * np.outer(geo(N - s[idx] + 1), qv[h])),
                         (dv, qk * np.outer(geo(N - s[idx] + 1), dov[h]))):
            g = got[0, idx, h].float().cpu().numpy()
            assert np.max(np.abs(g - ref)) <= BF16_TOL * np.max(np.abs(ref)) + 1e-6


def test_cuda_graph_replay_matches_eager(L):
    """bench.py replays the step from a CUDA graph: the captured fwd_local + bwd_local launches (with their
    programmatic-dependent-launch edges) must reproduce the eager results bit for bit."""
    p = synth.problem(10, 1, 4096, 4, 64, dtype="bf16")
    q, k, v, do = (to_dev(p[x], torch.bfloat16) for x in ("q", "k", "v", "do"))
    o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))
    cache, ws = L.alloc_cache(q), L.alloc_workspace(q)

    def step():
        L.fwd_local(q, k, v, p["lam"], o=o, kv_out=False, cache=cache, workspace=ws)
        L.bwd_local(q, k, v, p["lam"], do, cache, dq=dq, dk=dk, dv=dv, dkv_out=False, workspace=ws)

    step()
    torch.cuda.synchronize()
    eager = [t.clone() for t in (o, dq, dk, dv)]
    for t in (o, dq, dk, dv):
        t.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, (o, dq, dk, dv)):
        assert torch.equal(a, b)


# ---- config 4 (TNL-7B, 32 heads x 128, per-head decay, 128K tokens per rank) ---------------------------
def test_config4_heads_parity(L, oracle_mod):
    """32 heads x 128 with per-head lambda (config 4's head layout and segment plan family), 32K tokens:
    every element of every head against the oracle."""
    p = synth.problem(4, 1, 32768, 32, 128, dtype="bf16")
    res = run_sim_ring(L, p, 1, torch.bfloat16, 32768)
    errs = check_against_oracle(oracle_mod, p, res, BF16_TOL)
    print("config4 heads errors", errs)


def test_config4_rank_shape_closed_form(L):
    """Config 4's per-rank shard at full size (32 heads x 128, n_local = 131072, per-head lambda from the
    TNL recipe, the plan bench.py --config tnl7b times): constant inputs per head have closed forms
    (derived from Eq. 4), checked at sampled positions of every head."""
    N, H, D = 131072, 32, 128
    lam = synth.head_lambdas(H, None)
    rng = np.random.default_rng(4)
    qv, kv_, vv, dov = (synth.round_bf16(rng.standard_normal((H, D)).astype(np.float32) * 0.3) for _ in range(4))
    mk = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).cuda() \
        .view(1, 1, H, D).expand(1, N, H, D).contiguous()
    o, _, cache = L.fwd_local(mk(qv), mk(kv_), mk(vv), lam)
    dq, dk, dv, _ = L.bwd_local(mk(qv), mk(kv_), mk(vv), lam, mk(dov), cache)
    torch.cuda.synchronize()
    idx = np.array([0, 1, 127, 128, 4095, 65535, 100000, N - 1])
    s = idx.astype(np.float64) + 1
    got = {n: t[0, idx].float().cpu().numpy() for n, t in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv))}
    for h in range(H):
        l = float(lam[h])
        geo = (lambda n: n) if l == 1.0 else (lambda n: (1 - l ** n) / (1 - l))
        qk = float(qv[h].astype(np.float64) @ kv_[h]); vd = float(vv[h].astype(np.float64) @ dov[h])
        for name, ref in (("o", qk * np.outer(geo(s), vv[h])), ("dq", vd * np.outer(geo(s), kv_[h])),
                          ("dk", vd * np.outer(geo(N - s + 1), qv[h])), ("dv", qk * np.outer(geo(N - s + 1), dov[h]))):
            g = got[name][:, h]
            assert np.max(np.abs(g - ref)) <= BF16_TOL * np.max(np.abs(ref)) + 1e-6, (name, h)


def test_layer_trains_through_autograd(L):
    """A linear-attention layer (torch projections + lasp_attention) fits a fixed target: the library's
    forward / backward inside torch.autograd drive the loss down over a few optimiser steps."""
    torch.manual_seed(0)
    B, N, d, H, D = 1, 2048, 256, 4, 64
    qkv = torch.nn.Linear(d, 3 * H * D, bias=False).cuda()
    out = torch.nn.Linear(H * D, d, bias=False).cuda()
    opt = torch.optim.Adam(list(qkv.parameters()) + list(out.parameters()), lr=3e-3)
    lam = [0.5, 0.9, 0.99, 0.999]
    x = torch.randn(B, N, d, device="cuda")
    target = torch.randn(B, N, d, device="cuda") * 0.1
    losses = []
    for _ in range(30):
        q, k, v = qkv(x).view(B, N, 3, H, D).to(torch.bfloat16).unbind(2)
        o = L.lasp_attention(q.contiguous(), k.contiguous(), v.contiguous(), lam)
        loss = (out(o.float().reshape(B, N, H * D)) - target).square().mean()
        opt.zero_grad()
        loss.backward()
        opt.step()
        losses.append(loss.item())
    assert all(np.isfinite(losses)) and losses[-1] < 0.5 * losses[0], losses


def test_config5_longest_sequence_closed_form(L):
    """BASELINE configs[4]'s longest point on one GPU: TNL-1B shape (16 heads x 128), 2048K tokens (8.6 GB per
    tensor), per-head lambda; constant inputs per head have closed forms (Eq. 4), checked at sampled
    positions spread over the whole sequence for every head (no oracle run needed at this size)."""
    N, H, D = 2097152, 16, 128
    free, _ = torch.cuda.mem_get_info()
    if free < 80e9:
        pytest.skip("needs ~70 GB of free device memory")
    lam = synth.head_lambdas(H, None)
    rng = np.random.default_rng(5)
    qv, kv_, vv, dov = (synth.round_bf16(rng.standard_normal((H, D)).astype(np.float32) * 0.3) for _ in range(4))
    mk = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).cuda() \
        .view(1, 1, H, D).expand(1, N, H, D).contiguous()
    q, k, v = mk(qv), mk(kv_), mk(vv)
    o, _, cache = L.fwd_local(q, k, v, lam)
    idx = np.array([0, 1, 1000, 65535, 1048575, 1500000, N - 2, N - 1])
    o_s = o[0, idx].float().cpu().numpy()
    del o
    do = mk(dov)
    dq, dk, dv, _ = L.bwd_local(q, k, v, lam, do, cache)
    torch.cuda.synchronize()
    got = {"o": o_s, "dq": dq[0, idx].float().cpu().numpy(), "dk": dk[0, idx].float().cpu().numpy(),
           "dv": dv[0, idx].float().cpu().numpy()}
    s = idx.astype(np.float64) + 1
    for h in range(H):
        l = float(lam[h])
        geo = (lambda n: n) if l == 1.0 else (lambda n: (1 - l ** n) / (1 - l))
        qk = float(qv[h].astype(np.float64) @ kv_[h]); vd = float(vv[h].astype(np.float64) @ dov[h])
        for name, ref in (("o", qk * np.outer(geo(s), vv[h])), ("dq", vd * np.outer(geo(s), kv_[h])),
                          ("dk", vd * np.outer(geo(N - s + 1), qv[h])), ("dv", qk * np.outer(geo(N - s + 1), dov[h]))):
            g = got[name][:, h]
            assert np.max(np.abs(g - ref)) <= BF16_TOL * np.max(np.abs(ref)) + 1e-6, (name, h)


@pytest.mark.parametrize("case", range(12))
def test_random_shapes_sim_ring(L, oracle_mod, case):
    """Seeded random shapes: batch 1-3, heads 1-5, head_dim 32/64/128, 1-4 simulated ranks of ragged or
    block-aligned length, bf16 or fp32, random per-head lambda in (0.3, 1] (incl. exactly 1)."""
    rng = np.random.default_rng(1000 + case)
    B, H = int(rng.integers(1, 4)), int(rng.integers(1, 6))
    D = int(rng.choice([32, 64, 128]))
    T = int(rng.integers(1, 5))
    C = int(rng.choice([int(rng.integers(1, 400)), 128 * int(rng.integers(1, 4))]))
    dtype = "fp32" if case % 4 == 3 else "bf16"
    lam = rng.uniform(0.3, 1.0, H).astype(np.float32)
    lam[rng.integers(0, H)] = 1.0
    p = synth.problem(2000 + case, B, C * T, H, D, dtype=dtype)
    p["lam"] = lam
    res = run_sim_ring(L, p, T, torch.float32 if dtype == "fp32" else torch.bfloat16, C * T)
    check_against_oracle(oracle_mod, p, res, FP32_TOL if dtype == "fp32" else BF16_TOL)


_LONG = int(__import__("os").environ.get("LASP_LONG_SWEEP", "0"))


@pytest.mark.parametrize("case", range(100, 100 + _LONG))
def test_random_shapes_long_sweep(L, oracle_mod, case):
    """Opt-in (LASP_LONG_SWEEP=<count>): the same seeded random-shape generator as above over many more
    cases, with per-rank lengths up to 3000 tokens (several segments, ragged tails)."""
    rng = np.random.default_rng(7000 + case)
    B, H = int(rng.integers(1, 4)), int(rng.integers(1, 9))
    D = int(rng.choice([32, 64, 128]))
    T = int(rng.integers(1, 5))
    C = int(rng.choice([int(rng.integers(1, 3000)), 128 * int(rng.integers(1, 24))]))
    dtype = "fp32" if case % 5 == 4 else "bf16"
    lam = rng.uniform(0.3, 1.0, H).astype(np.float32)
    lam[rng.integers(0, H)] = 1.0
    p = synth.problem(9000 + case, B, C * T, H, D, dtype=dtype)
    p["lam"] = lam
    res = run_sim_ring(L, p, T, torch.float32 if dtype == "fp32" else torch.bfloat16, C * T)
    check_against_oracle(oracle_mod, p, res, FP32_TOL if dtype == "fp32" else BF16_TOL)


_PLAN = int(__import__("os").environ.get("LASP_PLAN_SWEEP", "0"))


@pytest.mark.parametrize("case", range(_PLAN))
def test_random_shapes_long_segment_plan(L, oracle_mod, case):
    """Opt-in (LASP_PLAN_SWEEP=<count>): head_dim-128 shapes large enough for the 28-block segment plan (B*H*2*nseg
    >= 296), random lengths with ragged last segments, against the fp64 oracle."""
    rng = np.random.default_rng(11000 + case)
    B = int(rng.integers(1, 3))
    H = int(rng.choice([8, 12, 16, 24]))
    nb_min = -(-296 // (2 * B * H)) * 28  # blocks for enough 28-block segments
    C = int(rng.integers(max(nb_min - 27, 1) * 128, max(nb_min, 160) * 128 + 1))
    lam = rng.uniform(0.3, 1.0, H).astype(np.float32)
    p = synth.problem(12000 + case, B, C, H, 128, dtype="bf16")
    p["lam"] = lam
    shape = L.api._shape(torch.empty((B, C, H, 128), dtype=torch.bfloat16, device="meta"))
    seg = L.segment_len(shape)
    res = run_sim_ring(L, p, 1, torch.bfloat16, C)
    check_against_oracle(oracle_mod, p, res, BF16_TOL)
    print(f"case {case}: B={B} H={H} C={C} seg_len={seg}")


_FOLD_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import synth, paper_2404_02882_b200 as L
out = {{}}
import os
# (B, H, D, C, forced segment length): small states; B*H*D*D/2 = 65536 float2 = 256 fold chunks for at most 148 CTAs
# (2 rounds); and segment counts on both sides of the prefix kernel's load batches (U = 8 / 16 / 24 / 40: 13, 21 and
# 52 segments, the last folded in two batches of at most 40)
for B, H, D, C, seg in ((2, 3, 64, 3 * 1024 + 384, 0), (2, 3, 128, 2 * 1024 + 256, 0), (2, 16, 64, 4096 + 640, 0),
                        (1, 2, 64, 13 * 128, 128), (1, 2, 128, 20 * 128 + 10, 128), (1, 2, 64, 51 * 128 + 40, 128)):
    if seg:
        os.environ["LASP_SEG_LEN"] = str(seg)
    else:
        os.environ.pop("LASP_SEG_LEN", None)
    p = synth.problem(77 + D + H + seg, B, C, H, D, dtype="bf16")
    q, k, v, do = (torch.from_numpy(np.ascontiguousarray(p[x])).cuda().to(torch.bfloat16) for x in ("q", "k", "v", "do"))
    g = torch.Generator().manual_seed(D)
    kv_in = torch.randn(B, H, D, D, generator=g).cuda()
    dkv_in = torch.randn(B, H, D, D, generator=g).cuda()
    o, kv_out, cache = L.fwd_local(q, k, v, p["lam"], kv_in)
    dq, dk, dv, dkv_out = L.bwd_local(q, k, v, p["lam"], do, cache, dkv_in)
    for n, t in zip(("o", "kv_out", "dq", "dk", "dv", "dkv_out"), (o, kv_out, dq, dk, dv, dkv_out)):
        out[f"{{n}}{{D}}_{{H}}_{{C}}"] = t.float().cpu().numpy()
np.savez({dst!r}, **out)
"""


@pytest.mark.parametrize("pdl", ["on", "off"])
def test_fused_prefix_fold_matches_separate_kernel(tmp_path, pdl):
    """The local path folds F2 / B2 into the following core launch (claimed chunks, PrefixFold); with
    LASP_NO_FUSED_FOLD=1 it runs the separate prefix kernel. Same arithmetic in the same order, so every
    output (including kv_out / dkv_out with a nonzero kv_in / dkv_in, D = 64 and 128, ragged segments,
    batch 2, a state large enough for two rounds of fold chunks per CTA) must agree bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for off in ("0", "1"):
        dst = str(tmp_path / f"fold{off}.npz")
        env = dict(os.environ, LASP_NO_FUSED_FOLD=off)
        if pdl == "off":  # launches without the programmatic-serialization attribute
            env["LASP_NO_PDL"] = "1"
        script = _FOLD_SCRIPT.format(root=root, tests=os.path.join(root, "tests"), dst=dst)
        subprocess.run([sys.executable, "-c", script], env=env, check=True, timeout=300)
        res[off] = np.load(dst)
    for key in res["0"].files:
        assert np.array_equal(res["0"][key], res["1"][key]), key


def test_concurrent_streams_fused_fold(L):
    """The fused prefix fold waits on a done-counter of claimed chunks, not on a per-CTA barrier, so two
    calls running at the same time on two streams (each with its own workspace; their core launches
    compete for the SMs) complete and give the same results as the same calls run one after the other."""
    shapes = [(1, 8192, 16, 64), (2, 4096, 4, 128)]
    runs = []
    for i, (B, C, H, D) in enumerate(shapes):
        p = synth.problem(90 + i, B, C, H, D, dtype="bf16")
        q, k, v, do = (to_dev(p[x], torch.bfloat16) for x in ("q", "k", "v", "do"))
        runs.append((p["lam"], q, k, v, do, L.alloc_workspace(q)))

    def call(r):
        lam, q, k, v, do, ws = r
        o, _, cache = L.fwd_local(q, k, v, lam, workspace=ws)
        dq, dk, dv, _ = L.bwd_local(q, k, v, lam, do, cache, workspace=ws)
        return [o, dq, dk, dv]

    ref = [[t.clone() for t in call(r)] for r in runs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in runs]
    for _ in range(5):
        outs = []
        for s, r in zip(streams, runs):
            with torch.cuda.stream(s):
                outs.append(call(r))
        torch.cuda.synchronize()
        for got, want in zip(outs, ref):
            for a, b in zip(got, want):
                assert torch.equal(a, b)


# ---- grouped-query / multi-query attention ---------------------------------
def run_sim_ring_gqa(L, p, T, n_global):
    """As run_sim_ring, with k, v (dk, dv, the states and lambda) on Hk < H heads."""
    C = n_global // T
    dev = {k: to_dev(p[k], torch.bfloat16) for k in ("q", "k", "v", "do")}
    lam = p["lam"]
    outs, caches, kv = [], [], None
    for r in range(T):
        sl = slice(r * C, (r + 1) * C)
        q, k, v = (dev[x][:, sl].contiguous() for x in ("q", "k", "v"))
        o, kv, cache = L.fwd_local(q, k, v, lam, kv_in=kv)
        outs.append(o)
        caches.append(cache)
    grads, dkv = [None] * T, None
    for r in range(T - 1, -1, -1):
        sl = slice(r * C, (r + 1) * C)
        q, k, v, do = (dev[x][:, sl].contiguous() for x in ("q", "k", "v", "do"))
        dq, dk, dv, dkv = L.bwd_local(q, k, v, lam, do, caches[r], dkv_in=dkv, check_state=True)
        grads[r] = (dq, dk, dv)
    torch.cuda.synchronize()
    cat = lambda ts: torch.cat(ts, dim=1).float().cpu().numpy()
    return cat(outs), cat([g[0] for g in grads]), cat([g[1] for g in grads]), cat([g[2] for g in grads])


@pytest.mark.parametrize("B,N,H,Hk,D,T", [(1, 1536, 4, 2, 64, 2),     # GQA, 2 ranks
                                          (1, 1000, 8, 1, 128, 1),    # MQA, ragged, head_dim 128
                                          (2, 2048, 6, 3, 64, 4),     # batch 2, 4 ranks
                                          (1, 3000, 8, 2, 128, 3),    # ragged ranks, several segments
                                          (1, 640, 4, 4, 64, 2)])     # Hk = H through the GQA API (= MHA)
def test_gqa_sim_ring_matches_oracle(L, oracle_mod, B, N, H, Hk, D, T):
    p = synth.problem(60 + H + Hk, B, N, H, D, dtype="bf16", kv_heads=Hk)
    got = run_sim_ring_gqa(L, p, T, N)
    refs = [oracle_mod.fwd_gqa(p["q"], p["k"], p["v"], p["lam"])] + \
        list(oracle_mod.bwd_gqa(p["q"], p["k"], p["v"], p["lam"], p["do"]))
    errs = {n: per_head_err(x, r) for n, x, r in zip(("o", "dq", "dk", "dv"), got, refs)}
    assert max(errs.values()) <= BF16_TOL, errs


@pytest.mark.parametrize("H,Hk,D", [(16, 4, 64), (16, 4, 128)])
def test_gqa_tnl_shapes_full_size(L, oracle_mod, H, Hk, D):
    """TNL-0.4B / TNL-1B layer shapes (32K tokens) with 4 kv-heads (G = 4), every element against the
    oracle's grouped-query recurrence."""
    N = 32768
    p = synth.problem(7, 1, N, H, D, dtype="bf16", kv_heads=Hk)
    got = run_sim_ring_gqa(L, p, 1, N)
    refs = [oracle_mod.fwd_gqa(p["q"], p["k"], p["v"], p["lam"])] + \
        list(oracle_mod.bwd_gqa(p["q"], p["k"], p["v"], p["lam"], p["do"]))
    errs = {n: per_head_err(x, r) for n, x, r in zip(("o", "dq", "dk", "dv"), got, refs)}
    assert max(errs.values()) <= BF16_TOL, errs


def test_gqa_deterministic_and_rejects_unsupported(L):
    from paper_2404_02882_b200._native import LaspError
    p = synth.problem(61, 1, 2000, 8, 64, dtype="bf16", kv_heads=2)
    a = run_sim_ring_gqa(L, p, 2, 2000)
    b = run_sim_ring_gqa(L, p, 2, 2000)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    q = torch.zeros((1, 128, 4, 32), dtype=torch.bfloat16, device="cuda")   # head_dim 32: CUDA-core path
    k = torch.zeros((1, 128, 2, 32), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(LaspError) as e:
        L.fwd_local(q, k, k, [0.9, 0.9])
    assert e.value.name == "LASP_ERR_UNSUPPORTED"
