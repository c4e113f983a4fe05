"""Pins for the fp64 oracle (oracle/) against things other than itself.

Each test states what pins what. Citations: P:n = PAPER.md line n,
S:n = SPEC.md line n. All CPU-only.
"""
import json
import os

import numpy as np
import pytest
import torch

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rand_problem(seed, B, N, H, D, lam=None):
    p = synth.problem(seed, B, N, H, D, dtype="fp32", lam=lam)
    return {k: p[k].astype(np.float64) if k != "lam" else p[k] for k in p}


def dense_mask(N, lam):
    """M_ij = lam^(i-j) for i>=j (Alg. 2) built with numpy power (not the oracle's
    repeated multiplication)."""
    i = np.arange(N)[:, None]
    j = np.arange(N)[None, :]
    e = np.where(i >= j, i - j, 0).astype(np.float64)
    return np.where(i >= j, np.power(np.float64(lam), e), 0.0)


def dense_fwd(q, k, v, lam):
    """Eq. 2 without Norm: O = [(Q K^T) (.) M] V, per (b, h), numpy fp64."""
    B, N, H, D = q.shape
    o = np.zeros_like(q)
    for b in range(B):
        for h in range(H):
            M = dense_mask(N, float(np.float64(np.float32(lam[h]))))
            o[b, :, h] = ((q[b, :, h] @ k[b, :, h].T) * M) @ v[b, :, h]
    return o


def dense_torch_grads(q, k, v, lam, do):
    """torch fp64 autograd of L = sum(O * dO) on the dense masked form (pin 2)."""
    tq, tk, tv = (torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in (q, k, v))
    B, N, H, D = q.shape
    outs = []
    for h in range(H):
        M = torch.tensor(dense_mask(N, float(np.float64(np.float32(lam[h])))))
        s = torch.einsum("bid,bjd->bij", tq[:, :, h], tk[:, :, h]) * M
        outs.append(torch.einsum("bij,bjd->bid", s, tv[:, :, h]))
    o = torch.stack(outs, dim=2)
    (o * torch.tensor(do)).sum().backward()
    return tq.grad.numpy(), tk.grad.numpy(), tv.grad.numpy()


def rel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / den) if den > 0 else float(np.max(np.abs(x)))


# ---------------------------------------------------------------------------------------------
# pin 1: dense masked form (Eq. 2 without Norm) -- oracle forward, S:694 criterion 1
@pytest.mark.parametrize("lam", [1.0, 0.99, 0.9, 0.5])
@pytest.mark.parametrize("N,D", [(16, 4), (64, 16), (256, 32)])
def test_fwd_matches_dense_masked_form(oracle_mod, lam, N, D):
    for seed in range(2):
        p = rand_problem(seed, 1, N, 2, D, lam=lam)
        o = oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])
        ref = dense_fwd(p["q"], p["k"], p["v"], p["lam"])
        assert rel(o, ref) <= 1e-12


def test_fwd_per_head_lambdas_batch(oracle_mod):
    p = rand_problem(3, 2, 96, 4, 8)  # per-head TNL recipe, B=2
    o = oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])
    assert rel(o, dense_fwd(p["q"], p["k"], p["v"], p["lam"])) <= 1e-12


# pin 2: fp64 autograd of the dense form -- oracle backward
@pytest.mark.parametrize("lam", [1.0, 0.95, 0.5])
def test_bwd_matches_torch_autograd(oracle_mod, lam):
    p = rand_problem(7, 2, 48, 2, 8, lam=lam)
    dq, dk, dv = oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])
    rq, rk, rv = dense_torch_grads(p["q"], p["k"], p["v"], p["lam"], p["do"])
    for x, r in ((dq, rq), (dk, rk), (dv, rv)):
        assert rel(x, r) <= 1e-12


# pin 2b: the paper's masked closed forms via numpy, full sequence T=1
def test_bwd_matches_paper_masked_products(oracle_mod):
    p = rand_problem(11, 1, 40, 1, 6, lam=0.8)
    q, k, v, do = (p[x][0, :, 0] for x in ("q", "k", "v", "do"))
    M = dense_mask(40, float(np.float64(np.float32(0.8))))
    dq_ref = ((do @ v.T) * M) @ k
    dk_ref = ((do @ v.T) * M).T @ q
    dv_ref = ((q @ k.T) * M).T @ do
    dq, dk, dv = oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])
    assert rel(dq[0, :, 0], dq_ref) <= 1e-12
    assert rel(dk[0, :, 0], dk_ref) <= 1e-12
    assert rel(dv[0, :, 0], dv_ref) <= 1e-12


# pin 3: central finite differences of L = sum(O * dO)
def test_bwd_matches_finite_differences(oracle_mod):
    p = rand_problem(5, 1, 12, 1, 3, lam=0.9)
    dq, dk, dv = oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])
    eps = 1e-6

    def loss(q, k, v):
        return float(np.sum(oracle_mod.fwd(q, k, v, p["lam"]) * p["do"]))

    for name, g in (("q", dq), ("k", dk), ("v", dv)):
        fd = np.zeros_like(g)
        base = {x: p[x].copy() for x in ("q", "k", "v")}
        it = np.nditer(base[name], flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            plus = {x: base[x].copy() for x in base}
            minus = {x: base[x].copy() for x in base}
            plus[name][idx] += eps
            minus[name][idx] -= eps
            fd[idx] = (loss(plus["q"], plus["k"], plus["v"]) - loss(minus["q"], minus["k"], minus["v"])) / (2 * eps)
        assert rel(g, fd) <= 1e-5


# pin 4: SPEC worked examples (tests/golden/spec_examples.json, each with its citation)
def _arr(x):
    a = np.asarray(x, dtype=np.float64)
    return a.reshape(1, a.shape[0], 1, a.shape[1])


@pytest.mark.parametrize("key", ["fwd_n1", "fwd_lambda1_n2", "fwd_lambda_half_n3"])
def test_golden_forward(oracle_mod, key):
    g = GOLD[key]
    o = oracle_mod.fwd(_arr(g["q"]), _arr(g["k"]), _arr(g["v"]), [g["lam"]])
    np.testing.assert_allclose(o[0, :, 0], np.asarray(g["o"]), rtol=0, atol=1e-15)


def test_golden_backward_n1(oracle_mod):
    g = GOLD["bwd_n1"]
    dq, dk, dv = oracle_mod.bwd(_arr(g["q"]), _arr(g["k"]), _arr(g["v"]), [g["lam"]], _arr(g["do"]))
    np.testing.assert_allclose(dq[0, :, 0], g["dq"], atol=1e-15)
    np.testing.assert_allclose(dk[0, :, 0], g["dk"], atol=1e-15)
    np.testing.assert_allclose(dv[0, :, 0], g["dv"], atol=1e-15)


def test_golden_build_decay(oracle_mod):
    g = GOLD["build_decay_half_c3"]
    mask, lf, lr, lc = oracle_mod.build_decay(g["C"], g["lam"])
    np.testing.assert_array_equal(mask, g["mask"])
    np.testing.assert_array_equal(lf, g["lam_fwd"])
    np.testing.assert_array_equal(lr, g["lam_rev"])
    assert lc == g["lam_C"]


def test_golden_dkv_update_c1(oracle_mod):
    g = GOLD["dkv_update_c1"]
    _, lf, _, lc = oracle_mod.build_decay(1, g["lam"])
    out = oracle_mod.dkv_update(np.array(g["dkv_next"]), np.array(g["q"]), np.array(g["do"]), lf, lc)
    np.testing.assert_array_equal(out, g["dkv"])


def test_golden_table1_volume(oracle_mod):
    """Table 1 LASP row: one hop carries B*d^2/h elements; at B=1, d=2048, h=16 that is
    262144. The oracle's rank-simulated Alg. 2/3 report their own message size, compared with the
    printed number (d = H*D, so D = d/h = 128)."""
    g = GOLD["table1_lasp_volume"]
    H, D = g["h"], g["d"] // g["h"]
    T, N = 4, 8
    z = np.zeros((g["B"], N, H, D))
    o, cache, hops, elems = oracle_mod.lasp_fwd_sim(z, z, z, [0.9] * H, T)
    _, _, _, bhops, belems = oracle_mod.lasp_bwd_sim(z, z, z, [0.9] * H, z, cache, T)
    assert (hops, bhops) == (T - 1, T - 1)
    assert elems == g["elements"] and belems == g["elements"]


# normwise_err (reading A14) grades every GPU parity check: pinned on hand-computed values so that a
# mean instead of a max, a sum in the denominator or a missing abs fails
def test_normwise_err_known_values(oracle_mod):
    ref = np.array([[1.0, -4.0], [2.0, 0.5]])
    x = ref.copy()
    assert oracle_mod.normwise_err(x, ref) == 0.0
    x[1, 1] += 0.2                       # one element off by 0.2; max|ref| = 4 (a negative entry)
    assert oracle_mod.normwise_err(x, ref) == pytest.approx(0.05, abs=1e-15)
    x[0, 0] -= 0.4                       # the max error, with a negative sign
    assert oracle_mod.normwise_err(x, ref) == pytest.approx(0.1, abs=1e-15)
    # mean-based or sum-based variants give different values on the same input
    assert oracle_mod.normwise_err(x, ref) != pytest.approx(np.mean(np.abs(x - ref)) / np.max(np.abs(ref)))
    assert oracle_mod.normwise_err(x, ref) != pytest.approx(np.max(np.abs(x - ref)) / np.sum(np.abs(ref)))
    # all-zero reference: the absolute error is reported (no division by zero)
    assert oracle_mod.normwise_err(np.array([0.0, 3.0]), np.zeros(2)) == 3.0
    assert oracle_mod.normwise_err(np.zeros(3), np.zeros(3)) == 0.0
    # scale invariance: the metric is relative to the tensor's own magnitude
    assert oracle_mod.normwise_err(1e6 * x, 1e6 * ref) == pytest.approx(0.1, rel=1e-12)
    # bf16-rounded copy of a random tensor: error within 2^-9 of the max (RNE, reading A13)
    r = np.random.default_rng(0).standard_normal(1000)
    xb = torch.tensor(r, dtype=torch.float32).to(torch.bfloat16).double().numpy()
    e = oracle_mod.normwise_err(xb, r)
    assert 0 < e <= 2.0 ** -9
    # shape mismatch is an error, not a silent broadcast
    with pytest.raises(ValueError):
        oracle_mod.normwise_err(np.zeros((2, 3)), np.zeros((3, 2)))
    with pytest.raises(ValueError):
        oracle_mod.normwise_err(np.zeros(3), np.zeros((1, 3)))


# pin 5: closed forms for constant inputs (derived from Eq. 4), any N
@pytest.mark.parametrize("lam", [1.0, 0.999, 0.9, 0.5])
def test_constant_input_closed_forms(oracle_mod, lam):
    N, D = 4096, 3
    rng = np.random.default_rng(0)
    qv, kv_, vv, dov = (rng.standard_normal(D) for _ in range(4))
    q = np.broadcast_to(qv, (1, N, 1, D)).copy()
    k = np.broadcast_to(kv_, (1, N, 1, D)).copy()
    v = np.broadcast_to(vv, (1, N, 1, D)).copy()
    do = np.broadcast_to(dov, (1, N, 1, D)).copy()
    l64 = float(np.float64(np.float32(lam)))
    s = np.arange(1, N + 1, dtype=np.float64)  # 1-based position
    geo = (lambda n: n) if l64 == 1.0 else (lambda n: (1.0 - l64 ** n) / (1.0 - l64))
    o = oracle_mod.fwd(q, k, v, [lam])
    o_ref = (qv @ kv_) * np.outer(geo(s), vv)
    assert rel(o[0, :, 0], o_ref) <= 1e-12
    dq, dk, dv = oracle_mod.bwd(q, k, v, [lam], do)
    assert rel(dq[0, :, 0], (vv @ dov) * np.outer(geo(s), kv_)) <= 1e-12
    assert rel(dk[0, :, 0], (vv @ dov) * np.outer(geo(N - s + 1), qv)) <= 1e-12
    assert rel(dv[0, :, 0], (qv @ kv_) * np.outer(geo(N - s + 1), dov)) <= 1e-12


# pin 6: Euler identity -- L is linear in each of Q, K, V, so <X, dX> = L for X in {Q,K,V}
def test_euler_identity(oracle_mod):
    p = rand_problem(2, 1, 512, 3, 16)
    o = oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])
    dq, dk, dv = oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])
    L = np.sum(o * p["do"])
    for x, g in ((p["q"], dq), (p["k"], dk), (p["v"], dv)):
        assert abs(np.sum(x * g) - L) <= 1e-11 * max(1.0, abs(L))


# pin 7: causality
def test_causality(oracle_mod):
    p = rand_problem(4, 1, 128, 2, 8)
    o = oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])
    for cut in (0, 17, 64, 127):
        k2, v2 = p["k"].copy(), p["v"].copy()
        k2[:, cut + 1:] = 0
        v2[:, cut + 1:] = 0
        o2 = oracle_mod.fwd(p["q"], k2, v2, p["lam"])
        np.testing.assert_array_equal(o2[:, :cut + 1], o[:, :cut + 1])


# pin 8: chunk-size / rank-count invariance of Alg. 2/3 in the rank-simulated mode
@pytest.mark.parametrize("lam", [1.0, 0.99, 0.9, 0.5])
def test_rank_simulated_matches_definition(oracle_mod, lam):
    N = 256
    p = rand_problem(9, 2, N, 2, 8, lam=lam)
    o_ref = oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])
    g_ref = oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])
    for T in (1, 2, 4, 8, 16, 64, 256):
        o, cache, hops, elems = oracle_mod.lasp_fwd_sim(p["q"], p["k"], p["v"], p["lam"], T)
        assert rel(o, o_ref) <= 1e-10
        assert hops == T - 1 and elems == 2 * 2 * 8 * 8
        dq, dk, dv, bh, be = oracle_mod.lasp_bwd_sim(p["q"], p["k"], p["v"], p["lam"], p["do"], cache, T)
        assert bh == T - 1 and be == elems
        for x, r in zip((dq, dk, dv), g_ref):
            assert rel(x, r) <= 1e-10


def test_cache_holds_state_entering_each_rank(oracle_mod):
    """cache[t] = KV_in(t) = sum_{g < tC} lam^(tC-1-g) k_g v_g^T (reading A4), by brute force."""
    N, T, D = 64, 4, 5
    p = rand_problem(13, 1, N, 1, D, lam=0.9)
    _, cache, _, _ = oracle_mod.lasp_fwd_sim(p["q"], p["k"], p["v"], p["lam"], T)
    l64 = float(np.float64(np.float32(0.9)))
    C = N // T
    k, v = p["k"][0, :, 0], p["v"][0, :, 0]
    for t in range(T):
        ref = np.zeros((D, D))
        for g in range(t * C):
            ref += l64 ** (t * C - 1 - g) * np.outer(k[g], v[g])
        np.testing.assert_allclose(cache[t, 0, 0], ref, rtol=1e-12, atol=1e-12)


def test_partition_and_domain_errors(oracle_mod):
    p = rand_problem(0, 1, 30, 1, 4)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.lasp_fwd_sim(p["q"], p["k"], p["v"], p["lam"], 4)  # 4 does not divide 30
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.fwd(p["q"], p["k"], p["v"], [1.5])  # lambda outside (0, 1]
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.fwd(p["q"], p["k"], p["v"], [0.0])


# pin 9: lambda = 1, T = 1 -> torch.tril(Q K^T) V (plain linear attention)
def test_lambda_one_is_tril_linear_attention(oracle_mod):
    p = rand_problem(1, 1, 200, 1, 16, lam=1.0)
    q, k, v = (torch.tensor(p[x][0, :, 0]) for x in ("q", "k", "v"))
    ref = (torch.tril(q @ k.T) @ v).numpy()
    o = oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])
    assert rel(o[0, :, 0], ref) <= 1e-12


# pin 10: protocol -- T-1 hops of B*H*D*D elements per direction, independent of N
def test_protocol_independent_of_n(oracle_mod):
    T, B, H, D = 4, 1, 2, 4
    seen = set()
    for N in (256, 1024, 4096):
        p = rand_problem(0, B, N, H, D)
        o, cache, hops, elems = oracle_mod.lasp_fwd_sim(p["q"], p["k"], p["v"], p["lam"], T)
        _, _, _, bh, be = oracle_mod.lasp_bwd_sim(p["q"], p["k"], p["v"], p["lam"], p["do"], cache, T)
        seen.add((hops, elems, bh, be))
    assert seen == {(T - 1, B * H * D * D, T - 1, B * H * D * D)}


# pin 12: head independence -- h heads equal h single-head runs, bitwise
def test_head_independence_bitwise(oracle_mod):
    p = rand_problem(6, 1, 100, 4, 8)
    o = oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"])
    g = oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])
    for h in range(4):
        sl = (slice(None), slice(None), slice(h, h + 1))
        o1 = oracle_mod.fwd(p["q"][sl], p["k"][sl], p["v"][sl], p["lam"][h:h + 1])
        np.testing.assert_array_equal(o1, o[sl])
        g1 = oracle_mod.bwd(p["q"][sl], p["k"][sl], p["v"][sl], p["lam"][h:h + 1], p["do"][sl])
        for a, b in zip(g1, g):
            np.testing.assert_array_equal(a, b[sl])


# ---- single-chunk ops vs brute-force sums of their defining equations ----------------------
def _chunk(seed, C, D):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((C, D)) for _ in range(4)] + [rng.standard_normal((D, D))]


def test_chunk_intra_fwd_is_dense_on_isolated_chunk(oracle_mod):
    Q, K, V, _, _ = _chunk(1, 8, 3)
    mask, _, _, _ = oracle_mod.build_decay(8, 0.7)
    ref = dense_fwd(Q[None, :, None], K[None, :, None], V[None, :, None], [np.float32(0.7)])[0, :, 0]
    assert rel(oracle_mod.intra_fwd(Q, K, V, mask), ref) <= 1e-13


def test_chunk_inter_terms_brute_force(oracle_mod):
    """Second summands of Eq. 8, Eq. 16, Eq. 19, Eq. 22."""
    C, D, lam = 6, 3, 0.8
    l64 = float(np.float64(np.float32(lam)))
    Q, K, V, dO, S = _chunk(2, C, D)
    _, lf, lr, lc = oracle_mod.build_decay(C, lam)
    # O_inter row s: lam^(s+1) q_s^T KV_{t-1}   (s 0-based)
    ref = np.stack([l64 ** (s + 1) * (Q[s] @ S) for s in range(C)])
    assert rel(oracle_mod.inter_fwd(Q, S, lf), ref) <= 1e-14
    ref = np.stack([l64 ** (s + 1) * (S @ dO[s]) for s in range(C)])
    assert rel(oracle_mod.inter_bwd_q(dO, S, lf), ref) <= 1e-14
    ref = np.stack([l64 ** (C - 1 - s) * (S @ V[s]) for s in range(C)])
    assert rel(oracle_mod.inter_bwd_k(V, S, lr), ref) <= 1e-14
    ref = np.stack([l64 ** (C - 1 - s) * (K[s] @ S) for s in range(C)])
    assert rel(oracle_mod.inter_bwd_v(K, S, lr), ref) <= 1e-14


def test_chunk_state_updates_brute_force(oracle_mod):
    """Eq. 12 and Eq. 21 as defining sums: KV_t = sum lam^(C-1-s) k v^T + lam^C KV_{t-1};
    dKV_t = sum lam^(s+1) q do^T + lam^C dKV_{t+1}."""
    C, D, lam = 7, 4, 0.6
    l64 = float(np.float64(np.float32(lam)))
    Q, K, V, dO, S = _chunk(3, C, D)
    _, lf, lr, lc = oracle_mod.build_decay(C, lam)
    ref = l64 ** C * S + sum(l64 ** (C - 1 - s) * np.outer(K[s], V[s]) for s in range(C))
    assert rel(oracle_mod.kv_update(S, K, V, lr, lc), ref) <= 1e-14
    ref = l64 ** C * S + sum(l64 ** (s + 1) * np.outer(Q[s], dO[s]) for s in range(C))
    assert rel(oracle_mod.dkv_update(S, Q, dO, lf, lc), ref) <= 1e-14


def test_chunk_intra_bwd_matches_autograd(oracle_mod):
    C, D = 9, 4
    Q, K, V, dO, _ = _chunk(4, C, D)
    mask, _, _, _ = oracle_mod.build_decay(C, 0.75)
    dq, dk, dv = oracle_mod.intra_bwd(Q, K, V, dO, mask)
    rq, rk, rv = dense_torch_grads(Q[None, :, None], K[None, :, None], V[None, :, None], [np.float32(0.75)],
                                   dO[None, :, None])
    for a, r in ((dq, rq), (dk, rk), (dv, rv)):
        assert rel(a, r[0, :, 0]) <= 1e-13


def test_dkv_chain_matches_definition(oracle_mod):
    """Iterating Eq. 21 from the last chunk reproduces dKV_t = sum_{s > tC} lam^(s-tC) q_s do_s^T
    with the 0-based reading A3 (exponent starts at 1)."""
    N, C, D, lam = 24, 6, 3, 0.85
    l64 = float(np.float64(np.float32(lam)))
    rng = np.random.default_rng(8)
    Q, dO = rng.standard_normal((N, D)), rng.standard_normal((N, D))
    _, lf, _, lc = oracle_mod.build_decay(C, lam)
    dkv = np.zeros((D, D))
    for t in range(N // C - 1, -1, -1):
        dkv = oracle_mod.dkv_update(dkv, Q[t * C:(t + 1) * C], dO[t * C:(t + 1) * C], lf, lc)
        ref = sum(l64 ** (g - t * C + 1) * np.outer(Q[g], dO[g]) for g in range(t * C, N))
        assert rel(dkv, ref) <= 1e-13


# ---- grouped-query / multi-query attention (reading G1) -------------
def dense_torch_gqa(q, k, v, lam, do):
    """Dense masked form per query head with the group's key/value head (k, v expanded along heads by
    torch.repeat_interleave), O and the fp64 autograd gradients -- the expansion makes autograd sum dK, dV
    over the group's query heads. lam is per kv-head."""
    B, N, H, D = q.shape
    Hk = k.shape[2]
    G = H // Hk
    tq, tk, tv = (torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in (q, k, v))
    ke, ve = tk.repeat_interleave(G, dim=2), tv.repeat_interleave(G, dim=2)
    outs = []
    for h in range(H):
        M = torch.tensor(dense_mask(N, float(np.float64(np.float32(lam[h // G])))))
        s = torch.einsum("bid,bjd->bij", tq[:, :, h], ke[:, :, h]) * M
        outs.append(torch.einsum("bij,bjd->bid", s, ve[:, :, h]))
    o = torch.stack(outs, dim=2)
    (o * torch.tensor(do)).sum().backward()
    return o.detach().numpy(), tq.grad.numpy(), tk.grad.numpy(), tv.grad.numpy()


@pytest.mark.parametrize("H,Hk", [(4, 2), (6, 1), (8, 4)])
def test_gqa_matches_dense_autograd(oracle_mod, H, Hk):
    rng = np.random.default_rng(H * 10 + Hk)
    B, N, D = 2, 96, 8
    q, do = (rng.standard_normal((B, N, H, D)) for _ in range(2))
    k, v = (rng.standard_normal((B, N, Hk, D)) for _ in range(2))
    lam = rng.uniform(0.5, 1.0, Hk).astype(np.float32)
    lam[0] = 1.0
    o_ref, dq_ref, dk_ref, dv_ref = dense_torch_gqa(q, k, v, lam, do)
    o = oracle_mod.fwd_gqa(q, k, v, lam)
    dq, dk, dv = oracle_mod.bwd_gqa(q, k, v, lam, do)
    for x, r in ((o, o_ref), (dq, dq_ref), (dk, dk_ref), (dv, dv_ref)):
        assert x.shape == r.shape and rel(x, r) <= 1e-12


def test_gqa_one_group_is_mha_bitwise(oracle_mod):
    """G = 1 (Hk = H) is the pinned MHA recurrence, operation for operation."""
    p = rand_problem(12, 2, 70, 3, 5)
    o = oracle_mod.fwd_gqa(p["q"], p["k"], p["v"], p["lam"])
    g = oracle_mod.bwd_gqa(p["q"], p["k"], p["v"], p["lam"], p["do"])
    assert np.array_equal(o, oracle_mod.fwd(p["q"], p["k"], p["v"], p["lam"]))
    for a, b in zip(g, oracle_mod.bwd(p["q"], p["k"], p["v"], p["lam"], p["do"])):
        assert np.array_equal(a, b)


def test_mqa_is_mha_with_repeated_kv(oracle_mod):
    """Hk = 1: O equals the MHA oracle with k, v repeated for every head; dK, dV equal the MHA gradients
    summed over the heads (linearity of L in the shared k, v)."""
    rng = np.random.default_rng(5)
    B, N, H, D = 1, 130, 4, 6
    q, do = (rng.standard_normal((B, N, H, D)) for _ in range(2))
    k, v = (rng.standard_normal((B, N, 1, D)) for _ in range(2))
    lam = np.array([0.93], dtype=np.float32)
    kr, vr = np.repeat(k, H, axis=2), np.repeat(v, H, axis=2)
    o = oracle_mod.fwd_gqa(q, k, v, lam)
    dq, dk, dv = oracle_mod.bwd_gqa(q, k, v, lam, do)
    o_m = oracle_mod.fwd(q, kr, vr, np.repeat(lam, H))
    dq_m, dk_m, dv_m = oracle_mod.bwd(q, kr, vr, np.repeat(lam, H), do)
    assert rel(o, o_m) <= 1e-13 and rel(dq, dq_m) <= 1e-13
    assert rel(dk, dk_m.sum(axis=2, keepdims=True)) <= 1e-12
    assert rel(dv, dv_m.sum(axis=2, keepdims=True)) <= 1e-12


# ---- NEXT-3: Norm(.) (Eq. 2; reading N1) and the projection prologue (Alg. 2) ----------------
def test_norm_known_values_and_invariants(oracle_mod):
    o = np.array([[3.0, 4.0], [0.0, 0.0], [-1.0, 1.0]])
    y, r = oracle_mod.norm_fwd(o, eps=0.0 + 1e-300)
    np.testing.assert_allclose(y[0], [3 / np.sqrt(12.5), 4 / np.sqrt(12.5)], rtol=1e-15)
    np.testing.assert_allclose(y[2], [-1.0, 1.0], rtol=1e-15)      # mean square 1 already
    assert np.all(y[1] == 0.0)                                      # eps keeps the zero row finite
    rng = np.random.default_rng(3)
    x = rng.standard_normal((50, 64))
    y, r = oracle_mod.norm_fwd(x, eps=0.0)
    np.testing.assert_allclose(np.mean(y * y, axis=1), 1.0, rtol=1e-13)          # unit RMS
    y2, _ = oracle_mod.norm_fwd(7.5 * x, eps=0.0)
    np.testing.assert_allclose(y2, y, rtol=1e-13, atol=1e-15)                      # scale invariance
    dy = rng.standard_normal((50, 64))
    do = oracle_mod.norm_bwd(y, r, dy)
    np.testing.assert_allclose(np.sum(do * x, axis=1), 0.0, atol=1e-11)            # d/dc Norm(c x) = 0


def test_norm_matches_torch_rms_norm(oracle_mod):
    """The reading N1 normalization is exactly torch.nn.functional.rms_norm over the head dimension (a
    library routine), forward and backward (fp64 autograd)."""
    rng = np.random.default_rng(4)
    o = rng.standard_normal((2, 33, 3, 16))
    dy = rng.standard_normal(o.shape)
    y, r = oracle_mod.norm_fwd(o)
    t = torch.tensor(o, requires_grad=True)
    ty = torch.nn.functional.rms_norm(t, (16,), eps=oracle_mod.NORM_EPS)
    (ty * torch.tensor(dy)).sum().backward()
    assert rel(y, ty.detach().numpy()) <= 1e-14
    assert rel(oracle_mod.norm_bwd(y, r, dy), t.grad.numpy()) <= 1e-13


@pytest.mark.parametrize("H,Hk", [(2, 2), (4, 2)])
def test_layer_matches_dense_autograd(oracle_mod, H, Hk):
    """The NEXT-3 layer Y = Norm(LASP(X W_Q, X W_K, X W_V)) and its gradients (dX, dW_*) against torch fp64
    autograd of the dense masked form (Eq. 2 with the reading-N1 Norm)."""
    rng = np.random.default_rng(H + Hk)
    B, N, D = 2, 48, 8
    d = H * D
    x = rng.standard_normal((B, N, d))
    wq, wk, wv = (rng.standard_normal((d, h * D)) * d ** -0.5 for h in (H, Hk, Hk))
    dy = rng.standard_normal((B, N, H, D))
    lam = rng.uniform(0.6, 1.0, Hk).astype(np.float32)
    fw = oracle_mod.layer_fwd(x, wq, wk, wv, lam, H, Hk)
    dx, dwq, dwk, dwv = oracle_mod.layer_bwd(x, wq, wk, wv, lam, fw, dy)[:4]
    tx, tq, tk, tv = (torch.tensor(a, requires_grad=True) for a in (x, wq, wk, wv))
    q = (tx @ tq).reshape(B, N, H, D)
    k = (tx @ tk).reshape(B, N, Hk, D).repeat_interleave(H // Hk, dim=2)
    v = (tx @ tv).reshape(B, N, Hk, D).repeat_interleave(H // Hk, dim=2)
    outs = []
    for h in range(H):
        M = torch.tensor(dense_mask(N, float(np.float64(np.float32(lam[h // (H // Hk)])))))
        outs.append(torch.einsum("bij,bjd->bid", torch.einsum("bid,bjd->bij", q[:, :, h], k[:, :, h]) * M,
                                 v[:, :, h]))
    y = torch.nn.functional.rms_norm(torch.stack(outs, dim=2), (D,), eps=oracle_mod.NORM_EPS)
    (y * torch.tensor(dy)).sum().backward()
    assert rel(fw["y"], y.detach().numpy()) <= 1e-12
    for a, b in ((dx, tx.grad), (dwq, tq.grad), (dwk, tk.grad), (dwv, tv.grad)):
        assert rel(a, b.numpy()) <= 1e-11


def test_round_bf16_matches_torch_conversion(oracle_mod):
    """oracle.round_bf16 (reading N2) is torch's fp32 -> bf16 round-to-nearest-even (a library routine) after
    fp64 -> fp32, including ties, negative values, subnormal-range and large magnitudes."""
    rng = np.random.default_rng(11)
    a = np.concatenate([rng.standard_normal(20000) * 10.0 ** rng.integers(-30, 30, 20000),
                        [0.0, -0.0, 1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 3e38, 1e-40]])
    ref = torch.tensor(a, dtype=torch.float64).to(torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    got = oracle_mod.round_bf16(a)
    assert np.array_equal(got, ref)
    assert got[-5] == 1.0 and got[-4] == 1.0 + 2 ** -6  # ties to even: 1 + 2^-8 -> 1, 1 + 3*2^-8 -> 1 + 2^-6


def test_layer_bf16_points_round_exactly_the_materialized_tensors(oracle_mod):
    """bf16_points=True (reading N2) changes only the rounding of Q, K, V / Y, dO, dQ, dK, dV: with inputs whose
    projections are already bf16-exact (X, W with few significant bits), both modes agree to fp64 rounding."""
    rng = np.random.default_rng(5)
    B, N, H, D = 1, 40, 2, 8
    d = H * D
    x = rng.integers(-2, 3, (B, N, d)).astype(np.float64)
    wq, wk, wv = (rng.integers(-1, 2, (d, H * D)).astype(np.float64) / 8 for _ in range(3))
    dy = oracle_mod.round_bf16(rng.standard_normal((B, N, H, D)))
    lam = np.full(H, 0.75, np.float32)
    fa = oracle_mod.layer_fwd(x, wq, wk, wv, lam, H)
    fb = oracle_mod.layer_fwd(x, wq, wk, wv, lam, H, bf16_points=True)
    for n in ("q", "k", "v", "o", "y", "r"):
        assert np.array_equal(fa[n], fb[n]), n          # projections exact in bf16: identical forward
    ga = oracle_mod.layer_bwd(x, wq, wk, wv, lam, fa, dy)
    gb = oracle_mod.layer_bwd(x, wq, wk, wv, lam, fb, dy)
    assert np.array_equal(gb[4], oracle_mod.round_bf16(gb[4]))           # dO is bf16-valued
    assert rel(gb[4], ga[4]) <= 2 ** -8 and rel(gb[0], ga[0]) <= 5e-2   # the rounding of the fp64 chain (dX: cancellation)
    assert not np.array_equal(gb[4], ga[4])                              # ... but rounded


# ---- NEXT-4: generalised decay (Table 3 GLA / GateLoop row, App. A.4) --------------------
def _gla_inputs(seed, B, N, H, D, lo=0.0, hi=1.0):
    rng = np.random.default_rng(seed)
    q, k, v, do = (rng.standard_normal((B, N, H, D)) for _ in range(4))
    lg = -rng.uniform(lo, hi, (B, N, H, D))
    return q, k, v, lg, do


def test_gla_constant_decay_is_the_scalar_lambda_path(oracle_mod):
    """lg_t = log(lambda_h) for every token and channel is the TNL / RetNet row (Eq. 5): gla_fwd / gla_bwd
    equal the scalar-lambda oracle, and the decay gradient summed over a head's tokens and channels is
    dL/dlog(lambda), checked by finite differences of the (constant-decay) forward."""
    B, N, H, D = 2, 37, 3, 5
    q, k, v, _, do = _gla_inputs(1, B, N, H, D)
    lam = np.array([0.9, 0.5, 1.0], np.float32)
    lg = np.broadcast_to(np.log(lam.astype(np.float64))[None, None, :, None], (B, N, H, D)).copy()
    o = oracle_mod.gla_fwd(q, k, v, lg)
    assert rel(o, oracle_mod.fwd(q, k, v, lam)) <= 1e-13
    dq, dk, dv, dlg = oracle_mod.gla_bwd(q, k, v, lg, do)
    for a, b in zip((dq, dk, dv), oracle_mod.bwd(q, k, v, lam, do)):
        assert rel(a, b) <= 1e-13
    L = lambda x: np.sum(oracle_mod.gla_fwd(q, k, v, x) * do)
    for h in range(H):
        # one-sided second-order difference towards smaller log-decay (lambda = 1 has no room above)
        eps = 1e-5
        l1, l2 = lg.copy(), lg.copy()
        l1[:, :, h] -= eps
        l2[:, :, h] -= 2 * eps
        fd = (3 * L(lg) - 4 * L(l1) + L(l2)) / (2 * eps)
        assert abs(dlg[:, :, h].sum() - fd) <= 1e-6 * max(1.0, abs(fd)), (h, dlg[:, :, h].sum(), fd)


def _gla_dense_torch(q, k, v, lg):
    """Dense form of the GLA recurrence: o_t = sum_{i<=t} sum_d q_t[d] k_i[d] exp(sum_{s=i+1..t} lg_s[d]) v_i."""
    c = torch.cumsum(lg, dim=1)                                        # [B][N][H][D]
    N = q.shape[1]
    dec = torch.exp(c[:, :, None] - c[:, None, :])                     # [B][t][i][H][D] = exp(c_t - c_i)
    causal = torch.tril(torch.ones(N, N, dtype=q.dtype))[None, :, :, None, None]
    A = torch.einsum("bthd,bihd,btihd->bhti", q, k, dec * causal)      # exp(c_t - c_i) only for i <= t
    return torch.einsum("bhti,bihe->bthe", A, v)


def test_gla_matches_dense_form_and_fp64_autograd(oracle_mod):
    """Forward against the dense decay-product form; dQ, dK, dV and the decay gradient against torch fp64
    autograd of that dense form (a different evaluation order and a different gradient derivation)."""
    B, N, H, D = 2, 29, 2, 4
    q, k, v, lg, do = _gla_inputs(2, B, N, H, D, 0.0, 2.0)
    o = oracle_mod.gla_fwd(q, k, v, lg)
    tq, tk, tv, tl = (torch.tensor(a, requires_grad=True) for a in (q, k, v, lg))
    to = _gla_dense_torch(tq, tk, tv, tl)
    assert rel(o, to.detach().numpy()) <= 1e-12
    (to * torch.tensor(do)).sum().backward()
    got = oracle_mod.gla_bwd(q, k, v, lg, do)
    for a, t in zip(got, (tq, tk, tv, tl)):
        assert rel(a, t.grad.numpy()) <= 1e-11


def test_gla_decay_gradient_finite_differences(oracle_mod):
    """d L / d lg at single (token, head, channel) entries by central differences of the forward."""
    B, N, H, D = 1, 70, 1, 3      # spans two 64-token checkpoint chunks of the oracle's reverse sweep
    q, k, v, lg, do = _gla_inputs(3, B, N, H, D)
    dlg = oracle_mod.gla_bwd(q, k, v, lg, do)[3]
    eps = 1e-6
    for (t, d) in ((0, 0), (1, 2), (63, 1), (64, 0), (69, 2), (35, 1)):
        lp, lm = lg.copy(), lg.copy()
        lp[0, t, 0, d] += eps
        lm[0, t, 0, d] -= eps
        fd = (np.sum(oracle_mod.gla_fwd(q, k, v, lp) * do) - np.sum(oracle_mod.gla_fwd(q, k, v, lm) * do)) / (2 * eps)
        assert abs(dlg[0, t, 0, d] - fd) <= 1e-6 * max(1.0, abs(fd)), (t, d, dlg[0, t, 0, d], fd)
    assert np.all(dlg[0, 0] == 0.0)   # kv_{-1} = 0: the first token's decay multiplies nothing


def test_gla_causality_and_no_decay_is_linear_attention(oracle_mod):
    """lg = 0 (g = 1) is plain linear attention tril(Q K^T) V; changing tokens after t never changes o_t."""
    B, N, H, D = 1, 20, 2, 3
    q, k, v, lg, _ = _gla_inputs(4, B, N, H, D)
    o0 = oracle_mod.gla_fwd(q, k, v, np.zeros_like(lg))
    for h in range(H):
        ref = np.tril(q[0, :, h] @ k[0, :, h].T) @ v[0, :, h]
        assert rel(o0[0, :, h], ref) <= 1e-13
    o = oracle_mod.gla_fwd(q, k, v, lg)
    k2, lg2 = k.copy(), lg.copy()
    k2[:, 12:] += 1.0
    lg2[:, 12:] -= 0.5
    o2 = oracle_mod.gla_fwd(q, k2, v, lg2)
    assert np.array_equal(o[:, :12], o2[:, :12]) and not np.array_equal(o[:, 12:], o2[:, 12:])
