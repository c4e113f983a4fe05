"""GPU parity of the NEXT-3 layer: Q, K, V = X W (Alg. 2), LASP, Norm (Eq. 2 P:62,
reading N1) and all gradients, through lasp_layer_fwd / lasp_layer_bwd, against the fp64 oracle
(oracle.layer_fwd / layer_bwd) on the same synthetic inputs (synth.layer_problem).

Tolerance: normwise 2e-2 (BASELINE bf16 bar), the same as the core path, against the oracle chain with the
bf16 rounding points of reading N2 (Q, K, V, Y, dO, dQ, dK, dV rounded where the path stores them in bf16).
Without them the comparison measures the conditioning of Norm, not the kernels: a row whose RMS is small
against the magnitude of its terms turns the 2^-8 relative rounding of Q, K, V into a several-percent change
of that row of Y (N2; measured 8-14 % on such rows, profiles/r2g_layer_diag.txt). The GEMM outputs
Q, K, V are checked against the unrounded fp64 projection X W at the bf16 rounding bound 2^-8. Gradients
(dO and all that follows) get 4e-2: dO = r (dY - y (y . dY) / D) is largest on the rows with the largest r,
i.e. the smallest RMS of O, which are the rows where the kernel-internal bf16 roundings (P, u . c; not
reproducible by the oracle) are amplified by Norm's conditioning; those rows set the normwise denominator
of dQ (measured 2.2e-2 at TNL-1B, every forward quantity <= 6.2e-3)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
TOL = 2e-2        # forward: Y, rnorm
TOL_GRAD = 4e-2   # dO and everything downstream of the Norm backward (reading N2)


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_02882_b200 as lasp
    return lasp


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.bfloat16)


def per_head(x, ref):
    worst = 0.0
    for h in range(ref.shape[2]):
        den = np.max(np.abs(ref[:, :, h]))
        worst = max(worst, np.max(np.abs(x[:, :, h] - ref[:, :, h])) / den if den > 0 else 0.0)
    return worst


def rel(x, ref):
    return float(np.max(np.abs(np.asarray(x, np.float64) - ref)) / np.max(np.abs(ref)))


def run_layer(L, oracle_mod, B, N, H, Hk, D, d, seed=0):
    t = synth.layer_problem(seed, B, N, H, Hk, D, d)
    x, wq, wk, wv, dy = (dev(t[n]) for n in ("x", "w_q", "w_k", "w_v", "dy"))
    fw = L.layer_fwd(x, wq, wk, wv, t["lam"], H)
    g = L.layer_bwd(x, wq, wk, wv, t["lam"], fw, dy)
    torch.cuda.synchronize()
    ref = oracle_mod.layer_fwd(t["x"], t["w_q"], t["w_k"], t["w_v"], t["lam"], H, Hk, bf16_points=True)
    pure = oracle_mod.layer_fwd(t["x"], t["w_q"], t["w_k"], t["w_v"], t["lam"], H, Hk)
    rdx, rdwq, rdwk, rdwv, rdo, rdq, rdk, rdv = oracle_mod.layer_bwd(t["x"], t["w_q"], t["w_k"], t["w_v"], t["lam"], ref, t["dy"])
    qkv = max(per_head(fw[n].float().cpu().numpy(), pure[n]) for n in "qkv")
    assert qkv <= 2 ** -8 * 1.01, ("q, k, v against X W beyond the bf16 rounding bound", qkv)
    errs = {"y": per_head(fw["y"].float().cpu().numpy(), ref["y"]),
            "rnorm": rel(fw["rnorm"].cpu().numpy(), ref["r"]),
            "d_o": per_head(g["d_o"].float().cpu().numpy(), rdo),
            "dq": per_head(g["dq"].float().cpu().numpy(), rdq), "dk": per_head(g["dk"].float().cpu().numpy(), rdk),
            "dv": per_head(g["dv"].float().cpu().numpy(), rdv),
            "dx": rel(g["dx"].float().cpu().numpy(), rdx),
            "dw_q": rel(g["dw_q"].cpu().numpy(), rdwq), "dw_k": rel(g["dw_k"].cpu().numpy(), rdwk),
            "dw_v": rel(g["dw_v"].cpu().numpy(), rdwv)}
    return errs


@pytest.mark.parametrize("B,N,H,Hk,D,d", [(1, 1000, 4, 4, 64, 256),     # ragged, several segments
                                           (2, 640, 4, 2, 128, 512),    # batch 2, grouped queries, D = 128
                                           (1, 3000, 8, 8, 128, 1024)])
def test_layer_matches_oracle(L, oracle_mod, B, N, H, Hk, D, d):
    errs = run_layer(L, oracle_mod, B, N, H, Hk, D, d, seed=B + H + D)
    check(errs)


def check(errs):
    fwd = {n: e for n, e in errs.items() if n in ("y", "rnorm")}
    assert max(fwd.values()) <= TOL, errs
    assert max(errs.values()) <= TOL_GRAD, errs


@pytest.mark.parametrize("H,D", [(16, 64), (16, 128)])
def test_layer_tnl_shapes(L, oracle_mod, H, D):
    """TNL-0.4B (d = 1024) and TNL-1B (d = 2048) layer shapes at 32K tokens, every element of y, dO, dX and
    the weight gradients against the oracle."""
    errs = run_layer(L, oracle_mod, 1, 32768, H, H, D, H * D, seed=3)
    print("layer errors", errs)
    check(errs)


def test_layer_y_has_unit_rms(L):
    """Property at any size (reading N1): every (token, head) row of Y has mean square 1 / (1 + eps / ms(O))."""
    t = synth.layer_problem(9, 1, 8192, 8, 8, 128, 1024)
    fw = L.layer_fwd(*(dev(t[n]) for n in ("x", "w_q", "w_k", "w_v")), t["lam"], 8)
    y = fw["y"].float()
    ms = (y * y).mean(dim=-1)
    assert torch.allclose(ms, torch.ones_like(ms), atol=2e-2)


def test_layer_unrounded_gap_is_norm_conditioning(L, oracle_mod):
    """Against the unrounded fp64 chain (no reading N2) each row of Y stays within the first-order forward
    error bound of the arithmetic: |dY|_row <= 10 u kappa_row + u max|Y_row|, u = 2^-8 (bf16), where
    kappa_row = max_c O_abs[row, c] / rms(O[row]) and O_abs = LASP(|Q|, |K|, |V|) bounds the sum of the
    magnitudes of the terms of O (Q, K, V rounding 3u, P and u . c rounding 2u; Norm doubles a relative error
    of O's row, the stored bf16 Y adds u). So the larger gap on rows with small RMS is the conditioning
    of Norm, not an error of the kernels."""
    B, N, H, D, d = 1, 3000, 8, 128, 1024
    t = synth.layer_problem(137, B, N, H, H, D, d)
    fw = L.layer_fwd(*(dev(t[n]) for n in ("x", "w_q", "w_k", "w_v")), t["lam"], H)
    torch.cuda.synchronize()
    pure = oracle_mod.layer_fwd(t["x"], t["w_q"], t["w_k"], t["w_v"], t["lam"], H, H)
    o_abs = oracle_mod.fwd(np.abs(pure["q"]), np.abs(pure["k"]), np.abs(pure["v"]), t["lam"])
    u = 2.0 ** -8
    kappa = np.abs(o_abs).max(-1) / np.sqrt((pure["o"] ** 2).mean(-1))
    err = np.abs(fw["y"].float().cpu().numpy() - pure["y"]).max(-1)
    bound = 10 * u * kappa + u * np.abs(pure["y"]).max(-1)
    worst = np.unravel_index(np.argmax(err / bound), err.shape)
    print("unrounded chain: max row error", err.max(), "worst err / bound", (err / bound).max(), "at", worst,
          "kappa there", kappa[worst])
    assert np.all(err <= bound), (err[worst], bound[worst])
    assert err.max() > 2e-2  # the gap the bf16-points oracle removes is real at this shape


@pytest.mark.parametrize("exchange", ["ring", "p2p"])
def test_layer_over_loopback_ring(L, oracle_mod, exchange):
    """The NEXT-3 layer across a 2-rank ring (lasp_layer_fwd / lasp_layer_bwd with a loopback ctx; the ring over the
    in-process transport, or the P2P ring exchange): each rank projects its chunk, the state crosses the ring,
    Norm runs per token. The concatenated Y, dX and the sum over ranks of the weight gradients match the single-sequence oracle chain (reading N2)."""
    import threading
    B, N, H, D, T = 1, 1536, 4, 64, 2
    t = synth.layer_problem(44, B, N, H, H, D, H * D)
    C = N // T
    res, errs = [None] * T, []

    def rank(r):
        ring = None
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ring = L.Ring.loopback(r, T, f"layer-{exchange}")
                x = dev(t["x"][:, r * C:(r + 1) * C])
                wq, wk, wv = (dev(t[n]) for n in ("w_q", "w_k", "w_v"))
                dy = dev(t["dy"][:, r * C:(r + 1) * C])
                if exchange == "p2p":
                    # one step over the host transport first: a kernel's first launch (lazy module loading)
                    # synchronizes the context, which must not happen while the peer's hop kernel spins on
                    # this GPU (include/lasp.h, LASP_EXCHANGE_P2P)
                    L.layer_bwd(x, wq, wk, wv, t["lam"], L.layer_fwd(x, wq, wk, wv, t["lam"], H, ring), dy, ring)
                    s.synchronize()
                    ring.enable_p2p(B * H * D * D)
                fw = L.layer_fwd(x, wq, wk, wv, t["lam"], H, ring)
                g = L.layer_bwd(x, wq, wk, wv, t["lam"], fw, dy, ring)
            s.synchronize()
            res[r] = (fw["y"].float().cpu().numpy(), g["dx"].float().cpu().numpy(),
                      [g[n].cpu().numpy() for n in ("dw_q", "dw_k", "dw_v")])
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
    ths = [threading.Thread(target=rank, args=(r,)) for r in range(T)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errs, errs
    ref = oracle_mod.layer_fwd(t["x"], t["w_q"], t["w_k"], t["w_v"], t["lam"], H, H, bf16_points=True)
    rdx, rdwq, rdwk, rdwv = oracle_mod.layer_bwd(t["x"], t["w_q"], t["w_k"], t["w_v"], t["lam"], ref, t["dy"])[:4]
    y = np.concatenate([res[r][0] for r in range(T)], 1)
    dx = np.concatenate([res[r][1] for r in range(T)], 1)
    assert per_head(y, ref["y"]) <= TOL
    assert rel(dx, rdx) <= TOL_GRAD
    for i, rw in enumerate((rdwq, rdwk, rdwv)):
        assert rel(sum(res[r][2][i] for r in range(T)), rw) <= TOL_GRAD
