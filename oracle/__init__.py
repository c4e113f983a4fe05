"""fp64 CPU oracle for the LASP hot path (arXiv 2404.02882) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path
(``paper_2404_02882_b200``) never imports it and shares no code with it.

The arithmetic lives in ``lasp_oracle.c`` (plain C, fp64, pthreads over (batch, head));
this module only builds/loads it and marshals numpy arrays. Functions:

* ``fwd`` / ``bwd`` -- definition mode, the recurrences Eq. 5 and
  Eq. 13-14.
* ``fwd_gqa`` / ``bwd_gqa`` -- the same recurrences with H query heads sharing Hk key/value heads
  (multi-query / grouped-query attention).
* ``gla_fwd`` / ``gla_bwd`` -- generalised (per-token, per-channel) decay: the GLA / GateLoop row of
  Table 3 (App. A.4); recurrence and its reverse, the decay
  gradient from its definition.
* ``norm_fwd`` / ``norm_bwd`` / ``layer_fwd`` / ``layer_bwd`` -- the steps either side of the path
  (SURVEY §8(f) NEXT-3): Q, K, V = X W (Alg. 2) and Norm(.) of Eq. 2 read as per-head RMS
  normalization (reading N1).
* ``lasp_fwd_sim`` / ``lasp_bwd_sim`` -- Alg. 2 and Alg. 3 run
  literally with T simulated ranks, explicit messages and a KV cache.
* chunk ops (``build_decay``, ``intra_fwd``, ``inter_fwd``, ``kv_update``, ``intra_bwd``,
  ``inter_bwd_q/k/v``, ``dkv_update``) -- the single-chunk formulas of Alg. 2/3.

Every function is pinned in ``tests/test_oracle_pins.py`` against something other than
itself (dense masked form, fp64 autograd, finite differences, closed forms, SPEC worked
examples); see DESIGN.md "Oracle pins". No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lasp_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liblasp_oracle.so")
_lock = threading.Lock()
_lib = None

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile lasp_oracle.c with gcc (plain -O2, no fast-math: no reassociation)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lpthread", "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.oracle_fwd.argtypes = [_i64] * 4 + [_dp] * 3 + [_fp, _dp, ctypes.c_int]
            lib.oracle_bwd.argtypes = [_i64] * 4 + [_dp] * 3 + [_fp] + [_dp] * 4 + [ctypes.c_int]
            lib.oracle_norm_fwd.argtypes = [_i64, _i64, ctypes.c_double, _dp, _dp, _dp]
            lib.oracle_norm_bwd.argtypes = [_i64, _i64, _dp, _dp, _dp, _dp]
            lib.oracle_norm_fwd.restype = ctypes.c_int
            lib.oracle_norm_bwd.restype = ctypes.c_int
            lib.oracle_fwd_gqa.argtypes = [_i64] * 5 + [_dp] * 3 + [_fp, _dp, ctypes.c_int]
            lib.oracle_bwd_gqa.argtypes = [_i64] * 5 + [_dp] * 3 + [_fp] + [_dp] * 4 + [ctypes.c_int]
            lib.oracle_build_decay.argtypes = [_i64, ctypes.c_float, _dp, _dp, _dp, _dp]
            lib.oracle_intra_fwd.argtypes = [_i64, _i64] + [_dp] * 5
            lib.oracle_inter_fwd.argtypes = [_i64, _i64] + [_dp] * 4
            lib.oracle_kv_update.argtypes = [_i64, _i64, _dp, _dp, _dp, _dp, ctypes.c_double, _dp]
            lib.oracle_intra_bwd.argtypes = [_i64, _i64] + [_dp] * 8
            lib.oracle_inter_bwd_q.argtypes = [_i64, _i64] + [_dp] * 4
            lib.oracle_inter_bwd_k.argtypes = [_i64, _i64] + [_dp] * 4
            lib.oracle_inter_bwd_v.argtypes = [_i64, _i64] + [_dp] * 4
            lib.oracle_dkv_update.argtypes = [_i64, _i64, _dp, _dp, _dp, _dp, ctypes.c_double, _dp]
            lib.oracle_lasp_fwd_sim.argtypes = [_i64] * 5 + [_dp] * 3 + [_fp, _dp, _dp, _i64p, _i64p,
                                                                          ctypes.c_int]
            lib.oracle_lasp_bwd_sim.argtypes = [_i64] * 5 + [_dp] * 3 + [_fp, _dp, _dp] + [_dp] * 3 + \
                [_i64p, _i64p, ctypes.c_int]
            lib.oracle_gla_fwd.argtypes = [_i64] * 4 + [_dp] * 5 + [ctypes.c_int]
            lib.oracle_gla_bwd.argtypes = [_i64] * 4 + [_dp] * 9 + [ctypes.c_int]
            for fn in ("oracle_fwd", "oracle_bwd", "oracle_fwd_gqa", "oracle_bwd_gqa", "oracle_build_decay",
                       "oracle_gla_fwd", "oracle_gla_bwd",
                       "oracle_lasp_fwd_sim",
                       "oracle_lasp_bwd_sim"):
                getattr(lib, fn).restype = ctypes.c_int
            _lib = lib
    return _lib


class OracleError(RuntimeError):
    pass


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _lam(lam, H):
    lam = np.ascontiguousarray(np.broadcast_to(np.asarray(lam, dtype=np.float32), (H,)))
    return lam, lam.ctypes.data_as(_fp)


def _check(st):
    if st != 0:
        raise OracleError(f"oracle status {st}")


def _threads(nthreads):
    return int(nthreads or os.cpu_count() or 1)


def _shape4(x):
    x = np.asarray(x)
    if x.ndim != 4:
        raise ValueError("expected [B][N][H][D]")
    return x.shape


def fwd(q, k, v, lam, nthreads=None):
    """O of Eq. 4 via the recurrence Eq. 5; inputs [B][N][H][D], lam [H] (float32)."""
    B, N, H, D = _shape4(q)
    q, k, v = _f64(q), _f64(k), _f64(v)
    o = np.zeros_like(q)
    lam, lp = _lam(lam, H)
    _check(_load().oracle_fwd(B, N, H, D, _ptr(q), _ptr(k), _ptr(v), lp, _ptr(o), _threads(nthreads)))
    return o


def bwd(q, k, v, lam, do, nthreads=None):
    """(dQ, dK, dV) of L = sum(O * dO) via Eq. 13-14."""
    B, N, H, D = _shape4(q)
    q, k, v, do = _f64(q), _f64(k), _f64(v), _f64(do)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(q), np.zeros_like(q)
    lam, lp = _lam(lam, H)
    _check(_load().oracle_bwd(B, N, H, D, _ptr(q), _ptr(k), _ptr(v), lp, _ptr(do), _ptr(dq), _ptr(dk),
                              _ptr(dv), _threads(nthreads)))
    return dq, dk, dv


def fwd_gqa(q, k, v, lam, nthreads=None):
    """Grouped-query O: q [B][N][H][D], k, v [B][N][Hk][D], lam [Hk];
    q-head h reads kv-head h // (H/Hk), whose state kv_s = lam kv_{s-1} + k_s v_s^T is shared."""
    B, N, H, D = _shape4(q)
    Hk = _shape4(k)[2]
    q, k, v = _f64(q), _f64(k), _f64(v)
    o = np.zeros_like(q)
    lam, lp = _lam(lam, Hk)
    _check(_load().oracle_fwd_gqa(B, N, H, Hk, D, _ptr(q), _ptr(k), _ptr(v), lp, _ptr(o), _threads(nthreads)))
    return o


def bwd_gqa(q, k, v, lam, do, nthreads=None):
    """(dQ [B][N][H][D], dK, dV [B][N][Hk][D]) of L = sum(O * dO) for fwd_gqa."""
    B, N, H, D = _shape4(q)
    Hk = _shape4(k)[2]
    q, k, v, do = _f64(q), _f64(k), _f64(v), _f64(do)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    lam, lp = _lam(lam, Hk)
    _check(_load().oracle_bwd_gqa(B, N, H, Hk, D, _ptr(q), _ptr(k), _ptr(v), lp, _ptr(do), _ptr(dq), _ptr(dk),
                                  _ptr(dv), _threads(nthreads)))
    return dq, dk, dv


def gla_fwd(q, k, v, lg, nthreads=None):
    """Generalised decay (NEXT-4; Table 3 GLA / GateLoop row, App. A.4): O of the recurrence
    kv_t = Diag(exp(lg_t)) kv_{t-1} + k_t v_t^T, o_t = kv_t^T q_t. All inputs [B][N][H][D]; lg <= 0 is the
    log of the per-token, per-key-channel decay."""
    B, N, H, D = _shape4(q)
    q, k, v, lg = _f64(q), _f64(k), _f64(v), _f64(lg)
    o = np.zeros_like(q)
    _check(_load().oracle_gla_fwd(B, N, H, D, _ptr(q), _ptr(k), _ptr(v), _ptr(lg), _ptr(o), _threads(nthreads)))
    return o


def gla_bwd(q, k, v, lg, do, nthreads=None):
    """(dQ, dK, dV, dlg) of L = sum(O * dO) for gla_fwd; dlg_t[d] = g_t[d] sum_e dkv_t[d][e] kv_{t-1}[d][e] (the
    definition of the gradient through kv_t = Diag(g_t) kv_{t-1} + ...)."""
    B, N, H, D = _shape4(q)
    q, k, v, lg, do = _f64(q), _f64(k), _f64(v), _f64(lg), _f64(do)
    dq, dk, dv, dlg = (np.zeros_like(q) for _ in range(4))
    _check(_load().oracle_gla_bwd(B, N, H, D, _ptr(q), _ptr(k), _ptr(v), _ptr(lg), _ptr(do), _ptr(dq), _ptr(dk),
                                  _ptr(dv), _ptr(dlg), _threads(nthreads)))
    return dq, dk, dv, dlg


NORM_EPS = 1e-6  # DESIGN.md reading N1


def norm_fwd(o, eps=NORM_EPS):
    """Norm(O) of Eq. 2 read as per-head RMS normalization (reading N1): o [..][D] ->
    (y = o r, r = (mean_c o_c^2 + eps)^-1/2 with shape o.shape[:-1])."""
    o = _f64(o)
    D = o.shape[-1]
    rows = o.size // D if D else 0
    y, r = np.zeros_like(o), np.zeros(o.shape[:-1])
    _check(_load().oracle_norm_fwd(rows, D, float(eps), _ptr(o), _ptr(y), _ptr(r)))
    return y, r


def norm_bwd(y, r, dy):
    """dO = r (dY - y (y . dY) / D) per row, the gradient of norm_fwd."""
    y, r, dy = _f64(y), _f64(r), _f64(dy)
    D = y.shape[-1]
    out = np.zeros_like(y)
    _check(_load().oracle_norm_bwd(y.size // D, D, _ptr(y), _ptr(r), _ptr(dy), _ptr(out)))
    return out


def round_bf16(a):
    """Round to bfloat16 (ties to even), returned as float64: the precision of a tensor the bf16 path
    materializes (reading N2). fp64 -> fp32 (RNE) -> bf16 (RNE on the fp32 bits), the same two
    steps as a kernel that accumulates in fp32 and stores bf16 (the double rounding can differ from a direct
    fp64 -> bf16 rounding only when the fp32 step lands on a bf16 tie)."""
    f = np.ascontiguousarray(np.asarray(a, np.float64).astype(np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16  # RNE on the low 16 bits (finite inputs)
    return u.astype(np.uint32).view(np.float32).astype(np.float64).reshape(np.shape(a))


def layer_fwd(x, w_q, w_k, w_v, lam, H, Hk=None, eps=NORM_EPS, nthreads=None, bf16_points=False):
    """NEXT-3 layer: Alg. 2 line 'Calculate Q = X W_Q, K = X W_K, V = X W_V' (numpy matmul as the
    library step), LASP O (fwd / fwd_gqa), then Norm (reading N1). x [B][N][d], w_* [d][heads * D].
    bf16_points: Q, K, V (and in layer_bwd Y, dO, dQ, dK, dV) are rounded to bf16 where the bf16 path
    materializes them (reading N2); everything else stays fp64.
    Returns dict with q, k, v [B][N][heads][D], o, y, r."""
    x = _f64(x)
    B, N, d = x.shape
    Hk = Hk or H
    rnd = round_bf16 if bf16_points else (lambda t: t)
    q = rnd(x @ _f64(w_q)).reshape(B, N, H, -1)
    k = rnd(x @ _f64(w_k)).reshape(B, N, Hk, -1)
    v = rnd(x @ _f64(w_v)).reshape(B, N, Hk, -1)
    o = fwd_gqa(q, k, v, lam, nthreads) if Hk != H else fwd(q, k, v, lam, nthreads)
    y, r = norm_fwd(o, eps)
    return {"q": q, "k": k, "v": v, "o": o, "y": y, "r": r, "bf16_points": bf16_points}


def layer_bwd(x, w_q, w_k, w_v, lam, fw, dy, nthreads=None):
    """Gradients of sum(Y * dY) for layer_fwd: (dX [B][N][d], dW_Q, dW_K, dW_V [d][heads * D], dO, dQ, dK, dV).
    With fw from layer_fwd(bf16_points=True) the stored Y, the formed dO and dQ, dK, dV are rounded to bf16
    (reading N2), as the bf16 path stores them."""
    x = _f64(x)
    B, N, d = x.shape
    q, k, v = fw["q"], fw["k"], fw["v"]
    rnd = round_bf16 if fw.get("bf16_points") else (lambda t: t)
    do = rnd(norm_bwd(rnd(fw["y"]), fw["r"], dy))
    if k.shape[2] != q.shape[2]:
        dq, dk, dv = bwd_gqa(q, k, v, lam, do, nthreads)
    else:
        dq, dk, dv = bwd(q, k, v, lam, do, nthreads)
    dq, dk, dv = rnd(dq), rnd(dk), rnd(dv)
    dq2, dk2, dv2 = (t.reshape(B * N, -1) for t in (dq, dk, dv))
    x2 = x.reshape(B * N, d)
    dx = (dq2 @ _f64(w_q).T + dk2 @ _f64(w_k).T + dv2 @ _f64(w_v).T).reshape(B, N, d)
    return dx, x2.T @ dq2, x2.T @ dk2, x2.T @ dv2, do, dq, dk, dv


def lasp_fwd_sim(q, k, v, lam, T, nthreads=None):
    """Alg. 2 with T simulated ranks -> (O, cache [T][B][H][D][D], hops, elems_per_hop)."""
    B, N, H, D = _shape4(q)
    q, k, v = _f64(q), _f64(k), _f64(v)
    o = np.zeros_like(q)
    cache = np.zeros((T, B, H, D, D))
    lam, lp = _lam(lam, H)
    mc, me = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(_load().oracle_lasp_fwd_sim(B, N, H, D, T, _ptr(q), _ptr(k), _ptr(v), lp, _ptr(o), _ptr(cache),
                                       ctypes.byref(mc), ctypes.byref(me), _threads(nthreads)))
    return o, cache, mc.value, me.value


def lasp_bwd_sim(q, k, v, lam, do, cache, T, nthreads=None):
    """Alg. 3 with T simulated ranks -> (dQ, dK, dV, hops, elems_per_hop)."""
    B, N, H, D = _shape4(q)
    q, k, v, do, cache = _f64(q), _f64(k), _f64(v), _f64(do), _f64(cache)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(q), np.zeros_like(q)
    lam, lp = _lam(lam, H)
    mc, me = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(_load().oracle_lasp_bwd_sim(B, N, H, D, T, _ptr(q), _ptr(k), _ptr(v), lp, _ptr(do), _ptr(cache),
                                       _ptr(dq), _ptr(dk), _ptr(dv), ctypes.byref(mc), ctypes.byref(me),
                                       _threads(nthreads)))
    return dq, dk, dv, mc.value, me.value


# ---- single-chunk ops (one head, C x D) ----------------------------------------------------

def build_decay(C, lam):
    """(mask C x C, lam_fwd [C], lam_rev [C], lam_C) of Alg. 2 lines P:152-153 and Eq. 12."""
    mask, lf, lr = np.zeros((C, C)), np.zeros(C), np.zeros(C)
    lc = ctypes.c_double(0.0)
    _check(_load().oracle_build_decay(C, float(np.float32(lam)), _ptr(mask), _ptr(lf), _ptr(lr),
                                      ctypes.byref(lc)))
    return mask, lf, lr, lc.value


def intra_fwd(Q, K, V, mask):
    Q, K, V, mask = _f64(Q), _f64(K), _f64(V), _f64(mask)
    C, D = Q.shape
    out = np.zeros((C, D))
    _load().oracle_intra_fwd(C, D, _ptr(Q), _ptr(K), _ptr(V), _ptr(mask), _ptr(out))
    return out


def inter_fwd(Q, kv_prev, lam_fwd):
    Q, kv, lf = _f64(Q), _f64(kv_prev), _f64(lam_fwd)
    C, D = Q.shape
    out = np.zeros((C, D))
    _load().oracle_inter_fwd(C, D, _ptr(Q), _ptr(kv), _ptr(lf), _ptr(out))
    return out


def kv_update(kv_prev, K, V, lam_rev, lam_C):
    K, V, lr = _f64(K), _f64(V), _f64(lam_rev)
    C, D = K.shape
    kv = _f64(kv_prev) if kv_prev is not None else None
    out = np.zeros((D, D))
    _load().oracle_kv_update(C, D, _ptr(kv), _ptr(K), _ptr(V), _ptr(lr), float(lam_C), _ptr(out))
    return out


def intra_bwd(Q, K, V, dO, mask):
    Q, K, V, dO, mask = _f64(Q), _f64(K), _f64(V), _f64(dO), _f64(mask)
    C, D = Q.shape
    dq, dk, dv = np.zeros((C, D)), np.zeros((C, D)), np.zeros((C, D))
    _load().oracle_intra_bwd(C, D, _ptr(Q), _ptr(K), _ptr(V), _ptr(dO), _ptr(mask), _ptr(dq), _ptr(dk),
                             _ptr(dv))
    return dq, dk, dv


def inter_bwd_q(dO, kv_prev, lam_fwd):
    dO, kv, lf = _f64(dO), _f64(kv_prev), _f64(lam_fwd)
    C, D = dO.shape
    out = np.zeros((C, D))
    _load().oracle_inter_bwd_q(C, D, _ptr(dO), _ptr(kv), _ptr(lf), _ptr(out))
    return out


def inter_bwd_k(V, dkv_next, lam_rev):
    V, dkv, lr = _f64(V), _f64(dkv_next), _f64(lam_rev)
    C, D = V.shape
    out = np.zeros((C, D))
    _load().oracle_inter_bwd_k(C, D, _ptr(V), _ptr(dkv), _ptr(lr), _ptr(out))
    return out


def inter_bwd_v(K, dkv_next, lam_rev):
    K, dkv, lr = _f64(K), _f64(dkv_next), _f64(lam_rev)
    C, D = K.shape
    out = np.zeros((C, D))
    _load().oracle_inter_bwd_v(C, D, _ptr(K), _ptr(dkv), _ptr(lr), _ptr(out))
    return out


def dkv_update(dkv_next, Q, dO, lam_fwd, lam_C):
    Q, dO, lf = _f64(Q), _f64(dO), _f64(lam_fwd)
    C, D = Q.shape
    dkv = _f64(dkv_next) if dkv_next is not None else None
    out = np.zeros((D, D))
    _load().oracle_dkv_update(C, D, _ptr(dkv), _ptr(Q), _ptr(dO), _ptr(lf), float(lam_C), _ptr(out))
    return out


def normwise_err(x, ref):
    """max|x - ref| / max|ref| per tensor (reading A14)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if x.shape != ref.shape:
        raise ValueError(f"normwise_err: shape {x.shape} vs reference {ref.shape}")
    den = np.max(np.abs(ref)) if ref.size else 0.0
    num = np.max(np.abs(x - ref)) if ref.size else 0.0
    return float(num / den) if den > 0 else float(num)
