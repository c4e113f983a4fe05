"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of LASP's arithmetic: it only draws numbers. Both sides of every
parity check (the fp64 CPU oracle under ``oracle/`` and the CUDA path behind
``include/lasp.h``) receive exactly the bits produced here, so neither side generates
its own inputs.

Generator:
  u   = splitmix64(seed XOR tensor_id * 2**56 XOR flat_index) -> top 53 bits -> [0, 1)
  x   = (2u - 1) * sqrt(3) * scale          (unit variance times ``scale``)
  out = x rounded to fp32, then (for bf16 tensors) rounded to-nearest-even to bf16.

``flat_index`` is the element's index in the GLOBAL [B][N][H][D] tensor, so a rank that
owns tokens [r*C, (r+1)*C) can draw its shard without drawing the whole sequence.

Scales follow SURVEY.md §8(d): Q and K use D**-0.25 (q.k has unit variance), V and dO
use 1. Per-head decay for TNL-shaped workloads: lambda_h = 1 - 2**-(1 + 14 h/(H-1)),
which spans [0.5, 0.99997] (the paper gives no lambda values; the recipe exercises both the
fast-decay/underflow end and the long-memory end).
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "TENSOR_IDS", "splitmix64", "uniform", "draw", "round_bf16", "bf16_bits",
    "bits_to_f32", "head_lambdas", "problem", "head_decay_rates", "gla_problem",
]

# Fixed tensor ids (part of the recipe: changing them changes every fixture).
TENSOR_IDS = {"q": 1, "k": 2, "v": 3, "do": 4, "x": 5, "wq": 6, "wk": 7, "wv": 8, "dy": 9, "lg": 10}

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser applied elementwise to a uint64 array (counter-based)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, tensor_id: int, flat_index: np.ndarray) -> np.ndarray:
    """u in [0, 1) as float64 from the top 53 bits of splitmix64(seed ^ id<<56 ^ idx)."""
    key = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(tensor_id) << np.uint64(56))
    z = splitmix64(np.asarray(flat_index, dtype=np.uint64) ^ key)
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returned as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    out = u.astype(np.uint32).view(np.float32)
    # NaN/inf never occur in the recipe (|x| <= sqrt(3)); keep them untouched anyway.
    bad = ~np.isfinite(x)
    if bad.any():
        out = out.copy()
        out[bad] = x[bad]
    return out


def bf16_bits(x_bf16_valued_f32: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns of float32 values that are already bf16-representable."""
    x = np.ascontiguousarray(x_bf16_valued_f32, dtype=np.float32)
    return (x.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Inverse of bf16_bits."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def draw(name: str, seed: int, batch: int, n_global: int, heads: int, head_dim: int,
         dtype: str = "bf16", token_lo: int = 0, token_hi: int | None = None,
         scale: float | None = None) -> np.ndarray:
    """Draw tensor ``name`` ("q","k","v","do") as float32 with layout [B][tokens][H][D].

    Only tokens [token_lo, token_hi) of the global sequence of length ``n_global`` are drawn
    (a rank's shard). ``dtype`` "bf16" rounds to bf16 values; "fp32" keeps fp32.
    """
    if token_hi is None:
        token_hi = n_global
    if not (0 <= token_lo <= token_hi <= n_global):
        raise ValueError("bad token range")
    if scale is None:
        scale = head_dim ** -0.25 if name in ("q", "k") else 1.0
    tid = TENSOR_IDS[name]
    n = token_hi - token_lo
    out = np.empty((batch, n, heads, head_dim), dtype=np.float32)
    inner = heads * head_dim
    # chunk over (b, tokens) rows to bound temporary memory
    rows_per = max(1, (1 << 22) // max(inner, 1))
    for b in range(batch):
        for s0 in range(0, n, rows_per):
            s1 = min(n, s0 + rows_per)
            base = (b * n_global + token_lo + s0) * inner
            idx = np.arange(base, base + (s1 - s0) * inner, dtype=np.uint64)
            u = uniform(seed, tid, idx)
            x = ((2.0 * u - 1.0) * (math.sqrt(3.0) * scale)).astype(np.float32)
            out[b, s0:s1] = x.reshape(s1 - s0, heads, head_dim)
    if dtype == "bf16":
        out = round_bf16(out).reshape(out.shape)
    elif dtype != "fp32":
        raise ValueError(dtype)
    return out


def head_lambdas(heads: int, scalar: float | None = None) -> np.ndarray:
    """Per-head decay lambda_h as float32 (the boundary's precision, reading A8)."""
    if scalar is not None:
        return np.full(heads, scalar, dtype=np.float32)
    if heads == 1:
        return np.array([0.99], dtype=np.float32)
    h = np.arange(heads, dtype=np.float64)
    return (1.0 - 2.0 ** -(1.0 + 14.0 * h / (heads - 1))).astype(np.float32)


def problem(seed: int, batch: int, n_global: int, heads: int, head_dim: int,
            dtype: str = "bf16", lam: float | None = None, token_lo: int = 0,
            token_hi: int | None = None, with_do: bool = True, kv_heads: int | None = None) -> dict:
    """Convenience: q, k, v (and do) shards plus the float32 per-head lambda vector. ``kv_heads``
    (grouped-query attention): k, v are drawn with that many heads and lambda has one entry per kv-head."""
    hk = heads if kv_heads is None else kv_heads
    t = {nm: draw(nm, seed, batch, n_global, hk if nm in ("k", "v") else heads, head_dim, dtype, token_lo,
                  token_hi)
         for nm in (("q", "k", "v", "do") if with_do else ("q", "k", "v"))}
    t["lam"] = head_lambdas(hk, lam)
    return t


def _draw2(name: str, seed: int, rows: int, cols: int, scale: float, dtype: str, row_lo: int = 0,
           row_hi: int | None = None, row_total: int | None = None) -> np.ndarray:
    """A [rows][cols] matrix (rows [row_lo, row_hi) of a [row_total][cols] one) with the same generator."""
    row_hi = rows if row_hi is None else row_hi
    a = draw(name, seed, 1, row_total or rows, 1, cols, dtype, row_lo, row_hi, scale=scale)
    return a.reshape(row_hi - row_lo, cols)


def layer_problem(seed: int, batch: int, n_global: int, heads: int, kv_heads: int, head_dim: int, d_model: int,
                  token_lo: int = 0, token_hi: int | None = None, lam: float | None = None) -> dict:
    """Inputs of the NEXT-3 layer (projection + LASP + Norm): x [B][tokens][d_model] (unit variance),
    w_q [d][H*D], w_k, w_v [d][Hk*D] with scales d^-1/2 * D^-1/4 (q . k of unit variance, as the q, k recipe)
    and d^-1/2 (v), dy [B][tokens][H][D] (unit variance), all bf16-valued float32; lambda per kv-head."""
    token_hi = n_global if token_hi is None else token_hi
    n = token_hi - token_lo
    x = np.stack([_draw2("x", seed, n_global, d_model, 1.0, "bf16", b * n_global + token_lo,
                         b * n_global + token_hi, batch * n_global) for b in range(batch)])
    sq = d_model ** -0.5 * head_dim ** -0.25
    t = {"x": x.reshape(batch, n, d_model),
         "w_q": _draw2("wq", seed, d_model, heads * head_dim, sq, "bf16"),
         "w_k": _draw2("wk", seed, d_model, kv_heads * head_dim, sq, "bf16"),
         "w_v": _draw2("wv", seed, d_model, kv_heads * head_dim, d_model ** -0.5, "bf16"),
         "dy": draw("dy", seed, batch, n_global, heads, head_dim, "bf16", token_lo, token_hi),
         "lam": head_lambdas(kv_heads, lam)}
    return t


def head_decay_rates(heads: int) -> np.ndarray:
    """Mean per-token log-decay magnitude a_h of head h for the generalised-decay inputs: 2^-(1 + 9 h/(H-1))
    (0.5 .. ~0.001: from a few tokens of memory to ~1000; GLA-style gates sigmoid(x)^(1/16) sit near 0.05)."""
    if heads == 1:
        return np.array([0.05])
    return 2.0 ** -(1.0 + 9.0 * np.arange(heads, dtype=np.float64) / (heads - 1))


def gla_problem(seed: int, batch: int, n_global: int, heads: int, head_dim: int, token_lo: int = 0,
                token_hi: int | None = None) -> dict:
    """Inputs of the generalised-decay path (NEXT-4), all float32 [B][tokens][H][D]: q, k, v, do as ``draw``
    (fp32), and the log decay lg = -2 a_h u (u uniform in [0, 1), per token, head and key channel; mean -a_h)."""
    token_hi = n_global if token_hi is None else token_hi
    t = {nm: draw(nm, seed, batch, n_global, heads, head_dim, "fp32", token_lo, token_hi)
         for nm in ("q", "k", "v", "do")}
    n = token_hi - token_lo
    inner = heads * head_dim
    lg = np.empty((batch, n, heads, head_dim), dtype=np.float32)
    rate = head_decay_rates(heads)[None, :, None]
    for b in range(batch):
        base = (b * n_global + token_lo) * inner
        u = uniform(seed, TENSOR_IDS["lg"], np.arange(base, base + n * inner, dtype=np.uint64))
        lg[b] = (-2.0 * rate * u.reshape(n, heads, head_dim)).astype(np.float32)
    t["lg"] = lg
    return t
