"""Torch-facing wrappers of the LASP C ABI (marshalling only; all compute is in liblasp.so).

PyTorch is used for device memory, streams and process groups. Tensors use the boundary layout
[batch][n_local][heads][head_dim] (include/lasp.h); states are fp32 [batch][heads][D][D].

* ``fwd_local`` / ``bwd_local`` -- one rank's Alg. 2 / Alg. 3 compute without transport. k, v (and dk, dv)
  may have fewer heads than q (grouped-query / multi-query attention; lambda then has one entry per kv-head).
* ``Ring``                        -- Alg. 2 / Alg. 3 across a torch.distributed world (NCCL P2P).
* ``LaspAttention``               -- torch.autograd.Function over ``Ring`` or the local path.
* ``gla_fwd_local`` / ``gla_bwd_local`` / ``Ring.gla_fwd`` / ``Ring.gla_bwd`` -- generalised decay (SURVEY §8(f)
  NEXT-4, the GLA / GateLoop row of Table 3): per-token, per-key-channel decay exp(log_g), fp32.
* ``topology`` / ``sp_group`` / ``scatter_sequence`` -- data-sequence hybrid parallelism (Alg. 1): G = W/T
  sequence-parallel groups, one ring per group.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N

_DT = {torch.bfloat16: N.LASP_BF16, torch.float32: N.LASP_FP32}


def _shape(q: torch.Tensor, k: torch.Tensor | None = None) -> N.lasp_shape_t:
    """Boundary shape of q [B][C][H][D]; k [B][C][Hk][D] with Hk < H selects grouped-query attention."""
    if q.dim() != 4:
        raise ValueError("expected [batch][n_local][heads][head_dim]")
    if q.dtype not in _DT:
        raise TypeError("dtype must be bfloat16 or float32")
    B, C, H, D = q.shape
    Hk = 0 if k is None or k.shape[2] == H else int(k.shape[2])
    return N.shape(B, C, H, D, _DT[q.dtype], Hk)


def _lam(lam, heads: int):
    arr = np.ascontiguousarray(np.broadcast_to(np.asarray(
        lam.detach().cpu().numpy() if isinstance(lam, torch.Tensor) else lam, dtype=np.float32), (heads,)))
    return arr, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check_seq(*ts):
    ref = ts[0]
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda or t.shape != ref.shape or t.dtype != ref.dtype or not t.is_contiguous():
            raise ValueError("sequence tensors must be contiguous CUDA tensors of equal shape and dtype")


def _check_qkv(q, k, v, do=None):
    """q (and do) [B][C][H][D]; k, v [B][C][Hk][D] with Hk dividing H (Hk = H: multi-head)."""
    _check_seq(q, do)
    _check_seq(k, v)
    if (k.dim() != 4 or k.shape[:2] != q.shape[:2] or k.shape[3] != q.shape[3] or k.dtype != q.dtype
            or q.shape[2] % k.shape[2] != 0 or k.device != q.device):
        raise ValueError("k, v must be [B][C][Hk][D] like q with Hk dividing H (grouped-query attention)")


def _check_state(t, q, name):
    """kv_in / kv_out / dkv_in / dkv_out: fp32 [B][Hk][D][D], contiguous, on the device (include/lasp.h);
    ``q`` here is a tensor with the state's head count (k)."""
    if t is None:
        return
    B, _, H, D = q.shape
    if (not isinstance(t, torch.Tensor) or t.device != q.device or t.dtype != torch.float32
            or tuple(t.shape) != (B, H, D, D) or not t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor of shape {(B, H, D, D)} on {q.device}")


def _check_like(t, q, name):
    """Output sequence tensors: same shape, dtype and device as q, contiguous."""
    if (not isinstance(t, torch.Tensor) or t.device != q.device or t.dtype != q.dtype or t.shape != q.shape
            or not t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous {q.dtype} tensor of shape {tuple(q.shape)} on {q.device}")


def _check_buf(t, nbytes, name, device):
    if (not isinstance(t, torch.Tensor) or t.device != device or not t.is_contiguous()
            or t.numel() * t.element_size() < nbytes):
        raise ValueError(f"{name} must be a contiguous tensor of at least {nbytes} bytes on {device}")


def workspace_status(workspace: torch.Tensor) -> None:
    """Raise LaspError(LASP_ERR_STATE) if the last backward on ``workspace`` found a cache whose tag does not
    match (synchronizes the current stream; include/lasp.h lasp_workspace_status)."""
    N.check(N.lib().lasp_workspace_status(_p(workspace), _stream(workspace.device)))


def cache_bytes(shape: N.lasp_shape_t) -> int:
    return int(N.lib().lasp_cache_bytes(ctypes.byref(shape)))


def workspace_bytes(shape: N.lasp_shape_t) -> int:
    return int(N.lib().lasp_workspace_bytes(ctypes.byref(shape)))


def segment_len(shape: N.lasp_shape_t) -> int:
    return int(N.lib().lasp_segment_len(ctypes.byref(shape)))


def alloc_cache(q: torch.Tensor, k: torch.Tensor | None = None) -> torch.Tensor:
    """Caller-owned KV cache for q's shape (one per layer); pass k for grouped-query shapes."""
    return torch.empty(max(cache_bytes(_shape(q, k)), 16), dtype=torch.uint8, device=q.device)


def alloc_workspace(q: torch.Tensor, k: torch.Tensor | None = None) -> torch.Tensor:
    return torch.empty(max(workspace_bytes(_shape(q, k)), 16), dtype=torch.uint8, device=q.device)


def _state_like(k: torch.Tensor) -> torch.Tensor:
    B, _, Hk, D = k.shape
    return torch.empty((B, Hk, D, D), dtype=torch.float32, device=k.device)


def fwd_local(q, k, v, lam, kv_in=None, *, o=None, kv_out=True, cache=None, workspace=None):
    """Alg. 2 for one rank -> (o, kv_out or None, cache)."""
    _check_qkv(q, k, v)
    s = _shape(q, k)
    o = torch.empty_like(q) if o is None else o
    kv_out_t = _state_like(k) if kv_out is True else (kv_out if isinstance(kv_out, torch.Tensor) else None)
    cache = alloc_cache(q, k) if cache is None else cache
    workspace = alloc_workspace(q, k) if workspace is None else workspace
    _check_like(o, q, "o")
    _check_state(kv_in, k, "kv_in")
    _check_state(kv_out_t, k, "kv_out")
    _check_buf(cache, cache_bytes(s), "cache", q.device)
    _check_buf(workspace, workspace_bytes(s), "workspace", q.device)
    _, lp = _lam(lam, k.shape[2])
    N.check(N.lib().lasp_fwd_local(ctypes.byref(s), _p(q), _p(k), _p(v), lp, _p(kv_in), _p(o), _p(kv_out_t),
                                   _p(cache), _p(workspace), _stream(q.device)))
    return o, kv_out_t, cache


def bwd_local(q, k, v, lam, do, cache, dkv_in=None, *, dq=None, dk=None, dv=None, dkv_out=True, workspace=None,
              check_state=False):
    """Alg. 3 for one rank -> (dq, dk, dv, dkv_out or None). ``check_state``: synchronize and raise
    LaspError(LASP_ERR_STATE) if the cache's tag did not match (else a mismatch shows as NaN outputs)."""
    _check_qkv(q, k, v, do)
    s = _shape(q, k)
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    dkv_out_t = _state_like(k) if dkv_out is True else (dkv_out if isinstance(dkv_out, torch.Tensor) else None)
    workspace = alloc_workspace(q, k) if workspace is None else workspace
    for t, n, ref in ((dq, "dq", q), (dk, "dk", k), (dv, "dv", v)):
        _check_like(t, ref, n)
    _check_state(dkv_in, k, "dkv_in")
    _check_state(dkv_out_t, k, "dkv_out")
    _check_buf(cache, cache_bytes(s), "cache", q.device)
    _check_buf(workspace, workspace_bytes(s), "workspace", q.device)
    _, lp = _lam(lam, k.shape[2])
    N.check(N.lib().lasp_bwd_local(ctypes.byref(s), _p(q), _p(k), _p(v), lp, _p(do), _p(cache), _p(dkv_in),
                                   _p(dq), _p(dk), _p(dv), _p(dkv_out_t), _p(workspace), _stream(q.device)))
    if check_state:
        workspace_status(workspace)
    return dq, dk, dv, dkv_out_t


def ring_peers(rank: int, world: int, backward: bool) -> tuple[int, int]:
    """(recv_from, send_to) of the library's ring schedule (-1 = none); host-only."""
    a, b = ctypes.c_int(), ctypes.c_int()
    N.check(N.lib().lasp_ring_peers(rank, world, int(backward), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def topology(rank: int, world: int, sp_size: int) -> tuple[int, int, int]:
    """(group, group_rank, src_rank) of global ``rank`` with sequence-parallel size T = ``sp_size``
    (Alg. 1: G = W/T groups of T consecutive ranks, R_src = floor(R/T)*T); host-only."""
    g, r, s = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    N.check(N.lib().lasp_topology(rank, world, sp_size, ctypes.byref(g), ctypes.byref(r), ctypes.byref(s)))
    return g.value, r.value, s.value


def sp_group(sp_size: int):
    """This rank's sequence-parallel process group (a torch.distributed subgroup of T consecutive ranks).
    Every rank of the default group must call it (torch creates all G subgroups collectively)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    mine = topology(rank, world, sp_size)[0]
    groups = [dist.new_group(list(range(g * sp_size, (g + 1) * sp_size))) for g in range(world // sp_size)]
    return groups[mine]


def scatter_sequence(x, group, sp_size: int):
    """Alg. 1 lines 6-8: the group's source rank holds the whole [batch][N][heads][D] sequence ``x``
    (other ranks pass None), splits it into T chunks of C = N/T tokens and scatters chunk t to the rank
    with group_rank t. Returns this rank's chunk. LASP_ERR_PARTITION-style ValueError if T does not
    divide N."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    src = dist.get_global_rank(group, 0)
    meta = [None]
    if rank == 0:
        if x.shape[1] % sp_size != 0:
            raise ValueError(f"sequence length {x.shape[1]} is not divisible by sp_size {sp_size} (C = N/T)")
        meta = [(tuple(x.shape), x.dtype)]
    dist.broadcast_object_list(meta, src=src, group=group)
    shape, dtype = meta[0]
    C = shape[1] // sp_size
    dev = x.device if x is not None else (torch.device("cuda", torch.cuda.current_device())
                                          if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    out = torch.empty((shape[0], C) + tuple(shape[2:]), dtype=dtype, device=dev)
    chunks = [c.contiguous() for c in x.split(C, dim=1)] if rank == 0 else None
    dist.scatter(out, chunks, src=src, group=group)
    return out


class Ring:
    """The LASP ring over the default torch.distributed group: rank r owns tokens [rC, (r+1)C)
    (Alg. 1 with T = W). Rank 0 creates the NCCL id; torch broadcasts it."""

    def __init__(self, device=None, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self._group = group
        idbuf = ctypes.create_string_buffer(128)
        if self.rank == 0:
            N.check(N.lib().lasp_unique_id(idbuf))
        obj = [bytes(idbuf.raw)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        self._ctx = ctypes.c_void_p()
        N.check(N.lib().lasp_ctx_create(self.rank, self.world, obj[0], self.device.index or 0,
                                        ctypes.byref(self._ctx)))

    @classmethod
    def loopback(cls, rank: int, world: int, group: str, device=None) -> "Ring":
        """A ring context whose ranks are threads of this process on one GPU (in-process loopback
        transport instead of NCCL; for exercising the multi-rank path on a single device)."""
        self = cls.__new__(cls)
        self.rank, self.world = rank, world
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self._ctx = ctypes.c_void_p()
        self._loopback = True
        N.check(N.lib().lasp_ctx_create_loopback(rank, world, group.encode(), self.device.index or 0,
                                                 ctypes.byref(self._ctx)))
        return self

    def set_exchange(self, exchange: str) -> "Ring":
        """'ring' (the paper's T-1 hops, default), 'allgather' (one all-gather of the local states plus a
        local fold), 'p2p' (the ring with each hop one kernel over peer memory) or
        'p2p_allgather' (the all-gather as one kernel per direction over peer memory); the P2P ones need enable_p2p
        first."""
        mode = {"ring": N.LASP_EXCHANGE_RING, "allgather": N.LASP_EXCHANGE_ALLGATHER,
                "p2p": N.LASP_EXCHANGE_P2P, "p2p_allgather": N.LASP_EXCHANGE_P2P_ALLGATHER}[exchange]
        N.check(N.lib().lasp_ctx_set_exchange(self._ctx, mode))
        return self

    def enable_p2p(self, max_state_elems: int, group=None) -> "Ring":
        """Set up the P2P exchange (include/lasp.h lasp_ctx_p2p_setup / _connect): every rank allocates its flag /
        receive block for states of up to max_state_elems (batch * kv_heads * head_dim^2, the same on every
        rank); the CUDA IPC handles are exchanged with torch.distributed (all_gather_object over ``group``), or
        inside a loopback group without it. Selects the 'p2p' exchange."""
        h = ctypes.create_string_buffer(64)
        N.check(N.lib().lasp_ctx_p2p_setup(self._ctx, int(max_state_elems), h))
        if getattr(self, "_loopback", False):
            N.check(N.lib().lasp_ctx_p2p_connect(self._ctx, None))
        else:
            import torch.distributed as dist
            allh = [None] * self.world
            dist.all_gather_object(allh, h.raw, group=group if group is not None else getattr(self, "_group", None))
            N.check(N.lib().lasp_ctx_p2p_connect(self._ctx, b"".join(allh)))
        self._p2p = True
        return self.set_exchange("p2p")

    @classmethod
    def p2p_only(cls, max_state_elems: int, device=None, group=None) -> "Ring":
        """A ring over the torch.distributed world (or ``group``) WITHOUT NCCL: the P2P exchange only (CUDA IPC
        peer buffers; several processes may share one GPU, which NCCL refuses)."""
        import torch.distributed as dist
        self = cls.__new__(cls)
        self.rank = dist.get_rank(group) if group is not None else dist.get_rank()
        self.world = dist.get_world_size(group) if group is not None else dist.get_world_size()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self._group = group
        self._ctx = ctypes.c_void_p()
        N.check(N.lib().lasp_ctx_create_p2p(self.rank, self.world, self.device.index or 0, ctypes.byref(self._ctx)))
        return self.enable_p2p(max_state_elems, group)

    def close(self):
        if self._ctx:
            N.lib().lasp_ctx_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def protocol(self, q, k=None) -> tuple[int, int, int]:
        s = _shape(q, k)
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        N.check(N.lib().lasp_ctx_protocol(self._ctx, ctypes.byref(s), ctypes.byref(a), ctypes.byref(b),
                                          ctypes.byref(c)))
        return a.value, b.value, c.value

    def fwd(self, q, k, v, lam, *, o=None, cache=None, workspace=None):
        _check_qkv(q, k, v)
        s = _shape(q, k)
        o = torch.empty_like(q) if o is None else o
        cache = alloc_cache(q, k) if cache is None else cache
        workspace = alloc_workspace(q, k) if workspace is None else workspace
        _check_like(o, q, "o")
        _check_buf(cache, cache_bytes(s), "cache", q.device)
        _check_buf(workspace, workspace_bytes(s), "workspace", q.device)
        _, lp = _lam(lam, k.shape[2])
        N.check(N.lib().lasp_fwd(self._ctx, ctypes.byref(s), _p(q), _p(k), _p(v), lp, _p(o), _p(cache),
                                 _p(workspace), _stream(q.device)))
        return o, cache

    def bwd(self, q, k, v, lam, do, cache, *, dq=None, dk=None, dv=None, workspace=None, check_state=False):
        _check_qkv(q, k, v, do)
        s = _shape(q, k)
        dq = torch.empty_like(q) if dq is None else dq
        dk = torch.empty_like(k) if dk is None else dk
        dv = torch.empty_like(v) if dv is None else dv
        workspace = alloc_workspace(q, k) if workspace is None else workspace
        for t, n, ref in ((dq, "dq", q), (dk, "dk", k), (dv, "dv", v)):
            _check_like(t, ref, n)
        _check_buf(cache, cache_bytes(s), "cache", q.device)
        _check_buf(workspace, workspace_bytes(s), "workspace", q.device)
        _, lp = _lam(lam, k.shape[2])
        N.check(N.lib().lasp_bwd(self._ctx, ctypes.byref(s), _p(q), _p(k), _p(v), lp, _p(do), _p(cache), _p(dq),
                                 _p(dk), _p(dv), _p(workspace), _stream(q.device)))
        if check_state:
            workspace_status(workspace)
        return dq, dk, dv


# ---- NEXT-4: generalised decay (include/lasp.h lasp_gla_*) ------------------------------------------------------
def _gla_check(q, *ts):
    if q.dim() != 4 or q.dtype != torch.float32 or not q.is_cuda or not q.is_contiguous():
        raise ValueError("generalised decay: q must be a contiguous float32 CUDA tensor [B][C][H][D]")
    _check_seq(q, *ts)


def gla_cache_bytes(q) -> int:
    return int(N.lib().lasp_gla_cache_bytes(ctypes.byref(_shape(q))))


def gla_workspace_bytes(q) -> int:
    return int(N.lib().lasp_gla_workspace_bytes(ctypes.byref(_shape(q))))


def gla_alloc(q):
    """(cache, workspace) for the generalised-decay path at q's shape."""
    return (torch.empty(max(gla_cache_bytes(q), 16), dtype=torch.uint8, device=q.device),
            torch.empty(max(gla_workspace_bytes(q), 16), dtype=torch.uint8, device=q.device))


def gla_fwd_local(q, k, v, log_g, kv_in=None, *, o=None, kv_out=True, cache=None, workspace=None):
    """kv_t = Diag(exp(log_g_t)) kv_{t-1} + k_t v_t^T, o_t = kv_t^T q_t for one rank -> (o, kv_out or None, cache).
    All tensors float32 [B][C][H][D]; log_g <= 0."""
    _gla_check(q, k, v, log_g)
    s = _shape(q)
    o = torch.empty_like(q) if o is None else o
    kv_out_t = _state_like(k) if kv_out is True else (kv_out if isinstance(kv_out, torch.Tensor) else None)
    if cache is None or workspace is None:
        c2, w2 = gla_alloc(q)
        cache = c2 if cache is None else cache
        workspace = w2 if workspace is None else workspace
    _check_like(o, q, "o")
    _check_state(kv_in, k, "kv_in")
    _check_state(kv_out_t, k, "kv_out")
    _check_buf(cache, gla_cache_bytes(q), "cache", q.device)
    _check_buf(workspace, gla_workspace_bytes(q), "workspace", q.device)
    N.check(N.lib().lasp_gla_fwd_local(ctypes.byref(s), _p(q), _p(k), _p(v), _p(log_g), _p(kv_in), _p(o),
                                       _p(kv_out_t), _p(cache), _p(workspace), _stream(q.device)))
    return o, kv_out_t, cache


def gla_bwd_local(q, k, v, log_g, do, cache, dkv_in=None, *, dq=None, dk=None, dv=None, dlog_g=None, dkv_out=True,
                  workspace=None, check_state=False):
    """Gradients of sum(O * dO) for gla_fwd_local -> (dq, dk, dv, dlog_g, dkv_out or None)."""
    _gla_check(q, k, v, log_g, do)
    s = _shape(q)
    dq, dk, dv, dlog_g = (torch.empty_like(q) if t is None else t for t in (dq, dk, dv, dlog_g))
    dkv_out_t = _state_like(k) if dkv_out is True else (dkv_out if isinstance(dkv_out, torch.Tensor) else None)
    workspace = gla_alloc(q)[1] if workspace is None else workspace
    for t, n in ((dq, "dq"), (dk, "dk"), (dv, "dv"), (dlog_g, "dlog_g")):
        _check_like(t, q, n)
    _check_state(dkv_in, k, "dkv_in")
    _check_state(dkv_out_t, k, "dkv_out")
    _check_buf(cache, gla_cache_bytes(q), "cache", q.device)
    _check_buf(workspace, gla_workspace_bytes(q), "workspace", q.device)
    N.check(N.lib().lasp_gla_bwd_local(ctypes.byref(s), _p(q), _p(k), _p(v), _p(log_g), _p(do), _p(cache),
                                       _p(dkv_in), _p(dq), _p(dk), _p(dv), _p(dlog_g), _p(dkv_out_t), _p(workspace),
                                       _stream(q.device)))
    if check_state:
        workspace_status(workspace)
    return dq, dk, dv, dlog_g, dkv_out_t


def _ring_gla_fwd(self, q, k, v, log_g, *, o=None, cache=None, workspace=None):
    """Generalised-decay Alg. 2 across the ring (KV r -> r+1) -> (o, cache)."""
    _gla_check(q, k, v, log_g)
    s = _shape(q)
    o = torch.empty_like(q) if o is None else o
    if cache is None or workspace is None:
        c2, w2 = gla_alloc(q)
        cache = c2 if cache is None else cache
        workspace = w2 if workspace is None else workspace
    _check_like(o, q, "o")
    _check_buf(cache, gla_cache_bytes(q), "cache", q.device)
    _check_buf(workspace, gla_workspace_bytes(q), "workspace", q.device)
    N.check(N.lib().lasp_gla_fwd(self._ctx, ctypes.byref(s), _p(q), _p(k), _p(v), _p(log_g), _p(o), _p(cache),
                                 _p(workspace), _stream(q.device)))
    return o, cache


def _ring_gla_bwd(self, q, k, v, log_g, do, cache, *, workspace=None, check_state=False):
    """Generalised-decay Alg. 3 across the ring (dKV r+1 -> r) -> (dq, dk, dv, dlog_g)."""
    _gla_check(q, k, v, log_g, do)
    s = _shape(q)
    dq, dk, dv, dlg = (torch.empty_like(q) for _ in range(4))
    workspace = gla_alloc(q)[1] if workspace is None else workspace
    _check_buf(cache, gla_cache_bytes(q), "cache", q.device)
    _check_buf(workspace, gla_workspace_bytes(q), "workspace", q.device)
    N.check(N.lib().lasp_gla_bwd(self._ctx, ctypes.byref(s), _p(q), _p(k), _p(v), _p(log_g), _p(do), _p(cache),
                                 _p(dq), _p(dk), _p(dv), _p(dlg), _p(workspace), _stream(q.device)))
    if check_state:
        workspace_status(workspace)
    return dq, dk, dv, dlg


Ring.gla_fwd = _ring_gla_fwd
Ring.gla_bwd = _ring_gla_bwd


class LaspAttention(torch.autograd.Function):
    """O = LASP(Q, K, V; lambda) with the KV-state cache saved for backward.
    ``ring`` None runs the single-rank path (world size 1)."""

    @staticmethod
    def forward(ctx, q, k, v, lam, ring=None):
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        if ring is None:
            o, _, cache = fwd_local(q, k, v, lam, kv_out=False)
        else:
            o, cache = ring.fwd(q, k, v, lam)
        ctx.save_for_backward(q, k, v, cache)
        ctx.lam = lam
        ctx.ring = ring
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, cache = ctx.saved_tensors
        do = do.contiguous()
        if ctx.ring is None:
            dq, dk, dv, _ = bwd_local(q, k, v, ctx.lam, do, cache, dkv_out=False)
        else:
            dq, dk, dv = ctx.ring.bwd(q, k, v, ctx.lam, do, cache)
        return dq, dk, dv, None, None


def lasp_attention(q, k, v, lam, ring=None):
    return LaspAttention.apply(q, k, v, lam, ring)


class GlaAttention(torch.autograd.Function):
    """O = generalised-decay LASP(Q, K, V; log_g) (NEXT-4, the GLA / GateLoop row) with gradients for q, k, v and
    the log decay; the state cache is saved for backward. ``ring`` None runs the single-rank path."""

    @staticmethod
    def forward(ctx, q, k, v, log_g, ring=None):
        q, k, v, log_g = q.contiguous(), k.contiguous(), v.contiguous(), log_g.contiguous()
        if ring is None:
            o, _, cache = gla_fwd_local(q, k, v, log_g, kv_out=False)
        else:
            o, cache = ring.gla_fwd(q, k, v, log_g)
        ctx.save_for_backward(q, k, v, log_g, cache)
        ctx.ring = ring
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, log_g, cache = ctx.saved_tensors
        do = do.contiguous()
        if ctx.ring is None:
            dq, dk, dv, dlg, _ = gla_bwd_local(q, k, v, log_g, do, cache, dkv_out=False)
        else:
            dq, dk, dv, dlg = ctx.ring.gla_bwd(q, k, v, log_g, do, cache)
        return dq, dk, dv, dlg, None


def gla_attention(q, k, v, log_g, ring=None):
    return GlaAttention.apply(q, k, v, log_g, ring)


# ---- NEXT-3: the layer around the path (include/lasp.h lasp_layer_fwd / lasp_layer_bwd) ----------------------
def layer_workspace_bytes(shape: N.lasp_shape_t) -> int:
    return int(N.lib().lasp_layer_workspace_bytes(ctypes.byref(shape)))


def layer_fwd(x, w_q, w_k, w_v, lam, heads, ring=None, *, out=None, workspace=None):
    """Y = Norm(LASP(X W_Q, X W_K, X W_V)) for this rank's chunk x [B][C][d_model] (bf16); w_q [d][H*D],
    w_k, w_v [d][Hk*D]. Norm is the per-head RMS normalization of DESIGN.md reading N1. ``ring``: a Ring
    (the state arrives over the ring) or None (single rank). Returns a dict with q, k, v, y, rnorm, cache
    (all needed by layer_bwd)."""
    B, C, d = x.shape
    D = w_q.shape[1] // heads
    Hk = w_k.shape[1] // D
    if w_q.shape != (d, heads * D) or w_k.shape != (d, Hk * D) or w_v.shape != w_k.shape:
        raise ValueError("w_q must be [d_model][heads*D], w_k and w_v [d_model][kv_heads*D]")
    for t in (x, w_q, w_k, w_v):
        if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("layer tensors must be contiguous bf16 CUDA tensors")
    o = out or {}
    q = o.get("q") if o.get("q") is not None else torch.empty((B, C, heads, D), dtype=x.dtype, device=x.device)
    k = o.get("k") if o.get("k") is not None else torch.empty((B, C, Hk, D), dtype=x.dtype, device=x.device)
    v = o.get("v") if o.get("v") is not None else torch.empty_like(k)
    y = o.get("y") if o.get("y") is not None else torch.empty_like(q)
    rnorm = o.get("rnorm") if o.get("rnorm") is not None else torch.empty((B, C, heads), dtype=torch.float32,
                                                                           device=x.device)
    s = _shape(q, k)
    cache = o.get("cache") if o.get("cache") is not None else alloc_cache(q, k)
    if workspace is None:
        workspace = torch.empty(max(layer_workspace_bytes(s), 16), dtype=torch.uint8, device=x.device)
    _check_buf(workspace, layer_workspace_bytes(s), "workspace", x.device)
    _check_buf(cache, cache_bytes(s), "cache", x.device)
    _, lp = _lam(lam, Hk)
    ctx = ring._ctx if ring is not None else None
    N.check(N.lib().lasp_layer_fwd(ctx, ctypes.byref(s), d, _p(x), _p(w_q), _p(w_k), _p(w_v), lp, _p(q), _p(k),
                                   _p(v), _p(y), _p(rnorm), _p(cache), _p(workspace), _stream(x.device)))
    return {"q": q, "k": k, "v": v, "y": y, "rnorm": rnorm, "cache": cache, "workspace": workspace}


def layer_bwd(x, w_q, w_k, w_v, lam, fw, dy, ring=None, *, out=None):
    """Gradients of sum(Y * dY) for layer_fwd: returns dict dx, dw_q, dw_k, dw_v (fp32) and the intermediates
    d_o (= dL/dO, formed by the Norm backward inside the B1 kernel), dq, dk, dv."""
    q, k = fw["q"], fw["k"]
    B, C, d = x.shape
    o = out or {}
    d_o = o.get("d_o") if o.get("d_o") is not None else torch.empty_like(q)
    dq = o.get("dq") if o.get("dq") is not None else torch.empty_like(q)
    dk = o.get("dk") if o.get("dk") is not None else torch.empty_like(k)
    dv = o.get("dv") if o.get("dv") is not None else torch.empty_like(k)
    dx = o.get("dx") if o.get("dx") is not None else torch.empty_like(x)
    dws = [o.get(n) if o.get(n) is not None else torch.empty(w.shape, dtype=torch.float32, device=x.device)
           for n, w in (("dw_q", w_q), ("dw_k", w_k), ("dw_v", w_v))]
    _check_like(dy, q, "dy")
    s = _shape(q, k)
    _, lp = _lam(lam, k.shape[2])
    ctx = ring._ctx if ring is not None else None
    N.check(N.lib().lasp_layer_bwd(ctx, ctypes.byref(s), d, _p(x), _p(w_q), _p(w_k), _p(w_v), lp, _p(q), _p(k),
                                   _p(fw["v"]), _p(fw["y"]), _p(fw["rnorm"]), _p(dy), _p(fw["cache"]), _p(d_o),
                                   _p(dq), _p(dk), _p(dv), _p(dx), _p(dws[0]), _p(dws[1]), _p(dws[2]),
                                   _p(fw["workspace"]), _stream(x.device)))
    return {"dx": dx, "dw_q": dws[0], "dw_k": dws[1], "dw_v": dws[2], "d_o": d_o, "dq": dq, "dk": dk, "dv": dv}
