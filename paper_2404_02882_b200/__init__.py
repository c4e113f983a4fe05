"""B200-native LASP hot path (arXiv 2404.02882): chunked causal linear attention with per-head
decay, sequence-parallel over a KV-state P2P ring. The compute lives in liblasp.so (CUDA, sm_100a,
C ABI in include/lasp.h); this package only marshals arguments."""
from . import _native
from .api import (GlaAttention, LaspAttention, Ring, gla_attention, alloc_cache, alloc_workspace, bwd_local, cache_bytes, fwd_local,
                  gla_alloc, gla_bwd_local, gla_cache_bytes, gla_fwd_local, gla_workspace_bytes, layer_bwd, layer_fwd, layer_workspace_bytes,
                  lasp_attention, scatter_sequence, segment_len, sp_group, topology,
                  workspace_bytes, workspace_status)

__all__ = ["GlaAttention", "LaspAttention", "Ring", "gla_attention", "alloc_cache", "alloc_workspace", "bwd_local", "cache_bytes", "fwd_local",
           "gla_alloc", "gla_bwd_local", "gla_cache_bytes", "gla_fwd_local", "gla_workspace_bytes",
           "layer_bwd", "layer_fwd", "layer_workspace_bytes",
           "lasp_attention", "scatter_sequence", "segment_len", "sp_group", "topology", "workspace_bytes",
           "workspace_status", "_native"]
