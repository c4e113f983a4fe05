"""A TransNormerLLM-style linear-attention layer on the LASP library (usage example).

    x -> [Q, K, V] = x W_qkv -> LASP(Q, K, V; lambda_h) -> O W_o

The projections are plain torch Linear layers; the attention (forward and backward, with the KV-state
cache) runs in liblasp.so through `lasp_attention` (a torch.autograd.Function). One GPU:

    python examples/lasp_layer.py --tokens 32768

Sequence parallel over G GPUs of one node (rank r owns tokens [r C, (r+1) C), the KV state travels
r -> r+1 in the forward pass and the dKV state r+1 -> r in the backward pass, Alg. 2 / Alg. 3):

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 examples/lasp_layer.py --tokens 262144

Data-sequence hybrid (Alg. 1: G = W/T groups of T ranks, each group on its own sequence):

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 examples/lasp_layer.py --tokens 131072 --sp-size 4
"""
import argparse
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_02882_b200 as lasp  # noqa: E402


class LaspLayer(torch.nn.Module):
    def __init__(self, d_model: int, heads: int, head_dim: int, ring=None):
        super().__init__()
        self.h, self.dh, self.ring = heads, head_dim, ring
        self.qkv = torch.nn.Linear(d_model, 3 * heads * head_dim, bias=False)
        self.out = torch.nn.Linear(heads * head_dim, d_model, bias=False)
        # TNL-style per-head decay, fixed (not learned): lambda_h = 1 - 2^-(1 + 14 h / (H - 1)); kept as a
        # host fp32 array (the boundary takes lambda as fp32 on the host, reading A8), not a module buffer
        hs = np.arange(heads, dtype=np.float64)
        self.lam = (1 - 2 ** -(1 + 14 * hs / max(heads - 1, 1))).astype(np.float32)

    def forward(self, x):  # x: [batch][n_local][d_model]
        B, C, _ = x.shape
        q, k, v = self.qkv(x).view(B, C, 3, self.h, self.dh).unbind(2)  # [B][C][H][D] each
        o = lasp.lasp_attention(q.contiguous(), k.contiguous(), v.contiguous(), self.lam, self.ring)
        return self.out(o.reshape(B, C, self.h * self.dh))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=32768, help="sequence length (split over the ring)")
    ap.add_argument("--d-model", type=int, default=1024)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--head-dim", type=int, default=64)
    ap.add_argument("--sp-size", type=int, default=0, help="sequence-parallel size T (default: all ranks)")
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    ring, T = None, 1
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        T = args.sp_size or world
        group = lasp.sp_group(T) if T < world else None
        ring = lasp.Ring(torch.device("cuda", local), group=group) if T > 1 else None
    _, chunk, _ = lasp.topology(rank, world, T)
    C = args.tokens // T

    torch.manual_seed(0)
    layer = LaspLayer(args.d_model, args.heads, args.head_dim, ring).cuda().to(torch.bfloat16)
    opt = torch.optim.AdamW(layer.parameters(), lr=1e-4)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank // T)  # same sequence inside a group
    x_full = torch.randn(1, args.tokens, args.d_model, device="cuda", dtype=torch.bfloat16, generator=g)
    x = x_full[:, chunk * C:(chunk + 1) * C].contiguous()  # this rank's chunk (Alg. 1)
    for step in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        y = layer(x)
        loss = y.float().square().mean()
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        torch.cuda.synchronize()
        if rank == 0:
            print(f"step {step}: loss {loss.item():.5f}  {1e3 * (time.perf_counter() - t0):.2f} ms "
                  f"({world} rank(s), {C} tokens per rank)")
    if ring is not None:
        ring.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
