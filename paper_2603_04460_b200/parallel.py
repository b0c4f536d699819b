"""KV-head sharding of the VS-prefill layer across the GPUs of one node.

Every hot-path step is per KV head (indexer, selection, and the sparse attention of the Q
heads in the group), so a layer splits into independent shards with NO collective on the
data path. Rank r owns KV heads [r*Hkv/N, (r+1)*Hkv/N) and their Q heads. The only
collective is the optional all-gather that assembles the full output: each rank's O is
made head-major [Hq/N, n, d] so its shard is one contiguous send buffer, and
`all_gather_into_tensor` over NCCL (NVLink/NVSwitch) lands it as [Hq, n, d].
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def head_range(num_heads: int, rank: int, world: int) -> Tuple[int, int]:
    if num_heads % world:
        raise ValueError(f"{num_heads} heads do not split across {world} ranks")
    per = num_heads // world
    return rank * per, (rank + 1) * per


def shard_heads(x: torch.Tensor, rank: int, world: int, dim: int = 1) -> torch.Tensor:
    """Contiguous slice of the head dimension owned by `rank` (token-major [n, H, d] -> dim 1;
    per-head parameter tensors [H, ...] -> dim 0)."""
    lo, hi = head_range(x.shape[dim], rank, world)
    return x.narrow(dim, lo, hi - lo).contiguous()


def assemble_heads(o_shard: torch.Tensor, group=None) -> torch.Tensor:
    """[n, Hq/N, d] per rank -> [Hq, n, d] everywhere (head-major), one all-gather."""
    world = dist.get_world_size(group)
    oh = o_shard.permute(1, 0, 2).contiguous()
    full = torch.empty((world * oh.shape[0],) + tuple(oh.shape[1:]), dtype=oh.dtype, device=oh.device)
    dist.all_gather_into_tensor(full, oh, group=group)
    return full


def max_over_ranks(value: float, device) -> float:
    """Device-timed numbers are reported as the max over ranks."""
    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
