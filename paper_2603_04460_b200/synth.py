"""Synthetic attention layers with planted vertical-slash structure, generated on the GPU.

Same construction as the reference's datagen (reference datagen.hpp:61-115 with
theory.hpp:197 plant_slash_means), restated for many heads and long sequences and done in
torch on the device (the reference's `generate` also runs an O(n^2) f64 aggregation, which
is skipped here; the ground truth comes from K5 when needed):

* RoPE with interleaved pairs (2p, 2p+1), theta_p = base^(-2p/d) (reference rope.hpp:42-52).
* Slash structure: q_i = R(i)(mu_q + noise), k_j = R(j)(mu_k + noise) gives
  E[q_i . k_j] = sum_p r_p cos((i-j) theta_p - alpha_p). Planes are dealt round-robin to the
  planted offsets; a plane assigned to offset o* gets phase alpha_p = o* theta_p so all of its
  planes peak together at i - j = o*. Offset 0 (the local window) is always planted.
* Vertical structure: anchor keys are overwritten after rotation with a multiple of the
  normalised mean post-RoPE query (datagen.hpp:85-108), so a planted column scores high from
  every row; the slowest plane carries a query baseline (q_base, datagen.hpp:64-66).
* V is i.i.d. N(0, 1).
Each KV group draws its own offsets/anchors (inter-group divergence); the Q heads of a group
share mu_q (intra-group consistency), as observed in the paper.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import torch


@dataclasses.dataclass
class PlantConfig:
    n_offsets: int = 6            # planted slash offsets per KV group (besides offset 0)
    max_offset: int = 4096        # planted offsets drawn from [1, max_offset)
    n_anchors: int = 24           # planted vertical columns per KV group (besides token 0)
    plane_amp: float = 1.6        # |mu_q,p| = |mu_k,p| per rotated plane
    anchor_strength: float = 14.0
    q_base: float = 6.0
    noise_sigma: float = 0.6
    rope_base: float = 10000.0


def rope_angles(n: int, d: int, base: float, device) -> torch.Tensor:
    p = torch.arange(d // 2, device=device, dtype=torch.float64)
    theta = base ** (-2.0 * p / d)
    t = torch.arange(n, device=device, dtype=torch.float64)
    return torch.outer(t, theta)  # [n, d/2]


def apply_rope(x: torch.Tensor, ang: torch.Tensor) -> torch.Tensor:
    """x [n, H, d] f32; rotate interleaved pairs by ang [n, d/2] (rope.hpp:42-52)."""
    c = torch.cos(ang).float()[:, None, :]
    s = torch.sin(ang).float()[:, None, :]
    x0, x1 = x[..., 0::2], x[..., 1::2]
    out = torch.empty_like(x)
    out[..., 0::2] = x0 * c - x1 * s
    out[..., 1::2] = x0 * s + x1 * c
    return out


def planted_layer(n: int, hq: int, hkv: int, d: int = 128, seed: int = 0, cfg: Optional[PlantConfig] = None,
                  device="cuda") -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor, List[dict]]:
    """-> Q [n, hq, d], K [n, hkv, d], V [n, hkv, d] bf16 and the planted structure per group."""
    cfg = cfg or PlantConfig()
    dev = torch.device(device)
    g = torch.Generator(device="cpu").manual_seed(seed)
    grp = hq // hkv
    planes = d // 2
    ang = rope_angles(n, d, cfg.rope_base, dev)
    theta = (cfg.rope_base ** (-2.0 * torch.arange(planes, dtype=torch.float64) / d))
    mu_q = torch.zeros(hkv, d, dtype=torch.float64)
    mu_k = torch.zeros(hkv, d, dtype=torch.float64)
    plants = []
    for kv in range(hkv):
        offs = [0] + sorted(set(int(x) for x in torch.randint(1, max(2, min(cfg.max_offset, n)), (cfg.n_offsets,),
                                                                 generator=g).tolist()))
        # the slowest plane is reserved for the query baseline (datagen.hpp:57-66)
        for p in range(planes - 1):
            # E[q_i.k_j] on plane p = a^2 cos((i-j) theta_p - o theta_p): peaks at i - j = o
            o = offs[p % len(offs)]
            phase = o * float(theta[p])
            a = cfg.plane_amp
            mu_q[kv, 2 * p] = a
            mu_k[kv, 2 * p] = a * math.cos(phase)
            mu_k[kv, 2 * p + 1] = a * math.sin(phase)
        mu_q[kv, d - 2] += cfg.q_base
        anchors = sorted(set([0] + [int(x) for x in torch.randint(1, max(2, n), (cfg.n_anchors,), generator=g)]))
        plants.append(dict(offsets=offs, anchors=anchors))
    gen = torch.Generator(device=dev).manual_seed(seed + 1)
    q0 = torch.randn(n, hq, d, device=dev, generator=gen) * cfg.noise_sigma
    q0 += mu_q.to(dev).float().repeat_interleave(grp, dim=0)[None]
    k0 = torch.randn(n, hkv, d, device=dev, generator=gen) * cfg.noise_sigma + mu_k.to(dev).float()[None]
    q = apply_rope(q0, ang)
    k = apply_rope(k0, ang)
    del q0, k0
    for kv in range(hkv):
        mq = q[:, kv * grp:(kv + 1) * grp].mean(dim=(0, 1))
        mq = mq / mq.norm().clamp_min(1e-9)
        idx = torch.tensor(plants[kv]["anchors"], device=dev)
        k[idx, kv] = cfg.anchor_strength * mq
    v = torch.randn(n, hkv, d, device=dev, generator=gen)
    return q.to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16), plants
