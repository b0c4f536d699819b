"""Synthetic attention layers with planted vertical-slash structure, generated on the GPU.

Same construction as the reference's datagen (reference datagen.hpp:61-115 with
theory.hpp:197 plant_slash_means), restated for many heads and long sequences and done in
torch on the device (the reference's `generate` also runs an O(n^2) f64 aggregation; here
the ground truth comes from K5 when needed):

* RoPE with interleaved pairs (2p, 2p+1), theta_p = base^(-2p/d) (reference rope.hpp:42-52).
* Slash structure: q_i = R(i)(mu_q + noise), k_j = R(j)(mu_k + noise) gives
  E[q_i . k_j] = sum_p a_p^2 cos((i - j - o_p) theta_p): a rotated plane p assigned to offset
  o_p peaks at i - j = o_p. The mid/low-frequency planes build the local window (o_p = 0);
  groups of high-frequency planes build sharp long-range stripes.
* Vertical structure: every query carries q_base on the last plane, which is left unrotated
  (NoPE), and anchor keys are overwritten with a multiple of that direction, so a planted
  column scores high from every row at any distance. This is datagen.hpp:85-108's "anchor
  aligned with the mean query" made position-free: at 128k the reference's slowest RoPE
  plane rotates by ~15 rad and no longer gives a coherent mean query. Token 0 is the sink.
* V is i.i.d. N(0, 1).

Two seeds, mirroring how a real model behaves: `head_seed` fixes each KV
group's structure (its stripe offsets and mean vectors — a property of the "weights"), while
`prompt_seed` draws the noise and the anchor positions (content). The Q heads of a group share
mu_q (intra-group consistency); groups differ (inter-group divergence).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Tuple

import torch


@dataclasses.dataclass
class PlantConfig:
    n_stripes: int = 1            # long-range slash offsets per KV group
    stripe_range: Tuple[int, int] = (256, 8192)
    stripe_planes: int = 16       # fast planes per stripe (planes 0 .. n_stripes*stripe_planes-1)
    stripe_amp: float = 3.3
    local_amp: float = 2.1        # amplitude of the remaining rotated planes (peak at offset 0)
    n_anchors: int = 16           # vertical heavy hitters per KV group (plus the sink, token 0)
    anchor_strength: float = 36.0
    sink_strength: float = 41.0
    q_base: float = 6.0           # query component on the unrotated (NoPE) plane
    noise_sigma: float = 0.5
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


def head_structure(hkv: int, d: int, n: int, head_seed: int, cfg: PlantConfig):
    """Per KV group: stripe offsets and the (mu_q, mu_k) mean vectors."""
    g = torch.Generator(device="cpu").manual_seed(head_seed)
    planes = d // 2
    theta = cfg.rope_base ** (-2.0 * torch.arange(planes, dtype=torch.float64) / d)
    mu_q = torch.zeros(hkv, d, dtype=torch.float64)
    mu_k = torch.zeros(hkv, d, dtype=torch.float64)
    stripes = []
    lo, hi = cfg.stripe_range
    hi = max(lo + 1, min(hi, n))
    for kv in range(hkv):
        offs = sorted(int(x) for x in torch.randint(lo, hi, (cfg.n_stripes,), generator=g))
        stripes.append(offs)
        assign = {}
        for s, o in enumerate(offs):
            for j in range(cfg.stripe_planes):
                assign[s + j * len(offs)] = (o, cfg.stripe_amp)  # interleave stripes over the fast planes
        for p in range(planes - 1):  # the last plane is the unrotated (NoPE) sink channel
            o, a = assign.get(p, (0, cfg.local_amp))
            ph = o * float(theta[p])
            mu_q[kv, 2 * p] = a
            mu_k[kv, 2 * p] = a * math.cos(ph)
            mu_k[kv, 2 * p + 1] = a * math.sin(ph)
        mu_q[kv, d - 2] = cfg.q_base
    return mu_q, mu_k, stripes


def planted_layer(n: int, hq: int, hkv: int, d: int = 128, seed: int = 0, cfg: Optional[PlantConfig] = None,
                  device="cuda", head_seed: Optional[int] = None, gen_device=None,
                  ) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor, List[dict]]:
    """-> Q [n, hq, d], K [n, hkv, d], V [n, hkv, d] bf16 on `device` and the planted structure
    per group. `seed` is the prompt seed; `head_seed` (default: 1000003) fixes the heads'
    structure. `gen_device` (default: `device`) is where the values are drawn and computed:
    "cpu" gives the same bits on every machine and process (torch's CPU generator and
    unfused elementwise ops), so a CPU-only process (bench.py's reference arm) and a GPU
    process see the identical layer."""
    cfg = cfg or PlantConfig()
    if gen_device is not None and torch.device(gen_device) != torch.device(device):
        q, k, v, plants = planted_layer(n, hq, hkv, d, seed, cfg, gen_device, head_seed)
        return q.to(device), k.to(device), v.to(device), plants
    dev = torch.device(device)
    hs = 1000003 if head_seed is None else head_seed
    mu_q, mu_k, stripes = head_structure(hkv, d, n, hs, cfg)
    grp = hq // hkv
    gp = torch.Generator(device="cpu").manual_seed(seed)
    plants = []
    for kv in range(hkv):
        anchors = sorted(set(int(x) for x in torch.randint(1, max(2, n), (cfg.n_anchors,), generator=gp)))
        plants.append(dict(stripes=stripes[kv], anchors=[0] + anchors))
    ang = rope_angles(n, d, cfg.rope_base, dev)
    ang[:, -1] = 0.0  # NoPE plane: the sink/anchor channel does not rotate (position-free heavy hitters)
    gen = torch.Generator(device=dev).manual_seed(seed + 1)
    q = torch.randn(n, hq, d, device=dev, generator=gen).mul_(cfg.noise_sigma)
    q += mu_q.to(dev).float().repeat_interleave(grp, dim=0)[None]
    q = apply_rope(q, ang)
    k = torch.randn(n, hkv, d, device=dev, generator=gen).mul_(cfg.noise_sigma)
    k += mu_k.to(dev).float()[None]
    k = apply_rope(k, ang)
    del ang
    # heavy hitters: keys on the NoPE channel, which every query carries with weight q_base
    # (the long-sequence analogue of datagen.hpp:85-108's "aligned with the mean query")
    u = torch.zeros(d, device=dev)
    u[d - 2] = 1.0
    for kv in range(hkv):
        idx = torch.tensor(plants[kv]["anchors"][1:], device=dev, dtype=torch.long)
        if len(idx):
            k[idx, kv] = cfg.anchor_strength * u + k[idx, kv] * 0.1
        k[0, kv] = cfg.sink_strength * u
    v = torch.randn(n, hkv, d, device=dev, generator=gen)
    return q.to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16), plants
