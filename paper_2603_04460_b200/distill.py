"""VSIndexer distillation on the GPU (§4.2).

Trains the indexer of every KV head against K5's ground-truth aggregates with the
reference's objective and optimiser (reference indexer.hpp):
  * loss  = D_KL(pred_v || target_v + eps) + D_KL(pred_s || target_s + eps)  (kl_loss :138-149,
            forward direction, eps = 1e-8 smoothing in the log denominator)
  * AdamW, beta = (0.9, 0.999), eps 1e-8, decoupled weight decay 0.01      (optimizer_step :347-363)
  * linear warmup to lr_peak then cosine to 0                                (learning_rate :322-329)
  * init make_indexer_params: W_U ~ U(+-1/sqrt(2d)), heads and biases 0      (:53-64)
The forward matches K1 (X = [K | V], SiLU, two heads, Reverse slash mapping, softmax over n)
and runs in fp32 torch with autograd: this is the offline training half of the paper, not the
prefill hot path (the product forward is the sm_100a K1 kernel, fed the bf16 copy of W_U).
Samples are visited round-robin, one prompt per optimiser step (train_custom :388-427).
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import torch

from . import IndexerParams


def _forward(k: torch.Tensor, v: torch.Tensor, w_u, b_u, w_v, b_v, w_s, b_s, reverse: bool = True):
    """k, v [n, H, d] -> (log pred_v, log pred_s) [H, n]."""
    x = torch.cat([k.float(), v.float()], dim=2).permute(1, 0, 2)  # [H, n, 2d]
    y = torch.baddbmm(b_u[:, None, :], x, w_u)                       # [H, n, d_h]
    z = torch.nn.functional.silu(y)
    lv = torch.bmm(z, w_v[:, :, None])[..., 0] + b_v[:, None]
    ls = torch.bmm(z, w_s[:, :, None])[..., 0] + b_s[:, None]
    if reverse:
        ls = ls.flip(1)
    return torch.log_softmax(lv, dim=1), torch.log_softmax(ls, dim=1)


def kl_forward(logp: torch.Tensor, target: torch.Tensor, eps: float = 1e-8) -> torch.Tensor:
    """sum_i p_i (log p_i - log(t_i + eps)) per head (kl_loss, indexer.hpp:138-149)."""
    p = logp.exp()
    return (p * (logp - torch.log(target.double().float() + eps))).sum(dim=1)


def learning_rate(step: int, steps: int, warmup: int, lr_peak: float) -> float:
    if step < warmup:
        return lr_peak * (step + 1) / warmup
    span = max(steps - warmup, 1)
    return lr_peak * 0.5 * (1.0 + math.cos(math.pi * (step - warmup) / span))


def distill_indexer(samples: Sequence[Tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]], d_h: int,
                    steps: int = 300, lr_peak: float = 3e-3, warmup: int = 30, weight_decay: float = 0.01,
                    eps: float = 1e-8, seed: int = 1, reverse: bool = True, log_every: int = 0
                    ) -> Tuple[IndexerParams, List[float]]:
    """samples: (K [n,H,d], V [n,H,d], target_v [H,n], target_s [H,n]) per prompt, all on one
    device. Returns bf16/fp32 IndexerParams for the K1 kernel and the per-step losses."""
    k0 = samples[0][0]
    dev = k0.device
    hkv, d = k0.shape[1], k0.shape[2]
    g = torch.Generator(device="cpu").manual_seed(seed)
    lim = 1.0 / math.sqrt(2 * d)
    w_u = ((torch.rand(hkv, 2 * d, d_h, generator=g) * 2 - 1) * lim).to(dev).requires_grad_()
    b_u = torch.zeros(hkv, d_h, device=dev, requires_grad=True)
    w_v = torch.zeros(hkv, d_h, device=dev, requires_grad=True)
    w_s = torch.zeros(hkv, d_h, device=dev, requires_grad=True)
    b_v = torch.zeros(hkv, device=dev, requires_grad=True)
    b_s = torch.zeros(hkv, device=dev, requires_grad=True)
    params = [w_u, b_u, w_v, b_v, w_s, b_s]
    opt = torch.optim.AdamW(params, lr=lr_peak, betas=(0.9, 0.999), eps=1e-8, weight_decay=weight_decay)
    losses = []
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        for step in range(steps):
            k, v, tv, ts = samples[step % len(samples)]
            for pg in opt.param_groups:
                pg["lr"] = learning_rate(step, steps, warmup, lr_peak)
            lpv, lps = _forward(k, v, w_u, b_u, w_v, b_v, w_s, b_s, reverse)
            loss_h = kl_forward(lpv, tv, eps) + kl_forward(lps, ts, eps)
            loss = loss_h.sum()
            opt.zero_grad(set_to_none=True)
            loss.backward()
            opt.step()
            losses.append(float(loss_h.mean().item()) if (log_every and step % log_every == 0) or step == steps - 1
                          else float("nan"))
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
    with torch.no_grad():
        out = IndexerParams(w_u.detach().to(torch.bfloat16).contiguous(), b_u.detach().contiguous(),
                            w_v.detach().contiguous(), b_v.detach().contiguous(), w_s.detach().contiguous(),
                            b_s.detach().contiguous())
    return out, losses


def eval_kl(params: IndexerParams, k, v, tv, ts, eps: float = 1e-8, reverse: bool = True) -> torch.Tensor:
    """Per-head held-out loss of fixed params (evaluate_loss, indexer.hpp:440-451) in fp32."""
    with torch.no_grad():
        lpv, lps = _forward(k, v, params.w_u.float(), params.b_u, params.w_v, params.b_v, params.w_s, params.b_s,
                            reverse)
        return kl_forward(lpv, tv, eps) + kl_forward(lps, ts, eps)
