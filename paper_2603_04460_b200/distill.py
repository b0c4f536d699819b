"""VSIndexer distillation on the GPU (§4.2).

`IndexerTrainer` / `distill_indexer` run on the hand-written sm_100a kernels of csrc/train.cu
through the C ABI (vsp_indexer_loss_grad: K1 forward + fp64 KL softmax + tcgen05 backward
GEMMs; vsp_adamw_step), with fp32 master weights and the bf16 copy the K1 forward reads.
`distill_indexer_torch` is the same objective in fp32 torch autograd, kept as the test
reference for the kernels.

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

import ctypes
import math
from typing import List, Optional, Sequence, Tuple

import torch

from . import IndexerParams, _check, _context, _need_cuda, _ptr, _stream, _workspace, load_library


class _AdamW(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("adam_eps", ctypes.c_double), ("weight_decay", ctypes.c_double)]


def _bind(lib):
    vp, i, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    lib.vsp_indexer_grad_workspace_size.restype = ctypes.c_size_t
    lib.vsp_indexer_grad_workspace_size.argtypes = [i, i, i]
    lib.vsp_indexer_loss_grad.argtypes = [vp, vp, vp, i, i, i, i, vp, vp, vp, vp, vp, vp, i, vp, vp, ctypes.c_double,
                                          vp, vp, vp, vp]
    lib.vsp_adamw_step.argtypes = [vp, vp, vp, vp, vp, i64, i64, ctypes.POINTER(_AdamW), vp, i64, vp]
    return lib


class IndexerTrainer:
    """Flat fp32 master parameters of every KV head's indexer, in the C ABI's gradient layout
    W_U [hkv, 2d, d_h] | b_U | w_v | w_s [hkv, d_h] | b_v | b_s [hkv], plus AdamW moments and
    the bf16 W_U copy. Init = make_indexer_params (indexer.hpp:53-64): W_U ~ U(+-1/sqrt(2d)),
    heads and biases zero."""

    def __init__(self, hkv: int, d: int, d_h: int, device, seed: int = 1):
        self.hkv, self.d, self.d_h = hkv, d, d_h
        self.nw, self.nv = hkv * 2 * d * d_h, hkv * d_h
        self.count = self.nw + 3 * self.nv + 2 * hkv
        dev = torch.device(device)
        g = torch.Generator(device="cpu").manual_seed(seed)
        lim = 1.0 / math.sqrt(2 * d)
        self.flat = torch.zeros(self.count, device=dev)
        self.flat[:self.nw] = ((torch.rand(self.nw, generator=g) * 2 - 1) * lim).to(dev)
        self.m = torch.zeros_like(self.flat)
        self.v = torch.zeros_like(self.flat)
        self.grads = torch.zeros_like(self.flat)
        self.w_u_bf16 = self.flat[:self.nw].view(hkv, 2 * d, d_h).to(torch.bfloat16)
        self.loss = torch.zeros(hkv, device=dev)
        self._lib = _bind(load_library())

    def view(self, name: str) -> torch.Tensor:
        nw, nv, h = self.nw, self.nv, self.hkv
        o = {"w_u": (0, nw), "b_u": (nw, nv), "w_v": (nw + nv, nv), "w_s": (nw + 2 * nv, nv),
             "b_v": (nw + 3 * nv, h), "b_s": (nw + 3 * nv + h, h)}[name]
        t = self.flat[o[0]:o[0] + o[1]]
        if name == "w_u":
            return t.view(h, 2 * self.d, self.d_h)
        return t.view(h, self.d_h) if name in ("b_u", "w_v", "w_s") else t

    def params(self) -> IndexerParams:
        """The current weights as the K1 kernel takes them (W_U bf16, the rest fp32)."""
        return IndexerParams(self.w_u_bf16, self.view("b_u"), self.view("w_v"), self.view("b_v"), self.view("w_s"),
                             self.view("b_s"))

    def loss_grad(self, k, v, target_v, target_s, eps: float = 1e-8, reverse: bool = True):
        """indexer_backward_loss for every head (vsp_indexer_loss_grad) -> per-head loss [hkv];
        the flat gradient lands in self.grads."""
        _need_cuda(k, v, target_v, target_s)
        n = k.shape[0]
        dev = k.device
        ws = _workspace(dev, self._lib.vsp_indexer_grad_workspace_size(n, self.hkv, self.d_h))
        _check(self._lib.vsp_indexer_loss_grad(
            _context(dev), _ptr(k), _ptr(v), n, self.hkv, self.d, self.d_h, _ptr(self.w_u_bf16), _ptr(self.view("b_u")),
            _ptr(self.view("w_v")), _ptr(self.view("b_v")), _ptr(self.view("w_s")), _ptr(self.view("b_s")),
            0 if reverse else 1, _ptr(target_v.contiguous()), _ptr(target_s.contiguous()), float(eps), _ptr(self.loss),
            _ptr(self.grads), _ptr(ws), _stream(dev)))
        return self.loss

    def adamw(self, step_index: int, lr: float, beta1: float = 0.9, beta2: float = 0.999, adam_eps: float = 1e-8,
              weight_decay: float = 0.01):
        """optimizer_step (indexer.hpp:347-363) on all parameters; refreshes the bf16 W_U."""
        cfg = _AdamW(lr, beta1, beta2, adam_eps, weight_decay)
        dev = self.flat.device
        _check(self._lib.vsp_adamw_step(_context(dev), _ptr(self.flat), _ptr(self.grads), _ptr(self.m), _ptr(self.v),
                                        self.count, int(step_index), ctypes.byref(cfg), _ptr(self.w_u_bf16), self.nw,
                                        _stream(dev)))


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
                    eps: float = 1e-8, seed: int = 1, reverse: bool = True, log_every: int = 0,
                    stats: Optional[dict] = None) -> Tuple[IndexerParams, List[float]]:
    """samples: (K [n,H,d], V [n,H,d], target_v [H,n], target_s [H,n]) per prompt, all on one
    device. Samples are visited round-robin, one per optimiser step (train_custom :388-427);
    every step is one vsp_indexer_loss_grad + one vsp_adamw_step. Returns the trained
    IndexerParams (bf16 W_U for K1) and the per-step mean losses (nan where not logged).
    stats (optional) receives step_ms: device time per step (CUDA events over the loop)."""
    k0 = samples[0][0]
    tr = IndexerTrainer(k0.shape[1], k0.shape[2], d_h, k0.device, seed=seed)
    losses = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for step in range(steps):
        k, v, tv, ts = samples[step % len(samples)]
        loss = tr.loss_grad(k, v, tv, ts, eps=eps, reverse=reverse)
        tr.adamw(step, learning_rate(step, steps, warmup, lr_peak), weight_decay=weight_decay)
        logged = (log_every and step % log_every == 0) or step == steps - 1
        losses.append(float(loss.mean().item()) if logged else float("nan"))
    ev1.record()
    if stats is not None:
        torch.cuda.synchronize()
        stats["step_ms"] = ev0.elapsed_time(ev1) / max(steps, 1)
    return tr.params(), losses


def distill_indexer_torch(samples: Sequence[Tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]], d_h: int,
                          steps: int = 300, lr_peak: float = 3e-3, warmup: int = 30, weight_decay: float = 0.01,
                          eps: float = 1e-8, seed: int = 1, reverse: bool = True, log_every: int = 0
                          ) -> Tuple[IndexerParams, List[float]]:
    """The same objective in fp32 torch autograd (test reference for the kernels)."""
    k0 = samples[0][0]
    dev = k0.device
    hkv, d = k0.shape[1], k0.shape[2]
    g = torch.Generator(device="cpu").manual_seed(seed)
    lim = 1.0 / math.sqrt(2 * d)
    w_u = ((torch.rand(hkv * 2 * d * d_h, generator=g) * 2 - 1) * lim).view(hkv, 2 * d, d_h).to(dev).requires_grad_()
    b_u = torch.zeros(hkv, d_h, device=dev, requires_grad=True)
    w_v = torch.zeros(hkv, d_h, device=dev, requires_grad=True)
    w_s = torch.zeros(hkv, d_h, device=dev, requires_grad=True)
    b_v = torch.zeros(hkv, device=dev, requires_grad=True)
    b_s = torch.zeros(hkv, device=dev, requires_grad=True)
    params = [w_u, b_u, w_v, b_v, w_s, b_s]
    opt = torch.optim.AdamW(params, lr=lr_peak, betas=(0.9, 0.999), eps=1e-8, weight_decay=weight_decay)
    losses = []
    for step in range(steps):
        k, v, tv, ts = samples[step % len(samples)]
        for pg in opt.param_groups:
            pg["lr"] = learning_rate(step, steps, warmup, lr_peak)
        lpv, lps = _forward(k, v, w_u, b_u, w_v, b_v, w_s, b_s, reverse)
        loss_h = kl_forward(lpv, tv, eps) + kl_forward(lps, ts, eps)
        opt.zero_grad(set_to_none=True)
        loss_h.sum().backward()
        opt.step()
        losses.append(float(loss_h.mean().item()) if (log_every and step % log_every == 0) or step == steps - 1
                      else float("nan"))
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
