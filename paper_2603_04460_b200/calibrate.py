"""Offline preparation of a VS-prefill layer: distill the indexer on training prompts and
pick the cumulative-threshold budget (tau_v, tau_s) that reaches a recall target.

This is the paper's recipe (§4.2-4.3): ground-truth aggregates from full attention
(K5 over K4's LSE), KL distillation of the VSIndexer, then adaptive top-k selection whose
thresholds are fixed hyper-parameters. Calibration measures recall exactly on the device
(mean_i exp(LSE_sparse - LSE_dense), attention.hpp:198-215) on a TRAINING prompt; the
bench then reports the recall it actually gets on its held-out prompt.
"""
from __future__ import annotations

import itertools
from typing import List, Optional, Sequence, Tuple

import torch

from . import (BudgetConfig, IndexerParams, aggregate_streaming, attention_recall, blockwise_attention,
               indexer_forward, select_pattern, sparse_attention, sparse_tile_stats)
from .distill import distill_indexer

DEFAULT_TAUS = (0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9)


def ground_truth(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor):
    """-> (A_v, A_s) [Hkv, n] group-mean normalised aggregates and the dense LSE [Hq, n]."""
    _, lse = blockwise_attention(q, k, v)
    a_v, a_s = aggregate_streaming(q, k, lse=lse)
    return a_v, a_s, lse


def train_indexer(prompts: Sequence[Tuple[torch.Tensor, torch.Tensor, torch.Tensor]], d_h: int, steps: int = 200,
                  lr_peak: float = 3e-3, seed: int = 1) -> Tuple[IndexerParams, List[float]]:
    samples = []
    for q, k, v in prompts:
        a_v, a_s, _ = ground_truth(q, k, v)
        samples.append((k, v, a_v, a_s))
    return distill_indexer(samples, d_h=d_h, steps=steps, lr_peak=lr_peak, warmup=max(1, steps // 10), seed=seed,
                           log_every=max(1, steps // 10))


def calibrate_budget(q, k, v, params: IndexerParams, recall_target: float = 0.9,
                     taus: Sequence[float] = DEFAULT_TAUS, min_budget: int = 1,
                     max_budget: Optional[int] = None) -> Tuple[BudgetConfig, dict]:
    """Grid over (tau_v, tau_s); keep the cheapest pattern (fewest KV tiles) whose recall
    reaches the target on this prompt. Falls back to the highest-recall point."""
    n, hq, d = q.shape
    hkv = k.shape[1]
    _, lse_d = blockwise_attention(q, k, v)
    a_v, a_s = indexer_forward(k, v, params)
    o = torch.empty_like(q)
    lse = torch.empty_like(lse_d)
    best, best_any = None, None
    for tv, ts in itertools.product(taus, taus):
        b = BudgetConfig(tv, ts, min_budget, max_budget)
        pat = select_pattern(a_v, a_s, b)
        sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse)
        tiles, dense_tiles = sparse_tile_stats(n, hkv, pat.i_v.shape[1], q.device)
        rec = float(attention_recall(lse, lse_d).mean().item())
        pt = dict(tau_v=tv, tau_s=ts, recall=rec, tiles=tiles, tile_density=tiles / dense_tiles)
        if best_any is None or rec > best_any[1]["recall"]:
            best_any = (b, pt)
        if rec >= recall_target and (best is None or tiles < best[1]["tiles"]):
            best = (b, pt)
    return best if best is not None else best_any
