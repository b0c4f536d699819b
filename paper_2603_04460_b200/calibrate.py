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
                  lr_peak: float = 3e-3, seed: int = 1, stats: Optional[dict] = None
                  ) -> Tuple[IndexerParams, List[float]]:
    """K5 ground truth of each prompt, then distillation on the sm_100a training kernels.
    stats (optional) receives ground_truth_ms (K4 LSE + K5 per prompt) and step_ms."""
    samples = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for q, k, v in prompts:
        a_v, a_s, _ = ground_truth(q, k, v)
        samples.append((k, v, a_v, a_s))
    ev1.record()
    out = distill_indexer(samples, d_h=d_h, steps=steps, lr_peak=lr_peak, warmup=max(1, steps // 10), seed=seed,
                          log_every=max(1, steps // 10), stats=stats)
    if stats is not None:
        stats["ground_truth_ms"] = ev0.elapsed_time(ev1) / max(len(prompts), 1)
    return out


def calibrate_budget(q, k=None, v=None, params: IndexerParams = None, recall_target: float = 0.9,
                     taus: Sequence[float] = DEFAULT_TAUS, min_budget: int = 1,
                     max_budget: Optional[int] = None, cliff_weight: float = 0.25,
                     aggregate: str = "mean") -> Tuple[List[BudgetConfig], dict]:
    """Per KV head, grid over (tau_v, tau_s); then pick one grid point per head so that the
    total KV-tile count is minimal while the MEAN recall over heads reaches the target (the
    paper's accuracy target is an average; heads trade budget). Solved with a Lagrangian
    sweep: for multiplier lam each head minimises tiles - lam * recall, and lam is bisected
    to the cheapest feasible point. Returns one BudgetConfig per KV head (select_pattern
    accepts per-head budgets) and a summary. With several validation prompts each grid point
    is scored by the mean (aggregate="mean") or the worst case (most tiles, least recall) over
    them; the tile cost also weighs the next-higher grid neighbours by cliff_weight (below)."""
    prompts = [(q, k, v)] if torch.is_tensor(q) else list(q)  # one prompt or a list of them
    n, hq, d = prompts[0][0].shape
    hkv = prompts[0][1].shape[1]
    grp = hq // hkv
    grid = list(itertools.product(taus, taus))
    worst = {}  # (g, grid index) -> [tiles, recall]
    dense_tiles = 1
    for pq, pk, pv in prompts:
        _, lse_d = blockwise_attention(pq, pk, pv)
        a_v, a_s = indexer_forward(pk, pv, params)
        o = torch.empty_like(pq)
        lse = torch.empty_like(lse_d)
        for gi, (tv, ts) in enumerate(grid):
            pat = select_pattern(a_v, a_s, BudgetConfig(tv, ts, min_budget, max_budget))
            sparse_attention(pq, pk, pv, pat, validate=False, out=o, lse=lse)
            _, dense_tiles, per_head = sparse_tile_stats(n, hkv, pat.i_v.shape[1], pq.device, per_head=True)
            rec_q = attention_recall(lse, lse_d).view(hkv, grp).mean(dim=1).tolist()
            for g in range(hkv):
                w = worst.setdefault((g, gi), [0, 1.0, 0.0, 0.0, 0])
                w[0] = max(w[0], per_head[g])
                w[1] = min(w[1], rec_q[g])
                w[2] += per_head[g]
                w[3] += rec_q[g]
                w[4] += 1
    if aggregate == "mean":  # expected tiles and recall over the validation prompts
        for w in worst.values():
            w[0], w[1] = w[2] / w[4], w[3] / w[4]
    # Cliff-aware cost: a cumulative threshold just below a plateau of the score mass is
    # fragile — on another prompt the same tau can need thousands more indices. A grid point
    # is charged its expected tile count if, with probability cliff_weight per direction, the
    # prompt shifts the mass by one grid step (its next-higher neighbour's worst count).
    ti = {t: i for i, t in enumerate(taus)}
    gidx = {(tv, ts): gi for gi, (tv, ts) in enumerate(grid)}

    def cost(g, tv, ts):
        base = worst[(g, gidx[(tv, ts)])][0]
        if not cliff_weight:
            return base
        up_v = worst[(g, gidx[(taus[min(ti[tv] + 1, len(taus) - 1)], ts)])][0]
        up_s = worst[(g, gidx[(tv, taus[min(ti[ts] + 1, len(taus) - 1)])])][0]
        return base + cliff_weight * (max(up_v - base, 0) + max(up_s - base, 0))

    points = [[(cost(g, tv, ts), worst[(g, gi)][1], tv, ts) for gi, (tv, ts) in enumerate(grid)]
              for g in range(hkv)]

    def pick(lam):
        return [min(pts, key=lambda p: (p[0] - lam * p[1], -p[1])) for pts in points]

    def mean_recall(ch):
        return sum(c[1] for c in ch) / hkv

    hi = float(dense_tiles) * 1e3
    chosen = pick(hi)
    if mean_recall(chosen) >= recall_target:
        lo = 0.0
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            if mean_recall(pick(mid)) >= recall_target:
                hi = mid
            else:
                lo = mid
        chosen = pick(hi)
    else:  # unreachable target: the highest-recall point per head
        chosen = [max(pts, key=lambda p: (p[1], -p[0])) for pts in points]
    budgets = [BudgetConfig(c[2], c[3], min_budget, max_budget) for c in chosen]
    summary = dict(recall=sum(c[1] for c in chosen) / hkv,
                   tile_density=sum(worst[(g, gidx[(c[2], c[3])])][0] for g, c in enumerate(chosen)) / dense_tiles,
                   per_head=[dict(tau_v=c[2], tau_s=c[3], recall=round(c[1], 4)) for c in chosen])
    return budgets, summary
