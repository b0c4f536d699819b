"""Distillation generalisation check: train on P prompts, calibrate tau on a validation
prompt, evaluate recall / tile density / speedup on a held-out prompt."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_04460_b200 as vsp  # noqa: E402
from paper_2603_04460_b200 import calibrate, distill  # noqa: E402
from paper_2603_04460_b200.synth import planted_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--prompts", type=int, nargs="+", default=[2, 6])
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--lr", type=float, default=3e-3)
ap.add_argument("--hkv", type=int, default=8)
args = ap.parse_args()
n, hq, hkv = args.n, 4 * args.hkv, args.hkv


def layer(seed):
    q, k, v, _ = planted_layer(n, hq, hkv, seed=seed)
    return q, k, v


val = layer(7)
test = layer(2026)
_, lse_d = vsp.blockwise_attention(*test)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
vsp.blockwise_attention(*test)
e1.record()
torch.cuda.synchronize()
dense_ms = e0.elapsed_time(e1)
gt_test = calibrate.ground_truth(*test)
for P in args.prompts:
    t0 = time.time()
    prompts = [layer(100 + i) for i in range(P)]
    params, losses = calibrate.train_indexer(prompts, 1024, steps=args.steps, lr_peak=args.lr)
    train_s = time.time() - t0
    kl = distill.eval_kl(params, test[1], test[2], gt_test[0], gt_test[1]).mean().item()
    budget, pt = calibrate.calibrate_budget(*val, params, 0.9)
    a_v, a_s = vsp.indexer_forward(test[1], test[2], params)
    pat = vsp.select_pattern(a_v, a_s, budget)
    o, lse = vsp.sparse_attention(*test, pat, validate=False)
    tiles, dt = vsp.sparse_tile_stats(n, hkv, pat.i_v.shape[1], test[0].device)
    e0.record()
    vsp.sparse_attention(*test, pat, validate=False, out=o, lse=lse)
    e1.record()
    torch.cuda.synchronize()
    rec = vsp.attention_recall(lse, lse_d).mean().item()
    print(f"P={P} steps={args.steps} train {train_s:.1f}s loss {losses[0]:.3f}->{losses[-1]:.3f} heldout KL {kl:.3f} | "
          f"val-calibrated tau={[(b.tau_v, b.tau_s) for b in budget]} val recall {pt['recall']:.3f} | TEST recall {rec:.4f} "
          f"tile density {tiles / dt:.4f} k_v {pat.k_v.float().mean():.0f} k_s {pat.k_s.float().mean():.0f} "
          f"speedup {dense_ms / e0.elapsed_time(e1):.2f}x")
    # oracle selection on ground truth for reference
    pat_gt = vsp.select_pattern(gt_test[0], gt_test[1], budget)
    vsp.sparse_attention(*test, pat_gt, validate=False, out=o, lse=lse)
    print(f"   (ground-truth scores at same tau: recall {vsp.attention_recall(lse, lse_d).mean().item():.4f})")
