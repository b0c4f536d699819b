"""Minimal driver for ncu: runs the VS-prefill path (and K4 dense) a few times on a planted
layer with a fixed budget so each kernel can be captured by name."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_04460_b200 as vsp  # noqa: E402
from paper_2603_04460_b200.synth import planted_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--what", default="all", choices=["all", "dense", "sparse", "indexer", "select", "aggregate"])
ap.add_argument("--tau-v", type=float, default=0.3)
ap.add_argument("--tau-s", type=float, default=0.5)
args = ap.parse_args()
n = args.n
q, k, v, _ = planted_layer(n, 32, 8, seed=2026)
g = torch.Generator().manual_seed(1)
params = vsp.make_indexer_params(8, 128, 1024, g, head_sigma=0.3)
budget = vsp.BudgetConfig(args.tau_v, args.tau_s, 1, None)
for _ in range(args.iters):
    if args.what in ("all", "indexer", "select", "sparse"):
        a_v, a_s = vsp.indexer_forward(k, v, params)
    if args.what in ("all", "select", "sparse"):
        # ground-truth-like structured scores for a realistic sparse pattern
        _, lse = vsp.blockwise_attention(q, k, v) if args.what != "select" else (None, None)
        if lse is not None:
            a_v, a_s = vsp.aggregate_streaming(q, k, lse=lse)
        pat = vsp.select_pattern(a_v, a_s, budget)
    if args.what in ("all", "sparse"):
        vsp.sparse_attention(q, k, v, pat, validate=False)
    if args.what in ("all", "dense"):
        vsp.blockwise_attention(q, k, v)
    if args.what == "aggregate":
        _, lse = vsp.blockwise_attention(q, k, v)
        vsp.aggregate_streaming(q, k, lse=lse)
torch.cuda.synchronize()
print("done")
