"""C2 (32k) calibration variants: held-out recall / tile density / speed-up per (aggregate, margin)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tools"))
import torch
import bench_configs as bc
from paper_2603_04460_b200 import calibrate
from paper_2603_04460_b200.synth import planted_layer

n = 32768
prompts = [planted_layer(n, 32, 8, seed=100 + i)[:3] for i in range(12)]
params, _ = calibrate.train_indexer(prompts, 1024, steps=900)
del prompts
vals = [planted_layer(n, 32, 8, seed=1100 + i)[:3] for i in range(6)]
q, k, v, _ = planted_layer(n, 32, 8, seed=2026)
for agg, margin in [("mean", 0.05), ("mean", 0.08), ("worst", 0.0), ("worst", 0.02), ("worst", 0.03)]:
    budget, pt = calibrate.calibrate_budget(vals, params=params, recall_target=0.9 + margin, aggregate=agg)
    r = bc.layer_stats(q, k, v, params, budget)
    print(json.dumps({"aggregate": agg, "margin": margin, "recall": r["recall"], "tile_density": r["tile_density"],
                      "speedup_vs_dense": r["speedup_vs_dense"], "tau": [[b.tau_v, b.tau_s] for b in budget]}))
