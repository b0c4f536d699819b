"""Explore planted-structure configs: ground truth (K5) -> oracle-indexer selection ->
recall / element density / tile density / speedup, all on the GPU."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_04460_b200 as vsp  # noqa: E402
from paper_2603_04460_b200.synth import PlantConfig, planted_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--cfg", type=str, default="{}")
ap.add_argument("--taus", type=str, default="[[0.3,0.3],[0.4,0.5],[0.5,0.6],[0.6,0.7],[0.7,0.8],[0.8,0.9],[0.9,0.9]]")
args = ap.parse_args()
cfg = PlantConfig(**json.loads(args.cfg))
n = args.n
q, k, v, plants = planted_layer(n, 32, 8, seed=1, cfg=cfg)
o_d, lse_d = vsp.blockwise_attention(q, k, v)
a_v, a_s = vsp.aggregate_streaming(q, k, lse=lse_d)
torch.cuda.synchronize()
anchor_mass = sum(float(a_v[g, torch.tensor(plants[g]["anchors"], device="cuda")].sum()) for g in range(8)) / 8
local = float(a_s[:, :256].sum(1).mean())
stripe = 0.0
for g in range(8):
    for o in plants[g]["stripes"]:
        stripe += float(a_s[g, max(0, o - 8):o + 9].sum())
stripe /= 8
print(f"cfg={cfg}\n n={n} anchor_mass(v)={anchor_mass:.3f} local<256(s)={local:.3f} stripes+-8(s)={stripe:.3f}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
vsp.blockwise_attention(q, k, v, out=o_d, lse=lse_d)
e1.record()
torch.cuda.synchronize()
dense_ms = e0.elapsed_time(e1)
for tv, ts in json.loads(args.taus):
    pat = vsp.select_pattern(a_v, a_s, vsp.BudgetConfig(tv, ts, 1, None))
    o, lse = vsp.sparse_attention(q, k, v, pat, validate=False)
    tiles, dense_tiles = vsp.sparse_tile_stats(n, 8, pat.i_v.shape[1], q.device)
    e0.record()
    vsp.sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rec = vsp.attention_recall(lse, lse_d).mean().item()
    print(f"  tau_v {tv:.2f} tau_s {ts:.2f}: k_v {pat.k_v.float().mean():8.1f} k_s {pat.k_s.float().mean():8.1f} "
          f"recall {rec:.4f} tile_density {tiles / dense_tiles:.4f} speedup {dense_ms / ms:6.2f}x")
