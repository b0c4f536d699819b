"""Slash offsets and tile classes of the bench's held-out pattern (config[2])."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2603_04460_b200 as vsp
args = bench.parse([])
dev = torch.device("cuda", 0)
params, budget, _ = bench.prepare_indexer(args, dev, 0, 1)
q, k, v = (x.to(dev) for x in bench.synth_layer(args, "cpu"))
o, lse, pat = vsp.vs_prefill(q, k, v, params, budget)
torch.cuda.synchronize()
out = {}
for g in range(args.hkv):
    iv, is_ = pat.lists(g)
    out[g] = {"k_v": len(iv), "k_s": len(is_), "offsets": is_[:40]}
vsp.sparse_attention(q, k, v, pat, validate=False)
tiles, dense, per_head = vsp.sparse_tile_stats(args.n, args.hkv, pat.i_v.shape[1], dev, per_head=True)
counts = vsp.sparse_tile_counts(args.n, args.hkv, pat.i_v.shape[1], dev).cpu()
for g in range(args.hkv):
    iv, is_ = pat.lists(g)
    nq = counts.shape[1]
    vt = sum(( (sum(1 for j in iv if j <= min(qb*128+127, args.n-1)) + 127) // 128) for qb in range(0, nq, 64)) * 64
    out[g]["tiles"] = int(per_head[g]); out[g]["approx_vertical_tiles"] = int(vt)
print(json.dumps({"tiles": tiles, "dense": dense, "heads": out}))
