"""Run the bench layer (config[2]) through vs_prefill a few times for the package at VSP_ROOT
(ncu target for kernel-level A/B of two builds on the same inputs)."""
import os, sys
sys.path.insert(0, os.environ.get("VSP_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2603_04460_b200 as vsp
args = bench.parse([])
dev = torch.device("cuda", 0)
params, budget, _ = bench.prepare_indexer(args, dev, 0, 1)
q, k, v = (x.to(dev) for x in bench.synth_layer(args, "cpu"))
o = torch.empty_like(q)
lse = torch.empty(args.hq, args.n, device=dev)
for _ in range(int(os.environ.get("REPS", "5"))):
    vsp.vs_prefill(q, k, v, params, budget, out=o, lse=lse)
torch.cuda.synchronize()
print("lib", vsp.lib_path)
