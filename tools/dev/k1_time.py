"""K1 (indexer scoring) device time at 128k, 8 KV heads, d_h = 1024 (CUDA events, median of reps)."""
import os, sys, json, statistics
sys.path.insert(0, os.environ.get("VSP_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import torch
import paper_2603_04460_b200 as vsp
n, hkv = 131072, 8
g = torch.Generator().manual_seed(3)
k = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
v = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
params = vsp.make_indexer_params(hkv, 128, 1024, torch.Generator().manual_seed(4), head_sigma=0.3)
for _ in range(3):
    vsp.indexer_forward(k, v, params)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); vsp.indexer_forward(k, v, params); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"root": os.environ.get("VSP_ROOT", "."), "k1_plus_softmax_ms_median": statistics.median(ts), "min": min(ts)}))
