"""One K4 launch and one K3 dense-switch launch on the C1 layer (for an ncu side-by-side)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2603_04460_b200 as vsp
from paper_2603_04460_b200.synth import planted_layer
n = 4096
q, k, v, _ = planted_layer(n, 32, 8, seed=1)
params = vsp.make_indexer_params(8, 128, 1024, torch.Generator().manual_seed(1), head_sigma=0.3)
a_v, a_s = vsp.indexer_forward(k, v, params)
pat = vsp.select_pattern(a_v, a_s, vsp.BudgetConfig(0.9, 0.9, 256, 256))
for _ in range(3):
    o, l = vsp.blockwise_attention(q, k, v)
    o2, l2 = vsp.sparse_attention(q, k, v, pat, validate=False, dense_switch=True)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("pair")
vsp.blockwise_attention(q, k, v, out=o, lse=l)
vsp.sparse_attention(q, k, v, pat, validate=False, out=o2, lse=l2, dense_switch=True)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
