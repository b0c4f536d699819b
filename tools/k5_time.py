"""Time K5 pass 2 alone (CUDA events) at a given n, 32Q/8KV."""
import os, sys, torch
sys.path.insert(0, os.environ.get("VSP_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2603_04460_b200 as vsp
from paper_2603_04460_b200.synth import planted_layer
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v, _ = planted_layer(n, 32, 8, seed=1)
_, lse = vsp.blockwise_attention(q, k, v)
res = vsp.aggregate_streaming(q, k, lse=lse)
torch.cuda.synchronize()
w = torch.arange(n, device=q.device, dtype=torch.float64)
fp = [float((r.double() * w).sum()) for r in (res if isinstance(res, (tuple, list)) else (res,))]
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    vsp.aggregate_streaming(q, k, lse=lse)
b.record()
torch.cuda.synchronize()
print(os.environ.get("VSP_K5_DEBUG", "0"), n, a.elapsed_time(b) / 3, "ms", "fingerprint", ["%.6e" % x for x in fp])
