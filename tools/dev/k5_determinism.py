"""Repeat K5 on the same inputs and report how the outputs differ (bit-reproducibility probe)."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.environ.get("VSP_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2603_04460_b200 as vsp  # noqa: E402
from paper_2603_04460_b200.synth import planted_layer  # noqa: E402


def h(t):
    return hashlib.sha1(t.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:10]


n = int(sys.argv[1])
q, k, v, _ = planted_layer(n, 32, 8, seed=5)
_, lse = vsp.blockwise_attention(q, k, v)
outs = []
for i in range(3):
    a_v, a_s = vsp.aggregate_streaming(q, k, lse=lse)
    torch.cuda.synchronize()
    outs.append((a_v.clone(), a_s.clone()))
    print(i, h(a_v), h(a_s), "zeros", int((a_s == 0).sum()), "sum", float(a_s.double().sum()), flush=True)
for i in (1, 2):
    d = outs[0][1] != outs[i][1]
    idx = d.nonzero()
    print("run", i, "differs at", int(d.sum()), "entries; heads", sorted(set(idx[:, 0].tolist()))[:8],
          "first offsets", idx[:8, 1].tolist())
