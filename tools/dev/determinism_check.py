"""Bit-reproducibility probe of the preparation chain (ground truth -> distillation step ->
indexer scores): prints checksums; run it in two processes and compare the lines."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_04460_b200 as vsp  # noqa: E402
from paper_2603_04460_b200 import calibrate, distill  # noqa: E402
from paper_2603_04460_b200.synth import planted_layer  # noqa: E402


def h(t):
    return hashlib.sha1(t.detach().contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:12]


n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q, k, v, _ = planted_layer(n, 32, 8, seed=5)
print("inputs", h(q), h(k), h(v))
_, lse = vsp.blockwise_attention(q, k, v)
print("lse", h(lse))
tv, ts, _ = calibrate.ground_truth(q, k, v)
print("targets", h(tv), h(ts))
tr = distill.IndexerTrainer(8, 128, 1024, "cuda", seed=1)
print("init", h(tr.flat))
loss = tr.loss_grad(k, v, tv, ts)
print("loss", h(loss), "grads", h(tr.grads))
tr.adamw(0, 1e-3)
a_v, a_s = vsp.indexer_forward(k, v, tr.params())
print("scores", h(a_v), h(a_s))
