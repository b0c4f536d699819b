"""Quick device timing of K4 dense / K3 sparse attention (CUDA events, warm, L2-flushed)."""
import argparse
import math
import os
import sys

sys.path.insert(0, os.environ.get("VSP_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch

import paper_2603_04460_b200 as vsp

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[4096, 32768, 131072])
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--iters", type=int, default=5)

args = ap.parse_args()

dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)


def timeit(fn):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(args.iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), sorted(ts)[len(ts) // 2]


for n in args.n:
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn(n, args.hq, 128, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(n, args.hkv, 128, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(n, args.hkv, 128, device=dev, generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(args.hq, n, device=dev)
    best, med = timeit(lambda: vsp.blockwise_attention(q, k, v, out=o, lse=lse))
    flops = 4 * 128 * args.hq * n * (n + 1) / 2
    print(f"dense n={n} hq={args.hq}: best {best:.3f} ms med {med:.3f} ms  "
          f"{flops / best / 1e9:.1f} TFLOP/s (causal alg)  tok/s {n / best * 1e3:.3e}")
