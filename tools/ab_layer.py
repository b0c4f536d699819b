"""Alternating A/B of the unfused three-call layer and vsp_vs_prefill (one process, one call
per sample, strictly alternating so clock/power drift hits both arms equally).

    python tools/ab_layer.py [--pairs 40] [--hpc 0] [bench.py options]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.environ.get("VSP_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_04460_b200 as vsp  # noqa: E402


def main():
    pairs, hpc = 40, 0
    argv = sys.argv[1:]
    for key in ("--pairs", "--hpc"):
        if key in argv:
            i = argv.index(key)
            if key == "--pairs":
                pairs = int(argv[i + 1])
            else:
                hpc = int(argv[i + 1])
            del argv[i:i + 2]
    sys.argv = [sys.argv[0]] + argv
    args = bench.parse()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    params, budget, _ = bench.prepare_indexer(args, dev, 0, 1)
    q, k, v = bench.synth_layer(args, dev)
    o = torch.empty_like(q)
    lse = torch.empty(args.hq, args.n, device=dev)

    def unfused():
        a_v, a_s = vsp.indexer_forward(k, v, params)
        pat = vsp.select_pattern(a_v, a_s, budget)
        vsp.sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse)

    def fused():
        vsp.vs_prefill(q, k, v, params, budget, heads_per_chunk=hpc, out=o, lse=lse)

    def attn_only(pat):
        vsp.sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse)

    a_v, a_s = vsp.indexer_forward(k, v, params)
    pat = vsp.select_pattern(a_v, a_s, budget)
    arms = {"unfused": unfused, "fused": fused, "attn": lambda: attn_only(pat)}
    t = {name: [] for name in arms}
    for fn in arms.values():
        fn()
        fn()
    torch.cuda.synchronize()
    for _ in range(pairs):
        for name, fn in arms.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            t[name].append(a.elapsed_time(b))
    print(json.dumps({name: {"median": round(statistics.median(x), 4), "min": round(min(x), 4),
                             "mean": round(statistics.fmean(x), 4)} for name, x in t.items()}))


if __name__ == "__main__":
    main()
