"""Interleaved A/B timing of the layer schedules on the bench workload (one process, same
clocks): unfused (three operator calls) vs vsp_vs_prefill with several chunk schedules.
Prints one JSON line with the median ms of each variant over R interleaved rounds.

    python tools/sched_sweep.py [--rounds 7] [--variants unfused,0,1,2,8]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_04460_b200 as vsp  # noqa: E402


def main():
    extra = {"--rounds": "7", "--variants": "unfused,0,1,2,8"}
    argv = sys.argv[1:]
    for key in list(extra):
        if key in argv:
            i = argv.index(key)
            extra[key] = argv[i + 1]
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

    fns = {}
    for name in extra["--variants"].split(","):
        if name == "unfused":
            fns[name] = unfused
        elif name == "units":  # vsp_vs_prefill_units over all heads: scoring, then one K3 launch per head
            o_h = torch.empty(args.hq, args.n, 128, dtype=q.dtype, device=dev)
            all_units = [(g, 0, (args.n + 127) // 128) for g in range(args.hkv)]
            fns[name] = lambda o_h=o_h, u=all_units: vsp.vs_prefill_units(q, k, v, params, budget, u, out=o_h, lse=lse)
        elif name == "attn":
            a_v, a_s = vsp.indexer_forward(k, v, params)
            pat = vsp.select_pattern(a_v, a_s, budget)
            fns[name] = lambda pat=pat: vsp.sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse)
        else:
            h = int(name)
            fns[name] = lambda h=h: vsp.vs_prefill(q, k, v, params, budget, heads_per_chunk=h, out=o, lse=lse)
    times = {name: [] for name in fns}
    for fn in fns.values():
        fn()
    torch.cuda.synchronize()
    for _ in range(int(extra["--rounds"])):
        for name, fn in fns.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                fn()
            b.record()
            torch.cuda.synchronize()
            times[name].append(a.elapsed_time(b) / 3)
    print(json.dumps({name: round(statistics.median(t), 4) for name, t in times.items()}))
    print(json.dumps({"min": {name: round(min(t), 4) for name, t in times.items()}}))


if __name__ == "__main__":
    main()
