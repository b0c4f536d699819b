"""Device time of the bench's sparse attention call (plan + K3) for the package at VSP_ROOT,
on the bench's held-out layer and its selected pattern. The pattern is cached in a file so
that several builds can be timed in alternating processes on the same inputs:

    python tools/k3_ab.py --pattern gpurun_out/pat.pt [--reps 20]      # prints one JSON line
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
    argv = sys.argv[1:]
    opts = {"--pattern": "gpurun_out/pat.pt", "--reps": "20", "--dense": "0", "--layer": "0"}
    for key in list(opts):
        if key in argv:
            i = argv.index(key)
            opts[key] = argv[i + 1]
            del argv[i:i + 2]
    sys.argv = [sys.argv[0]] + argv
    args = bench.parse()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    path = opts["--pattern"]
    if not os.path.exists(path):
        params, budget, _ = bench.prepare_indexer(args, dev, 0, 1)
        _, k, v = (x.to(dev) for x in bench.synth_layer(args, "cpu"))
        a_v, a_s = vsp.indexer_forward(k, v, params)
        pat = vsp.select_pattern(a_v, a_s, budget)
        torch.save({f: getattr(pat, f).cpu() for f in ("i_v", "k_v", "i_s", "k_s")}, path)
        del k, v
    saved = torch.load(path)
    pat = vsp.SelectedIndices(*(saved[f].to(dev) for f in ("i_v", "k_v", "i_s", "k_s")))
    q, k, v = (x.to(dev) for x in bench.synth_layer(args, "cpu"))
    o = torch.empty_like(q)
    lse = torch.empty(args.hq, args.n, device=dev)
    k3 = opts["--layer"] == "1"
    if k3:  # the bench step (K1 -> K2 -> plan -> K3 in one call), K3 bracketed by CUDA events
        params, budget, _ = bench.prepare_indexer(args, dev, 0, 1)
        fn = lambda: vsp.vs_prefill(q, k, v, params, budget, out=o, lse=lse)  # noqa: E731
    elif opts["--dense"] == "1":
        fn = lambda: vsp.blockwise_attention(q, k, v, out=o, lse=lse)  # noqa: E731
    else:
        fn = lambda: vsp.sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse)  # noqa: E731
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if k3:
        vsp.attn_timing(True, dev)
    ts = []
    for _ in range(int(opts["--reps"])):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    rec = {"root": os.environ.get("VSP_ROOT", "."), "lib": vsp.lib_path, "median_ms": round(statistics.median(ts), 4),
           "min_ms": round(min(ts), 4)}
    if k3:
        k3_ms, k3_n = vsp.attn_timing_read(dev)
        rec["k3_ms"] = round(k3_ms / max(k3_n, 1), 4)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
