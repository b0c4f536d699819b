"""Per-rank step times of the two multi-GPU splits of the 128k layer, measured on ONE B200.

Each rank of an N-GPU job runs independent work (no collective on the data path), so the
N-GPU step time is the max over ranks of that rank's own step. This tool times every rank's
share on the single GPU (CUDA events, warm, same clocks) for N = 1, 2, 4, 8 and reports the
predicted step (max over ranks) and tokens/s for
  heads    : KV-head sharding (each rank vs_prefill on Hkv/N heads, the north-star split)
  balanced : cost-balanced (KV head, query-block) units (vs_prefill_units, replicated inputs)
  spread   : every head's query blocks split evenly by cost across the ranks (vs_prefill_units)
The cost table of the balanced split comes from a separate validation prompt (not the timed
one). Prints one JSON line.

    python tools/scaling_sim.py [--cost-prompts K] [--cta-overhead C] [--head-overhead H] [bench.py options]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_04460_b200 as vsp  # noqa: E402
from paper_2603_04460_b200 import parallel  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    argv = sys.argv[1:]
    opts = {"--cost-prompts": "1", "--cta-overhead": "2.0", "--head-overhead": "2500"}
    for key in list(opts):
        if key in argv:
            i = argv.index(key)
            opts[key] = argv[i + 1]
            del argv[i:i + 2]
    sys.argv = [sys.argv[0]] + argv
    args = bench.parse()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    params, budget, _ = bench.prepare_indexer(args, dev, 0, 1)
    n, hq, hkv = args.n, args.hq, args.hkv
    # cost table: mean tile counts of the first K validation prompts (K = --cost-prompts)
    tables = []
    for i in range(int(opts["--cost-prompts"])):
        qv, kv_, vv = bench.synth_layer(args, dev, seed=args.seed + 201 + i)
        a_v, a_s = vsp.indexer_forward(kv_, vv, params)
        pat = vsp.select_pattern(a_v, a_s, budget)
        vsp.sparse_attention(qv, kv_, vv, pat, validate=False)
        tables.append(vsp.sparse_tile_counts(n, hkv, pat.i_v.shape[1], dev).double())
        del qv, kv_, vv
    cost = sum(tables) / len(tables)
    q, k, v = bench.synth_layer(args, dev)
    o_full = torch.empty(hq, n, 128, dtype=q.dtype, device=dev)
    lse_full = torch.empty(hq, n, device=dev)
    # the held-out prompt's own table (what the split should have predicted)
    a_v, a_s = vsp.indexer_forward(k, v, params)
    pat_h = vsp.select_pattern(a_v, a_s, budget)
    vsp.sparse_attention(q, k, v, pat_h, validate=False)
    held = vsp.sparse_tile_counts(n, hkv, pat_h.i_v.shape[1], dev)
    out = {"n": n, "hq": hq, "hkv": hkv, "cost_prompts": len(tables),
           "cta_overhead": float(opts["--cta-overhead"]), "head_overhead": float(opts["--head-overhead"]),
           "tiles_per_head_prompts": [t.sum(1).tolist() for t in tables],
           "tiles_per_head_heldout": held.sum(1).tolist(), "splits": {}}
    for world in (1, 2, 4, 8):
        # heads: rank r = vs_prefill on its KV heads
        t_heads = []
        for r in range(world):
            qs, ks, vs = (parallel.shard_heads(t, r, world) for t in (q, k, v))
            ps = vsp.IndexerParams(*(parallel.shard_heads(t, r, world, dim=0)
                                     for t in (params.w_u, params.b_u, params.w_v, params.b_v, params.w_s, params.b_s)))
            bs = budget[r * hkv // world:(r + 1) * hkv // world]
            slab, lslab = parallel.head_slab(o_full, r, world), parallel.head_slab(lse_full, r, world)
            t_heads.append(timed(lambda: vsp.vs_prefill(qs, ks, vs, ps, bs, out=slab, lse=lslab, head_major=True)))
            del qs, ks, vs
        # heads_cost: whole KV heads placed by the predicted cost (what bench.py --head-placement cost does)
        hsets = parallel.balanced_head_sets(cost.sum(1) + float(opts["--head-overhead"]), world)
        grp = hq // hkv
        t_hc = []
        for hs in hsets:
            kvi = torch.tensor(hs, device=dev)
            qi = torch.tensor(parallel.q_heads_of(hs, grp), device=dev)
            qs, ks, vs = q.index_select(1, qi), k.index_select(1, kvi), v.index_select(1, kvi)
            ps = vsp.IndexerParams(*(t.index_select(0, kvi)
                                     for t in (params.w_u, params.b_u, params.w_v, params.b_v, params.w_s, params.b_s)))
            bs = [budget[g] for g in hs]
            o_r = torch.empty(len(qi), n, 128, dtype=q.dtype, device=dev)
            l_r = torch.empty(len(qi), n, device=dev)
            t_hc.append(timed(lambda: vsp.vs_prefill(qs, ks, vs, ps, bs, out=o_r, lse=l_r, head_major=True)))
            del qs, ks, vs, o_r, l_r
        # balanced: rank r = vs_prefill_units on its units (full inputs)
        units = parallel.balanced_units(cost, world, cta_overhead=float(opts["--cta-overhead"]),
                                        head_overhead=float(opts["--head-overhead"]))
        t_bal = [timed(lambda u=u: vsp.vs_prefill_units(q, k, v, params, budget, u, out=o_full, lse=lse_full))
                 for u in units]
        # spread: every head's query blocks split across the ranks (every rank scores every head)
        sunits = parallel.spread_units(cost, world, cta_overhead=float(opts["--cta-overhead"]))
        t_spr = [timed(lambda u=u: vsp.vs_prefill_units(q, k, v, params, budget, u, out=o_full, lse=lse_full))
                 for u in sunits]
        out["splits"][world] = {
            "spread_ms_per_rank": [round(x, 3) for x in t_spr], "spread_step_ms": round(max(t_spr), 3),
            "spread_tok_s": n / (max(t_spr) * 1e-3),
            "heads_ms_per_rank": [round(x, 3) for x in t_heads], "heads_step_ms": round(max(t_heads), 3),
            "heads_cost_ms_per_rank": [round(x, 3) for x in t_hc], "heads_cost_step_ms": round(max(t_hc), 3),
            "heads_cost_sets": hsets,
            "heads_tok_s": n / (max(t_heads) * 1e-3),
            "balanced_ms_per_rank": [round(x, 3) for x in t_bal], "balanced_step_ms": round(max(t_bal), 3),
            "balanced_tok_s": n / (max(t_bal) * 1e-3), "balanced_units": units}
    base_h = out["splits"][1]["heads_step_ms"]
    for world, s in out["splits"].items():
        s["heads_speedup"] = round(base_h / s["heads_step_ms"], 2)
        s["heads_cost_speedup"] = round(base_h / s["heads_cost_step_ms"], 2)
        s["balanced_speedup"] = round(base_h / s["balanced_step_ms"], 2)
        s["spread_speedup"] = round(base_h / s["spread_step_ms"], 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
