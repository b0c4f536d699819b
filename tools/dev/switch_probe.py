"""K3 in dense-switch mode vs K4 on identical tiles: is the gap per item or per tile?"""
import os, sys, json
sys.path.insert(0, os.environ.get("VSP_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import torch
import paper_2603_04460_b200 as vsp


def ev(fn, reps=20):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for n in [int(x) for x in os.environ.get("PROBE_N", "4096,16384,32768").split(",")]:
    hq, hkv = 32, 8
    g = torch.Generator().manual_seed(1)
    q = torch.randn(n, hq, 128, generator=g).to(torch.bfloat16).cuda()
    k = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    cap = n + 1
    # every offset 0..n-1 selected as slash: all blocks dense
    i_v = torch.zeros(hkv, cap, dtype=torch.int32, device="cuda")
    k_v = torch.zeros(hkv, dtype=torch.int32, device="cuda")
    i_s = torch.arange(cap, dtype=torch.int32, device="cuda").repeat(hkv, 1)
    k_s = torch.full((hkv,), n, dtype=torch.int32, device="cuda")
    pat = vsp.SelectedIndices(i_v, k_v, i_s, k_s)
    if os.environ.get("PROBE_RANDOM"):  # C1-like: 256 random verticals and offsets (0 included)
        gg = torch.Generator().manual_seed(7)
        iv = [torch.sort(torch.randperm(n, generator=gg)[:256]).values for _ in range(hkv)]
        is_ = [torch.sort(torch.cat([torch.zeros(1, dtype=torch.long), 1 + torch.randperm(n - 1, generator=gg)[:255]])).values for _ in range(hkv)]
        i_v = torch.zeros(hkv, cap, dtype=torch.int32); i_s = torch.zeros(hkv, cap, dtype=torch.int32)
        for h in range(hkv):
            i_v[h, :256] = iv[h].int(); i_s[h, :256] = is_[h].int()
        pat = vsp.SelectedIndices(i_v.cuda(), torch.full((hkv,), 256, dtype=torch.int32, device="cuda"),
                                  i_s.cuda(), torch.full((hkv,), 256, dtype=torch.int32, device="cuda"))
    o, l = vsp.blockwise_attention(q, k, v)
    sw = os.environ.get("VSP_ROOT") is None  # the base build may predate dense_switch
    o2, l2 = vsp.sparse_attention(q, k, v, pat, validate=False, **({"dense_switch": True} if sw else {}))
    torch.cuda.synchronize()
    same = bool(torch.equal(o, o2) and torch.equal(l, l2)) if not os.environ.get("PROBE_RANDOM") else None
    td = ev(lambda: vsp.blockwise_attention(q, k, v, out=o, lse=l))
    ts = ev(lambda: vsp.sparse_attention(q, k, v, pat, validate=False, out=o2, lse=l2, **({"dense_switch": True} if sw else {})))
    tm = ev(lambda: vsp.sparse_attention(q, k, v, pat, validate=False, out=o2, lse=l2))
    print(json.dumps({"n": n, "k4_ms": td, "switch_ms": ts, "masked_full_ms": tm, "switch_equals_k4": same,
                      "ratio": td / ts}), flush=True)
