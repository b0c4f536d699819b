"""Dump the bench's held-out vertical-slash pattern (i_v/i_s per KV head) and K3 tile counts
to gpurun_out/pattern_128k.npz for CPU-side analysis (tile census)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2603_04460_b200 as vsp  # noqa: E402


def main():
    args = bench.parse()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    params, budget, _ = bench.prepare_indexer(args, dev, 0, 1)
    q, k, v = (t.to(dev) for t in bench.synth_layer(args, "cpu"))  # the timed prompt, drawn as bench.py does
    a_v, a_s = vsp.indexer_forward(k, v, params)
    pat = vsp.select_pattern(a_v, a_s, budget)
    vsp.sparse_attention(q, k, v, pat, validate=False)
    tiles = vsp.sparse_tile_counts(args.n, args.hkv, pat.i_v.shape[1], dev)
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez_compressed("gpurun_out/pattern_128k.npz", i_v=pat.i_v.cpu().numpy(), k_v=pat.k_v.cpu().numpy(),
                        i_s=pat.i_s.cpu().numpy(), k_s=pat.k_s.cpu().numpy(), tiles=tiles.cpu().numpy())
    print("k_v", pat.k_v.tolist(), "k_s", pat.k_s.tolist(), "tiles", int(tiles.sum()))
    for g in range(args.hkv):
        print(g, sorted(pat.i_s[g, :int(pat.k_s[g])].tolist()))


if __name__ == "__main__":
    main()
