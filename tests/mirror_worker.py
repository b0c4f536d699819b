"""One rank of the mirrored-output KV-head split (tests/test_gpu_mirrors.py launches two on
one GPU): the full-layer output buffers are CUDA-IPC allocations, each rank's attention
epilogue stores its Q-head slab into its own buffer and into the other rank's (mapped with
vsp_ipc_open), then a barrier; the assembled buffer must equal the one-process layer bit for
bit. Exit code 0 = match."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_04460_b200 as vsp  # noqa: E402
from paper_2603_04460_b200 import parallel  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n, hq, hkv = int(os.environ.get("MIRROR_N", "1536")), 8, 4
    g = torch.Generator(device="cpu").manual_seed(5)
    q = (torch.randn(n, hq, 128, generator=g) * 0.7).to(torch.bfloat16).to(dev)
    k = (torch.randn(n, hkv, 128, generator=g) * 0.7).to(torch.bfloat16).to(dev)
    v = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).to(dev)
    params = vsp.make_indexer_params(hkv, 128, 256, torch.Generator().manual_seed(9), head_sigma=0.5)
    budget = vsp.BudgetConfig(0.6, 0.7, 1, None)
    o_ref, l_ref, _ = vsp.vs_prefill(q, k, v, params, budget, head_major=True)

    obytes, lbytes = hq * n * 128 * 2, hq * n * 4
    mine = [vsp.IpcBuffer(obytes, dev), vsp.IpcBuffer(lbytes, dev)]
    handles = [None] * world
    dist.all_gather_object(handles, [mine[0].handle, mine[1].handle])
    peers = [(vsp.IpcBuffer.open(h[0], obytes, dev), vsp.IpcBuffer.open(h[1], lbytes, dev))
             for r, h in enumerate(handles) if r != rank]
    lo, hi = parallel.head_range(hkv, rank, world)
    qlo, qhi = lo * (hq // hkv), hi * (hq // hkv)
    slab_o, slab_l = qlo * n * 128 * 2, qlo * n * 4
    o_full, l_full = mine[0].tensor(torch.bfloat16, (hq, n, 128)), mine[1].tensor(torch.float32, (hq, n))
    o_full.zero_()
    l_full.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    sub = vsp.IndexerParams(*(t[lo:hi] for t in (params.w_u, params.b_u, params.w_v, params.b_v, params.w_s,
                                                   params.b_s)))
    vsp.vs_prefill(q[:, qlo:qhi].contiguous(), k[:, lo:hi].contiguous(), v[:, lo:hi].contiguous(), sub, budget,
                   out=o_full[qlo:qhi], lse=l_full[qlo:qhi], head_major=True,
                   mirrors=[(po.ptr + slab_o, pl.ptr + slab_l) for po, pl in peers])
    torch.cuda.synchronize()
    dist.barrier()  # every rank's mirrored stores have landed
    ok = torch.equal(o_full, o_ref) and torch.equal(l_full, l_ref)
    print(f"rank {rank}: assembled == one-process layer: {ok}", flush=True)
    for po, pl in peers:
        po.close()
        pl.close()
    dist.barrier()
    for b in mine:
        b.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
