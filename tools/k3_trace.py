"""K3 pipeline timeline: clock64 stamps of CTA 0's events per tile (attn_fwd.cu, -DVSP_K3_TRACE).

    python tools/k3_trace.py --build                 # here: package copy in _exp_trace/ built with the probe
    python tools/k3_trace.py --pattern gpurun_out/pat.pt [--dense 1]   # on the GPU: prints a JSON summary

Events (per head w and global tile G): 0 MMA issues PV_w(G-1) second half + S_w(G); 1 K tile G
landed (MMA side); 2 softmax saw S_w(G); 3 softmax finished load/mask/max/rescale; 4 P first
half published; 5 P complete; 6 MMA saw the first half of P_w(G).
"""
import json
import os
import shutil
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TRACE_ROOT = os.path.join(ROOT, "_exp_trace")
TILES = 8192


def build():
    dst = os.path.join(TRACE_ROOT, "paper_2603_04460_b200")
    shutil.rmtree(TRACE_ROOT, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2603_04460_b200"), dst,
                    ignore=shutil.ignore_patterns("_objs", "*.so", "__pycache__"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(TRACE_ROOT, "include"))
    sys.path.insert(0, TRACE_ROOT)
    from paper_2603_04460_b200 import _build  # the copy
    _build.FLAGS.append("-DVSP_K3_TRACE")
    print(_build.build())


def main():
    argv = sys.argv[1:]
    if "--build" in argv:
        build()
        return
    opts = {"--pattern": "gpurun_out/pat.pt", "--dense": "0"}
    for key in list(opts):
        if key in argv:
            i = argv.index(key)
            opts[key] = argv[i + 1]
            del argv[i:i + 2]
    sys.argv = [sys.argv[0]] + argv
    sys.path.insert(0, TRACE_ROOT)
    sys.path.insert(1, ROOT)
    import ctypes
    import numpy as np
    import torch
    import bench
    import paper_2603_04460_b200 as vsp
    assert vsp.lib_path.startswith(TRACE_ROOT), vsp.lib_path
    args = bench.parse()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    saved = torch.load(opts["--pattern"])
    pat = vsp.SelectedIndices(*(saved[f].to(dev) for f in ("i_v", "k_v", "i_s", "k_s")))
    q, k, v = (x.to(dev) for x in bench.synth_layer(args, "cpu"))
    o = torch.empty_like(q)
    lse = torch.empty(args.hq, args.n, device=dev)
    if opts["--dense"] == "1":
        fn = lambda: vsp.blockwise_attention(q, k, v, out=o, lse=lse)  # noqa: E731
    else:
        fn = lambda: vsp.sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse)  # noqa: E731
    fn()
    fn()
    torch.cuda.synchronize()
    lib = vsp.load_library()
    buf = np.zeros(12 * 2 * TILES, dtype=np.uint64)
    lib.vsp_k3_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    rc = lib.vsp_k3_trace_read(buf.ctypes.data, buf.nbytes)
    assert rc == 0, rc
    ev = buf.reshape(12, 2, TILES).astype(np.int64)
    n_t = int(max(np.nonzero(ev[2, 0])[0].max(), 1))
    os.makedirs("gpurun_out", exist_ok=True)
    np.save("gpurun_out/k3_trace_%s.npy" % ("dense" if opts["--dense"] == "1" else "sparse"), ev[:, :, :n_t + 1])

    def med(xs):
        xs = [x for x in xs if 0 < x < 10**6]
        return round(float(statistics.median(xs)), 1) if xs else None

    G = range(2, n_t - 1)
    out = {"tiles_cta0": int(n_t), "mode": "dense" if opts["--dense"] == "1" else "sparse"}
    for w in (0, 1):
        out[f"w{w}"] = {
            "softmax_busy (S seen -> P full)": med([ev[5, w, g] - ev[2, w, g] for g in G]),
            "softmax_max (S seen -> max done)": med([ev[3, w, g] - ev[2, w, g] for g in G]),
            "exp_half1 (max done -> P half)": med([ev[4, w, g] - ev[3, w, g] for g in G]),
            "exp_half2 (P half -> P full)": med([ev[5, w, g] - ev[4, w, g] for g in G]),
            "softmax_idle (P full(G-1) -> S seen(G))": med([ev[2, w, g] - ev[5, w, g - 1] for g in G]),
            "S_latency (S issue -> S seen)": med([ev[2, w, g] - ev[0, w, g] for g in G]),
            "mma_sees_half_after_arrive": med([ev[6, w, g] - ev[4, w, g] for g in G]),
            "mma_issue_after_full_arrive": med([ev[0, w, g + 1] - ev[5, w, g] for g in G]),
        }
    out["tile_period (S_0 issue to S_0 issue)"] = med([ev[0, 0, g + 1] - ev[0, 0, g] for g in G])
    out["k_tile_ready_before_S0_issue"] = med([ev[0, 0, g] - ev[1, 0, g] for g in G])
    out["model_tensor_clk_per_tile (2 heads, SS S 8x96 + TS PV 8x71.5)"] = 2 * (8 * 96.3 + 8 * 71.5)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
