"""K2 (selection) phase timeline: globaltimer stamps of every CTA's phase boundaries
(select.cu, -DVSP_SELECT_TRACE), on the bench layer's logits (config[2], 128k) and at C1 (4k).

    python tools/k2_trace.py --build     # here: package copy in _exp_k2trace/ built with the probe
    python tools/k2_trace.py             # on the GPU: prints per-phase medians (us) over CTAs

Events: 0 start, 1 slice loaded, 2 softmax done, 3/5/7/9 histogram pass p done, 4/6/8/10 scan
of pass p done, 11 before compaction, 12 compaction done, 13 final cluster sync done.
"""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TRACE_ROOT = os.environ.get("K2_TRACE_ROOT", os.path.join(ROOT, "_exp_k2trace"))
EV = 18


def build():
    dst = os.path.join(TRACE_ROOT, "paper_2603_04460_b200")
    shutil.rmtree(TRACE_ROOT, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2603_04460_b200"), dst,
                    ignore=shutil.ignore_patterns("_objs", "*.so", "__pycache__"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(TRACE_ROOT, "include"))
    sys.path.insert(0, TRACE_ROOT)
    from paper_2603_04460_b200 import _build  # the copy
    _build.FLAGS.append("-DVSP_SELECT_TRACE")
    for a in sys.argv[1:]:
        if a.startswith("-D"):
            _build.FLAGS.append(a)
    print(_build.build())


def run(n, budget_fn, label):
    import ctypes
    import numpy as np
    import torch
    import paper_2603_04460_b200 as vsp
    hkv = 8
    g = torch.Generator().manual_seed(3)
    k = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    params = vsp.make_indexer_params(hkv, 128, 1024, torch.Generator().manual_seed(4), head_sigma=0.3)
    a_v, a_s = vsp.indexer_forward(k, v, params)
    budget = budget_fn()
    # keep the clocks up: a second of dense GEMMs right before the traced calls (an idle B200
    # parks its SM clock far below max, and a 100 us kernel does not ramp it)
    x = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    import time
    t_end = time.time() + float(os.environ.get("K2_WARM_S", "0"))
    while time.time() < t_end:
        for _ in range(10):
            x @ x
        torch.cuda.synchronize()
    for _ in range(3):
        vsp.select_pattern(a_v, a_s, budget)
    torch.cuda.synchronize()
    buf = np.zeros(4096 * EV, dtype=np.uint64)
    lib = vsp.load_library()
    lib.vsp_k2_trace_read(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(buf.nbytes))
    ctas = 2 * hkv * int(os.environ.get("K2_CLUSTER", "8"))
    t = buf[: ctas * EV].reshape(ctas, EV).astype(np.int64)
    # phase events are SM clocks; 16/17 the globaltimer (ns) around the whole CTA
    mhz = float(np.median((t[:, 13] - t[:, 0]) / (t[:, 17] - t[:, 16]))) * 1e3
    t = np.concatenate([(t[:, :16] / (mhz / 1e3)).astype(np.int64), t[:, 16:]], axis=1)  # -> ns
    t0 = t[:, 16].min()
    out = {"config": label, "n": n}
    names = {1: "load", 2: "softmax", 3: "hist0", 4: "scan0", 5: "hist1", 6: "scan1", 7: "hist2", 8: "scan2",
             9: "hist3", 10: "scan3", 11: "pre_compact", 12: "compact", 13: "end"}
    prev = t[:, 0]
    for e in range(1, 14):
        col = t[:, e]
        if (col == 0).all():
            continue
        out[names[e]] = round(float(np.median(col - prev)) / 1e3, 2)
        prev = col
    # inside pass 0: 2 -> 14 element loop, 14 -> 15 slot merges, 15 -> 13 block sync (13 is
    # overwritten by the final cluster sync unless this is a probe build)
    out["p0_loop"] = round(float(np.median(t[:, 14] - t[:, 2])) / 1e3, 2)
    out["p0_merge"] = round(float(np.median(t[:, 15] - t[:, 14])) / 1e3, 2)
    out["total_us"] = round(float(np.median(t[:, 13] - t[:, 0])) / 1e3, 2)
    out["span_us"] = round(float(t[:, 17].max() - t0) / 1e3, 2)
    out["sm_mhz"] = round(mhz, 0)
    sc = np.zeros(4096 * 8, dtype=np.uint64)
    lib.vsp_k2_scan_read(ctypes.c_void_p(sc.ctypes.data), ctypes.c_size_t(sc.nbytes))
    sc = sc[: ctas * 8].reshape(ctas, 8).astype(np.int64)
    out["last_scan_cycles"] = [int(np.median(sc[:, e] - sc[:, e - 1])) for e in range(1, 6)]
    print(json.dumps(out))


def main():
    if "--build" in sys.argv:
        build()
        return
    sys.path.insert(0, TRACE_ROOT)
    import paper_2603_04460_b200 as vsp
    run(131072, lambda: vsp.BudgetConfig(0.3, 0.6, 1, None), "128k adaptive")
    run(4096, lambda: vsp.BudgetConfig(0.9, 0.9, 256, 256), "4k fixed top-k 256")


if __name__ == "__main__":
    main()
