"""Measurement of the SURVEY §8f kernels at the headline geometry (n = 131072, 32 Q / 8 KV heads,
d = 128, d_h = 1024) against their rooflines (MEASURED_PEAKS.json), CUDA events on the
launching stream, after warm-up, median of reps. One JSON line per kernel.

  * RoPE feed (`vsp_apply_rope`, rope.hpp:63-79): HBM-bound; algorithmic bytes = read + write of
    Q and K once = 2 * (|Q| + |K|) (out of place; in place the same bytes).
  * recall harness (`vsp_recall_from_lse`, attention.hpp:198-215): HBM-bound; bytes = the two
    fp32 LSE arrays [Hq, n].
  * distillation step (`vsp_indexer_loss_grad` + `vsp_adamw_step`, indexer.hpp:265-272, :347-363):
    tensor-bound; algorithmic FLOPs = forward GEMM + recomputed Y in the backward + dW_U =
    3 * 2 n (2d) d_h per KV head (the two-head epilogue and the KL terms are O(n d_h)).

Usage (GPU): python tools/f_rows_bench.py [--n 131072]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_04460_b200 as vsp  # noqa: E402
from paper_2603_04460_b200.distill import IndexerTrainer  # noqa: E402


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except OSError:  # B200_PROFILING.md fallback
        return {"hbm_gbs": 7700.0, "bf16_tflops": 2250.0, "bf16_tflops_sustained": 2250.0}, "nominal fallback"


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--d-h", type=int, default=1024)
    args = ap.parse_args()
    n, hq, hkv, d = args.n, args.hq, args.hkv, 128
    dev = torch.device("cuda", 0)
    pk, pk_src = peaks()
    hbm = pk["hbm_gbs"]
    tf = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    g = torch.Generator(device=dev).manual_seed(1)
    q = torch.randn(n, hq, d, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(n, hkv, d, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(n, hkv, d, device=dev, generator=g).to(torch.bfloat16)
    out = []

    # ---- RoPE feed: Q and K in one pass (out of place and in place; both styles)
    qo, ko = torch.empty_like(q), torch.empty_like(k)
    lib = vsp.load_library()
    ctx = vsp._context(dev)
    byts = 2 * (q.numel() + k.numel()) * 2
    for style in ("interleaved", "half_split"):
        cfg = vsp.RopeConfig(d, 10000.0, style)
        for inplace in (False, True):
            qa, ka = (q.clone(), k.clone()) if inplace else (q, k)
            dst_q, dst_k = (qa, ka) if inplace else (qo, ko)

            def rope():
                vsp._check(lib.vsp_apply_rope(ctx, vsp._ptr(qa), vsp._ptr(ka), vsp._ptr(dst_q), vsp._ptr(dst_k), n,
                                              hq, hkv, d, None, float(cfg.base),
                                              0 if style == "interleaved" else 1, vsp._stream(dev)))
            med, best = timed(rope)
            gbs = byts / (med * 1e-3) / 1e9
            out.append({"kernel": f"rope_{style}" + ("_inplace" if inplace else ""), "ms": med, "ms_min": best,
                        "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                     "algorithmic_bytes": byts}})
            del qa, ka

    # ---- recall harness (exact, from the two LSEs)
    ls = torch.randn(hq, n, device=dev) - 1.0
    ld = ls + torch.rand(hq, n, device=dev)
    med, best = timed(lambda: vsp.attention_recall(ls, ld))
    byts = 2 * hq * n * 4
    gbs = byts / (med * 1e-3) / 1e9
    out.append({"kernel": "recall_from_lse", "ms": med, "ms_min": best,
                "note": "includes the [Hq] result allocation of the Python call",
                "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                             "algorithmic_bytes": byts}})

    # ---- one distillation step of every KV head (loss + gradients, then AdamW)
    tr = IndexerTrainer(hkv, d, args.d_h, dev, seed=3)
    tv = torch.softmax(torch.randn(hkv, n, device=dev, generator=g), dim=1)
    ts_ = torch.softmax(torch.randn(hkv, n, device=dev, generator=g), dim=1)
    step_i = [0]

    def train_step():
        tr.loss_grad(k, v, tv, ts_)
        tr.adamw(step_i[0], 1e-3)
        step_i[0] += 1
    med, best = timed(train_step, reps=10)
    flops = 3 * 2.0 * n * (2 * d) * args.d_h * hkv
    tfs = flops / (med * 1e-3) / 1e12
    med_lg, _ = timed(lambda: tr.loss_grad(k, v, tv, ts_), reps=10)
    out.append({"kernel": "distill_step (loss_grad + adamw)", "ms": med, "ms_min": best, "loss_grad_ms": med_lg,
                "roofline": {"bound": "tensor", "achieved": tfs, "peak": tf, "unit": "TFLOP/s", "frac": tfs / tf,
                             "algorithmic_flops": flops}})
    for r in out:
        r.update({"n": n, "hq": hq, "hkv": hkv, "d": d, "d_h": args.d_h, "peak_source": pk_src})
        print(json.dumps(r))


if __name__ == "__main__":
    main()
