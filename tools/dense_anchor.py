"""Anchor the speed-up denominator: K4 (our dense causal kernel, vsp_dense_attn_fwd) against
the vendor/library dense causal attention kernels available in this image, on the same bf16
inputs (32 Q / 8 KV heads, d = 128) at n = 32k and 128k.

Each backend is tried independently (a missing or failing one is reported, not fatal); its
output is compared with K4's so every line is the same problem. Times are CUDA-event device
times of warm launches (median of `reps`). TFLOP/s uses the causal dense count
4 * d * n(n+1)/2 per Q head (the same algorithmic count bench.py uses).

Backends: torch SDPA (cuDNN / flash / efficient), flash_attn 2.8 (FA2), the FlashAttention-4
CuTe-DSL sm_100 kernel shipped in vllm.vllm_flash_attn.cute, and flashinfer's single prefill.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_04460_b200 as vsp  # noqa: E402


def ev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[32768, 131072])
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    hq, hkv, d = 32, 8, 128
    dev = torch.device("cuda:0")
    for n in args.n:
        g = torch.Generator(device=dev).manual_seed(n)
        q = torch.randn(n, hq, d, device=dev, generator=g).to(torch.bfloat16)
        k = torch.randn(n, hkv, d, device=dev, generator=g).to(torch.bfloat16)
        v = torch.randn(n, hkv, d, device=dev, generator=g).to(torch.bfloat16)
        flops = 4.0 * d * n * (n + 1) / 2 * hq
        o_ref = torch.empty_like(q)
        lse = torch.empty(hq, n, device=dev)
        scale = d ** -0.5

        def k4():
            vsp.blockwise_attention(q, k, v, out=o_ref, lse=lse)

        res = []

        def run(name, fn, get_out):
            try:
                ms = ev_time(fn, args.reps)
                out = get_out()
                diff = float((out.float() - o_ref.float()).abs().max())
                res.append({"backend": name, "ms": ms, "tflops": flops / (ms * 1e-3) / 1e12, "max_abs_diff_vs_k4": diff})
            except Exception as e:  # noqa: BLE001 — a backend that cannot run is reported, not fatal
                res.append({"backend": name, "error": f"{type(e).__name__}: {str(e)[:300]}"})
            torch.cuda.synchronize()

        run("ours K4 (attn_fwd_kernel<false>)", k4, lambda: o_ref)

        # torch SDPA wants [b, h, s, d]; GQA through enable_gqa
        qt, kt, vt = (x.permute(1, 0, 2).unsqueeze(0).contiguous() for x in (q, k, v))
        from torch.nn.attention import SDPBackend, sdpa_kernel
        box = {}
        for name, be in (("torch sdpa cuDNN", SDPBackend.CUDNN_ATTENTION), ("torch sdpa flash", SDPBackend.FLASH_ATTENTION),
                         ("torch sdpa efficient", SDPBackend.EFFICIENT_ATTENTION)):
            def f(be=be):
                with sdpa_kernel([be]):
                    box["o"] = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True, enable_gqa=True)
            run(name, f, lambda: box["o"][0].permute(1, 0, 2))
            box.clear()

        try:
            import flash_attn
            def fa2():
                box["o"] = flash_attn.flash_attn_func(q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0), causal=True)
            run("flash_attn 2.8 (FA2)", fa2, lambda: box["o"][0])
        except Exception as e:  # noqa: BLE001
            res.append({"backend": "flash_attn 2.8 (FA2)", "error": f"import: {e}"})
        box.clear()

        try:
            from vllm.vllm_flash_attn.cute.interface import flash_attn_func as fa4_func
            def fa4():
                r = fa4_func(q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0), causal=True, softmax_scale=scale)
                box["o"] = r[0] if isinstance(r, tuple) else r
            run("FlashAttention-4 CuTe sm100 (vllm_flash_attn.cute)", fa4, lambda: box["o"][0])
        except Exception as e:  # noqa: BLE001
            res.append({"backend": "FlashAttention-4 CuTe sm100 (vllm_flash_attn.cute)", "error": f"import: {str(e)[:300]}"})
        box.clear()

        try:
            import flashinfer
            for be in ("auto", "cutlass", "trtllm-gen", "fa2"):
                def fi(be=be):
                    box["o"] = flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True, sm_scale=scale, backend=be)
                run(f"flashinfer single_prefill backend={be}", fi, lambda: box["o"])
                box.clear()
        except Exception as e:  # noqa: BLE001
            res.append({"backend": "flashinfer", "error": f"import: {str(e)[:300]}"})
        print(json.dumps({"n": n, "hq": hq, "hkv": hkv, "d": d, "causal": True, "flops": flops,
                          "gpu": torch.cuda.get_device_name(0), "results": res}), flush=True)
        del q, k, v, qt, kt, vt, o_ref, lse
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
