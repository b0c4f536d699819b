#!/usr/bin/env python
"""bench.py — VS-prefill hot path on B200 (BASELINE.json config[2]).

One step = one layer of the VS-prefill path on this rank's KV heads:
    K1 indexer scores -> K2 adaptive selection -> K3 fused VS sparse attention
at LLaMA-3.1-8B attention geometry (32 Q / 8 KV heads, d=128), n = 131072, synthetic
planted-structure Q/K/V (paper_2603_04460_b200/synth.py, drawn on the CPU so every process
sees the same bits), inputs resident in HBM (Q alone is 1.07 GB > the 126 MB L2, so no
flush is needed between steps).

The indexer parameters and per-head budgets come from bench_data/ (written by
`python bench.py --prep fresh --save-prep`: KL distillation of the VSIndexer on 12 training
prompts and budget calibration on 6 validation prompts, on the GPU). Both arms load the same
file, so they run the same layer with the same indexer and budgets.

Multi-GPU (torchrun, one rank per GPU): KV heads are sharded 8/N per rank with no
collective on the data path; value = n / max-over-ranks step time
(strong scaling: the layer is fixed, heads split). The NCCL all-gather that assembles O is
timed separately (`allgather_ms`). `--shard balanced|spread` split (KV head, query block)
units instead; their assembly (vsp_assemble_units, NCCL broadcasts) is timed the same way.

`--impl reference` runs the reference's own CPU implementation (oracle/_ref: the unmodified
reference headers) on a bounded sample of the same layer, in a CPU-only process (no CUDA,
no libvsp_gpu.so): its own full-length indexer scoring and selection once (measured), then
per step select_pattern on all n and sparse_attention on rows [0, 4096) and [0, 8192),
extrapolated to the layer (ReferenceLayer).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# A/B hook: VSP_ROOT=<dir> benches the package copy under <dir> (same inputs, same process setup)
if os.environ.get("VSP_ROOT"):
    sys.path.insert(0, os.path.abspath(os.environ["VSP_ROOT"]))
if ROOT not in sys.path:  # tools may put another build of the package ahead (A/B)
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "prefill attn tokens/s @128k LLaMA-8B geom, 1/2/4/8 B200; speedup vs own dense"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
PREP_DIR = os.path.join(ROOT, "bench_data")
# bump when synth.py / the preparation recipe changes what a given seed produces
SYNTH_TAG = "planted-v1 (synth.py PlantConfig defaults); timed prompt drawn on the CPU"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--d-h", type=int, default=1024)
    ap.add_argument("--indexer", choices=["distilled", "random"], default="distilled")
    ap.add_argument("--prep", choices=["auto", "load", "fresh"], default="auto",
                    help="indexer + budgets: load bench_data/ (auto: when it matches these flags, else "
                         "prepare on the GPU), or prepare fresh")
    ap.add_argument("--save-prep", action="store_true", help="write the fresh preparation to bench_data/")
    ap.add_argument("--train-prompts", type=int, default=12)
    ap.add_argument("--val-prompts", type=int, default=6)
    ap.add_argument("--calib-aggregate", choices=["mean", "worst"], default="mean",
                    help="score calibration grid points by the mean or the worst case over validation prompts")
    ap.add_argument("--distill-steps", type=int, default=900)
    ap.add_argument("--recall-target", type=float, default=0.9)
    ap.add_argument("--calib-margin", type=float, default=0.035,
                    help="calibrate the budget for recall_target + margin on the validation prompts")
    ap.add_argument("--tau-step", type=float, default=0.1,
                    help="grid step of the per-head (tau_v, tau_s) calibration over (0, 1)")
    ap.add_argument("--tau-v", type=float, default=None, help="fix tau_v (skips calibration)")
    ap.add_argument("--tau-s", type=float, default=None)
    ap.add_argument("--min-budget", type=int, default=1)
    ap.add_argument("--max-budget", type=int, default=-1)
    ap.add_argument("--head-sigma", type=float, default=0.3, help="random indexer head scale")
    ap.add_argument("--seed", type=int, default=2026)
    ap.add_argument("--ref-rows", type=int, default=8192,
                    help="reference sample: sparse_attention row prefixes rows/2 and rows per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard", choices=["auto", "heads", "balanced", "spread"], default="auto",
                    help="multi-GPU split: KV heads (north star; auto), or cost-balanced (KV head, query-block) "
                         "units with replicated inputs, or spread (every head split across the ranks)")
    ap.add_argument("--head-placement", choices=["cost", "contiguous"], default="cost",
                    help="heads split at N>1: whole KV heads placed by predicted cost (default) or contiguous slabs")
    ap.add_argument("--assemble", choices=["nccl", "mirror"], default="nccl",
                    help="heads split at N>1: assemble O with an NCCL all-gather after the layer (timed "
                         "separately), or inside K3 — every rank's epilogue also stores its slab into the other "
                         "ranks' outputs (CUDA IPC over NVLink; vsp_vs_prefill_mirrored) — inside the timed step")
    ap.add_argument("--heads-per-chunk", type=int, default=0,
                    help="KV heads per pipeline chunk of vsp_vs_prefill (indexer/select of chunk c+1 overlap attention of c)")
    ap.add_argument("--e2e-heads-per-chunk", type=int, default=0)
    return ap.parse_args(argv)


# --------------------------------------------------------------------------- helpers

def k3_traffic():
    """DRAM bytes (read + write) per K3 launch from the committed `ncu --set full` capture of
    this bench's timed region (profiles/k3_traffic.json, written by tools/k3_traffic.py), or None."""
    path = os.path.join(ROOT, "profiles", "k3_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)["bytes_per_launch"]
    except Exception:
        return None


def peaks():
    try:
        with open(PEAKS) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML every 2 ms (the
    timed region of a default run is only tens of milliseconds), nvidia-smi as a fallback."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # [sm_mhz, max_mhz, reason flags...]
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._nvml = (pynvml, h, bits, mx)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            pynvml, h, bits, mx = self._nvml
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append([float(sm), float(mx)] + [bool(r & b) for b in bits])
            return
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            f = [x.strip() for x in out.stdout.strip().split(",")]
            if f[0].replace(".", "").isdigit() and f[1].replace(".", "").isdigit():
                self.rows.append([float(f[0]), float(f[1])] + [x == "Active" for x in f[2:6]])

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(0.002 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows),
                "sm_min_mhz": min(sm), "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def pairs_prefix(iv: np.ndarray, is_: np.ndarray, rows: int) -> int:
    """Covered causal pairs (i, j), i < rows, of one KV head's pattern (ascending lists):
    sum_v (rows - v) + sum_o (rows - o) - #{(v, o): v + o < rows} (vertical/slash overlap)."""
    iv = np.asarray(iv, np.int64)
    is_ = np.asarray(is_, np.int64)
    iv = iv[iv < rows]
    is_ = is_[is_ < rows]
    a = int((rows - iv).sum()) + int((rows - is_).sum())
    ov = int(np.searchsorted(is_, rows - 1 - iv, side="right").sum()) if len(iv) else 0
    return a - ov


def covered_pairs(pat, n: int, hkv: int) -> np.ndarray:
    """Exact covered (i, j) pairs per KV head of a (device) VS pattern."""
    return np.array([pairs_prefix(*pat.lists(g), n) for g in range(hkv)], np.int64)


def synth_layer(args, device, seed=None, gen_device=None):
    """One prompt of the planted layer, all heads. The timed prompt (seed = args.seed) is
    drawn with gen_device="cpu" in both arms, so they attend the identical layer."""
    from paper_2603_04460_b200.synth import planted_layer
    q, k, v, _ = planted_layer(args.n, args.hq, args.hkv, seed=args.seed if seed is None else seed, device=device,
                               gen_device=gen_device)
    return q, k, v


def shard(x, r, world, dim):
    size = x.shape[dim] // world
    return x.narrow(dim, r * size, size).contiguous()


# --------------------------------------------------------------------------- preparation

PREP_KEYS = ("n", "hq", "hkv", "d_h", "seed", "indexer", "train_prompts", "val_prompts", "distill_steps",
             "recall_target", "calib_margin", "tau_step", "calib_aggregate", "min_budget", "max_budget",
             "head_sigma", "tau_v", "tau_s")


def prep_key(args) -> dict:
    key = {k: getattr(args, k) for k in PREP_KEYS}
    key["synth"] = SYNTH_TAG
    return key


def prep_path(args) -> str:
    return os.path.join(PREP_DIR, f"prep_{args.indexer}_n{args.n}_h{args.hq}x{args.hkv}_dh{args.d_h}.npz")


def save_prep(args, params, budgets, info) -> str:
    """bf16 W_U as its raw 16-bit patterns, the fp32 rest, per-head (tau_v, tau_s), and the
    preparation's provenance; ~3.5 MB compressed for the bench config."""
    os.makedirs(PREP_DIR, exist_ok=True)
    path = prep_path(args)
    meta = {"key": prep_key(args), "info": info}
    np.savez_compressed(path, w_u=params.w_u.contiguous().view(torch.int16).cpu().numpy(),
                        b_u=params.b_u.float().cpu().numpy(), w_v=params.w_v.float().cpu().numpy(),
                        b_v=params.b_v.float().cpu().numpy(), w_s=params.w_s.float().cpu().numpy(),
                        b_s=params.b_s.float().cpu().numpy(),
                        tau=np.array([[t[0], t[1]] for t in budgets], np.float64), meta=json.dumps(meta))
    return path


def load_prep(args):
    """-> (numpy params with W_U as f32 [hkv, 2d, d_h], [(tau_v, tau_s)] per KV head, info) or
    None when bench_data/ holds no preparation made with these flags."""
    path = prep_path(args)
    if not os.path.exists(path):
        return None
    z = np.load(path, allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    if meta["key"] != prep_key(args):
        return None
    w_u = (z["w_u"].astype(np.int32).astype(np.uint32) << 16).view(np.float32)  # bf16 bits -> f32
    prm = dict(w_u=w_u, b_u=z["b_u"], w_v=z["w_v"], b_v=z["b_v"], w_s=z["w_s"], b_s=z["b_s"])
    budgets = [(float(a), float(b)) for a, b in z["tau"]]
    info = dict(meta["info"])
    info["prep_file"] = os.path.relpath(path, ROOT)
    return prm, budgets, info


def params_to_device(prm: dict, dev):
    import paper_2603_04460_b200 as vsp
    t = {k: torch.from_numpy(np.ascontiguousarray(x)) for k, x in prm.items()}
    return vsp.IndexerParams(t["w_u"].to(torch.bfloat16).to(dev), t["b_u"].float().to(dev), t["w_v"].float().to(dev),
                             t["b_v"].float().to(dev), t["w_s"].float().to(dev), t["b_s"].float().to(dev))


def params_to_numpy(params) -> dict:
    return {f: getattr(params, f).float().cpu().numpy() for f in ("w_u", "b_u", "w_v", "b_v", "w_s", "b_s")}


def random_params(args):
    """The reference's make_indexer_params with N(0, head_sigma^2) heads, on the CPU."""
    import paper_2603_04460_b200 as vsp  # pure torch here: the library is not loaded
    g = torch.Generator().manual_seed(args.seed + 7)
    return vsp.make_indexer_params(args.hkv, 128, args.d_h, g, head_sigma=args.head_sigma, device="cpu")


def prepare_gpu(args, device):
    """Indexer parameters and per-head budgets of every KV head, prepared on the GPU.
    distilled: KL distillation on `train_prompts` other prompts of the same heads (K5 ground
    truth); budgets calibrated on `val_prompts` further prompts to reach recall_target +
    calib_margin. random: make_indexer_params with N(0, head_sigma^2) heads. The timed prompt
    is never seen. Returns (params on device, [(tau_v, tau_s)], info)."""
    import paper_2603_04460_b200 as vsp
    from paper_2603_04460_b200 import calibrate
    info = {}
    t0 = time.time()
    if args.indexer == "random":
        params = params_to_device(params_to_numpy(random_params(args)), device)
        info["indexer"] = f"random-init VSIndexer (make_indexer_params), heads ~ N(0, {args.head_sigma}^2)"
    else:
        prompts = [synth_layer(args, device, seed=args.seed + 101 + i) for i in range(args.train_prompts)]
        tstats = {}
        params, losses = calibrate.train_indexer(prompts, args.d_h, steps=args.distill_steps, stats=tstats)
        del prompts
        info["indexer"] = (f"VSIndexer distilled on GPU (KL to K5 ground truth, AdamW, {args.distill_steps} steps; "
                           f"sm_100a loss/backward/AdamW kernels) on {args.train_prompts} training prompts of the "
                           f"same heads; held-out prompt timed")
        info["distill_loss_first_last"] = [x for x in losses if x == x][:1] + [losses[-1]]
        info["distill_step_ms"] = round(tstats.get("step_ms", float("nan")), 3)
        info["ground_truth_ms_per_prompt"] = round(tstats.get("ground_truth_ms", float("nan")), 2)
    if args.tau_v is not None and args.tau_s is not None:
        budgets = [(args.tau_v, args.tau_s)] * args.hkv
        info["budget_source"] = "fixed by flags"
    else:
        vals = [synth_layer(args, device, seed=args.seed + 201 + i) for i in range(args.val_prompts)]
        taus = tuple(round(args.tau_step * i, 4) for i in range(1, int(round(1 / args.tau_step))))
        bl, pt = calibrate.calibrate_budget(vals, params=params, taus=taus, aggregate=args.calib_aggregate,
                                            recall_target=args.recall_target + args.calib_margin,
                                            min_budget=args.min_budget,
                                            max_budget=None if args.max_budget < 0 else args.max_budget)
        budgets = [(b.tau_v, b.tau_s) for b in bl]
        info["budget_source"] = (f"per-KV-head (tau_v, tau_s) on a {args.tau_step} grid, calibrated on "
                                 f"{args.val_prompts} validation prompts "
                                 f"({args.calib_aggregate}, cliff-weighted tiles) for mean recall >= "
                                 f"{args.recall_target} + {args.calib_margin}: "
                                 f"recall {pt['recall']:.4f}, tile density {pt['tile_density']:.4f}")
        del vals
    info["prep_s"] = round(time.time() - t0, 1)
    return params, budgets, info


def obtain_prep(args, device):
    """(params on device, [(tau_v, tau_s)] per KV head, info): bench_data/ when it matches the
    flags (--prep auto|load), else prepared on the GPU (--prep auto|fresh)."""
    if args.prep != "fresh":
        got = load_prep(args)
        if got is not None:
            prm, budgets, info = got
            return params_to_device(prm, device), budgets, info
        if args.prep == "load":
            raise SystemExit(f"--prep load: {os.path.relpath(prep_path(args), ROOT)} missing or made with other flags")
    params, budgets, info = prepare_gpu(args, device)
    if args.save_prep:
        info["prep_file"] = os.path.relpath(save_prep(args, params, budgets, info), ROOT)
    return params, budgets, info


def prepare_indexer(args, device, rank=0, world=1):
    """For tools/: (params, [BudgetConfig] of this rank's KV heads, info) via obtain_prep."""
    import paper_2603_04460_b200 as vsp
    params, budgets, info = obtain_prep(args, device)
    per = args.hkv // world
    params = vsp.IndexerParams(*[shard(getattr(params, f), rank, world, 0)
                                 for f in ("w_u", "b_u", "w_v", "b_v", "w_s", "b_s")])
    mx = None if args.max_budget < 0 else args.max_budget
    return params, [vsp.BudgetConfig(tv, ts, args.min_budget, mx)
                    for tv, ts in budgets[rank * per:(rank + 1) * per]], info


def workload_config(args, world, budgets, info) -> dict:
    """The `config` of the JSON line — identical in both arms for the same flags."""
    balanced = args.shard in ("balanced", "spread")
    return {
        "workload": ("config[2]: LLaMA-3.1-8B attention geometry single layer, "
                     + (("every head split across ranks (spread units)" if args.shard == "spread"
                         else "cost-balanced (KV head, query-block) units") if balanced else "KV-head sharded")),
        "n": args.n, "hq": args.hq, "hkv": args.hkv, "d": 128, "d_h": args.d_h,
        "indexer": info.get("indexer"),
        "budget": {"tau_v": [b[0] for b in budgets], "tau_s": [b[1] for b in budgets], "min": args.min_budget,
                   "max": args.max_budget, "source": info.get("budget_source")},
        "prep": {k_: v_ for k_, v_ in info.items() if k_ not in ("indexer", "budget_source")},
        "inputs": ("planted vertical-slash synthetic layer (synth.py, seed %d, drawn on the CPU), resident in HBM; "
                   "Q is 1.07 GB > L2 so no flush between steps" % args.seed),
        "parallelism": (f"{'spread' if args.shard == 'spread' else 'balanced'} units x{world} (replicated inputs, "
                        f"static cost table from a validation prompt)" if balanced else
                        f"kv-head shard x{world}" + (" (whole KV heads placed by the predicted cost of a validation "
                                                     "prompt, equal counts)" if world > 1 and args.head_placement == "cost"
                                                     else "") +
                        ("; O assembled inside the attention kernel (epilogue stores into the peers' outputs over "
                         "CUDA IPC, one 1-element all-reduce barrier per step), timed in the step"
                         if world > 1 and getattr(args, "assemble", "nccl") == "mirror" else "")),
    }


# --------------------------------------------------------------------------- reference arm

class ReferenceLayer:
    """The reference's CPU implementation (oracle/_ref/libvspref.so: the unmodified headers)
    on a bounded sample of the bench layer, threaded over heads with every host core.

    Setup (once, measured): the reference's own indexer_forward over the full sequence (all
    n tokens: its softmax is over n) and select_pattern on it — the pattern the reference
    itself attends with. A step then times, through the same API, select_pattern on the
    full-length scores and sparse_attention over query rows [0, rows/2) and [0, rows) with
    that pattern (causality makes these the layer's own output rows). The full layer's
    attention time is extrapolated from the two prefixes: each head's call time is fitted as
    alpha * rows + beta * covered pairs (alpha: the per-row merge_row_columns work and
    allocations of attention.hpp:158-166, beta: the d-long dot + axpy per covered pair), and
    the per-head estimates at n are scheduled over the threads the way the threaded call
    does (next head to the next free thread). Checked against a full-length reference run
    (n = 32768, 8 threads, rows = 4096; tools/ref_extrapolation_check.py): the estimate was
    0.78-0.93 of the measured 20.5 s, i.e. it errs towards overstating the reference's
    throughput; a plain covered-pair ratio of one prefix (also reported) was 2.0-2.3x too
    slow, because early rows carry few pairs."""

    def __init__(self, args, q, k, v, prm: dict, budgets, threads: int, rows: int):
        import oracle
        if not oracle.have_ref():
            raise RuntimeError("oracle/_ref/libvspref.so not built (needs /root/reference at build time)")
        self.lib = oracle.ref()
        self.n, self.rows, self.threads = args.n, min(rows, args.n), threads
        self.hq, self.grp = args.hq, args.hq // args.hkv
        self.min_b, self.max_b = args.min_budget, args.max_budget if args.max_budget >= 0 else -1
        self.tau_v = [b[0] for b in budgets]
        self.tau_s = [b[1] for b in budgets]
        self.prm = {f: np.asarray(x, np.float64) for f, x in prm.items()}
        self.k = k.float().numpy().astype(np.float64)
        self.v = v.float().numpy().astype(np.float64)
        self.q = q[: self.rows].float().numpy().astype(np.float64)
        t0 = time.perf_counter()
        self.pv, self.ps = self.lib.layer_indexer(self.k, self.v, self.prm, threads)
        t1 = time.perf_counter()
        self.iv, self.kv, self.is_, self.ks = self.lib.layer_select(self.pv, self.ps, self.tau_v, self.tau_s,
                                                                    self.min_b, self.max_b, threads)
        t2 = time.perf_counter()
        self.indexer_full_s, self.select_full_s = t1 - t0, t2 - t1
        lists = [(self.iv[g, : self.kv[g]], self.is_[g, : self.ks[g]]) for g in range(len(self.kv))]
        # covered pairs per Q head: the layer and the two prefixes
        self.pairs = {r: np.array([pairs_prefix(*lists[h // self.grp], r) for h in range(self.hq)], np.float64)
                      for r in (self.n, self.rows, self.rows // 2)}

    def lists(self, g):
        return self.iv[g, : self.kv[g]].tolist(), self.is_[g, : self.ks[g]].tolist()

    def _sparse(self, rows):
        hs = np.zeros(self.hq)
        t0 = time.perf_counter()
        self.lib.layer_sparse(self.q, self.k, self.v, self.iv, self.kv, self.is_, self.ks, rows=rows,
                              threads=self.threads, head_s=hs)
        return time.perf_counter() - t0, hs

    def _makespan(self, per_head):
        free = [0.0] * min(self.threads, len(per_head))
        for t in per_head:  # heads in order, each to the first free thread (parallel_heads)
            i = int(np.argmin(free))
            free[i] += t
        return max(free)

    def step(self, i: int) -> dict:
        n, r, h = self.n, self.rows, self.rows // 2
        t0 = time.perf_counter()
        self.lib.layer_select(self.pv, self.ps, self.tau_v, self.tau_s, self.min_b, self.max_b, self.threads)
        sel = time.perf_counter() - t0
        wa, ta = self._sparse(h)
        wb, tb = self._sparse(r)
        # alpha * rows * hq + beta * pairs = summed per-head call time, at both prefixes
        A = np.array([[h * self.hq, self.pairs[h].sum()], [r * self.hq, self.pairs[r].sum()]])
        alpha, beta = np.linalg.solve(A, np.array([ta.sum(), tb.sum()]))
        if not (alpha >= 0 and beta > 0):  # degenerate sample: fall back to the pair ratio
            alpha, beta = 0.0, tb.sum() / max(self.pairs[r].sum(), 1.0)
        attn = self._makespan(alpha * n + beta * self.pairs[n])
        layer = self.indexer_full_s + sel + attn
        naive = wb * self.pairs[n].sum() / max(self.pairs[r].sum(), 1.0)
        return {"step_s": sel + wa + wb, "layer_s": layer, "select_s": sel, "attn_est_s": attn,
                "attn_rows_s": wb, "attn_half_rows_s": wa, "alpha_s_per_row": alpha, "beta_s_per_pair": beta,
                "attn_naive_pair_ratio_s": naive}

    def describe(self, recs) -> dict:
        m = {k_: float(np.mean([x[k_] for x in recs])) for k_ in recs[0]}
        return {
            "cpu_model": cpu_model(), "threads": self.threads,
            "layer_s_est": m["layer_s"],
            "components_s": {"indexer_full_measured": self.indexer_full_s, "select_full": m["select_s"],
                             "sparse_attention_est": m["attn_est_s"]},
            "sample_s": {"sparse_rows": m["attn_rows_s"], "sparse_half_rows": m["attn_half_rows_s"]},
            "fit": {"alpha_s_per_row_head": m["alpha_s_per_row"], "beta_s_per_pair": m["beta_s_per_pair"],
                    "pairs_layer": int(self.pairs[self.n].sum()), "pairs_sample": int(self.pairs[self.rows].sum())},
            "attn_naive_pair_ratio_s": m["attn_naive_pair_ratio_s"],
            "k_v": self.kv.tolist(), "k_s": self.ks.tolist(),
        }

    def sample_text(self) -> str:
        return (f"reference API (oracle/_ref) on the same layer, {self.threads} threads over heads: its own "
                f"indexer_forward + select_pattern over all n={self.n} (measured once), then per step select_pattern "
                f"on all n and sparse_attention of all {self.hq} Q heads on rows [0,{self.rows // 2}) and "
                f"[0,{self.rows}); layer attention extrapolated per head (alpha*rows + beta*covered pairs)")


def reference_inputs(args):
    """The bench layer, its indexer and budgets in a CPU-only process (no CUDA, no libvsp_gpu.so)."""
    if args.indexer == "random" and args.tau_v is not None and args.tau_s is not None:
        prm = params_to_numpy(random_params(args))
        budgets = [(args.tau_v, args.tau_s)] * args.hkv
        info = {"indexer": f"random-init VSIndexer (make_indexer_params), heads ~ N(0, {args.head_sigma}^2)",
                "budget_source": "fixed by flags"}
    else:
        got = load_prep(args)
        if got is None:
            return None
        prm, budgets, info = got
    q, k, v = synth_layer(args, "cpu")
    return q, k, v, prm, budgets, info


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    got = reference_inputs(args)
    if got is None:
        print(json.dumps({"impl": "reference", "unavailable": f"{os.path.relpath(prep_path(args), ROOT)} missing or "
                          f"made with other flags (run: python bench.py --prep fresh --save-prep)"}), flush=True)
        return
    q, k, v, prm, budgets, info = got
    threads = host_threads()
    torch.set_num_threads(threads)
    ref = ReferenceLayer(args, q, k, v, prm, budgets, threads, args.ref_rows)
    for i in range(args.warmup):
        ref.step(i)
    recs = [ref.step(args.warmup + i) for i in range(args.steps)]
    t_layer = float(np.mean([r["layer_s"] for r in recs]))
    val = args.n / t_layer
    desc = ref.describe(recs)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean([r["step_s"] for r in recs])) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world, budgets, info),
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "sample": ref.sample_text(), **desc},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "ms_per_step is the measured sample step; value = n / the extrapolated full-layer time",
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: run N ranks on fewer GPUs (e.g. the N>1 code path on a 1-GPU box) with gloo
    if os.environ.get("VSP_BENCH_DEVICES"):
        local = local % int(os.environ["VSP_BENCH_DEVICES"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("VSP_BENCH_BACKEND", "nccl")
    # cross-rank reductions of host-side numbers: on the GPU for NCCL, on the CPU for gloo
    red_dev = dev if backend == "nccl" else torch.device("cpu")
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))
    balanced = args.shard in ("balanced", "spread")
    assert balanced or args.hkv % world == 0, "KV heads must divide across ranks"
    import paper_2603_04460_b200 as vsp
    from paper_2603_04460_b200 import parallel

    n = args.n
    grp = args.hq // args.hkv
    # every rank holds all heads' (identical, deterministic) indexers and budgets; a heads
    # rank keeps its slice, a unit rank the whole layer
    params_full, budgets_full, prep_info = obtain_prep(args, dev)
    srank, sworld = (0, 1) if balanced else (rank, world)
    hq_r, hkv_r = args.hq // sworld, args.hkv // sworld
    mx = None if args.max_budget < 0 else args.max_budget
    # heads split at N > 1: whole KV heads, equal counts, placed by the predicted cost of a
    # validation prompt (parallel.balanced_head_sets); my_kv = this rank's KV heads
    head_sets = None
    my_kv = list(range(srank * hkv_r, (srank + 1) * hkv_r))
    if not balanced and world > 1 and args.head_placement == "cost":
        qv, kv_, vv = synth_layer(args, dev, seed=args.seed + 201)
        budget_all = [vsp.BudgetConfig(tv, ts, args.min_budget, mx) for tv, ts in budgets_full]
        a_v, a_s = vsp.indexer_forward(kv_, vv, params_full)
        pat_v = vsp.select_pattern(a_v, a_s, budget_all)
        vsp.sparse_attention(qv, kv_, vv, pat_v, validate=False)
        head_cost = vsp.sparse_tile_counts(n, args.hkv, pat_v.i_v.shape[1], dev).sum(dim=1).double() + 2500.0
        del qv, kv_, vv, a_v, a_s, pat_v
        head_sets = parallel.balanced_head_sets(head_cost.cpu(), world)
        my_kv = head_sets[rank]
    kv_idx = torch.tensor(my_kv, dtype=torch.long)
    q_idx = torch.tensor(parallel.q_heads_of(my_kv, grp), dtype=torch.long)
    params = vsp.IndexerParams(*[getattr(params_full, f).index_select(0, kv_idx.to(getattr(params_full, f).device))
                                 .contiguous() for f in ("w_u", "b_u", "w_v", "b_v", "w_s", "b_s")])
    budget = [vsp.BudgetConfig(*budgets_full[g], args.min_budget, mx) for g in my_kv]
    units = all_units = None
    if balanced:
        # static cost table: per (head, block) tiles of a validation prompt (not the timed one)
        qv, kv_, vv = synth_layer(args, dev, seed=args.seed + 201)
        a_v, a_s = vsp.indexer_forward(kv_, vv, params)
        pat_v = vsp.select_pattern(a_v, a_s, budget)
        vsp.sparse_attention(qv, kv_, vv, pat_v, validate=False)
        cost = vsp.sparse_tile_counts(n, args.hkv, pat_v.i_v.shape[1], dev)
        del qv, kv_, vv, a_v, a_s, pat_v
        all_units = (parallel.spread_units(cost, world) if args.shard == "spread"
                     else parallel.balanced_units(cost, world))
        units = all_units[rank]
    # the timed prompt, drawn on the CPU (the reference arm draws the identical layer)
    q_host, k_host, v_host = synth_layer(args, "cpu")
    q = q_host.index_select(1, q_idx).contiguous().to(dev)
    k = k_host.index_select(1, kv_idx).contiguous().to(dev)
    v = v_host.index_select(1, kv_idx).contiguous().to(dev)
    if not (rank == 0 and world == 1 and not args.no_cpu_baseline):
        del q_host, k_host, v_host
    # O is written head-major straight into this rank's slab of the full [Hq, n, d] output
    # (VSP_O_HEAD_MAJOR): the slab is the in-place all-gather send buffer (parallel.py)
    mirror = world > 1 and not balanced and args.assemble == "mirror"
    mirrors = ipc_bufs = None
    if mirror:
        # the full outputs are CUDA-IPC allocations; every rank maps the others' and K3 stores
        # its slab (placement order) into all of them (vsp_vs_prefill_mirrored)
        obytes, lbytes = args.hq * n * 128 * 2, args.hq * n * 4
        ipc_bufs = [vsp.IpcBuffer(obytes, dev), vsp.IpcBuffer(lbytes, dev)]
        handles = [None] * world
        torch.distributed.all_gather_object(handles, [ipc_bufs[0].handle, ipc_bufs[1].handle])
        peers = [(vsp.IpcBuffer.open(h[0], obytes, dev), vsp.IpcBuffer.open(h[1], lbytes, dev))
                 for r_, h in enumerate(handles) if r_ != rank]
        slab_o, slab_l = rank * hq_r * n * 128 * 2, rank * hq_r * n * 4
        mirrors = [(po.ptr + slab_o, pl.ptr + slab_l) for po, pl in peers]
        o_full = ipc_bufs[0].tensor(torch.bfloat16, (args.hq, n, 128))
        lse_full = ipc_bufs[1].tensor(torch.float32, (args.hq, n))
        flag = torch.zeros(1, device=dev)
    else:
        o_full = torch.empty(args.hq, n, 128, dtype=q.dtype, device=dev)
        lse_full = torch.empty(args.hq, n, device=dev)
    o = parallel.head_slab(o_full, srank, sworld)
    lse = parallel.head_slab(lse_full, srank, sworld)

    hpc = args.heads_per_chunk

    def step():
        if balanced:
            # one C-ABI call (vsp_vs_prefill_units): scoring/selection/planning of the heads this
            # rank's units touch, then attention of exactly its units
            return vsp.vs_prefill_units(q, k, v, params, budget, units, out=o_full, lse=lse_full)
        # one C-ABI call (vsp_vs_prefill): K1 -> K2 -> plan -> K3 (automatic schedule unless --heads-per-chunk)
        _, _, pat = vsp.vs_prefill(q, k, v, params, budget, heads_per_chunk=hpc, out=o, lse=lse, head_major=True,
                                   mirrors=mirrors)
        if mirror:  # every rank's stores have landed once every rank's layer has finished
            if backend == "nccl":
                torch.distributed.all_reduce(flag)  # stream-ordered
            else:  # shared-GPU test mode (gloo)
                torch.cuda.synchronize()
                torch.distributed.barrier()
        return pat

    def step_unfused():
        a_v, a_s = vsp.indexer_forward(k, v, params)
        pat = vsp.select_pattern(a_v, a_s, budget)
        vsp.sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse, head_major=True)
        return pat

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(max(args.warmup, 1)):
        pat = step()
    torch.cuda.synchronize()

    # ---- timed region (device events; max over ranks)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" captures this region
        launches0 = vsp.kernel_launches()
        vsp.attn_timing(True, dev)  # CUDA events around every K3 launch inside the timed steps
        e0.record(stream)
        for _ in range(args.steps):
            pat = step()
        e1.record(stream)
        timed_launches = vsp.kernel_launches() - launches0  # libvsp_gpu.so's own launch counter
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        k3_total_ms, k3_launches = vsp.attn_timing_read(dev)
        vsp.attn_timing(False, dev)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ms_step = parallel.max_over_ranks(ms, red_dev) if world > 1 else ms

    # ---- component timings (same heads, untimed by the contract, for the roofline)
    def timed(fn, reps=3):
        fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    a_v, a_s = vsp.indexer_forward(k, v, params)
    pat = vsp.select_pattern(a_v, a_s, budget)
    ms_unfused = timed(step_unfused)
    ms_indexer = timed(lambda: vsp.indexer_forward(k, v, params))
    ms_select = timed(lambda: vsp.select_pattern(a_v, a_s, budget))
    ms_attn = timed(lambda: vsp.sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse, head_major=True))
    tiles, tiles_dense = vsp.sparse_tile_stats(n, hkv_r, pat.i_v.shape[1], dev)
    o_d = torch.empty_like(q)
    lse_d = torch.empty_like(lse)
    ms_dense = timed(lambda: vsp.blockwise_attention(q, k, v, out=o_d, lse=lse_d))
    vsp.sparse_attention(q, k, v, pat, validate=False, out=o, lse=lse, head_major=True)
    recall = float(vsp.attention_recall(lse, lse_d).mean().item())
    pairs_kv = covered_pairs(pat, n, hkv_r)
    pairs_q = int(pairs_kv.sum()) * grp
    dense_pairs = hq_r * n * (n + 1) // 2
    alg_flops = 4.0 * 128 * pairs_q
    # compulsory bytes of one K3 launch: read Q, K, V of these heads once, write O and LSE
    alg_bytes = (q.numel() + k.numel() + v.numel() + o.numel()) * 2 + lse.numel() * 4
    pk, pk_kind = peaks()
    peak_tf = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    # K3's own duration, measured live inside the timed steps (event pair around each launch)
    # (a balanced rank's K3 launches cover only its units: there the all-head call is used)
    live = bool(k3_launches) and not (balanced and world > 1)
    k3_ms = k3_total_ms / args.steps if live else ms_attn
    achieved_tf = alg_flops / (k3_ms * 1e-3) / 1e12
    tile_tf = 4.0 * 128 * 128 * 128 * tiles * grp / (k3_ms * 1e-3) / 1e12
    dense_tf = 4.0 * 128 * dense_pairs / (ms_dense * 1e-3) / 1e12
    kv_list = pat.k_v.cpu().tolist()
    ks_list = pat.k_s.cpu().tolist()

    # ---- output assembly over NCCL, reported separately (not inside the step)
    allgather_ms = None
    mirror_check = None
    if mirror:
        # every rank must hold identical slabs: compare per-slab checksums across the ranks
        step()
        torch.cuda.synchronize()
        sums = torch.stack([s_.double().sum() for s_ in o_full.view(torch.int16).float().chunk(world, 0)])
        sums = sums.to(red_dev)
        all_sums = [torch.zeros_like(sums) for _ in range(world)]
        torch.distributed.all_gather(all_sums, sums)
        mirror_check = bool(all(torch.equal(a.cpu(), all_sums[0].cpu()) for a in all_sums))
    elif world > 1 and backend == "nccl":
        comm = parallel.VspComm(dev)
        if balanced:  # unit regions broadcast by their owners (vsp_assemble_units)
            vsp.vs_prefill_units(q, k, v, params, budget, units, out=o_full, lse=lse_full)
            allgather_ms = timed(lambda: comm.assemble_units(o_full, lse_full, all_units, args.hkv), reps=3)
        elif head_sets is None:  # one in-place ncclAllGather of the head-major slabs (O and LSE)
            allgather_ms = timed(lambda: comm.allgather_heads(o_full, lse_full), reps=3)
        else:  # slabs in placement order, then one permutation into head order
            perm = torch.tensor([q for hs in head_sets for q in parallel.q_heads_of(hs, grp)], device=dev)
            o_out = torch.empty_like(o_full)
            lse_out = torch.empty_like(lse_full)

            def assemble():
                comm.allgather_heads(o_full, lse_full)
                o_out.index_copy_(0, perm, o_full)
                lse_out.index_copy_(0, perm, lse_full)

            allgather_ms = timed(assemble, reps=3)
        allgather_ms = parallel.max_over_ranks(allgather_ms, dev)
        comm.close()
    elif world > 1:  # shared-GPU test mode (VSP_BENCH_DEVICES, gloo): CPU-staged assembly
        o_c, l_c = o_full.cpu(), lse_full.cpu()
        if balanced:
            parallel.assemble_units(o_c, l_c, all_units, args.hkv)
        else:
            lo_h, hi_h = parallel.head_range(args.hq, rank, world)
            for t in (o_c, l_c):
                parts = list(t.chunk(world, 0))
                torch.distributed.all_gather(parts, t[lo_h:hi_h].clone())
                t.copy_(torch.cat(parts, 0))
        o_full.copy_(o_c)
        lse_full.copy_(l_c)

    # ---- e2e through the public API with host buffers (H2D inputs, D2H output every step)
    e2e = None
    if not args.no_e2e:
        qh = q.cpu().pin_memory()
        kh = k.cpu().pin_memory()
        vh = v.cpu().pin_memory()
        if balanced:  # head-major host output; only this rank's unit regions come back
            oh_ = torch.empty(o_full.shape, dtype=q.dtype).pin_memory()
            lse_h = torch.empty(lse_full.shape, dtype=lse.dtype).pin_memory()
        else:
            oh_ = torch.empty(q.shape, dtype=q.dtype).pin_memory()
            lse_h = torch.empty(lse.shape, dtype=lse.dtype).pin_memory()
        d2h_units = sum(grp * (min(hi * 128, n) - lo * 128) * (128 * 2 + 4) for _, lo, hi in (units or []))

        def e2e_step():
            if balanced:
                # replicated inputs: H2D of the whole layer, the rank's units, D2H of its regions
                q.copy_(qh, non_blocking=True)
                k.copy_(kh, non_blocking=True)
                v.copy_(vh, non_blocking=True)
                vsp.vs_prefill_units(q, k, v, params, budget, units, out=o_full, lse=lse_full)
                for g_, lo, hi in units:
                    hs = slice(g_ * grp, (g_ + 1) * grp)
                    rs = slice(lo * 128, min(hi * 128, n))
                    oh_[hs, rs].copy_(o_full[hs, rs], non_blocking=True)
                    lse_h[hs, rs].copy_(lse_full[hs, rs], non_blocking=True)
                return
            # one host-buffer C-ABI call: H2D of Q/K/V, K1->K2->K3, D2H of O and LSE, pipelined per chunk
            vsp.vs_prefill_host(qh, kh, vh, params, budget, heads_per_chunk=args.e2e_heads_per_chunk,
                                out=oh_, lse=lse_h, device=dev)

        e2e_step()
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e2e_t = a.elapsed_time(b) / args.steps
        e2e_t = parallel.max_over_ranks(e2e_t, red_dev) if world > 1 else e2e_t
        e2e = {"value": n / (e2e_t * 1e-3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(qh.numel() * 2 + kh.numel() * 2 + vh.numel() * 2),
               "d2h_bytes_per_step": int(d2h_units if balanced else oh_.numel() * 2 + lse_h.numel() * 4),
               "ms_per_step": float(e2e_t),
               "api": ("vs_prefill_units (pinned host Q/K/V in, this rank's O/LSE regions out)" if balanced else
                       "vsp_vs_prefill_host (pinned host Q/K/V in, host O/LSE out)"),
               "heads_per_chunk": args.e2e_heads_per_chunk}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = host_threads()
            ref = ReferenceLayer(args, q_host, k_host, v_host, params_to_numpy(params_full), budgets_full, threads,
                                 args.ref_rows)
            rec = ref.step(0)
            agree = []
            for g in range(args.hkv):  # the reference's own pattern vs this build's (same inputs)
                gv, gs = (set(x) for x in pat.lists(g))
                rv, rs = (set(x) for x in ref.lists(g))
                agree.append([round(len(gv & rv) / max(len(gv | rv), 1), 4),
                              round(len(gs & rs) / max(len(gs | rs), 1), 4)])
            cpu = {"value": n / rec["layer_s"], "unit": "tokens/s", "cores": threads, "kind": "reference",
                   "sample": ref.sample_text() + "; one step", **ref.describe([rec]),
                   "pattern_jaccard_vs_gpu": agree}
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": "tokens/s", "cores": host_threads(), "kind": "reference",
                   "sample": f"failed: {ex}"}

    if rank == 0:
        cfg = workload_config(args, world, budgets_full, prep_info)
        line = {
            "metric": METRIC, "value": n / (ms_step * 1e-3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": cfg,
            "units_this_rank": units,
            "speedup_vs_dense": ms_dense / ms_attn, "dense_ms": ms_dense, "vs_attn_ms": ms_attn,
            "unfused_ms": ms_unfused, "heads_per_chunk": hpc,
            "indexer_ms": ms_indexer, "select_ms": ms_select, "recall": recall,
            "density": pairs_q / dense_pairs, "tile_density": tiles / tiles_dense,
            "k_v": kv_list, "k_s": ks_list, "dense_tflops": dense_tf, "allgather_ms": allgather_ms,
            "assembly": ("mirrored K3 stores (inside the step)" if mirror else
                         ("NCCL after the step (allgather_ms)" if world > 1 else None)),
            "mirror_check": mirror_check,
            "roofline": {"bound": "tensor", "kernel": "vs_attn_fwd (K3)", "achieved": achieved_tf,
                         "peak": peak_tf, "unit": "TFLOP/s", "frac": achieved_tf / peak_tf,
                         "traffic": k3_traffic(), "algorithmic_bytes": alg_bytes,
                         "peak_kind": f"{pk_kind} bf16 sustained",
                         "executed_tile_tflops": tile_tf, "executed_tile_frac": tile_tf / peak_tf,
                         "kernel_ms": k3_ms, "timing": ("CUDA events around each K3 launch inside the timed steps "
                                                        f"({k3_launches} launches)") if live
                         else "separate all-head sparse_attention calls (plan + K3)"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": timed_launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
