"""B200-native VS-prefill path (arxiv 2603.04460) behind the reference's operator API.

Host-side mirror of the reference's hot-path functions (namespace ``vsp`` in
/root/reference/proj/include/vsprefill) over the C ABI in include/vsp_gpu.h, which
dispatches to hand-written sm_100a kernels (tcgen05/TMEM/TMA). Torch tensors are used
only as device-memory carriers. There is no CPU fallback: every call fails loudly when
the extension (libvsp_gpu.so) or an sm_100 device is missing.

    reference                                  here
    ---------------------------------------    ------------------------------------
    vsp::indexer_forward   indexer.hpp:116      indexer_forward(k, v, params)
    vsp::select_pattern    sparsity.hpp:105     select_pattern(a_v, a_s, budget)
    vsp::sparse_attention  attention.hpp:150    sparse_attention(q, k, v, pattern)
    vsp::blockwise_attention attention.hpp:96   blockwise_attention(q, k, v)
    vsp::aggregate_streaming vsaggregate.hpp:62 aggregate_streaming(q, k)
      + combine_scores     vsaggregate.hpp:133    (group reduce fused)
    vsp::attention_recall  attention.hpp:198    attention_recall(lse_sparse, lse_dense)
    vsp::apply_rope        rope.hpp:63          apply_rope(x, positions, cfg) / apply_rope_qk(q, k, ...)

Tensors are batched over heads: Q [n, Hq, 128], K/V [n, Hkv, 128] bf16 (Q head h reads
KV head h // (Hq // Hkv)); one VS pattern per KV head, shared by its Q heads.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
import os
from typing import Optional, Sequence, Tuple

import torch

__all__ = [
    "VspError", "BudgetConfig", "IndexerParams", "SelectedIndices", "make_indexer_params",
    "indexer_forward", "select_pattern", "sparse_attention", "blockwise_attention",
    "aggregate_streaming", "attention_recall", "RopeConfig", "apply_rope", "apply_rope_qk", "vs_prefill", "vs_prefill_host", "vs_prefill_unfused", "vs_prefill_units", "sparse_tile_counts", "lib_path", "load_library",
    "topk_indices", "combine_scores", "merge_row_columns", "merge_path_partition", "IpcBuffer",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_PKG, "libvsp_gpu.so")

VSP_OK, VSP_EINVAL, VSP_ERUNTIME, VSP_ECUDA, VSP_ENCCL = range(5)
VSP_VALIDATE, VSP_O_HEAD_MAJOR, VSP_DENSE_SWITCH = 1, 2, 4


class VspError(ValueError):
    """VSP_EINVAL: the reference would have thrown std::invalid_argument (same text)."""


class VspRuntimeError(RuntimeError):
    """VSP_ECUDA / VSP_ERUNTIME / VSP_ENCCL."""


class _Budget(ctypes.Structure):
    _fields_ = [("tau_v", ctypes.c_double), ("tau_s", ctypes.c_double),
                ("min_budget", ctypes.c_int64), ("max_budget", ctypes.c_int64)]


_lib = None


def load_library():
    """Load libvsp_gpu.so (building it first if absent). Raises if it cannot be had."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        from . import _build
        _build.build()
    lib = ctypes.CDLL(lib_path)
    vp, i, f, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_size_t
    lib.vsp_last_error.restype = ctypes.c_char_p
    lib.vsp_version.restype = ctypes.c_char_p
    lib.vsp_kernel_launches.restype = ctypes.c_longlong
    lib.vsp_attn_timing.argtypes = [vp, i]
    lib.vsp_attn_timing_read.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i)]
    lib.vsp_create.argtypes = [ctypes.POINTER(vp), i]
    lib.vsp_destroy.argtypes = [vp]
    lib.vsp_indexer_workspace_size.restype = sz
    lib.vsp_indexer_workspace_size.argtypes = [i, i, i]
    lib.vsp_indexer_scores.argtypes = [vp, vp, vp, i, i, i, i, vp, vp, vp, vp, vp, vp, i, vp, vp, vp, vp, vp, vp]
    lib.vsp_select_workspace_size.restype = sz
    lib.vsp_select_workspace_size.argtypes = [i, i]
    lib.vsp_select.argtypes = [vp, vp, vp, i, i, ctypes.POINTER(_Budget), vp, vp, vp, vp, i, vp, i, vp]
    lib.vsp_vs_attn_workspace_size.restype = sz
    lib.vsp_vs_attn_workspace_size.argtypes = [i, i, i]
    lib.vsp_vs_attn_fwd.argtypes = [vp, vp, vp, vp, i, i, i, i, vp, vp, vp, vp, i, f, vp, vp, vp, i, vp]
    lib.vsp_dense_attn_fwd.argtypes = [vp, vp, vp, vp, i, i, i, i, f, vp, vp, vp]
    lib.vsp_aggregate_workspace_size.restype = sz
    lib.vsp_aggregate_workspace_size.argtypes = [i, i]
    lib.vsp_vs_aggregate.argtypes = [vp, vp, vp, i, i, i, i, f, vp, i, i, vp, vp, vp, vp]
    lib.vsp_recall_from_lse.argtypes = [vp, vp, vp, i, i, vp, vp]
    lib.vsp_vs_attn_tile_stats.argtypes = [vp, i, i, i, vp, ctypes.POINTER(ctypes.c_int64), vp]
    lib.vsp_vs_prefill_host_workspace_size.restype = sz
    lib.vsp_vs_prefill_host_workspace_size.argtypes = [i, i, i, i]
    lib.vsp_vs_prefill_host.argtypes = ([vp, vp, vp, vp, i, i, i, i, i, vp, vp, vp, vp, vp, vp, i,
                                         ctypes.POINTER(_Budget), vp, vp, vp, vp, vp, i, vp])
    lib.vsp_vs_prefill_workspace_size.restype = sz
    lib.vsp_vs_prefill_workspace_size.argtypes = [i, i, i, i]
    lib.vsp_vs_prefill.argtypes = ([vp, vp, vp, vp, i, i, i, i, i, vp, vp, vp, vp, vp, vp, i,
                                    ctypes.POINTER(_Budget), vp, vp, vp, vp, vp, vp, i, vp, vp, vp, i, i, vp])
    lib.vsp_vs_prefill_mirrored.argtypes = ([vp, vp, vp, vp, i, i, i, i, i, vp, vp, vp, vp, vp, vp, i,
                                             ctypes.POINTER(_Budget), vp, vp, vp, vp, vp, vp, i, vp, vp, vp, i, i,
                                             i, vp, vp, vp])
    lib.vsp_ipc_alloc.argtypes = [vp, sz, ctypes.POINTER(vp), ctypes.c_char_p]
    lib.vsp_ipc_open.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(vp)]
    lib.vsp_ipc_close.argtypes = [vp]
    lib.vsp_ipc_free.argtypes = [vp]
    lib.vsp_apply_rope.argtypes = [vp, vp, vp, vp, vp, i, i, i, i, vp, ctypes.c_double, i, vp]
    lib.vsp_vs_attn_tile_counts.argtypes = [vp, i, i, i, vp, vp, vp]
    lib.vsp_vs_prefill_units.argtypes = ([vp, vp, vp, vp, i, i, i, i, i, vp, vp, vp, vp, vp, vp, i,
                                          ctypes.POINTER(_Budget), vp, vp, vp, vp, vp, vp, i, vp, vp, vp, vp, i, i, vp])
    lib.vsp_merge_path_partition.argtypes = [vp, ctypes.c_int64, vp, ctypes.c_int64, ctypes.c_int64, vp]
    lib.vsp_merge_row_columns.argtypes = [vp, vp, i, vp, i, vp, i, vp, vp, i, i, vp]
    lib.vsp_topk_workspace_size.restype = sz
    lib.vsp_topk_workspace_size.argtypes = [i]
    lib.vsp_topk_indices.argtypes = [vp, vp, i, i, vp, vp, i, vp, vp]
    lib.vsp_combine_scores.argtypes = [vp, vp, vp, i, i, i, vp, vp, vp]
    _lib = lib
    return lib


def _check(rc: int):
    if rc == VSP_OK:
        return
    msg = _lib.vsp_last_error().decode()
    if rc == VSP_EINVAL:
        raise VspError(msg)
    raise VspRuntimeError(msg)


_ctx: dict = {}


def _context(device: torch.device):
    lib = load_library()
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _ctx:
        h = ctypes.c_void_p()
        _check(lib.vsp_create(ctypes.byref(h), idx))
        _ctx[idx] = h
    return _ctx[idx]


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


_ws_cache: dict = {}


def _workspace(device, nbytes: int) -> torch.Tensor:
    """Scratch for the calls on the current stream (one buffer per (device, stream), so calls
    on different streams may overlap; the C ABI's contract is one workspace per in-flight call)."""
    dev = torch.device(device)
    key = (str(dev), torch.cuda.current_stream(dev).cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def _need_cuda(*ts: torch.Tensor):
    for t in ts:
        if not t.is_cuda:
            raise VspRuntimeError("vsp: tensors must live on an sm_100 CUDA device (no CPU fallback)")


# ---------------------------------------------------------------------- data types

@dataclasses.dataclass
class BudgetConfig:
    """sparsity.hpp:22-36. max_budget None = no maximum."""
    tau_v: float = 0.9
    tau_s: float = 0.9
    min_budget: int = 1
    max_budget: Optional[int] = None

    def _c(self) -> _Budget:
        return _Budget(self.tau_v, self.tau_s, int(self.min_budget),
                       -1 if self.max_budget is None else int(self.max_budget))


@dataclasses.dataclass
class IndexerParams:
    """indexer.hpp:34-49, batched over KV heads. w_u [Hkv, 2d, d_h] bf16 (rows 0..d-1
    multiply K, d..2d-1 multiply V), b_u/w_v/w_s [Hkv, d_h] fp32, b_v/b_s [Hkv] fp32."""
    w_u: torch.Tensor
    b_u: torch.Tensor
    w_v: torch.Tensor
    b_v: torch.Tensor
    w_s: torch.Tensor
    b_s: torch.Tensor

    @property
    def d_h(self) -> int:
        return self.w_u.shape[2]


@dataclasses.dataclass
class SelectedIndices:
    """sparsity.hpp:38-46, batched: i_v/i_s [Hkv, cap] int32, k_v/k_s [Hkv] int32."""
    i_v: torch.Tensor
    k_v: torch.Tensor
    i_s: torch.Tensor
    k_s: torch.Tensor

    def lists(self, g: int):
        kv, ks = int(self.k_v[g]), int(self.k_s[g])
        return self.i_v[g, :kv].cpu().tolist(), self.i_s[g, :ks].cpu().tolist()


def make_indexer_params(hkv: int, d: int, d_h: int, generator: torch.Generator, head_sigma: float = 0.0,
                        device="cuda") -> IndexerParams:
    """make_indexer_params (indexer.hpp:53-64) batched: W_U ~ U(+-1/sqrt(2d)); heads zero
    (exactly uniform scores) unless head_sigma > 0 (heads ~ N(0, sigma^2))."""
    lim = 1.0 / math.sqrt(2 * d)
    w_u = (torch.rand(hkv, 2 * d, d_h, generator=generator) * 2 - 1) * lim
    w_v = torch.randn(hkv, d_h, generator=generator) * head_sigma
    w_s = torch.randn(hkv, d_h, generator=generator) * head_sigma
    z = torch.zeros(hkv, d_h)
    return IndexerParams(w_u.to(device=device, dtype=torch.bfloat16), z.to(device), w_v.to(device),
                         torch.zeros(hkv, device=device), w_s.to(device), torch.zeros(hkv, device=device))


@dataclasses.dataclass
class RopeConfig:
    """rope.hpp:13-39 (theta_p = base^(-2p/head_dim)), plus the pairing style: "interleaved"
    (2p, 2p+1), the reference's, or "half_split" (p, p + d/2) for HF checkpoints."""
    head_dim: int = 128
    base: float = 10000.0
    style: str = "interleaved"

    def __post_init__(self):
        if self.head_dim < 2 or self.head_dim % 2 != 0:
            raise VspError("rope head_dim must be even and >= 2")
        if not self.base > 0.0:
            raise VspError("rope base must be positive")
        if self.style not in ("interleaved", "half_split"):
            raise VspError("rope style must be 'interleaved' or 'half_split'")

    def theta(self, p: int) -> float:
        return self.base ** (-2.0 * p / self.head_dim)


# ---------------------------------------------------------------------- operators

def apply_rope_qk(q: Optional[torch.Tensor], k: Optional[torch.Tensor], positions: Optional[torch.Tensor] = None,
                  cfg: Optional[RopeConfig] = None, inplace: bool = False):
    """The RoPE feed before the path: apply_rope (rope.hpp:63-79) on Q [n, Hq, d] and K
    [n, Hkv, d] bf16 in ONE HBM pass (vsp_apply_rope). positions: int64 [n] on the device,
    or None for t = row index. Returns (Q', K') (the inputs themselves when inplace)."""
    ref = q if q is not None else k
    _need_cuda(*(t for t in (q, k) if t is not None))
    n, _, d = ref.shape
    cfg = cfg or RopeConfig(d)
    if cfg.head_dim != d:
        raise VspError("apply_rope: column count != head_dim")
    if positions is not None:
        if positions.numel() != n:
            raise VspError("apply_rope: positions length != row count")
        positions = positions.to(device=ref.device, dtype=torch.int64).contiguous()
    qo = None if q is None else (q if inplace else torch.empty_like(q))
    ko = None if k is None else (k if inplace else torch.empty_like(k))
    lib = load_library()
    _check(lib.vsp_apply_rope(_context(ref.device), _ptr(q), _ptr(k), _ptr(qo), _ptr(ko), n,
                              0 if q is None else q.shape[1], 0 if k is None else k.shape[1], d, _ptr(positions),
                              float(cfg.base), 0 if cfg.style == "interleaved" else 1, _stream(ref.device)))
    return qo, ko


def apply_rope(x: torch.Tensor, positions: Optional[torch.Tensor] = None, cfg: Optional[RopeConfig] = None,
               inplace: bool = False) -> torch.Tensor:
    """apply_rope (rope.hpp:63-79) for every head of x [n, H, d] bf16."""
    return apply_rope_qk(x, None, positions, cfg, inplace)[0]


def indexer_forward(k: torch.Tensor, v: torch.Tensor, p: IndexerParams, mapping: str = "reverse",
                    want_logits: bool = False):
    """indexer_forward (indexer.hpp:116-120) for every KV head -> (A_v, A_s) [Hkv, n] fp32
    (+ logits_v, logits_s when want_logits)."""
    _need_cuda(k, v)
    n, hkv, d = k.shape
    lib = load_library()
    dev = k.device
    a_v = torch.empty(hkv, n, device=dev, dtype=torch.float32)
    a_s = torch.empty_like(a_v)
    lv = torch.empty_like(a_v) if want_logits else None
    ls = torch.empty_like(a_v) if want_logits else None
    ws = _workspace(dev, lib.vsp_indexer_workspace_size(n, hkv, p.d_h))
    _check(lib.vsp_indexer_scores(_context(dev), _ptr(k), _ptr(v), n, hkv, d, p.d_h, _ptr(p.w_u), _ptr(p.b_u),
                                  _ptr(p.w_v), _ptr(p.b_v), _ptr(p.w_s), _ptr(p.b_s),
                                  0 if mapping == "reverse" else 1, _ptr(a_v), _ptr(a_s), _ptr(lv), _ptr(ls),
                                  _ptr(ws), _stream(dev)))
    return (a_v, a_s, lv, ls) if want_logits else (a_v, a_s)


def select_pattern(a_v: torch.Tensor, a_s: torch.Tensor, budget, validate: bool = False) -> SelectedIndices:
    """select_pattern (sparsity.hpp:105-114) per KV head. budget: BudgetConfig or a list of
    them (one per KV head, e.g. per-layer/per-head budgets)."""
    _need_cuda(a_v, a_s)
    hkv, n = a_v.shape
    budgets = list(budget) if isinstance(budget, (list, tuple)) else [budget] * hkv
    arr = (_Budget * hkv)(*[b._c() for b in budgets])
    lib = load_library()
    dev = a_v.device
    cap = n + 1
    i_v = torch.empty(hkv, cap, device=dev, dtype=torch.int32)
    i_s = torch.empty_like(i_v)
    k_v = torch.empty(hkv, device=dev, dtype=torch.int32)
    k_s = torch.empty_like(k_v)
    ws = _workspace(dev, lib.vsp_select_workspace_size(n, hkv))
    _check(lib.vsp_select(_context(dev), _ptr(a_v.contiguous()), _ptr(a_s.contiguous()), n, hkv, arr, _ptr(i_v),
                          _ptr(k_v), _ptr(i_s), _ptr(k_s), cap, _ptr(ws), 1 if validate else 0, _stream(dev)))
    return SelectedIndices(i_v, k_v, i_s, k_s)


def sparse_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, pattern: SelectedIndices,
                     validate: bool = True, out: Optional[torch.Tensor] = None,
                     lse: Optional[torch.Tensor] = None, head_major: bool = False,
                     dense_switch: bool = False):
    """sparse_attention (attention.hpp:150-194) for every Q head -> (O [n, Hq, d] bf16,
    LSE [Hq, n] fp32). validate=True reproduces the reference's checks and messages
    (merge.hpp:21-26, attention.hpp:161-163) at the cost of one stream sync.
    head_major=True writes O as [Hq, n, d] (the reference's per-head matrices).
    dense_switch=True (opt-in, not the reference's semantics): query blocks whose pattern
    already visits every causal tile run unmasked causal attention (VSP_DENSE_SWITCH)."""
    _need_cuda(q, k, v)
    n, hq, d = q.shape
    hkv = k.shape[1]
    lib = load_library()
    dev = q.device
    o = out if out is not None else (torch.empty(hq, n, d, dtype=q.dtype, device=dev) if head_major
                                     else torch.empty_like(q))
    lse = lse if lse is not None else torch.empty(hq, n, device=dev, dtype=torch.float32)
    cap = pattern.i_v.shape[1]
    ws = _workspace(dev, lib.vsp_vs_attn_workspace_size(n, hkv, cap))
    _check(lib.vsp_vs_attn_fwd(_context(dev), _ptr(q), _ptr(k), _ptr(v), n, hq, hkv, d, _ptr(pattern.i_v),
                               _ptr(pattern.k_v), _ptr(pattern.i_s), _ptr(pattern.k_s), cap,
                               1.0 / math.sqrt(d), _ptr(o), _ptr(lse), _ptr(ws),
                               (1 if validate else 0) | (VSP_O_HEAD_MAJOR if head_major else 0)
                               | (VSP_DENSE_SWITCH if dense_switch else 0), _stream(dev)))
    return o, lse


def sparse_tile_stats(n: int, hkv: int, cap: int, device, per_head: bool = False) -> tuple:
    """(KV tiles visited by the last sparse_attention on `device`, tiles dense would visit)
    summed over query blocks and KV heads [, tiles per KV head]. Synchronises the stream."""
    lib = load_library()
    ws = _workspace(device, 0)  # the current stream's scratch, which holds that call's plan
    out = (ctypes.c_int64 * (2 + hkv))()
    _check(lib.vsp_vs_attn_tile_stats(_context(device), n, hkv, cap, _ptr(ws), out, _stream(device)))
    if per_head:
        return int(out[0]), int(out[1]), [int(out[2 + g]) for g in range(hkv)]
    return int(out[0]), int(out[1])


def blockwise_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: Optional[torch.Tensor] = None,
                        lse: Optional[torch.Tensor] = None):
    """blockwise_attention (attention.hpp:96-145): dense causal, every Q head."""
    _need_cuda(q, k, v)
    n, hq, d = q.shape
    hkv = k.shape[1]
    lib = load_library()
    dev = q.device
    o = out if out is not None else torch.empty_like(q)
    lse = lse if lse is not None else torch.empty(hq, n, device=dev, dtype=torch.float32)
    _check(lib.vsp_dense_attn_fwd(_context(dev), _ptr(q), _ptr(k), _ptr(v), n, hq, hkv, d, 1.0 / math.sqrt(d),
                                  _ptr(o), _ptr(lse), _stream(dev)))
    return o, lse


def aggregate_streaming(q: torch.Tensor, k: torch.Tensor, lse: Optional[torch.Tensor] = None,
                        reduce: str = "mean", normalized: bool = True):
    """aggregate_streaming (vsaggregate.hpp:62-127) for every Q head, group-reduced per KV
    head with combine_scores (vsaggregate.hpp:133-157) -> (A_v, A_s) [Hkv, n] fp32."""
    _need_cuda(q, k)
    n, hq, d = q.shape
    hkv = k.shape[1]
    lib = load_library()
    dev = q.device
    a_v = torch.empty(hkv, n, device=dev, dtype=torch.float32)
    a_s = torch.empty_like(a_v)
    ws = _workspace(dev, lib.vsp_aggregate_workspace_size(n, hq))
    _check(lib.vsp_vs_aggregate(_context(dev), _ptr(q), _ptr(k), n, hq, hkv, d, 1.0 / math.sqrt(d), _ptr(lse),
                                0 if reduce == "mean" else 1, int(normalized), _ptr(a_v), _ptr(a_s), _ptr(ws),
                                _stream(dev)))
    return a_v, a_s


def attention_recall(lse_sparse: torch.Tensor, lse_dense: torch.Tensor) -> torch.Tensor:
    """attention_recall (attention.hpp:198-215) without the n x n matrix: row i's covered
    mass is exp(LSE_sparse_i - LSE_dense_i). Returns recall per Q head [Hq] fp32."""
    _need_cuda(lse_sparse, lse_dense)
    hq, n = lse_sparse.shape
    dev = lse_sparse.device
    out = torch.empty(hq, device=dev, dtype=torch.float32)
    _check(load_library().vsp_recall_from_lse(_context(dev), _ptr(lse_sparse), _ptr(lse_dense), n, hq, _ptr(out),
                                              _stream(dev)))
    return out


def topk_indices(scores: torch.Tensor, k) -> torch.Tensor:
    """topk_indices (sparsity.hpp:83-97) per row of scores [rows, n] (or [n]) fp32, any sign:
    the k largest, ties to the lower index, ascending -> int32 [rows, max k] (row r filled up
    to k[r]; k an int or one per row)."""
    _need_cuda(scores)
    one = scores.dim() == 1
    x = scores.reshape(1, -1) if one else scores
    x = x.contiguous().float()
    rows, n = x.shape
    ks = [int(k)] * rows if isinstance(k, int) else [int(t) for t in k]
    lib = load_library()
    cap = max(max(ks), 1) if ks else 1
    out = torch.zeros(rows, cap, dtype=torch.int32, device=x.device)
    karr = (ctypes.c_int * max(rows, 1))(*ks)
    ws = _workspace(x.device, lib.vsp_topk_workspace_size(rows))
    _check(lib.vsp_topk_indices(_context(x.device), _ptr(x), n, rows, ctypes.cast(karr, ctypes.c_void_p), _ptr(out),
                                cap, _ptr(ws), _stream(x.device)))
    return out[0] if one else out


def combine_scores(vertical: torch.Tensor, slash: torch.Tensor, reduce: str = "mean"):
    """combine_scores (vsaggregate.hpp:133-157): per-head scores [heads, n] -> the group's
    [n] (mean keeps normalisation, sum gives the raw total; f64 accumulation in head order)."""
    _need_cuda(vertical, slash)
    if vertical.dim() != 2 or vertical.shape != slash.shape:
        raise VspError("combine_scores: length mismatch")
    heads, n = vertical.shape
    v_out = torch.empty(n, dtype=torch.float32, device=vertical.device)
    s_out = torch.empty_like(v_out)
    lib = load_library()
    _check(lib.vsp_combine_scores(_context(vertical.device), _ptr(vertical.contiguous().float()),
                                  _ptr(slash.contiguous().float()), heads, n, 0 if reduce == "mean" else 1,
                                  _ptr(v_out), _ptr(s_out), _stream(vertical.device)))
    return v_out, s_out


def merge_row_columns(i_v: torch.Tensor, i_s: torch.Tensor, rows, validate: bool = True):
    """merge_row_columns (merge.hpp:18-56) on the device for query rows `rows` (int or 1-D
    int tensor / list) under one KV head's ascending lists i_v, i_s (int32 device tensors)
    -> list of int32 tensors (one ascending column set per row)."""
    _need_cuda(i_v, i_s)
    dev = i_v.device
    one = isinstance(rows, int)
    r = torch.as_tensor([rows] if one else rows, dtype=torch.int32).to(dev)
    count = r.numel()
    cap = i_v.numel() + i_s.numel()
    out = torch.empty(count, max(cap, 1), dtype=torch.int32, device=dev)
    lens = torch.empty(count, dtype=torch.int32, device=dev)
    lib = load_library()
    _check(lib.vsp_merge_row_columns(_context(dev), _ptr(i_v.int().contiguous()), i_v.numel(),
                                     _ptr(i_s.int().contiguous()), i_s.numel(), _ptr(r), count, _ptr(out),
                                     _ptr(lens), max(cap, 1), VSP_VALIDATE if validate else 0, _stream(dev)))
    res = [out[t, : int(lens[t])] for t in range(count)]
    return res[0] if one else res


def merge_path_partition(a, b, p: int):
    """merge_path_partition (merge.hpp:69-95): p + 1 (a_idx, b_idx) cut points of the merge of
    ascending a and b, a-first ties (host; the device row merge uses the same search)."""
    import numpy as np
    av = np.ascontiguousarray(np.asarray(a, dtype=np.int64).reshape(-1))
    bv = np.ascontiguousarray(np.asarray(b, dtype=np.int64).reshape(-1))
    cuts = np.zeros(2 * (max(int(p), 1) + 1), np.int64)
    lib = load_library()
    _check(lib.vsp_merge_path_partition(ctypes.c_void_p(av.ctypes.data), len(av), ctypes.c_void_p(bv.ctypes.data),
                                        len(bv), int(p), ctypes.c_void_p(cuts.ctypes.data)))
    return [tuple(int(x) for x in c) for c in cuts.reshape(-1, 2)]


def vs_prefill(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, params: IndexerParams, budget,
               mapping: str = "reverse", heads_per_chunk: int = 0, out: Optional[torch.Tensor] = None,
               lse: Optional[torch.Tensor] = None, head_major: bool = False, dense_switch: bool = False,
               mirrors=None):
    """The whole VS-prefill hot path of one layer in ONE C-ABI call (vsp_vs_prefill):
    indexer -> selection -> sparse attention; heads_per_chunk=0 runs them in order on the
    current stream, heads_per_chunk>0 pipelines KV-head chunks so that the
    scoring/selection/planning of chunk c+1 overlaps chunk c's attention. Mirrors
    `vsprefill select` + `vsprefill attend` (tools/vsprefill.cpp:154-185) on device.
    Same results as indexer_forward + select_pattern + sparse_attention.
    head_major=True writes O as [Hq, n, d] (e.g. a slab of the full output on a shard rank).
    dense_switch=True: see sparse_attention (opt-in; off = the reference's semantics).
    mirrors: optional list of (o_ptr, lse_ptr) device addresses (ints or tensors) laid out like
    `out` / `lse` — e.g. the same slab of other ranks' outputs mapped with IpcBuffer.open: the
    attention epilogue stores every O tile and LSE row there too (vsp_vs_prefill_mirrored).
    Returns (O, LSE, SelectedIndices)."""
    _need_cuda(q, k, v)
    n, hq, d = q.shape
    hkv = k.shape[1]
    budgets = list(budget) if isinstance(budget, (list, tuple)) else [budget] * hkv
    if len(budgets) != hkv:
        raise VspError("vs_prefill: one BudgetConfig per KV head required")
    arr = (_Budget * hkv)(*[b._c() for b in budgets])
    lib = load_library()
    dev = q.device
    cap = n + 1
    a_v = torch.empty(hkv, n, device=dev, dtype=torch.float32)
    a_s = torch.empty_like(a_v)
    i_v = torch.empty(hkv, cap, device=dev, dtype=torch.int32)
    i_s = torch.empty_like(i_v)
    k_v = torch.empty(hkv, device=dev, dtype=torch.int32)
    k_s = torch.empty_like(k_v)
    o = out if out is not None else (torch.empty(hq, n, d, dtype=q.dtype, device=dev) if head_major
                                     else torch.empty_like(q))
    lse = lse if lse is not None else torch.empty(hq, n, device=dev, dtype=torch.float32)
    ws = _workspace(dev, lib.vsp_vs_prefill_workspace_size(n, hkv, params.d_h, cap))
    flags = (VSP_O_HEAD_MAJOR if head_major else 0) | (VSP_DENSE_SWITCH if dense_switch else 0)
    if mirrors:
        addr = lambda x: None if x is None else (x.data_ptr() if isinstance(x, torch.Tensor) else int(x))
        om = (ctypes.c_void_p * len(mirrors))(*[addr(m[0]) for m in mirrors])
        lm = (ctypes.c_void_p * len(mirrors))(*[addr(m[1]) for m in mirrors])
        _check(lib.vsp_vs_prefill_mirrored(
            _context(dev), _ptr(q), _ptr(k), _ptr(v), n, hq, hkv, d, params.d_h, _ptr(params.w_u), _ptr(params.b_u),
            _ptr(params.w_v), _ptr(params.b_v), _ptr(params.w_s), _ptr(params.b_s), 0 if mapping == "reverse" else 1,
            arr, _ptr(a_v), _ptr(a_s), _ptr(i_v), _ptr(k_v), _ptr(i_s), _ptr(k_s), cap, _ptr(o), _ptr(lse), _ptr(ws),
            int(heads_per_chunk), flags, len(mirrors), ctypes.cast(om, ctypes.c_void_p),
            ctypes.cast(lm, ctypes.c_void_p), _stream(dev)))
        return o, lse, SelectedIndices(i_v, k_v, i_s, k_s)
    _check(lib.vsp_vs_prefill(_context(dev), _ptr(q), _ptr(k), _ptr(v), n, hq, hkv, d, params.d_h,
                              _ptr(params.w_u), _ptr(params.b_u), _ptr(params.w_v), _ptr(params.b_v),
                              _ptr(params.w_s), _ptr(params.b_s), 0 if mapping == "reverse" else 1, arr,
                              _ptr(a_v), _ptr(a_s), _ptr(i_v), _ptr(k_v), _ptr(i_s), _ptr(k_s), cap, _ptr(o),
                              _ptr(lse), _ptr(ws), int(heads_per_chunk),
                              (VSP_O_HEAD_MAJOR if head_major else 0) | (VSP_DENSE_SWITCH if dense_switch else 0),
                              _stream(dev)))
    return o, lse, SelectedIndices(i_v, k_v, i_s, k_s)


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (torch.as_tensor wraps it, no copy)."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "strides": None, "version": 3}
        self._owner = owner


class IpcBuffer:
    """Device memory another process can map (vsp_ipc_alloc / vsp_ipc_open): the KV-head split's
    full-layer output, into which every rank's attention epilogue stores its slab directly
    (vs_prefill(mirrors=...)). `handle` (64 bytes) travels to the other ranks, which call
    IpcBuffer.open(handle, nbytes, device)."""

    def __init__(self, nbytes: int, device, _ptr_handle=None):
        self.device = torch.device(device)
        self.nbytes = int(nbytes)
        lib = load_library()
        ptr = ctypes.c_void_p()
        if _ptr_handle is None:
            hbuf = ctypes.create_string_buffer(64)
            _check(lib.vsp_ipc_alloc(_context(self.device), self.nbytes, ctypes.byref(ptr), hbuf))
            self.handle, self.opened = hbuf.raw, False
        else:
            self.handle = bytes(_ptr_handle)
            _check(lib.vsp_ipc_open(_context(self.device), self.handle, ctypes.byref(ptr)))
            self.opened = True
        self.ptr = int(ptr.value)

    @classmethod
    def open(cls, handle: bytes, nbytes: int, device) -> "IpcBuffer":
        return cls(nbytes, device, _ptr_handle=handle)

    def tensor(self, dtype: torch.dtype, shape, offset_bytes: int = 0) -> torch.Tensor:
        """A torch view of [offset, offset + numel * itemsize) (bf16 through an int16 view)."""
        numel = 1
        for x in shape:
            numel *= int(x)
        item = torch.empty((), dtype=dtype).element_size()
        if offset_bytes + numel * item > self.nbytes:
            raise VspError("IpcBuffer.tensor: view exceeds the buffer")
        code = {torch.bfloat16: "<i2", torch.float16: "<f2", torch.float32: "<f4", torch.int32: "<i4"}[dtype]
        t = torch.as_tensor(_CudaArray(self.ptr + offset_bytes, shape, code, self), device=self.device)
        return t.view(dtype) if dtype == torch.bfloat16 else t

    def close(self):
        if self.ptr:
            lib = load_library()
            _check(lib.vsp_ipc_close(ctypes.c_void_p(self.ptr)) if self.opened else
                   lib.vsp_ipc_free(ctypes.c_void_p(self.ptr)))
            self.ptr = 0


class _Unit(ctypes.Structure):
    _fields_ = [("g", ctypes.c_int32), ("qb_lo", ctypes.c_int32), ("qb_hi", ctypes.c_int32)]


def kernel_launches() -> int:
    """Kernels libvsp_gpu.so has launched in this process (vsp_kernel_launches)."""
    return int(load_library().vsp_kernel_launches())


def attn_timing(enable: bool, device=None) -> None:
    """Bracket every K3 launch of the layer entry points with CUDA events (vsp_attn_timing)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    _check(load_library().vsp_attn_timing(_context(dev), 1 if enable else 0))


def attn_timing_read(device=None) -> Tuple[float, int]:
    """-> (summed K3 milliseconds, K3 launches) since attn_timing(True) or the last read."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ms, cnt = ctypes.c_double(), ctypes.c_int()
    _check(load_library().vsp_attn_timing_read(_context(dev), ctypes.byref(ms), ctypes.byref(cnt)))
    return ms.value, cnt.value


def sparse_tile_counts(n: int, hkv: int, cap: int, device) -> torch.Tensor:
    """Per (KV head, query block) tile counts [hkv, ceil(n/128)] of the last sparse_attention
    plan on this device's workspace (vsp_vs_attn_tile_counts) — the cost table of a balanced
    split. Call it right after sparse_attention (like sparse_tile_stats)."""
    lib = load_library()
    dev = torch.device(device)
    num_qb = (n + 127) // 128
    out = torch.empty(hkv * num_qb, dtype=torch.int32)
    ws = _workspace(dev, 0)
    _check(lib.vsp_vs_attn_tile_counts(_context(dev), n, hkv, cap, _ptr(ws), ctypes.c_void_p(out.data_ptr()),
                                       _stream(dev)))
    return out.view(hkv, num_qb)


def vs_prefill_units(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, params: IndexerParams, budget, units,
                     out: torch.Tensor, lse: torch.Tensor, mapping: str = "reverse"):
    """A rank's share of a balanced multi-GPU split (vsp_vs_prefill_units): `units` is a list of
    (KV head, qb_lo, qb_hi); Q/K/V and params cover ALL heads; O is head-major [Hq, n, d] and
    only the units' (head, row) regions are written. Returns the device SelectedIndices (valid
    for the heads the units touch)."""
    _need_cuda(q, k, v)
    n, hq, d = q.shape
    hkv = k.shape[1]
    budgets = list(budget) if isinstance(budget, (list, tuple)) else [budget] * hkv
    if len(budgets) != hkv:
        raise VspError("vs_prefill_units: one BudgetConfig per KV head required")
    if out.shape != (hq, n, d):
        raise VspError("vs_prefill_units: out must be head-major [Hq, n, d]")
    arr = (_Budget * hkv)(*[b._c() for b in budgets])
    ua = (_Unit * max(len(units), 1))(*[_Unit(int(g), int(lo), int(hi)) for g, lo, hi in units])
    lib = load_library()
    dev = q.device
    cap = n + 1
    a_v = torch.empty(hkv, n, device=dev, dtype=torch.float32)
    a_s = torch.empty_like(a_v)
    i_v = torch.empty(hkv, cap, device=dev, dtype=torch.int32)
    i_s = torch.empty_like(i_v)
    k_v = torch.zeros(hkv, device=dev, dtype=torch.int32)
    k_s = torch.zeros_like(k_v)
    ws = _workspace(dev, lib.vsp_vs_prefill_workspace_size(n, hkv, params.d_h, cap))
    _check(lib.vsp_vs_prefill_units(_context(dev), _ptr(q), _ptr(k), _ptr(v), n, hq, hkv, d, params.d_h,
                                    _ptr(params.w_u), _ptr(params.b_u), _ptr(params.w_v), _ptr(params.b_v),
                                    _ptr(params.w_s), _ptr(params.b_s), 0 if mapping == "reverse" else 1, arr,
                                    _ptr(a_v), _ptr(a_s), _ptr(i_v), _ptr(k_v), _ptr(i_s), _ptr(k_s), cap, _ptr(out),
                                    _ptr(lse), _ptr(ws), ua, len(units), VSP_O_HEAD_MAJOR, _stream(dev)))
    return SelectedIndices(i_v, k_v, i_s, k_s)


def vs_prefill_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, params: IndexerParams, budget,
                    mapping: str = "reverse", heads_per_chunk: int = 0, out: Optional[torch.Tensor] = None,
                    lse: Optional[torch.Tensor] = None, budgets_out: bool = False, device=None):
    """vs_prefill from HOST tensors (pinned CPU memory for overlap), like the reference's
    own operators which take host vectors: one C-ABI call (vsp_vs_prefill_host) that pipelines
    H2D copies, scoring/selection, attention and the D2H of O — per query-row range
    (heads_per_chunk=0: K/V first, then Q ranges) or per KV-head chunk (heads_per_chunk>0).
    Returns (O, LSE) as host tensors (+ (k_v, k_s) host tensors when budgets_out).
    Stream-ordered: synchronise the current stream before reading the results."""
    for t in (q, k, v):
        if t.is_cuda or not t.is_contiguous():
            raise VspError("vs_prefill_host: q, k, v must be contiguous host tensors")
    n, hq, d = q.shape
    hkv = k.shape[1]
    budgets = list(budget) if isinstance(budget, (list, tuple)) else [budget] * hkv
    if len(budgets) != hkv:
        raise VspError("vs_prefill: one BudgetConfig per KV head required")
    arr = (_Budget * hkv)(*[b._c() for b in budgets])
    lib = load_library()
    dev = torch.device(device) if device is not None else params.w_u.device
    o = out if out is not None else torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
    lse = lse if lse is not None else torch.empty(hq, n, dtype=torch.float32, pin_memory=True)
    kv = torch.empty(hkv, dtype=torch.int32, pin_memory=True) if budgets_out else None
    ks = torch.empty(hkv, dtype=torch.int32, pin_memory=True) if budgets_out else None
    key = (str(dev), torch.cuda.current_stream(dev).cuda_stream, "host")
    need = lib.vsp_vs_prefill_host_workspace_size(n, hq, hkv, params.d_h)
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < need:
        ws = _ws_cache[key] = torch.empty(need, dtype=torch.uint8, device=dev)
    _check(lib.vsp_vs_prefill_host(_context(dev), _ptr(q), _ptr(k), _ptr(v), n, hq, hkv, d, params.d_h,
                                   _ptr(params.w_u), _ptr(params.b_u), _ptr(params.w_v), _ptr(params.b_v),
                                   _ptr(params.w_s), _ptr(params.b_s), 0 if mapping == "reverse" else 1, arr,
                                   _ptr(o), _ptr(lse), _ptr(kv), _ptr(ks), _ptr(ws), int(heads_per_chunk),
                                   _stream(dev)))
    return (o, lse, kv, ks) if budgets_out else (o, lse)


def vs_prefill_unfused(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, params: IndexerParams, budget,
                       mapping: str = "reverse"):
    """vs_prefill as three separate operator calls (indexer_forward, select_pattern,
    sparse_attention) on one stream: the parity twin of the fused call."""
    a_v, a_s = indexer_forward(k, v, params, mapping)
    pat = select_pattern(a_v, a_s, budget)
    o, lse = sparse_attention(q, k, v, pat, validate=False)
    return o, lse, pat
