"""Shared helpers for the parity tests: seeded inputs, bf16 <-> f64 views, and per-head
oracle runs (the oracle package is the checker; the product path never calls it)."""
from __future__ import annotations

import numpy as np
import torch

import oracle


def qkv(n, hq, hkv, d=128, seed=0, device="cuda", scale=1.0):
    g = torch.Generator().manual_seed(seed)
    q = (torch.randn(n, hq, d, generator=g) * scale).to(torch.bfloat16)
    k = (torch.randn(n, hkv, d, generator=g) * scale).to(torch.bfloat16)
    v = torch.randn(n, hkv, d, generator=g).to(torch.bfloat16)
    return q.to(device), k.to(device), v.to(device)


def f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def oracle_dense(q, k, v, block=64):
    """Per-head oracle of blockwise_attention on the same bf16 values -> (O [n,hq,d], LSE [hq,n])."""
    n, hq, d = q.shape
    hkv = k.shape[1]
    grp = hq // hkv
    qn, kn, vn = f64(q), f64(k), f64(v)
    o = np.zeros((n, hq, d))
    lse = np.zeros((hq, n))
    port = oracle.port()
    for h in range(hq):
        g = h // grp
        o[:, h], lse[h] = port.blockwise_attention(qn[:, h], kn[:, g], vn[:, g], block=block, want_lse=True)
    return o, lse


def oracle_sparse(q, k, v, lists, block=32):
    """lists: per KV head (i_v, i_s) python lists."""
    n, hq, d = q.shape
    hkv = k.shape[1]
    grp = hq // hkv
    qn, kn, vn = f64(q), f64(k), f64(v)
    o = np.zeros((n, hq, d))
    lse = np.zeros((hq, n))
    port = oracle.port()
    for h in range(hq):
        g = h // grp
        iv, is_ = lists[g]
        o[:, h], lse[h] = port.sparse_attention(qn[:, h], kn[:, g], vn[:, g], iv, is_, block=block, want_lse=True)
    return o, lse


def pattern_tensors(lists, n, device="cuda"):
    """Per-KV-head (i_v, i_s) lists -> SelectedIndices with cap n + 1."""
    from paper_2603_04460_b200 import SelectedIndices
    hkv = len(lists)
    cap = n + 1
    i_v = torch.zeros(hkv, cap, dtype=torch.int32)
    i_s = torch.zeros(hkv, cap, dtype=torch.int32)
    k_v = torch.zeros(hkv, dtype=torch.int32)
    k_s = torch.zeros(hkv, dtype=torch.int32)
    for g, (iv, is_) in enumerate(lists):
        i_v[g, : len(iv)] = torch.tensor(list(iv), dtype=torch.int32)
        i_s[g, : len(is_)] = torch.tensor(list(is_), dtype=torch.int32)
        k_v[g] = len(iv)
        k_s[g] = len(is_)
    return SelectedIndices(i_v.to(device), k_v.to(device), i_s.to(device), k_s.to(device))


def assert_attn_close(o_gpu, lse_gpu, o_ref, lse_ref, max_tol=2e-2, mean_tol=2e-3, lse_tol=1e-3):
    """Stated tolerances (bf16 P and O, fp32 accumulation vs the f64 reference)."""
    og = f64(o_gpu)
    err = np.abs(og - o_ref)
    assert np.isfinite(og).all(), "non-finite output"
    assert err.max() <= max_tol, f"O max|d| {err.max():.3e} > {max_tol}"
    assert err.mean() <= mean_tol, f"O mean|d| {err.mean():.3e} > {mean_tol}"
    if lse_gpu is not None:
        le = np.abs(f64(lse_gpu) - lse_ref)
        assert le.max() <= lse_tol, f"LSE max|d| {le.max():.3e} > {lse_tol}"
