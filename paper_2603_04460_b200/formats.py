"""The reference's interchange formats over the C ABI (csrc/formats.cpp).

    reference                                        here
    ---------------------------------------------    ------------------------------------------
    vsp::write_tensor / read_tensor / read_vector    write_tensor / read_tensor / read_vector
        tensor_io.hpp:49-88 (VSTN, f64)
    vsp::save_checkpoint / load_checkpoint           save_checkpoint / load_checkpoint
        indexer.hpp:450-499 (VSCK, one KV head)        (+ load_checkpoints: stack KV heads onto the GPU)
    vsp::write_indices / read_indices                write_indices / read_indices
        sparsity.hpp:187-245 ("V:"/"S:" text)          (+ patterns_from_files: onto the GPU)

Errors keep the reference's exception types and texts: std::runtime_error ->
VspRuntimeError, std::invalid_argument -> VspError. The files are byte-identical to the
reference writers' (tests/test_formats.py checks against files the reference wrote).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import IndexerParams, SelectedIndices, _check, load_library

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_bound = False


def _lib():
    global _bound
    lib = load_library()
    if not _bound:
        c, i, i64, u64, f64 = ctypes.c_char_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        ip = ctypes.POINTER(ctypes.c_int)
        lib.vsp_tensor_header.argtypes = [c, ip, _u64p, i]
        lib.vsp_read_tensor.argtypes = [c, i, _f64p, u64]
        lib.vsp_write_tensor.argtypes = [c, i, _u64p, _f64p]
        lib.vsp_checkpoint_header.argtypes = [c, ip, ip]
        lib.vsp_load_checkpoint.argtypes = [c, i, i, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p]
        lib.vsp_save_checkpoint.argtypes = [c, i, i, _f64p, _f64p, _f64p, f64, _f64p, f64]
        lib.vsp_write_indices.argtypes = [c, _i64p, i64, _i64p, i64]
        lib.vsp_read_indices.argtypes = [c, _i64p, _i64p, _i64p, _i64p, i64]
        _bound = True
    return lib


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ---------------------------------------------------------------------- VSTN tensors

def tensor_shape(path) -> Tuple[int, ...]:
    """The dims of a VSTN file (read_tensor_header, tensor_io.hpp:26-42)."""
    lib = _lib()
    nd = ctypes.c_int()
    dims = (ctypes.c_uint64 * 64)()
    _check(lib.vsp_tensor_header(_path(path), ctypes.byref(nd), dims, 64))
    if nd.value > 64:
        raise NotImplementedError("VSTN rank > 64")
    return tuple(int(dims[t]) for t in range(nd.value))


def _read(path, rank: int) -> np.ndarray:
    lib = _lib()
    nd = ctypes.c_int()
    dims = (ctypes.c_uint64 * 64)()
    rc = lib.vsp_tensor_header(_path(path), ctypes.byref(nd), dims, 64)
    _check(rc)
    shape = tuple(int(dims[t]) for t in range(min(nd.value, 64)))
    count = int(np.prod(shape, dtype=np.uint64)) if (rank <= 0 or nd.value == rank) else 0
    out = np.empty(count, dtype=np.float64)
    _check(lib.vsp_read_tensor(_path(path), rank, out.ctypes.data_as(_f64p), count))
    return out.reshape(shape)


def read_tensor(path) -> np.ndarray:
    """vsp::read_tensor (tensor_io.hpp:66-77): a rank-2 f64 matrix."""
    return _read(path, 2)


def read_vector(path) -> np.ndarray:
    """vsp::read_vector (tensor_io.hpp:79-88): a rank-1 f64 vector."""
    return _read(path, 1)


def read_tensor_any(path) -> np.ndarray:
    """A VSTN file of any rank (the format allows it; the reference reads ranks 1 and 2)."""
    return _read(path, 0)


def write_tensor(path, x) -> None:
    """vsp::write_tensor (tensor_io.hpp:49-64): matrices as rank 2, vectors as rank 1 (any
    rank is written as-is). Torch tensors (any device/dtype) are widened to f64 on the host."""
    if isinstance(x, torch.Tensor):
        x = x.detach().to("cpu", torch.float64).numpy()
    a = _f64(x)
    dims = (ctypes.c_uint64 * max(a.ndim, 1))(*a.shape)
    _check(_lib().vsp_write_tensor(_path(path), a.ndim, dims, a.ctypes.data_as(_f64p)))


# ---------------------------------------------------------------------- VSCK checkpoints

def load_checkpoint(path) -> dict:
    """vsp::load_checkpoint (indexer.hpp:476-499) for one KV head: f64 numpy arrays
    {w_u [2d, d_h], b_u, w_v, b_v, w_s, b_s, d_h}."""
    lib = _lib()
    d, dh = ctypes.c_int(), ctypes.c_int()
    _check(lib.vsp_checkpoint_header(_path(path), ctypes.byref(d), ctypes.byref(dh)))
    d, dh = d.value, dh.value
    w_u = np.empty((2 * d, dh))
    b_u, w_v, w_s = np.empty(dh), np.empty(dh), np.empty(dh)
    b_v, b_s = ctypes.c_double(), ctypes.c_double()
    _check(lib.vsp_load_checkpoint(_path(path), d, dh, w_u.ctypes.data_as(_f64p), b_u.ctypes.data_as(_f64p),
                                   w_v.ctypes.data_as(_f64p), ctypes.byref(b_v), w_s.ctypes.data_as(_f64p),
                                   ctypes.byref(b_s)))
    return {"w_u": w_u, "b_u": b_u, "w_v": w_v, "b_v": b_v.value, "w_s": w_s, "b_s": b_s.value, "d_h": dh}


def save_checkpoint(params, path, head: int = 0) -> None:
    """vsp::save_checkpoint (indexer.hpp:450-474). `params` is a dict as load_checkpoint
    returns, or an IndexerParams (then KV head `head` is written; bf16 W_U widens exactly)."""
    if isinstance(params, IndexerParams):
        params = {"w_u": params.w_u[head].double().cpu().numpy(), "b_u": params.b_u[head].double().cpu().numpy(),
                  "w_v": params.w_v[head].double().cpu().numpy(), "b_v": float(params.b_v[head]),
                  "w_s": params.w_s[head].double().cpu().numpy(), "b_s": float(params.b_s[head])}
    w_u = _f64(params["w_u"])
    b_u, w_v, w_s = _f64(params["b_u"]), _f64(params["w_v"]), _f64(params["w_s"])
    in_dim, dh = w_u.shape
    if not (b_u.shape == (dh,) and w_v.shape == (dh,) and w_s.shape == (dh,)):
        from . import VspError
        raise VspError("indexer params: inconsistent shapes")
    if in_dim % 2:
        from . import VspError
        raise VspError("save_checkpoint: in_dim must be 2d")
    _check(_lib().vsp_save_checkpoint(_path(path), in_dim // 2, dh, w_u.ctypes.data_as(_f64p),
                                      b_u.ctypes.data_as(_f64p), w_v.ctypes.data_as(_f64p), float(params["b_v"]),
                                      w_s.ctypes.data_as(_f64p), float(params["b_s"])))


def load_checkpoints(paths: Sequence, device="cuda") -> IndexerParams:
    """One VSCK checkpoint per KV head -> the batched device IndexerParams the kernels take
    (W_U rounded to bf16, the rest fp32)."""
    ck = [load_checkpoint(p) for p in paths]
    st = lambda key: torch.from_numpy(np.stack([c[key] for c in ck]))  # noqa: E731
    return IndexerParams(st("w_u").to(device=device, dtype=torch.bfloat16), st("b_u").float().to(device),
                         st("w_v").float().to(device), torch.tensor([c["b_v"] for c in ck]).float().to(device),
                         st("w_s").float().to(device), torch.tensor([c["b_s"] for c in ck]).float().to(device))


def save_checkpoints(params: IndexerParams, paths: Sequence) -> None:
    """Write each KV head of `params` to its own VSCK file."""
    for g, p in enumerate(paths):
        save_checkpoint(params, p, head=g)


# ---------------------------------------------------------------------- index text

def write_indices(path, i_v, i_s=None) -> None:
    """vsp::write_indices (sparsity.hpp:192-205). Either (path, i_v, i_s) lists, or
    (path, SelectedIndices, g) for KV head g of a device pattern."""
    if isinstance(i_v, SelectedIndices):
        i_v, i_s = i_v.lists(0 if i_s is None else int(i_s))
    a = np.ascontiguousarray(np.asarray(i_v, dtype=np.int64).reshape(-1))
    b = np.ascontiguousarray(np.asarray(i_s, dtype=np.int64).reshape(-1))
    _check(_lib().vsp_write_indices(_path(path), a.ctypes.data_as(_i64p), a.size, b.ctypes.data_as(_i64p), b.size))


def read_indices(path) -> Tuple[list, list]:
    """vsp::read_indices (sparsity.hpp:234-245) -> (i_v, i_s) ascending lists."""
    lib = _lib()
    cap = max(os.path.getsize(path), 1) if os.path.exists(path) else 1
    a = np.empty(cap, dtype=np.int64)
    b = np.empty(cap, dtype=np.int64)
    kv, ks = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.vsp_read_indices(_path(path), a.ctypes.data_as(_i64p), ctypes.byref(kv), b.ctypes.data_as(_i64p),
                                ctypes.byref(ks), cap))
    return a[:kv.value].tolist(), b[:ks.value].tolist()


def patterns_from_files(paths: Sequence, n: int, device="cuda", cap: Optional[int] = None) -> SelectedIndices:
    """Index files (one per KV head) -> the device SelectedIndices that sparse_attention takes."""
    cap = cap or n + 1
    hkv = len(paths)
    i_v = torch.zeros(hkv, cap, dtype=torch.int32)
    i_s = torch.zeros_like(i_v)
    k_v = torch.zeros(hkv, dtype=torch.int32)
    k_s = torch.zeros_like(k_v)
    for g, p in enumerate(paths):
        a, b = read_indices(p)
        if len(a) > cap or len(b) > cap:
            from . import VspError
            raise VspError("patterns_from_files: more indices than cap")
        i_v[g, :len(a)] = torch.tensor(a, dtype=torch.int32)
        i_s[g, :len(b)] = torch.tensor(b, dtype=torch.int32)
        k_v[g], k_s[g] = len(a), len(b)
    return SelectedIndices(i_v.to(device), k_v.to(device), i_s.to(device), k_s.to(device))
