"""TEST INFRASTRUCTURE ONLY — the CPU checker for the sm_100a VS-prefill path.

Two libraries, both f64 and single-threaded per head:
  * ``port()`` — vsp_oracle.c, a plain-C restatement of the reference hot path
    (every function cites the reference file:line it follows);
  * ``ref()``  — oracle/_ref/libvspref.so: the UNMODIFIED reference headers from
    /root/reference/proj/include wrapped in extern "C" (ref_shim.cpp). Built only
    where /root/reference exists; the .so travels to the GPU box with the repo.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this package. The product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libvsp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvspref.so")

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64
_cp = ctypes.c_char_p


class OracleError(ValueError):
    """Mirrors the reference's std::invalid_argument (same message text)."""


def build(quiet: bool = True) -> None:
    r = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + r.stdout + r.stderr)


def _bind(lib, prefix: str):
    sig = {
        "merge_row_columns": (_i64, [_i64p, _i64, _i64p, _i64, _i64, _i64p, _cp, ctypes.c_size_t]),
        "merge_path_partition": (ctypes.c_int, [_i64p, _i64, _i64p, _i64, _i64, _i64p, _cp, ctypes.c_size_t]),
        "cumulative_budget": (ctypes.c_int, [_f64p, _i64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                             _i64, _i64, _i64p, _cp, ctypes.c_size_t]),
        "topk_indices": (ctypes.c_int, [_f64p, _i64, _i64, _i64p, _cp, ctypes.c_size_t]),
        "select_pattern": (ctypes.c_int, [_f64p, _f64p, _i64, ctypes.c_double, ctypes.c_double, _i64, _i64,
                                          _i64p, _i64p, _i64p, _i64p, _cp, ctypes.c_size_t]),
        "indexer_forward": (ctypes.c_int, [_i64, _i64, _f64p, _i64, _f64p, _i64, _i64, _f64p, _f64p, _f64p,
                                           ctypes.c_double, _f64p, ctypes.c_double, ctypes.c_int,
                                           _f64p, _f64p, _f64p, _f64p, _cp, ctypes.c_size_t]),
        "aggregate_streaming": (ctypes.c_int, [_i64, _i64, _f64p, _i64, _f64p, _i64, _i64, ctypes.c_int,
                                               _f64p, _f64p, _cp, ctypes.c_size_t]),
        "apply_rope": (ctypes.c_int, [_i64, _i64, _f64p, _i64, _i64p, ctypes.c_double, _f64p, _i64, _cp,
                                      ctypes.c_size_t]),
        "indexer_backward": (ctypes.c_int, [_i64, _i64, _f64p, _i64, _f64p, _i64, _i64, _f64p, _f64p, _f64p,
                                            ctypes.c_double, _f64p, ctypes.c_double, ctypes.c_int, _f64p, _f64p,
                                            ctypes.c_double, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p,
                                            _cp, ctypes.c_size_t]),
    }
    if prefix == "vso_":
        lib.vso_adamw_step.restype = None
        lib.vso_adamw_step.argtypes = [_i64, _f64p, _f64p, _f64p, _f64p, _i64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double]
        sig["blockwise_attention"] = (ctypes.c_int, [_i64, _i64, _f64p, _i64, _f64p, _i64, _f64p, _i64, _i64,
                                                     _f64p, _i64, _f64p, _cp, ctypes.c_size_t])
        sig["sparse_attention"] = (ctypes.c_int, [_i64, _i64, _f64p, _i64, _f64p, _i64, _f64p, _i64, _i64p, _i64,
                                                  _i64p, _i64, _i64, _f64p, _i64, _f64p, _cp, ctypes.c_size_t])
        sig["combine_scores"] = (None, [_i64, _i64, _f64p, _f64p, ctypes.c_int, _f64p, _f64p])
    else:
        sig["blockwise_attention"] = (ctypes.c_int, [_i64, _i64, _f64p, _i64, _f64p, _i64, _f64p, _i64, _i64,
                                                     _f64p, _i64, _cp, ctypes.c_size_t])
        sig["sparse_attention"] = (ctypes.c_int, [_i64, _i64, _f64p, _i64, _f64p, _i64, _f64p, _i64, _i64p, _i64,
                                                  _i64p, _i64, _i64, _f64p, _i64, _cp, ctypes.c_size_t])
        sig["combine_scores"] = (ctypes.c_int, [_i64, _i64, _f64p, _f64p, ctypes.c_int, _f64p, _f64p, _cp,
                                                ctypes.c_size_t])
        sig["attention_recall"] = (ctypes.c_int, [_i64, _i64, _f64p, _i64, _f64p, _i64, _i64p, _i64, _i64p, _i64,
                                                  _f64p, _cp, ctypes.c_size_t])
        sig["layer_vs_prefill"] = (ctypes.c_int, [_i64, _i64, _i64, _i64, _f64p, _f64p, _f64p, _i64, _f64p, _f64p,
                                                  _f64p, _f64p, _f64p, _f64p, _f64p, _f64p,
                                                  _i64, _i64, _i64, ctypes.c_int, _f64p, _i64p, _i64p, _cp,
                                                  ctypes.c_size_t])
        sig["layer_dense"] = (ctypes.c_int, [_i64, _i64, _i64, _i64, _f64p, _f64p, _f64p, _i64, ctypes.c_int,
                                             _f64p, _cp, ctypes.c_size_t])
        sig["layer_indexer"] = (ctypes.c_int, [_i64, _i64, _i64, _f64p, _f64p, _i64, _f64p, _f64p, _f64p, _f64p,
                                               _f64p, _f64p, ctypes.c_int, _f64p, _f64p, _f64p, _cp,
                                               ctypes.c_size_t])
        sig["layer_select"] = (ctypes.c_int, [_i64, _i64, _f64p, _f64p, _f64p, _f64p, _i64, _i64, _i64,
                                              ctypes.c_int, _i64p, _i64p, _i64p, _i64p, _cp, ctypes.c_size_t])
        sig["layer_sparse"] = (ctypes.c_int, [_i64, _i64, _i64, _i64, _f64p, _f64p, _f64p, _i64p, _i64p, _i64p,
                                              _i64p, _i64, _i64, ctypes.c_int, _f64p, _f64p, _cp, ctypes.c_size_t])
    for name, (res, args) in sig.items():
        fn = getattr(lib, prefix + name)
        fn.restype = res
        fn.argtypes = args
    return lib


def _f(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_f64p)


def _i(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


class _Oracle:
    """numpy front-end over either library; per-head functions take [n, d] arrays."""

    def __init__(self, so: str, prefix: str):
        if not os.path.exists(so):
            build()
        if not os.path.exists(so):
            raise FileNotFoundError(so)
        self.lib = _bind(ctypes.CDLL(so), prefix)
        self.p = prefix
        self.is_ref = prefix == "vspref_"

    def _call(self, name, *args):
        err = ctypes.create_string_buffer(512)
        rc = getattr(self.lib, self.p + name)(*args, err, 512)
        return rc, err.value.decode()

    def _check(self, rc, msg):
        if rc != 0:
            raise OracleError(msg)

    # ---- merge
    def merge_row_columns(self, iv, is_, i):
        iv = np.ascontiguousarray(iv, np.int64)
        is_ = np.ascontiguousarray(is_, np.int64)
        out = np.zeros(len(iv) + len(is_) + 1, np.int64)
        rc, msg = self._call("merge_row_columns", _i(iv), len(iv), _i(is_), len(is_), int(i), _i(out))
        if rc < 0:
            raise OracleError(msg)
        return out[:rc].copy()

    def merge_path_partition(self, a, b, p):
        a = np.ascontiguousarray(a, np.int64)
        b = np.ascontiguousarray(b, np.int64)
        cuts = np.zeros(2 * (max(p, 1) + 1), np.int64)
        rc, msg = self._call("merge_path_partition", _i(a), len(a), _i(b), len(b), int(p), _i(cuts))
        self._check(rc, msg)
        return [tuple(c) for c in cuts.reshape(-1, 2)]

    # ---- attention (one head; q/k/v [n, d] f64)
    def blockwise_attention(self, q, k, v, block=64, want_lse=False):
        q, k, v = (np.ascontiguousarray(x, np.float64) for x in (q, k, v))
        n, d = q.shape
        o = np.zeros((n, d))
        if self.is_ref:
            rc, msg = self._call("blockwise_attention", n, d, _f(q), d, _f(k), d, _f(v), d, block, _f(o), d)
            self._check(rc, msg)
            return o
        lse = np.zeros(n)
        rc, msg = self._call("blockwise_attention", n, d, _f(q), d, _f(k), d, _f(v), d, block, _f(o), d, _f(lse))
        self._check(rc, msg)
        return (o, lse) if want_lse else o

    def sparse_attention(self, q, k, v, iv, is_, block=32, want_lse=False):
        q, k, v = (np.ascontiguousarray(x, np.float64) for x in (q, k, v))
        iv = np.ascontiguousarray(iv, np.int64)
        is_ = np.ascontiguousarray(is_, np.int64)
        n, d = q.shape
        o = np.zeros((n, d))
        if self.is_ref:
            rc, msg = self._call("sparse_attention", n, d, _f(q), d, _f(k), d, _f(v), d, _i(iv), len(iv), _i(is_),
                                 len(is_), block, _f(o), d)
            self._check(rc, msg)
            return o
        lse = np.zeros(n)
        rc, msg = self._call("sparse_attention", n, d, _f(q), d, _f(k), d, _f(v), d, _i(iv), len(iv), _i(is_),
                             len(is_), block, _f(o), d, _f(lse))
        self._check(rc, msg)
        return (o, lse) if want_lse else o

    def attention_recall(self, q, k, iv, is_):
        assert self.is_ref
        q, k = (np.ascontiguousarray(x, np.float64) for x in (q, k))
        iv = np.ascontiguousarray(iv, np.int64)
        is_ = np.ascontiguousarray(is_, np.int64)
        n, d = q.shape
        r = np.zeros(1)
        rc, msg = self._call("attention_recall", n, d, _f(q), d, _f(k), d, _i(iv), len(iv), _i(is_), len(is_), _f(r))
        self._check(rc, msg)
        return float(r[0])

    # ---- selection
    def cumulative_budget(self, scores, tau, tau_v=0.9, tau_s=0.9, min_budget=1, max_budget=-1):
        s = np.ascontiguousarray(scores, np.float64)
        k = np.zeros(1, np.int64)
        rc, msg = self._call("cumulative_budget", _f(s), len(s), float(tau), float(tau_v), float(tau_s),
                             int(min_budget), int(max_budget), _i(k))
        self._check(rc, msg)
        return int(k[0])

    def topk_indices(self, scores, k):
        s = np.ascontiguousarray(scores, np.float64)
        out = np.zeros(max(int(k), 1), np.int64)
        rc, msg = self._call("topk_indices", _f(s), len(s), int(k), _i(out))
        self._check(rc, msg)
        return out[: int(k)].copy()

    def select_pattern(self, sv, ss, tau_v=0.9, tau_s=0.9, min_budget=1, max_budget=-1):
        sv = np.ascontiguousarray(sv, np.float64)
        ss = np.ascontiguousarray(ss, np.float64)
        n = len(sv)
        iv = np.zeros(n + 1, np.int64)
        is_ = np.zeros(n + 1, np.int64)
        kv = np.zeros(1, np.int64)
        ks = np.zeros(1, np.int64)
        rc, msg = self._call("select_pattern", _f(sv), _f(ss), n, float(tau_v), float(tau_s), int(min_budget),
                             int(max_budget), _i(iv), _i(kv), _i(is_), _i(ks))
        self._check(rc, msg)
        return iv[: kv[0]].copy(), is_[: ks[0]].copy()

    # ---- indexer (one KV head): params dict with w_u [2d, d_h], b_u, w_v, b_v, w_s, b_s
    def indexer_forward(self, k, v, params, reverse=True):
        k, v = (np.ascontiguousarray(x, np.float64) for x in (k, v))
        n, d = k.shape
        w_u = np.ascontiguousarray(params["w_u"], np.float64)
        d_h = w_u.shape[1]
        b_u, w_v, w_s = (np.ascontiguousarray(params[x], np.float64) for x in ("b_u", "w_v", "w_s"))
        outs = [np.zeros(n) for _ in range(4)]
        rc, msg = self._call("indexer_forward", n, d, _f(k), d, _f(v), d, d_h, _f(w_u), _f(b_u), _f(w_v),
                             float(params["b_v"]), _f(w_s), float(params["b_s"]), int(bool(reverse)),
                             *[_f(o) for o in outs])
        self._check(rc, msg)
        return dict(logits_v=outs[0], logits_s=outs[1], pred_v=outs[2], pred_s=outs[3])

    # ---- aggregation (one head)
    def aggregate_streaming(self, q, k, block=64, normalized=True):
        q, k = (np.ascontiguousarray(x, np.float64) for x in (q, k))
        n, d = q.shape
        vert = np.zeros(n)
        sl = np.zeros(n)
        rc, msg = self._call("aggregate_streaming", n, d, _f(q), d, _f(k), d, int(block), int(bool(normalized)),
                             _f(vert), _f(sl))
        self._check(rc, msg)
        return vert, sl

    def apply_rope(self, x, positions=None, base=10000.0):
        """x [n, d] f64 -> rotated copy (rope.hpp:63-79)."""
        x = np.ascontiguousarray(x, np.float64)
        n, d = x.shape
        out = np.zeros_like(x)
        pos = None if positions is None else np.ascontiguousarray(positions, np.int64)
        rc, msg = self._call("apply_rope", n, d, _f(x), d, None if pos is None else _i(pos), float(base), _f(out), d)
        self._check(rc, msg)
        return out

    def indexer_backward(self, k, v, params, target_v, target_s, eps=1e-8, reverse=True):
        """-> (loss, grads dict) of the KL distillation loss for one head (indexer.hpp:158-272)."""
        k, v = (np.ascontiguousarray(x, np.float64) for x in (k, v))
        n, d = k.shape
        w_u = np.ascontiguousarray(params["w_u"], np.float64)
        d_h = w_u.shape[1]
        b_u, w_v, w_s = (np.ascontiguousarray(params[x], np.float64) for x in ("b_u", "w_v", "w_s"))
        tv, ts = (np.ascontiguousarray(x, np.float64) for x in (target_v, target_s))
        g = {"w_u": np.zeros_like(w_u), "b_u": np.zeros(d_h), "w_v": np.zeros(d_h), "w_s": np.zeros(d_h)}
        loss, gbv, gbs = np.zeros(1), np.zeros(1), np.zeros(1)
        rc, msg = self._call("indexer_backward", n, d, _f(k), d, _f(v), d, d_h, _f(w_u), _f(b_u), _f(w_v),
                             float(params["b_v"]), _f(w_s), float(params["b_s"]), 1 if reverse else 0, _f(tv), _f(ts),
                             float(eps), _f(loss), _f(g["w_u"]), _f(g["b_u"]), _f(g["w_v"]), _f(gbv), _f(g["w_s"]),
                             _f(gbs))
        self._check(rc, msg)
        g["b_v"], g["b_s"] = float(gbv[0]), float(gbs[0])
        return float(loss[0]), g

    def combine_scores(self, verts, slashes, mean=True):
        v = np.ascontiguousarray(np.stack(verts), np.float64)
        s = np.ascontiguousarray(np.stack(slashes), np.float64)
        h, n = v.shape
        vo = np.zeros(n)
        so = np.zeros(n)
        if self.is_ref:
            rc, msg = self._call("combine_scores", h, n, _f(v), _f(s), int(bool(mean)), _f(vo), _f(so))
            self._check(rc, msg)
        else:
            getattr(self.lib, "vso_combine_scores")(h, n, _f(v), _f(s), int(bool(mean)), _f(vo), _f(so))
        return vo, so

    # ---- whole layer through the reference API (ref only), threaded over heads
    def layer_vs_prefill(self, q, k, v, params, tau_v, tau_s, min_budget, max_budget, block=32, threads=1):
        """tau_v / tau_s: scalars or one value per KV head."""
        assert self.is_ref
        n, hq, d = q.shape
        hkv = k.shape[1]
        tau_v = np.ascontiguousarray(np.broadcast_to(np.asarray(tau_v, np.float64), (hkv,)))
        tau_s = np.ascontiguousarray(np.broadcast_to(np.asarray(tau_s, np.float64), (hkv,)))
        q, k, v = (np.ascontiguousarray(x, np.float64) for x in (q, k, v))
        w_u = np.ascontiguousarray(params["w_u"], np.float64)
        d_h = w_u.shape[2]
        b_u, w_v, w_s, b_v, b_s = (np.ascontiguousarray(params[x], np.float64) for x in ("b_u", "w_v", "w_s",
                                                                                            "b_v", "b_s"))
        o = np.zeros((n, hq, d))
        kv = np.zeros(hkv, np.int64)
        ks = np.zeros(hkv, np.int64)
        rc, msg = self._call("layer_vs_prefill", n, hq, hkv, d, _f(q), _f(k), _f(v), d_h, _f(w_u), _f(b_u), _f(w_v),
                             _f(b_v), _f(w_s), _f(b_s), _f(tau_v), _f(tau_s), int(min_budget),
                             int(max_budget), int(block), int(threads), _f(o), _i(kv), _i(ks))
        self._check(rc, msg)
        return o, kv, ks

    def layer_dense(self, q, k, v, block=64, threads=1):
        assert self.is_ref
        n, hq, d = q.shape
        hkv = k.shape[1]
        q, k, v = (np.ascontiguousarray(x, np.float64) for x in (q, k, v))
        o = np.zeros((n, hq, d))
        rc, msg = self._call("layer_dense", n, hq, hkv, d, _f(q), _f(k), _f(v), int(block), int(threads), _f(o))
        self._check(rc, msg)
        return o


    # ---- the layer in stages (ref only): bounded samples for bench.py's reference arm
    def layer_indexer(self, k, v, params, threads=1, head_s=None):
        """indexer_forward of every KV head over all rows of k/v [len, hkv, d] -> (A_v, A_s) [hkv, len].
        head_s (optional f64 [hkv]) receives each head's call time on its worker thread."""
        assert self.is_ref
        ln, hkv, d = k.shape
        k, v = (np.ascontiguousarray(x, np.float64) for x in (k, v))
        w_u = np.ascontiguousarray(params["w_u"], np.float64)
        b_u, w_v, w_s, b_v, b_s = (np.ascontiguousarray(params[x], np.float64)
                                   for x in ("b_u", "w_v", "w_s", "b_v", "b_s"))
        pv = np.zeros((hkv, ln))
        ps = np.zeros((hkv, ln))
        rc, msg = self._call("layer_indexer", ln, hkv, d, _f(k), _f(v), w_u.shape[2], _f(w_u), _f(b_u), _f(w_v),
                             _f(b_v), _f(w_s), _f(b_s), int(threads), _f(pv), _f(ps),
                             _f(head_s) if head_s is not None else None)
        self._check(rc, msg)
        return pv, ps

    def layer_select(self, pred_v, pred_s, tau_v, tau_s, min_budget=1, max_budget=-1, threads=1):
        """select_pattern of every KV head -> (i_v [hkv, cap], k_v [hkv], i_s, k_s), cap = n + 1."""
        assert self.is_ref
        pred_v, pred_s = (np.ascontiguousarray(x, np.float64) for x in (pred_v, pred_s))
        hkv, n = pred_v.shape
        tau_v = np.ascontiguousarray(np.broadcast_to(np.asarray(tau_v, np.float64), (hkv,)))
        tau_s = np.ascontiguousarray(np.broadcast_to(np.asarray(tau_s, np.float64), (hkv,)))
        cap = n + 1
        iv = np.zeros((hkv, cap), np.int64)
        is_ = np.zeros((hkv, cap), np.int64)
        kv = np.zeros(hkv, np.int64)
        ks = np.zeros(hkv, np.int64)
        rc, msg = self._call("layer_select", n, hkv, _f(pred_v), _f(pred_s), _f(tau_v), _f(tau_s), int(min_budget),
                             int(max_budget), cap, int(threads), _i(iv), _i(kv), _i(is_), _i(ks))
        self._check(rc, msg)
        return iv, kv, is_, ks

    def layer_sparse(self, q, k, v, iv, kv, is_, ks, rows=None, block=32, threads=1, head_s=None):
        """sparse_attention of every Q head over rows [0, rows) (q/k/v hold at least `rows`
        tokens) with per-KV-head patterns (i_v [hkv, cap] ...) -> O [rows, hq, d]."""
        assert self.is_ref
        rows = q.shape[0] if rows is None else rows
        _, hq, d = q.shape
        hkv = k.shape[1]
        q, k, v = (np.ascontiguousarray(x[:rows], np.float64) for x in (q, k, v))
        iv, kv, is_, ks = (np.ascontiguousarray(x, np.int64) for x in (iv, kv, is_, ks))
        o = np.zeros((rows, hq, d))
        rc, msg = self._call("layer_sparse", rows, hq, hkv, d, _f(q), _f(k), _f(v), _i(iv), _i(kv), _i(is_), _i(ks),
                             iv.shape[1], int(block), int(threads), _f(o), _f(head_s) if head_s is not None else None)
        self._check(rc, msg)
        return o


_cache: dict = {}


def port() -> _Oracle:
    if "port" not in _cache:
        _cache["port"] = _Oracle(PORT_SO, "vso_")
    return _cache["port"]


def ref() -> _Oracle:
    """The reference itself (raises FileNotFoundError if it was never built)."""
    if "ref" not in _cache:
        _cache["ref"] = _Oracle(REF_SO, "vspref_")
    return _cache["ref"]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


# ---------------------------------------------------------------------- interchange formats
# The reference's own VSTN / VSCK / index-text writers and readers (tensor_io.hpp,
# indexer.hpp:450-499, sparsity.hpp:187-245) through oracle/_ref; used only to pin the
# C-ABI implementations in csrc/formats.cpp (tests/test_formats.py, make_format_golden.py).

class RefFormats:
    """Returns (kind, value): kind "ok" or the reference's exception type
    ("invalid_argument" / "runtime_error") with its message as value."""

    def __init__(self):
        lib = ctypes.CDLL(REF_SO)
        cp, sz, i64, f64 = ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_double
        lib.vspref_write_matrix.argtypes = [cp, i64, i64, _f64p, cp, sz]
        lib.vspref_write_vector.argtypes = [cp, i64, _f64p, cp, sz]
        lib.vspref_read_tensor.argtypes = [cp, ctypes.c_int, _i64p, _f64p, i64, cp, sz]
        lib.vspref_save_checkpoint.argtypes = [cp, i64, i64, _f64p, _f64p, _f64p, f64, _f64p, f64, cp, sz]
        lib.vspref_load_checkpoint.argtypes = [cp, _i64p, i64, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, cp, sz]
        lib.vspref_write_indices.argtypes = [cp, _i64p, i64, _i64p, i64, cp, sz]
        lib.vspref_read_indices.argtypes = [cp, _i64p, _i64p, _i64p, _i64p, i64, cp, sz]
        self.lib = lib

    @staticmethod
    def _res(rc, err, value=None):
        if rc == 0:
            return "ok", value
        return ("invalid_argument" if rc == 1 else "runtime_error"), err.value.decode()

    def write_matrix(self, path, m):
        m = np.ascontiguousarray(m, np.float64)
        err = ctypes.create_string_buffer(512)
        return self._res(self.lib.vspref_write_matrix(os.fsencode(path), m.shape[0], m.shape[1], _f(m), err, 512), err)

    def write_vector(self, path, v):
        v = np.ascontiguousarray(v, np.float64)
        err = ctypes.create_string_buffer(512)
        return self._res(self.lib.vspref_write_vector(os.fsencode(path), v.size, _f(v), err, 512), err)

    def read(self, path, rank):
        cap = max(os.path.getsize(path) // 8, 1) if os.path.exists(path) else 1
        shape = np.zeros(2, np.int64)
        data = np.zeros(cap, np.float64)
        err = ctypes.create_string_buffer(512)
        rc = self.lib.vspref_read_tensor(os.fsencode(path), rank, _i(shape), _f(data), cap, err, 512)
        if rc:
            return self._res(rc, err)
        shp = (int(shape[0]), int(shape[1])) if rank == 2 else (int(shape[0]),)
        return "ok", data[:int(np.prod(shp))].reshape(shp)

    def save_checkpoint(self, path, w_u, b_u, w_v, b_v, w_s, b_s):
        w_u = np.ascontiguousarray(w_u, np.float64)
        b_u, w_v, w_s = (np.ascontiguousarray(x, np.float64) for x in (b_u, w_v, w_s))
        err = ctypes.create_string_buffer(512)
        rc = self.lib.vspref_save_checkpoint(os.fsencode(path), w_u.shape[0], w_u.shape[1], _f(w_u), _f(b_u),
                                             _f(w_v), float(b_v), _f(w_s), float(b_s), err, 512)
        return self._res(rc, err)

    def load_checkpoint(self, path):
        dims = np.zeros(2, np.int64)
        err = ctypes.create_string_buffer(512)
        z = np.zeros(1)
        bv, bs = np.zeros(1), np.zeros(1)
        rc = self.lib.vspref_load_checkpoint(os.fsencode(path), _i(dims), 0, _f(z), _f(z), _f(z), _f(bv), _f(z),
                                             _f(bs), err, 512)
        if rc:
            return self._res(rc, err)
        in_dim, dh = int(dims[0]), int(dims[1])
        w_u, b_u, w_v, w_s = np.zeros((in_dim, dh)), np.zeros(dh), np.zeros(dh), np.zeros(dh)
        rc = self.lib.vspref_load_checkpoint(os.fsencode(path), _i(dims), dh, _f(w_u), _f(b_u), _f(w_v), _f(bv),
                                             _f(w_s), _f(bs), err, 512)
        return self._res(rc, err, {"w_u": w_u, "b_u": b_u, "w_v": w_v, "b_v": float(bv[0]), "w_s": w_s,
                                   "b_s": float(bs[0])})

    def write_indices(self, path, iv, is_):
        a = np.ascontiguousarray(iv, np.int64)
        b = np.ascontiguousarray(is_, np.int64)
        err = ctypes.create_string_buffer(512)
        return self._res(self.lib.vspref_write_indices(os.fsencode(path), _i(a), a.size, _i(b), b.size, err, 512),
                         err)

    def read_indices(self, path):
        cap = max(os.path.getsize(path), 1) if os.path.exists(path) else 1
        a, b = np.zeros(cap, np.int64), np.zeros(cap, np.int64)
        kv, ks = np.zeros(1, np.int64), np.zeros(1, np.int64)
        err = ctypes.create_string_buffer(512)
        rc = self.lib.vspref_read_indices(os.fsencode(path), _i(a), _i(kv), _i(b), _i(ks), cap, err, 512)
        return self._res(rc, err, (a[:int(kv[0])].tolist(), b[:int(ks[0])].tolist()))


def ref_formats() -> RefFormats:
    if "fmt" not in _cache:
        _cache["fmt"] = RefFormats()
    return _cache["fmt"]


def adamw_step(p, g, m, v, step_index, lr, beta1=0.9, beta2=0.999, adam_eps=1e-8, weight_decay=0.01):
    """optimizer_step (indexer.hpp:347-363) on flat f64 arrays, in place (the C restatement)."""
    lib = port().lib
    lib.vso_adamw_step(p.size, _f(p), _f(g), _f(m), _f(v), int(step_index), float(lr), beta1, beta2, adam_eps,
                       weight_decay)


def ref_optimizer_step(d, d_h, p, g, m, v, step, steps, warmup, lr_peak):
    """The reference's optimizer_step on one head (flat W_U | b_U | w_v | b_v | w_s | b_s), in place."""
    lib = ctypes.CDLL(REF_SO)
    f = lib.vspref_optimizer_step
    f.argtypes = [_i64, _i64, _f64p, _f64p, _f64p, _f64p, _i64, _i64, _i64, ctypes.c_double, _cp, ctypes.c_size_t]
    err = ctypes.create_string_buffer(512)
    if f(d, d_h, _f(p), _f(g), _f(m), _f(v), step, steps, warmup, lr_peak, err, 512):
        raise OracleError(err.value.decode())


def ref_learning_rate(step, steps, warmup, lr_peak):
    lib = ctypes.CDLL(REF_SO)
    lib.vspref_learning_rate.restype = ctypes.c_double
    lib.vspref_learning_rate.argtypes = [_i64, _i64, _i64, ctypes.c_double]
    return lib.vspref_learning_rate(step, steps, warmup, lr_peak)
