"""Config-level parity: the whole GPU layer against the reference itself at BASELINE.json's
parity config C1, and against the masked-softmax oracle on sampled rows of the 128k bench
layer (config[2]) with the bench's real distilled pattern.

C1 (BASELINE.json configs[0]): one attention layer, Qwen3-4B geometry (32 Q /
8 KV heads, d = 128), n = 4096, N(0, 1) Q/K/V in bf16 (the CPU side gets the same values
widened to f64), random-init VSIndexer with d_h = 1024 (make_indexer_params, indexer.hpp:53-64,
heads ~ N(0, 0.3^2)), fixed top-k budget min = max = 256. Every output is compared with the
UNMODIFIED reference (oracle/_ref), run on all heads with host threads:
  * A_v / A_s and the logits vs indexer_forward (indexer.hpp:116-120): logits |d| <= 3e-2,
    A relative <= 5e-2 on entries >= 1e-6;
  * I_v / I_s bit-exact vs select_pattern (sparsity.hpp:105-114) fed the GPU scores widened
    to f64, and close to the reference's own selection on its own f64 scores;
  * O vs sparse_attention (attention.hpp:150-194) on the same pattern and vs
    blockwise_attention (:96-145) for the dense kernel: max |d| <= 2e-2, mean <= 2e-3; LSE vs
    the pinned C restatement (the reference returns no LSE): |d| <= 1e-3;
  * the one-call layer (vsp_vs_prefill) equals the operator chain bit for bit.
"""
import concurrent.futures as cf
import os
import sys

import numpy as np
import pytest
import torch

import oracle
from helpers import f64

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def vsp():
    import paper_2603_04460_b200 as m
    m.load_library()
    return m


def _threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _pool_map(fn, items):
    with cf.ThreadPoolExecutor(max_workers=min(_threads(), len(items))) as ex:  # ctypes drops the GIL
        return list(ex.map(fn, items))


@pytest.fixture(scope="module")
def c1(vsp):
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    n, hq, hkv, d_h, k_top = 4096, 32, 8, 1024, 256
    g = torch.Generator().manual_seed(41)
    q = torch.randn(n, hq, 128, generator=g).to(torch.bfloat16).cuda()
    k = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    params = vsp.make_indexer_params(hkv, 128, d_h, torch.Generator().manual_seed(42), head_sigma=0.3)
    budget = vsp.BudgetConfig(0.9, 0.9, k_top, k_top)
    a_v, a_s, l_v, l_s = vsp.indexer_forward(k, v, params, want_logits=True)
    pat = vsp.select_pattern(a_v, a_s, budget)
    o, lse = vsp.sparse_attention(q, k, v, pat)
    o_d, lse_d = vsp.blockwise_attention(q, k, v)
    o1, lse1, pat1 = vsp.vs_prefill(q, k, v, params, budget)
    torch.cuda.synchronize()
    prm = {f: f64(getattr(params, f)) for f in ("w_u", "b_u", "w_v", "b_v", "w_s", "b_s")}
    return dict(n=n, hq=hq, hkv=hkv, k_top=k_top, q=q, k=k, v=v, params=params, prm=prm, a_v=a_v, a_s=a_s,
                l_v=l_v, l_s=l_s, pat=pat, o=o, lse=lse, o_d=o_d, lse_d=lse_d, o1=o1, lse1=lse1, pat1=pat1)


def test_c1_indexer_vs_reference(c1):
    ref = oracle.ref()
    kn, vn = f64(c1["k"]), f64(c1["v"])
    prm = c1["prm"]

    def head(gi):
        p = {f: (x[gi] if x.ndim > 1 else float(x[gi])) for f, x in prm.items()}
        return ref.indexer_forward(kn[:, gi], vn[:, gi], p)

    outs = _pool_map(head, list(range(c1["hkv"])))
    for gi, r in enumerate(outs):
        for name, got, want in (("logit_v", c1["l_v"][gi], r["logits_v"]), ("logit_s", c1["l_s"][gi], r["logits_s"])):
            err = np.abs(f64(got) - want).max()
            assert err <= 3e-2, f"head {gi} {name} max|d| {err:.3e}"
        for name, got, want in (("A_v", c1["a_v"][gi], r["pred_v"]), ("A_s", c1["a_s"][gi], r["pred_s"])):
            got = f64(got)
            m = want >= 1e-6
            rel = (np.abs(got - want)[m] / want[m]).max()
            assert rel <= 5e-2, f"head {gi} {name} rel {rel:.3e}"
            assert abs(got.sum() - 1.0) <= 1e-6


def test_c1_selection_bit_exact_vs_reference(c1):
    ref = oracle.ref()
    k_top = c1["k_top"]
    iv, kv, is_, ks = ref.layer_select(f64(c1["a_v"]), f64(c1["a_s"]), 0.9, 0.9, k_top, k_top, threads=_threads())
    for gi in range(c1["hkv"]):
        got_v, got_s = c1["pat"].lists(gi)
        assert got_v == iv[gi, : kv[gi]].tolist(), f"head {gi} I_v"
        assert got_s == is_[gi, : ks[gi]].tolist(), f"head {gi} I_s"
        assert kv[gi] == k_top and ks[gi] in (k_top, k_top + 1)


def test_c1_selection_close_to_reference_own_scores(c1):
    """The reference's whole front half in f64 (its own scores, its own selection) picks
    nearly the same sets: only entries whose score rank crosses position 256 under the bf16
    rounding of K/V/W_U may differ."""
    ref = oracle.ref()
    pv, ps = ref.layer_indexer(f64(c1["k"]), f64(c1["v"]), c1["prm"], threads=_threads())
    iv, kv, is_, ks = ref.layer_select(pv, ps, 0.9, 0.9, c1["k_top"], c1["k_top"], threads=_threads())
    for gi in range(c1["hkv"]):
        got_v, got_s = (set(x) for x in c1["pat"].lists(gi))
        jv = len(got_v & set(iv[gi, : kv[gi]].tolist())) / len(got_v | set(iv[gi, : kv[gi]].tolist()))
        js = len(got_s & set(is_[gi, : ks[gi]].tolist())) / len(got_s | set(is_[gi, : ks[gi]].tolist()))
        assert jv >= 0.9 and js >= 0.9, (gi, jv, js)


def test_c1_sparse_attention_vs_reference(c1):
    ref = oracle.ref()
    pat = c1["pat"]
    cap = pat.i_v.shape[1]
    iv = pat.i_v.cpu().numpy().astype(np.int64)
    is_ = pat.i_s.cpu().numpy().astype(np.int64)
    kv = pat.k_v.cpu().numpy().astype(np.int64)
    ks = pat.k_s.cpu().numpy().astype(np.int64)
    assert iv.shape[1] == cap
    o_ref = ref.layer_sparse(f64(c1["q"]), f64(c1["k"]), f64(c1["v"]), iv, kv, is_, ks, threads=_threads())
    err = np.abs(f64(c1["o"]) - o_ref)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3, (err.max(), err.mean())
    # LSE: the reference returns O only; its pinned C restatement returns the row LSE
    port = oracle.port()
    qn, kn, vn = f64(c1["q"]), f64(c1["k"]), f64(c1["v"])
    grp = c1["hq"] // c1["hkv"]

    def head(h):
        gi = h // grp
        l_v, l_s = pat.lists(gi)
        return port.sparse_attention(qn[:, h], kn[:, gi], vn[:, gi], l_v, l_s, want_lse=True)[1]

    lse_ref = np.stack(_pool_map(head, list(range(c1["hq"]))))
    le = np.abs(f64(c1["lse"]) - lse_ref).max()
    assert le <= 1e-3, le


def test_c1_dense_attention_vs_reference(c1):
    o_ref = oracle.ref().layer_dense(f64(c1["q"]), f64(c1["k"]), f64(c1["v"]), block=64, threads=_threads())
    err = np.abs(f64(c1["o_d"]) - o_ref)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3, (err.max(), err.mean())


def test_c1_one_call_layer_equals_operator_chain(c1):
    assert torch.equal(c1["pat1"].k_v, c1["pat"].k_v) and torch.equal(c1["pat1"].k_s, c1["pat"].k_s)
    for gi in range(c1["hkv"]):
        assert c1["pat1"].lists(gi) == c1["pat"].lists(gi)
    assert torch.equal(c1["o1"], c1["o"]) and torch.equal(c1["lse1"], c1["lse"])


def _event_ms(fn, reps=20, rounds=5):
    """Device time per call: `reps` calls back to back between two events (the host runs
    ahead, so host-side launch cost is not counted), median over `rounds`."""
    fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / reps)
    return float(np.median(times))


def test_c1_dense_switch_rows_and_speed(vsp, c1):
    """VSP_DENSE_SWITCH (opt-in): a query block whose vertical-slash tiles would
    visit every causal tile (plan count == qb + 1) runs unmasked causal attention, so its rows
    equal the dense kernel's (blockwise_attention, attention.hpp:96-145) bit for bit; every
    other block keeps the exact sparse result. At C1 (tile density ~0.99, random pattern) the
    masked call costs ~1.35x K4's time; with the switch it must reach 0.80x K4's speed (measured
    0.88-0.91 on B200 boxes: the K3 kernel itself runs ~8% behind K4 on identical tiles at this size —
    more instructions and i-cache misses — plus the 7.6 us planning launch)."""
    q, k, v, pat = c1["q"], c1["k"], c1["v"], c1["pat"]
    n, hq, hkv = c1["n"], c1["hq"], c1["hkv"]
    grp = hq // hkv
    o_sw, lse_sw = vsp.sparse_attention(q, k, v, pat, validate=False, dense_switch=True)
    counts = vsp.sparse_tile_counts(n, hkv, pat.i_v.shape[1], q.device).cpu()  # [hkv, num_qb]
    torch.cuda.synchronize()
    num_qb = (n + 127) // 128
    dense = counts == torch.arange(1, num_qb + 1).unsqueeze(0)
    assert dense.float().mean() > 0.9, "C1's random pattern should put almost every block in dense mode"
    for g in range(hkv):
        for qb in range(num_qb):
            r = slice(qb * 128, min(n, qb * 128 + 128))
            want_o, want_l = (c1["o_d"], c1["lse_d"]) if dense[g, qb] else (c1["o"], c1["lse"])
            hs = slice(g * grp, (g + 1) * grp)
            assert torch.equal(o_sw[r, hs], want_o[r, hs]), (g, qb, bool(dense[g, qb]))
            assert torch.equal(lse_sw[hs, r], want_l[hs, r]), (g, qb, bool(dense[g, qb]))
    o_buf, l_buf = torch.empty_like(o_sw), torch.empty_like(lse_sw)
    t_dense = _event_ms(lambda: vsp.blockwise_attention(q, k, v, out=o_buf, lse=l_buf))
    t_sw = _event_ms(lambda: vsp.sparse_attention(q, k, v, pat, validate=False, out=o_buf, lse=l_buf,
                                                  dense_switch=True))
    assert t_dense / t_sw >= 0.80, f"dense-switch call {t_sw:.4f} ms vs K4 {t_dense:.4f} ms"


# --------------------------------------------------------------------------- 128k sampled rows

def _masked_softmax_rows(qrows, kn, vn, iv, is_, rows, scale):
    """Exact f64 masked softmax of the given rows: columns = merge_row_columns (the pinned
    C restatement of merge.hpp:18-56), then softmax over q_i . k_j * scale (attention.hpp:150-194)."""
    port = oracle.port()
    o = np.zeros((len(rows), vn.shape[1]))
    lse = np.zeros(len(rows))
    for t, i in enumerate(rows):
        cols = port.merge_row_columns(iv, is_, int(i))
        s = kn[cols] @ qrows[t] * scale
        m = s.max()
        w = np.exp(s - m)
        lse[t] = m + np.log(w.sum())
        o[t] = (w[:, None] * vn[cols]).sum(0) / w.sum()
    return o, lse


def test_bench_layer_128k_sampled_rows_vs_oracle(vsp):
    """The bench's own layer (config[2]: n = 131072, 32/8 heads, distilled indexer and per-head
    budgets from bench_data/, the held-out prompt): 64 rows per Q head spread over the
    sequence, GPU O / LSE vs the exact masked softmax of the same pattern."""
    sys.path.insert(0, ROOT)
    import bench
    args = bench.parse([])
    got = bench.load_prep(args)
    if got is None:
        pytest.skip("bench_data/ holds no preparation for the default bench flags")
    prm, budgets, _ = got
    dev = torch.device("cuda")
    params = bench.params_to_device(prm, dev)
    budget = [vsp.BudgetConfig(tv, ts, args.min_budget, None) for tv, ts in budgets]
    qh, kh, vh = bench.synth_layer(args, "cpu")
    q, k, v = qh.to(dev), kh.to(dev), vh.to(dev)
    o, lse, pat = vsp.vs_prefill(q, k, v, params, budget)
    torch.cuda.synchronize()
    n, hq, _ = q.shape
    hkv = k.shape[1]
    grp = hq // hkv
    rng = np.random.default_rng(7)
    base = np.linspace(0, n - 1, 64).astype(np.int64)
    rows = np.unique(np.clip(base + rng.integers(-60, 60, size=64), 0, n - 1))
    rows[0], rows[-1] = 0, n - 1
    rows = np.unique(rows)
    qn = qh[rows].float().numpy().astype(np.float64)  # [rows, hq, d]
    kn = kh.float().numpy().astype(np.float64)
    vn = vh.float().numpy().astype(np.float64)
    og = o[torch.from_numpy(rows).to(dev)].float().cpu().numpy()
    lg = lse[:, torch.from_numpy(rows).to(dev)].cpu().numpy()
    scale = 1.0 / np.sqrt(128.0)

    def head(h):
        gi = h // grp
        iv, is_ = pat.lists(gi)
        return _masked_softmax_rows(qn[:, h], kn[:, gi], vn[:, gi], np.array(iv), np.array(is_), rows, scale)

    res = _pool_map(head, list(range(hq)))
    worst_o, worst_l, mean_o = 0.0, 0.0, []
    for h, (o_ref, l_ref) in enumerate(res):
        e = np.abs(og[:, h] - o_ref)
        worst_o = max(worst_o, float(e.max()))
        mean_o.append(float(e.mean()))
        worst_l = max(worst_l, float(np.abs(lg[h] - l_ref).max()))
    assert worst_o <= 2e-2, worst_o
    assert float(np.mean(mean_o)) <= 2e-3, np.mean(mean_o)
    assert worst_l <= 1e-3, worst_l
    assert int(pat.k_v.max()) > 1000  # the real distilled pattern: thousands of verticals on some heads
