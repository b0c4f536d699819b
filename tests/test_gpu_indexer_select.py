"""GPU parity of K1 (indexer scoring) and K2 (selection) against the oracle.

K1 mirrors test_indexer.cpp: ZeroHeadsGiveUniformPredictions :101-111, SingleTokenIsCertain
:113-121, MatchesStraightLineOracle :123-142, SlashMappingAnchorsAtLastToken :144-167.
Tolerances (bf16 K, V, W_U; fp32 accumulation): logits |d| <= 3e-2, A relative <= 5e-2 on
entries >= 1e-6, and sum(A) = 1 +- 1e-6.

K2 mirrors test_sparsity.cpp (DyadicHandValues :22-32, ClampsToMinAndMax :34-46,
TopK.HandValuesWithTies :93-104, MatchesFullSortOracle :116-126, SelectPattern.* :133-167):
index sets must be BIT-EXACT with select_pattern run on the same fp32 scores widened to f64.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from helpers import f64

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))["cases"]


@pytest.fixture(scope="module")
def vsp():
    import paper_2603_04460_b200 as m
    m.load_library()
    return m


def _params(vsp, hkv, d_h, seed, sigma=0.3, bias=0.3):
    g = torch.Generator().manual_seed(seed)
    p = vsp.make_indexer_params(hkv, 128, d_h, g, head_sigma=sigma)
    p.b_u = (torch.randn(hkv, d_h, generator=g) * bias).cuda()
    p.b_v = torch.tensor([0.1 * (i + 1) for i in range(hkv)]).cuda()
    p.b_s = torch.tensor([-0.2 * (i + 1) for i in range(hkv)]).cuda()
    return p


def _oracle_indexer(k, v, p, g, reverse=True):
    prm = dict(w_u=f64(p.w_u[g]), b_u=f64(p.b_u[g]), w_v=f64(p.w_v[g]), b_v=float(p.b_v[g]), w_s=f64(p.w_s[g]),
               b_s=float(p.b_s[g]))
    return oracle.port().indexer_forward(f64(k[:, g]), f64(v[:, g]), prm, reverse=reverse)


@pytest.mark.parametrize("n,hkv,d_h,mapping", [(300, 2, 256, "reverse"), (1000, 1, 1024, "identity"),
                                               (129, 2, 512, "reverse")])
def test_indexer_matches_oracle(vsp, n, hkv, d_h, mapping):
    g = torch.Generator().manual_seed(n)
    k = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    p = _params(vsp, hkv, d_h, seed=n)
    a_v, a_s, lv, ls = vsp.indexer_forward(k, v, p, mapping=mapping, want_logits=True)
    torch.cuda.synchronize()
    for h in range(hkv):
        r = _oracle_indexer(k, v, p, h, reverse=(mapping == "reverse"))
        assert np.abs(f64(lv[h]) - r["logits_v"]).max() <= 3e-2
        assert np.abs(f64(ls[h]) - r["logits_s"]).max() <= 3e-2
        for got, want in ((a_v[h], r["pred_v"]), (a_s[h], r["pred_s"])):
            gg = f64(got)
            assert abs(gg.sum() - 1.0) <= 1e-6
            m = want >= 1e-6
            assert (np.abs(gg[m] - want[m]) / want[m]).max() <= 5e-2


def test_indexer_zero_heads_uniform_and_single_token(vsp):
    n, hkv = 777, 2
    g = torch.Generator().manual_seed(1)
    k = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    p = vsp.make_indexer_params(hkv, 128, 256, g, head_sigma=0.0)
    a_v, a_s = vsp.indexer_forward(k, v, p)
    want = np.float32(1.0 / n)
    assert (a_v.cpu().numpy() == want).all() and (a_s.cpu().numpy() == want).all()
    a_v1, a_s1 = vsp.indexer_forward(k[:1].contiguous(), v[:1].contiguous(), p)
    assert (a_v1.cpu().numpy() == 1.0).all() and (a_s1.cpu().numpy() == 1.0).all()


@pytest.mark.parametrize("n", [9, 4099, 300001])
def test_indexer_softmax_exact_normaliser(vsp, n):
    """A_v / A_s are the fp32 rounding of softmax(logits) with an fp64 normaliser (at n past
    the shared-memory-cached slice size too): compare with float64 softmax of the logits."""
    hkv = 1
    g = torch.Generator().manual_seed(n)
    k = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    p = vsp.make_indexer_params(hkv, 128, 256, g, head_sigma=1.0)
    a_v, a_s, lv, ls = vsp.indexer_forward(k, v, p, want_logits=True)
    for a, lg in ((a_v, lv), (a_s, ls)):
        want = torch.softmax(lg.double(), dim=1)
        got = a.double()
        assert abs(float(got.sum()) - 1.0) <= 1e-6
        # fp32 exp of the fp32 difference (x - max): relative error <= ~2^-24 * |x - max| + 2 ulp
        rel_tol = 4e-7 * max(1.0, float((lg - lg.max()).abs().max()))
        assert float(((got - want).abs() / want.clamp_min(1e-30)).max()) <= rel_tol


def test_indexer_slash_mapping_anchor(vsp):
    """One hidden unit carrying K feature 0 = t: Reverse puts silu(n-1-o) at offset o."""
    n, d_h = 40, 256
    k = torch.zeros(n, 1, 128)
    k[:, 0, 0] = torch.arange(n, dtype=torch.float32)
    k = k.to(torch.bfloat16).cuda()
    v = torch.zeros(n, 1, 128, dtype=torch.bfloat16, device="cuda")
    w_u = torch.zeros(1, 256, d_h)
    w_u[0, 0, 0] = 1.0
    z = torch.zeros(1, d_h, device="cuda")
    w_s = torch.zeros(1, d_h, device="cuda")
    w_s[0, 0] = 1.0
    p = vsp.IndexerParams(w_u.to(torch.bfloat16).cuda(), z, z.clone(), torch.zeros(1, device="cuda"), w_s,
                          torch.zeros(1, device="cuda"))
    silu = lambda x: x / (1 + math.exp(-x))  # noqa: E731
    _, a_rev, _, ls_rev = vsp.indexer_forward(k, v, p, "reverse", want_logits=True)
    _, a_id, _, ls_id = vsp.indexer_forward(k, v, p, "identity", want_logits=True)
    for o in range(n):
        assert abs(ls_rev[0, o].item() - silu(n - 1 - o)) <= 1e-4 * max(1, n - 1 - o)
        assert abs(ls_id[0, o].item() - silu(o)) <= 1e-4 * max(1, o)
    assert int(a_rev[0].argmax()) == 0 and int(a_id[0].argmax()) == n - 1


# ------------------------------------------------------------------------- selection

def _select_gpu(vsp, sv, ss, budget):
    a_v = torch.tensor(np.asarray(sv, np.float32)).reshape(1, -1).cuda()
    a_s = torch.tensor(np.asarray(ss, np.float32)).reshape(1, -1).cuda()
    pat = vsp.select_pattern(a_v, a_s, budget)
    return pat.lists(0)


def _budget(vsp, tau_v, tau_s, mn=1, mx=-1):
    return vsp.BudgetConfig(tau_v, tau_s, mn, None if mx < 0 else mx)


def test_select_golden_exact_cases(vsp):
    """Cases whose scores are exact in fp32 compare directly against the reference's output."""
    for c in GOLD["select_pattern"][:2]:
        iv, is_ = _select_gpu(vsp, c["sv"], c["ss"], _budget(vsp, c["tau_v"], c["tau_s"], c["min"], c["max"]))
        assert iv == c["i_v"] and is_ == c["i_s"]


def test_select_dyadic_budget_table(vsp):
    s = [0.5, 0.25, 0.125, 0.125]
    for tau, k in ((0.5, 1), (0.6, 2), (0.75, 2), (0.76, 3), (0.875, 3), (0.9, 4), (1.0, 4)):
        iv, _ = _select_gpu(vsp, s, s, _budget(vsp, tau, 0.5))
        assert len(iv) == k, (tau, iv)
    iv, _ = _select_gpu(vsp, s, s, _budget(vsp, 0.5, 0.5, 3))
    assert len(iv) == 3
    iv, _ = _select_gpu(vsp, s, s, _budget(vsp, 1.0, 0.5, 1, 2))
    assert iv == [0, 1]


def test_select_ties_low_index(vsp):
    # TopK.HandValuesWithTies via a budget pinned to k (min = max = k)
    for scores, k, want in (([0.2, 0.5, 0.2, 0.1], 2, [0, 1]), ([0.2, 0.5, 0.2, 0.1], 3, [0, 1, 2]),
                            ([0.3, 0.2, 0.2, 0.3], 2, [0, 3]), ([0.3, 0.2, 0.2, 0.3], 3, [0, 1, 3]),
                            ([0.1, 0.4, 0.4, 0.1], 2, [1, 2])):
        iv, is_ = _select_gpu(vsp, scores, scores, _budget(vsp, 0.5, 0.5, k, k))
        assert iv == want
        assert is_ == (want if want[0] == 0 else [0] + want)


def _check_against_oracle(vsp, a_v, a_s, budgets):
    pat = vsp.select_pattern(a_v, a_s, budgets)
    port = oracle.port()
    for g in range(a_v.shape[0]):
        b = budgets[g]
        want_v, want_s = port.select_pattern(f64(a_v[g]), f64(a_s[g]), b.tau_v, b.tau_s, b.min_budget,
                                             -1 if b.max_budget is None else b.max_budget)
        got_v, got_s = pat.lists(g)
        assert got_v == want_v.tolist(), f"head {g} vertical"
        assert got_s == want_s.tolist(), f"head {g} slash"
    return pat


@pytest.mark.parametrize("n", [1, 2, 37, 5000, 131072, 300001])
def test_select_matches_oracle_random(vsp, n):
    rng = np.random.default_rng(n)
    hkv = 4
    sig = torch.tensor(rng.uniform(0.1, 4.0, size=(hkv, 1)), dtype=torch.float64)
    # f64 softmax then fp32: sums stay within 1e-6 of 1 (the reference's check) at any n
    a_v = torch.softmax(torch.randn(hkv, n, generator=torch.Generator().manual_seed(n), dtype=torch.float64) * sig,
                        dim=1).float().cuda()
    a_s = torch.softmax(torch.randn(hkv, n, generator=torch.Generator().manual_seed(n + 1), dtype=torch.float64) * sig,
                        dim=1).float().cuda()
    budgets = [vsp.BudgetConfig(float(rng.uniform(0.05, 1.0)), float(rng.uniform(0.05, 1.0)),
                                int(rng.integers(1, 5)), None if g % 2 else int(rng.integers(5, 2 * n + 6)))
               for g in range(hkv)]
    _check_against_oracle(vsp, a_v, a_s, budgets)


def test_select_quantized_ties_vs_oracle(vsp):
    rng = np.random.default_rng(5)
    for n in (50, 3000, 131072):
        c = rng.integers(0, 8, size=(2, n)).astype(np.float64)
        c[:, 0] += 1
        a = (c / c.sum(axis=1, keepdims=True)).astype(np.float32)
        a_v = torch.tensor(a[:1]).cuda()
        a_s = torch.tensor(a[1:]).cuda()
        for tau in (0.1, 0.5, 0.93):
            _check_against_oracle(vsp, a_v, a_s, [vsp.BudgetConfig(tau, tau, 1, None)])
        # clamped budgets take the count radix-select path; ties straddle the cluster's slices
        _check_against_oracle(vsp, a_v, a_s, [vsp.BudgetConfig(0.1, 0.93, n // 3 + 1, None)])
        _check_against_oracle(vsp, a_v, a_s, [vsp.BudgetConfig(0.93, 0.5, 1, n // 5 + 2)])


def test_select_uniform_zero_heads(vsp):
    n = 1000
    a = torch.full((1, n), 1.0 / n, dtype=torch.float32, device="cuda")
    pat = _check_against_oracle(vsp, a, a, [vsp.BudgetConfig(0.9, 0.25, 1, None)])
    iv, is_ = pat.lists(0)
    assert iv == list(range(len(iv))) and is_ == list(range(len(is_)))


def test_select_exact_fallback_boundary(vsp):
    """tau chosen so the prefix mass hits tau - 1e-12 exactly: exercises the sequential-f64
    fallback (the fast path cannot prove the decision)."""
    s = [0.125] * 8
    for tau in (0.5 + 1e-12, 0.5 + 2e-12, 0.5 + 5e-13):
        iv, _ = _select_gpu(vsp, s, s, _budget(vsp, tau, 0.5))
        want = oracle.port().cumulative_budget(np.float64(np.float32(s)), tau)
        assert len(iv) == want, tau


def test_select_negative_zero_ranks_as_zero(vsp):
    """-0.0 passes validation (v >= 0) and compares equal to 0.0 in the reference
    (sparsity.hpp:60-97): it must rank below every positive score, ties to the lower index."""
    rng = np.random.default_rng(11)
    for n in (9, 4000, 70000):
        a = rng.random((2, n)).astype(np.float64)
        a[:, rng.choice(n, n // 3, replace=False)] = 0.0
        a /= a.sum(axis=1, keepdims=True)
        a = a.astype(np.float32)
        zeros = np.flatnonzero(a[0] == 0.0)
        a[0, zeros[::2]] = -0.0
        a[1, np.flatnonzero(a[1] == 0.0)] = -0.0
        assert np.signbit(a).any()
        a_v = torch.tensor(a[:1]).cuda()
        a_s = torch.tensor(a[1:]).cuda()
        for tau in (0.3, 0.99):
            _check_against_oracle(vsp, a_v, a_s, [vsp.BudgetConfig(tau, tau, 1, None)])
        # budgets reaching into the zero block: ties among +-0 go to the lower index
        _check_against_oracle(vsp, a_v, a_s, [vsp.BudgetConfig(0.5, 0.5, n - n // 6, None)])


def test_select_validation_messages(vsp):
    a = torch.tensor([[0.5, 0.6, -0.1]], device="cuda")
    ok = torch.tensor([[0.5, 0.25, 0.25]], device="cuda")
    with pytest.raises(vsp.VspError, match="negative score"):
        vsp.select_pattern(a, ok, vsp.BudgetConfig(), validate=True)
    bad = torch.tensor([[0.4, 0.4, 0.1]], device="cuda")
    with pytest.raises(vsp.VspError, match="do not sum to 1"):
        vsp.select_pattern(ok, bad, vsp.BudgetConfig(), validate=True)
    with pytest.raises(vsp.VspError, match="tau_v must be in"):
        vsp.select_pattern(ok, ok, vsp.BudgetConfig(tau_v=1.5))
    with pytest.raises(vsp.VspError, match="min_budget exceeds max_budget"):
        vsp.select_pattern(ok, ok, vsp.BudgetConfig(min_budget=5, max_budget=3))


def test_vs_prefill_end_to_end(vsp):
    """indexer -> select -> sparse attention on one layer; indices bit-exact vs oracle select on
    the GPU scores, O vs the oracle sparse attention on the GPU indices."""
    from helpers import assert_attn_close, oracle_sparse, qkv
    n, hq, hkv = 640, 4, 2
    q, k, v = qkv(n, hq, hkv, seed=42)
    p = _params(vsp, hkv, 256, seed=3, sigma=0.5)
    budget = vsp.BudgetConfig(0.5, 0.5, 1, None)
    o, lse, pat = vsp.vs_prefill(q, k, v, p, budget)
    a_v, a_s = vsp.indexer_forward(k, v, p)
    _check_against_oracle(vsp, a_v, a_s, [budget] * hkv)
    lists = [pat.lists(g) for g in range(hkv)]
    o_ref, lse_ref = oracle_sparse(q, k, v, lists)
    assert_attn_close(o, lse, o_ref, lse_ref)


@pytest.mark.parametrize("hpc", [1, 3, 4, 0])
def test_vs_prefill_fused_matches_unfused(vsp, hpc):
    """The pipelined one-call layer (vsp_vs_prefill, chunks on a side stream) is bit-identical
    to the three operator calls, including a ragged last chunk (hkv=4, 3 heads per chunk)
    and per-KV-head budgets."""
    from helpers import qkv
    n, hq, hkv = 1100, 8, 4
    q, k, v = qkv(n, hq, hkv, seed=7)
    p = _params(vsp, hkv, 256, seed=5, sigma=0.5)
    budgets = [vsp.BudgetConfig(0.3 + 0.15 * g, 0.6 - 0.1 * g, 1 + g, None if g != 2 else 40) for g in range(hkv)]
    o_f, lse_f, pat_f = vsp.vs_prefill(q, k, v, p, budgets, heads_per_chunk=hpc)
    o_u, lse_u, pat_u = vsp.vs_prefill_unfused(q, k, v, p, budgets)
    torch.cuda.synchronize()
    assert torch.equal(pat_f.k_v, pat_u.k_v) and torch.equal(pat_f.k_s, pat_u.k_s)
    for g in range(hkv):
        assert pat_f.lists(g) == pat_u.lists(g)
    assert torch.equal(o_f, o_u)
    assert torch.equal(lse_f, lse_u)


def test_vs_prefill_rejects_bad_budget_count(vsp):
    from helpers import qkv
    q, k, v = qkv(256, 4, 2, seed=1)
    p = _params(vsp, 2, 256, seed=1, sigma=0.5)
    with pytest.raises(vsp.VspError, match="one BudgetConfig per KV head"):
        vsp.vs_prefill(q, k, v, p, [vsp.BudgetConfig()] * 3)
    with pytest.raises(vsp.VspError, match="tau_s must be in"):
        vsp.vs_prefill(q, k, v, p, vsp.BudgetConfig(0.9, 0.0))


@pytest.mark.parametrize("hpc,n", [(0, 1100), (0, 5000), (1, 1100), (3, 1100)])
def test_vs_prefill_host_matches_device(vsp, hpc, n):
    """The host-buffer layer call (pipelined H2D / compute / D2H per query-row range (hpc 0)
    or per KV-head chunk) returns exactly the device call's O, LSE and budgets."""
    from helpers import qkv
    hq, hkv = 8, 4
    q, k, v = qkv(n, hq, hkv, seed=9)
    p = _params(vsp, hkv, 256, seed=6, sigma=0.5)
    budgets = [vsp.BudgetConfig(0.4 + 0.1 * g, 0.5, 1, None) for g in range(hkv)]
    o_d, lse_d, pat = vsp.vs_prefill(q, k, v, p, budgets)
    qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
    o_h, lse_h, kv_h, ks_h = vsp.vs_prefill_host(qh, kh, vh, p, budgets, heads_per_chunk=hpc, budgets_out=True)
    torch.cuda.synchronize()
    assert torch.equal(o_h, o_d.cpu())
    assert torch.equal(lse_h, lse_d.cpu())
    assert torch.equal(kv_h, pat.k_v.cpu()) and torch.equal(ks_h, pat.k_s.cpu())
    # pageable host memory is accepted too (copies are then synchronous)
    o_p, lse_p = vsp.vs_prefill_host(q.cpu(), k.cpu(), v.cpu(), p, budgets, heads_per_chunk=hpc)
    torch.cuda.synchronize()
    assert torch.equal(o_p, o_d.cpu())


def test_vs_prefill_host_rejects_device_tensors(vsp):
    from helpers import qkv
    q, k, v = qkv(256, 4, 2, seed=1)
    p = _params(vsp, 2, 256, seed=1, sigma=0.5)
    with pytest.raises(vsp.VspError, match="contiguous host tensors"):
        vsp.vs_prefill_host(q, k.cpu(), v.cpu(), p, vsp.BudgetConfig())


@pytest.mark.parametrize("n,hkv", [(129, 2), (300, 3), (641, 2), (4099, 3), (131072, 1)])
def test_indexer_cta_pairs_identical(vsp, n, hkv, monkeypatch):
    """VSP_K1_MC = 2 runs K1 on CTA pairs (cta_group::2, M = 256, each CTA holding half of every
    W_U stage); odd tile counts leave a phantom tile in a head's last pair. Same bits as one CTA
    per tile (identical K order of the fp32 accumulation), for both W_U stage depths
    (VSP_K1_STAGEK = 32 / 64 K-rows), and for the split-X layout (VSP_K1_SPLIT = 1: one X tile
    in four per-box-barrier boxes, 128 KB W_U ring)."""
    g = torch.Generator().manual_seed(n + hkv)
    k = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(n, hkv, 128, generator=g).to(torch.bfloat16).cuda()
    p = _params(vsp, hkv, 512, seed=n)
    outs = []
    for mc, sk, split in (("1", "32", "0"), ("1", "64", "0"), ("2", "32", "0"), ("2", "64", "0"), ("1", "32", "1")):
        monkeypatch.setenv("VSP_K1_MC", mc)
        monkeypatch.setenv("VSP_K1_STAGEK", sk)
        monkeypatch.setenv("VSP_K1_SPLIT", split)
        _, _, lv, ls = vsp.indexer_forward(k, v, p, want_logits=True)
        torch.cuda.synchronize()
        outs.append((lv.clone(), ls.clone()))
    for lv, ls in outs[1:]:
        assert torch.equal(lv, outs[0][0]) and torch.equal(ls, outs[0][1])
    assert bool(torch.isfinite(outs[0][0]).all())
