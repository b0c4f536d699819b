"""GPU parity of K4 (dense causal) and K3 (VS sparse) attention vs the f64 oracle.

Mirrors the reference's attention tests (tests/test_attention.cpp) at bf16/fp32 precision:
  FullVerticalEqualsFull :118-127, MatchesMaskedSoftmaxOracle :129-143,
  BlockSizeIrrelevant :145-155, UncoveredRowThrows :157-170,
  BlockwiseAttention.EquivalentToFullAcrossSizes :99-109, SPEC.md:153 (I_s={0} -> O=V).
Tolerances (stated): O max|d| <= 2e-2, mean|d| <= 2e-3, LSE max|d| <= 1e-3.
"""
import numpy as np
import pytest
import torch

from helpers import (assert_attn_close, f64, oracle_dense, oracle_sparse, pattern_tensors, qkv)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vsp():
    import paper_2603_04460_b200 as m
    m.load_library()
    return m


@pytest.mark.parametrize("n,hq,hkv", [(1, 2, 1), (7, 4, 2), (128, 4, 1), (300, 4, 2), (512, 8, 2),
                                     (1, 1, 1), (200, 4, 4), (300, 3, 1), (130, 6, 2)])  # MHA and odd groups
def test_dense_matches_oracle(vsp, n, hq, hkv):
    q, k, v = qkv(n, hq, hkv, seed=n)
    o, lse = vsp.blockwise_attention(q, k, v)
    torch.cuda.synchronize()
    o_ref, lse_ref = oracle_dense(q, k, v)
    assert_attn_close(o, lse, o_ref, lse_ref)


def test_dense_long_vs_torch(vsp):
    """n = 4096 (config 1 length), against torch fp32 SDPA on the same bf16 values."""
    n, hq, hkv = 4096, 8, 2
    q, k, v = qkv(n, hq, hkv, seed=7)
    o, lse = vsp.blockwise_attention(q, k, v)
    qf = q.float().permute(1, 0, 2)
    kf = k.float().repeat_interleave(hq // hkv, dim=1).permute(1, 0, 2)
    vf = v.float().repeat_interleave(hq // hkv, dim=1).permute(1, 0, 2)
    ref = torch.nn.functional.scaled_dot_product_attention(qf, kf, vf, is_causal=True).permute(1, 0, 2)
    err = (o.float() - ref).abs()
    assert err.max().item() <= 2e-2 and err.mean().item() <= 2e-3
    s = (qf @ kf.transpose(1, 2)) / np.sqrt(128)
    s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool, device=s.device), 1), float("-inf"))
    lse_ref = torch.logsumexp(s, dim=-1)
    assert (lse - lse_ref).abs().max().item() <= 1e-3


def _random_pattern(rng, n, kv, ks):
    iv = sorted(rng.choice(n, size=min(kv, n), replace=False).tolist())
    is_ = sorted(set(rng.choice(n, size=min(ks, n), replace=False).tolist()) | {0})
    return iv, is_


@pytest.mark.parametrize("n,hq,hkv,kv,ks", [(64, 2, 1, 5, 4), (300, 4, 2, 20, 12), (512, 4, 1, 40, 30),
                                            (700, 8, 2, 100, 60),
                                            (256, 2, 2, 10, 8), (300, 3, 1, 20, 12), (384, 6, 2, 30, 16)])
def test_sparse_matches_masked_oracle(vsp, n, hq, hkv, kv, ks):
    rng = np.random.default_rng(n)
    q, k, v = qkv(n, hq, hkv, seed=n + 1)
    lists = [_random_pattern(rng, n, kv, ks) for _ in range(hkv)]
    o, lse = vsp.sparse_attention(q, k, v, pattern_tensors(lists, n))
    torch.cuda.synchronize()
    o_ref, lse_ref = oracle_sparse(q, k, v, lists)
    assert_attn_close(o, lse, o_ref, lse_ref)


def test_sparse_clustered_offsets(vsp):
    """Local band + periodic offsets (the structured case the speed claim rests on)."""
    n, hq, hkv = 1024, 4, 1
    q, k, v = qkv(n, hq, hkv, seed=3)
    is_ = sorted(set(range(0, 64)) | set(range(256, 300)) | {511, 700})
    iv = [0, 1, 2, 3, 100, 101, 500, 900]
    o, lse = vsp.sparse_attention(q, k, v, pattern_tensors([(iv, is_)], n))
    o_ref, lse_ref = oracle_sparse(q, k, v, [(iv, is_)])
    assert_attn_close(o, lse, o_ref, lse_ref)


def test_sparse_many_ranges_plan(vsp):
    """>32 slash offsets per query block mixing tight clusters, isolated offsets and offsets
    beyond i0 (clipped intervals): exercises the warp-parallel range merge of vs_plan_kernel."""
    n, hq, hkv = 2048, 4, 2
    q, k, v = qkv(n, hq, hkv, seed=17)
    rng = np.random.default_rng(17)
    lists = []
    for g in range(hkv):
        is_ = set(range(0, 40)) | set(range(300, 333)) | set(rng.choice(n, size=150, replace=False).tolist())
        iv = sorted(rng.choice(n, size=70, replace=False).tolist())
        lists.append((iv, sorted(is_)))
    o, lse = vsp.sparse_attention(q, k, v, pattern_tensors(lists, n))
    o_ref, lse_ref = oracle_sparse(q, k, v, lists)
    assert_attn_close(o, lse, o_ref, lse_ref)


def test_full_vertical_equals_dense(vsp):
    n, hq, hkv = 384, 4, 1
    q, k, v = qkv(n, hq, hkv, seed=11)
    o_s, lse_s = vsp.sparse_attention(q, k, v, pattern_tensors([(list(range(n)), [0])], n))
    o_d, lse_d = vsp.blockwise_attention(q, k, v)
    assert (o_s.float() - o_d.float()).abs().max().item() <= 1e-2
    assert (lse_s - lse_d).abs().max().item() <= 1e-4


def test_diagonal_only_returns_v(vsp):
    """I_v = {}, I_s = {0}: every row attends only to itself -> O = V."""
    n, hq, hkv = 200, 2, 1
    q, k, v = qkv(n, hq, hkv, seed=5)
    o, _ = vsp.sparse_attention(q, k, v, pattern_tensors([([], [0])], n))
    for h in range(hq):
        assert torch.equal(o[:, h], v[:, 0])


def test_hand_pattern_block_irrelevant(vsp):
    """test_attention.cpp:145-155 pattern; the GPU result is one fixed blocking."""
    n, hq, hkv = 48, 2, 1
    q, k, v = qkv(n, hq, hkv, seed=9)
    lists = [([0, 3, 17, 39], [0, 2, 9])]
    o, lse = vsp.sparse_attention(q, k, v, pattern_tensors(lists, n))
    for block in (1, 7, 1000):
        o_ref, lse_ref = oracle_sparse(q, k, v, lists, block=block)
        assert_attn_close(o, lse, o_ref, lse_ref)


def test_uncovered_row_raises(vsp):
    n = 16
    q, k, v = qkv(n, 2, 1, seed=1)
    with pytest.raises(vsp.VspError, match="^uncovered query row 0$"):
        vsp.sparse_attention(q, k, v, pattern_tensors([([5], [3])], n))


def test_unsorted_raises(vsp):
    n = 16
    q, k, v = qkv(n, 2, 1, seed=1)
    with pytest.raises(vsp.VspError, match="i_v not strictly ascending"):
        vsp.sparse_attention(q, k, v, pattern_tensors([([3, 1], [0])], n))
    with pytest.raises(vsp.VspError, match="i_s not strictly ascending"):
        vsp.sparse_attention(q, k, v, pattern_tensors([([1], [0, 4, 4])], n))


def test_count_above_cap_is_einval_not_a_fault(vsp):
    """k_v / k_s larger than the list capacity: validation reports EINVAL (its scans stay
    inside the row) and the context stays usable."""
    n = 16
    q, k, v = qkv(n, 2, 1, seed=1)
    pat = pattern_tensors([([0, 3], [0, 1])], n)
    pat.k_v.fill_(n + 50)
    with pytest.raises(vsp.VspError, match="index count exceeds cap"):
        vsp.sparse_attention(q, k, v, pat)
    o, lse = vsp.sparse_attention(q, k, v, pattern_tensors([([0, 3], [0, 1])], n))
    torch.cuda.synchronize()
    assert torch.isfinite(lse).all()


def test_recall_from_lse_matches_reference_recall(vsp):
    import oracle
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    n, hq, hkv = 256, 2, 1
    q, k, v = qkv(n, hq, hkv, seed=21)
    lists = [([0, 5, 77], [0, 1, 2, 3, 40])]
    _, lse_s = vsp.sparse_attention(q, k, v, pattern_tensors(lists, n))
    _, lse_d = vsp.blockwise_attention(q, k, v)
    rec = vsp.attention_recall(lse_s, lse_d).cpu().numpy()
    qn, kn = f64(q), f64(k)
    for h in range(hq):
        ref = oracle.ref().attention_recall(qn[:, h], kn[:, 0], *lists[0])
        assert abs(rec[h] - ref) <= 1e-3


def test_launch_counter_attributes_kernels(vsp):
    """vsp_kernel_launches counts this library's launches: dense = one K4 launch; sparse =
    one planning launch (bitmaps, vertical gather, tile lists) + one persistent K3 launch."""
    n, hq, hkv = 300, 4, 2
    q, k, v = qkv(n, hq, hkv, seed=21)
    pat = pattern_tensors([([0, 5, 77], [0, 1, 9]), ([0, 200], [0, 3])], n)
    c0 = vsp.kernel_launches()
    vsp.blockwise_attention(q, k, v)
    c1 = vsp.kernel_launches()
    vsp.sparse_attention(q, k, v, pat, validate=False)
    c2 = vsp.kernel_launches()
    assert c1 - c0 == 1
    assert c2 - c1 == 2


def test_attn_timing_brackets_layer_k3_launches(vsp):
    """vsp_attn_timing: one event pair per K3 launch of the layer entry point."""
    from paper_2603_04460_b200.synth import planted_layer
    n, hq, hkv = 2048, 8, 4
    q, k, v, _ = planted_layer(n, hq, hkv, seed=4)
    g = torch.Generator().manual_seed(2)
    params = vsp.make_indexer_params(hkv, 128, 256, g, head_sigma=0.4)
    budget = vsp.BudgetConfig(0.5, 0.5, 1, None)
    vsp.attn_timing(True)
    for hpc in (0, 0, 1):  # one chunk, one chunk, four chunks
        vsp.vs_prefill(q, k, v, params, budget, heads_per_chunk=hpc)
    ms, cnt = vsp.attn_timing_read()
    vsp.attn_timing(False)
    assert cnt == 1 + 1 + 4
    assert ms > 0.0
    vsp.vs_prefill(q, k, v, params, budget)
    assert vsp.attn_timing_read() == (0.0, 0)


@pytest.mark.parametrize("hq,hkv", [(4, 4), (6, 2)])
def test_layer_call_mha_and_odd_groups(vsp, hq, hkv):
    """Group sizes 1 (MHA) and 3: the one-call layer equals the operator chain, and each Q head
    matches the oracle on its KV head's pattern."""
    n = 640
    q, k, v = qkv(n, hq, hkv, seed=31)
    g = torch.Generator().manual_seed(8)
    params = vsp.make_indexer_params(hkv, 128, 256, g, head_sigma=0.5)
    budget = vsp.BudgetConfig(0.5, 0.5, 1, None)
    a_v, a_s = vsp.indexer_forward(k, v, params)
    pat = vsp.select_pattern(a_v, a_s, budget)
    o_ref, lse_ref = vsp.sparse_attention(q, k, v, pat)
    o, lse, _ = vsp.vs_prefill(q, k, v, params, budget)
    assert torch.equal(o, o_ref) and torch.equal(lse, lse_ref)
    lists = [pat.lists(h) for h in range(hkv)]
    o_or, lse_or = oracle_sparse(q, k, v, lists)
    assert_attn_close(o, lse, o_or, lse_or)


def test_concurrent_dense_launches_on_two_streams(vsp):
    """The persistent kernel's work counter is per launch: overlapping launches on two
    streams give the same bits as back-to-back ones."""
    n, hq, hkv = 4096, 8, 2
    q1, k1, v1 = qkv(n, hq, hkv, seed=41)
    q2, k2, v2 = qkv(n, hq, hkv, seed=42)
    ref1 = vsp.blockwise_attention(q1, k1, v1)
    ref2 = vsp.blockwise_attention(q2, k2, v2)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            a = vsp.blockwise_attention(q1, k1, v1)
        with torch.cuda.stream(s2):
            b = vsp.blockwise_attention(q2, k2, v2)
        outs.append((a, b))
    torch.cuda.synchronize()
    for a, b in outs:
        assert torch.equal(a[0], ref1[0]) and torch.equal(a[1], ref1[1])
        assert torch.equal(b[0], ref2[0]) and torch.equal(b[1], ref2[1])


def test_concurrent_sparse_calls_on_two_streams(vsp):
    """Python-level workspaces are per stream: overlapping sparse calls stay correct."""
    n, hq, hkv = 2048, 8, 2
    rng = np.random.default_rng(5)
    q, k, v = qkv(n, hq, hkv, seed=43)
    pats = [pattern_tensors([_random_pattern(rng, n, 300, 40) for _ in range(hkv)], n) for _ in range(2)]
    refs = [vsp.sparse_attention(q, k, v, p) for p in pats]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            a = vsp.sparse_attention(q, k, v, pats[0], validate=False)
        with torch.cuda.stream(s2):
            b = vsp.sparse_attention(q, k, v, pats[1], validate=False)
        outs.append((a, b))
    torch.cuda.synchronize()
    for a, b in outs:
        assert torch.equal(a[0], refs[0][0]) and torch.equal(b[0], refs[1][0])


def test_tile_stats_and_counts_describe_the_last_plan(vsp):
    """sparse_tile_stats / sparse_tile_counts read the plan of the last sparse_attention on the
    current stream: totals agree, per-head sums agree, and sparse never exceeds dense."""
    n, hq, hkv = 1500, 4, 2
    rng = np.random.default_rng(12)
    q, k, v = qkv(n, hq, hkv, seed=12)
    pat = pattern_tensors([_random_pattern(rng, n, 200, 30) for _ in range(hkv)], n)
    vsp.sparse_attention(q, k, v, pat, validate=False)
    tiles, dense, per_head = vsp.sparse_tile_stats(n, hkv, n + 1, q.device, per_head=True)
    counts = vsp.sparse_tile_counts(n, hkv, n + 1, q.device)
    assert 0 < tiles <= dense
    assert sum(per_head) == tiles == int(counts.sum())
    assert counts.sum(1).tolist() == per_head


def test_multicast_clusters_bit_identical(vsp, monkeypatch):
    """K/V multicast (two-CTA clusters, group size 4) and independent CTAs give the same bits."""
    n, hq, hkv = 1500, 8, 2
    rng = np.random.default_rng(77)
    q, k, v = qkv(n, hq, hkv, seed=77)
    pat = pattern_tensors([_random_pattern(rng, n, 300, 40) for _ in range(hkv)], n)
    o_mc, lse_mc = vsp.sparse_attention(q, k, v, pat, validate=False)
    d_mc = vsp.blockwise_attention(q, k, v)
    monkeypatch.setenv("VSP_NO_MULTICAST", "1")
    o_1, lse_1 = vsp.sparse_attention(q, k, v, pat, validate=False)
    d_1 = vsp.blockwise_attention(q, k, v)
    assert torch.equal(o_mc, o_1) and torch.equal(lse_mc, lse_1)
    assert torch.equal(d_mc[0], d_1[0]) and torch.equal(d_mc[1], d_1[1])


@pytest.mark.parametrize("n,hq", [(1, 3), (7, 2), (4099, 5), (131075, 32)])
def test_recall_from_lse_cluster_sum_matches_fp64(vsp, n, hq):
    """vsp_recall_from_lse splits each head over an 8-CTA cluster (fixed slices, partials added
    in rank order): equal to the fp64 mean of exp(LSE_s - LSE_d), rounded once to fp32, and
    identical across calls."""
    g = torch.Generator().manual_seed(n)
    ld = torch.randn(hq, n, generator=g) * 3.0
    ls = ld - torch.rand(hq, n, generator=g) * 2.0
    rec = vsp.attention_recall(ls.cuda(), ld.cuda())
    rec2 = vsp.attention_recall(ls.cuda(), ld.cuda())
    want = torch.exp(ls.double() - ld.double()).mean(dim=1)
    assert torch.equal(rec, rec2)
    assert float(((rec.cpu().double() - want).abs() / want).max()) <= 2e-7
