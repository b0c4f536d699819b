"""Full-size (BASELINE config[2]: n = 131072, 32 Q / 8 KV heads, d = 128) properties of the
sparse attention path, where the f64 oracle is too slow to run. Size-independent identities:

* I_v = {}, I_s = {0} -> O = V exactly and LSE_i = scale * q_i . k_i;
* I_v = every column -> the dense causal result, bit for bit (FullVerticalEqualsFull,
  test_attention.cpp:118-127, here against K4 at full size);
* nested patterns: P1 subset of P2 subset of dense -> LSE1 <= LSE2 <= LSE_dense (a softmax
  denominator over a subset of the columns), i.e. recall = exp(LSE_s - LSE_d) in (0, 1];
* determinism: the persistent kernel's dynamic work order never changes a result;
* the one-call layer (vs_prefill) reproduces indexer -> select -> sparse_attention exactly.
"""
import math

import pytest
import torch

from helpers import pattern_tensors

pytestmark = pytest.mark.gpu

N, HQ, HKV, D = 131072, 32, 8, 128


@pytest.fixture(scope="module")
def vsp():
    import paper_2603_04460_b200 as m
    m.load_library()
    return m


@pytest.fixture(scope="module")
def layer():
    g = torch.Generator(device="cuda").manual_seed(2026)
    q = torch.randn(N, HQ, D, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(N, HKV, D, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(N, HKV, D, device="cuda", generator=g).to(torch.bfloat16)
    return q, k, v


def _pattern(seed, n_vert, offsets_per_head):
    """Sorted random verticals (plus column 0) and clustered slash offsets per KV head."""
    g = torch.Generator().manual_seed(seed)
    lists = []
    for h in range(HKV):
        iv = torch.unique(torch.cat([torch.zeros(1, dtype=torch.long),
                                     torch.randint(0, N, (n_vert,), generator=g)])).tolist()
        band = list(range(0, 16 + 4 * h))
        far = [int(x) for x in torch.randint(100, N // 2, (offsets_per_head,), generator=g)]
        clusters = [o + d for o in far for d in range(3)]
        lists.append((iv, sorted(set(band + clusters))))
    return lists


def test_fullsize_diagonal_only_is_v(vsp, layer):
    q, k, v = layer
    o, lse = vsp.sparse_attention(q, k, v, pattern_tensors([([], [0])] * HKV, N))
    grp = HQ // HKV
    for h in range(HQ):
        assert torch.equal(o[:, h], v[:, h // grp])
    s = (q.float() * k.float().repeat_interleave(grp, dim=1)).sum(-1).t() / math.sqrt(D)  # [HQ, n]
    assert (lse - s).abs().max().item() <= 1e-3 * s.abs().max().item() + 1e-4


def test_fullsize_full_vertical_equals_dense(vsp, layer):
    q, k, v = layer
    o_s, lse_s = vsp.sparse_attention(q, k, v, pattern_tensors([(range(N), [0])] * HKV, N))
    o_d, lse_d = vsp.blockwise_attention(q, k, v)
    assert torch.equal(o_s, o_d)
    assert torch.equal(lse_s, lse_d)


def test_fullsize_nested_patterns_bound_lse_and_are_deterministic(vsp, layer):
    q, k, v = layer
    small = _pattern(7, 600, 4)
    # superset: every vertical and offset of `small` plus more of both
    big = [(sorted(set(iv) | set(iv2)), sorted(set(is_) | set(is2)))
           for (iv, is_), (iv2, is2) in zip(small, _pattern(8, 3000, 10))]
    o1, lse1 = vsp.sparse_attention(q, k, v, pattern_tensors(small, N))
    o1b, lse1b = vsp.sparse_attention(q, k, v, pattern_tensors(small, N))
    assert torch.equal(o1, o1b) and torch.equal(lse1, lse1b)  # dynamic work order, same bits
    _, lse2 = vsp.sparse_attention(q, k, v, pattern_tensors(big, N))
    _, lse_d = vsp.blockwise_attention(q, k, v)
    assert torch.isfinite(o1.float()).all() and torch.isfinite(lse1).all()
    tol = 1e-3  # bf16 P and fp32 accumulation in different tile orders
    assert (lse1 - lse2).max().item() <= tol
    assert (lse2 - lse_d).max().item() <= tol
    recall = vsp.attention_recall(lse1, lse_d)
    assert 0.0 < recall.min().item() and recall.max().item() <= 1.0 + tol


def test_fullsize_layer_call_matches_operator_chain(vsp, layer):
    q, k, v = layer
    g = torch.Generator().manual_seed(3)
    params = vsp.make_indexer_params(HKV, D, 256, g, head_sigma=0.5)
    budgets = [vsp.BudgetConfig(0.3 + 0.05 * h, 0.6, 1, None) for h in range(HKV)]
    a_v, a_s = vsp.indexer_forward(k, v, params)
    pat = vsp.select_pattern(a_v, a_s, budgets)
    o_ref, lse_ref = vsp.sparse_attention(q, k, v, pat, validate=False)
    for hpc in (0, 3):
        o, lse, pat2 = vsp.vs_prefill(q, k, v, params, budgets, heads_per_chunk=hpc)
        assert torch.equal(pat2.k_v, pat.k_v) and torch.equal(pat2.k_s, pat.k_s)
        assert torch.equal(o, o_ref) and torch.equal(lse, lse_ref)
