"""GPU: the sharded-output path of SURVEY.md §8e on one B200.

* VSP_O_HEAD_MAJOR: K3 (and the one-call layer) write O as [Hq, n, d] bit-identical to the
  token-major result permuted — the reference's per-head n x d matrices (attention.hpp:150).
* A shard rank's call with out = its slab of the full head-major buffer writes exactly that
  slab (the in-place all-gather send buffer) and nothing else.
* vsp_allgather_heads through a world-1 NCCL communicator created by the C ABI (the only
  world the single-GPU box allows; the 2-rank id exchange and slab logic run on gloo in
  tests/test_host.py).
"""
import pytest
import torch

from helpers import qkv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vsp():
    import paper_2603_04460_b200 as m
    m.load_library()
    return m


def _params(vsp, hkv, seed):
    g = torch.Generator().manual_seed(seed)
    return vsp.make_indexer_params(hkv, 128, 256, g, head_sigma=0.5)


def test_head_major_sparse_attention_is_a_permutation(vsp):
    n, hq, hkv = 1000, 8, 4
    q, k, v = qkv(n, hq, hkv, seed=21)
    p = _params(vsp, hkv, 3)
    a_v, a_s = vsp.indexer_forward(k, v, p)
    pat = vsp.select_pattern(a_v, a_s, vsp.BudgetConfig(0.5, 0.6, 1, None))
    o_t, lse_t = vsp.sparse_attention(q, k, v, pat)
    o_h, lse_h = vsp.sparse_attention(q, k, v, pat, head_major=True)
    torch.cuda.synchronize()
    assert o_h.shape == (hq, n, 128)
    assert torch.equal(o_h, o_t.permute(1, 0, 2))
    assert torch.equal(lse_h, lse_t)


@pytest.mark.parametrize("world", [2, 4])
def test_shard_rank_writes_only_its_slab(vsp, world):
    from paper_2603_04460_b200 import parallel
    n, hq, hkv = 777, 8, 4
    q, k, v = qkv(n, hq, hkv, seed=22)
    p = _params(vsp, hkv, 4)
    budgets = [vsp.BudgetConfig(0.4, 0.5, 1, None)] * hkv
    o_ref, lse_ref, _ = vsp.vs_prefill(q, k, v, p, budgets)
    o_full = torch.full((hq, n, 128), float("nan"), dtype=torch.bfloat16, device="cuda")
    lse_full = torch.full((hq, n), float("nan"), device="cuda")
    for rank in range(world):  # every "rank" on this one GPU, each touching only its slab
        qs, ks, vs = (parallel.shard_heads(t, rank, world) for t in (q, k, v))
        ps = vsp.IndexerParams(*(parallel.shard_heads(t, rank, world, dim=0)
                                 for t in (p.w_u, p.b_u, p.w_v, p.b_v, p.w_s, p.b_s)))
        slab = parallel.head_slab(o_full, rank, world)
        lo, hi = parallel.head_range(hq, rank, world)
        before = o_full.clone()
        vsp.vs_prefill(qs, ks, vs, ps, budgets[: hkv // world], out=slab, lse=lse_full[lo:hi], head_major=True)
        torch.cuda.synchronize()
        outside = torch.ones(hq, dtype=torch.bool, device="cuda")
        outside[lo:hi] = False
        assert torch.equal(o_full[outside].isnan(), before[outside].isnan())
        assert not o_full[lo:hi].isnan().any()
    assert torch.equal(o_full, o_ref.permute(1, 0, 2))
    assert torch.equal(lse_full, lse_ref)


def test_allgather_heads_world1_through_c_abi(vsp):
    from paper_2603_04460_b200 import parallel
    comm = parallel.VspComm(torch.device("cuda", 0))
    o = torch.randn(8, 300, 128, device="cuda").bfloat16()
    lse = torch.randn(8, 300, device="cuda")
    o0, l0 = o.clone(), lse.clone()
    comm.allgather_heads(o, lse)
    torch.cuda.synchronize()
    assert torch.equal(o, o0) and torch.equal(lse, l0)
    with pytest.raises(vsp.VspError, match="bad arguments"):
        comm.allgather_heads(torch.empty(0, 0, 0, device="cuda", dtype=torch.bfloat16))
    comm.close()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_balanced_units_reassemble_the_layer_bit_exact(vsp, world):
    """Virtual ranks on one GPU: each runs vs_prefill_units on its balanced units; the union
    of their head-major O / LSE regions equals the one-call layer exactly."""
    from paper_2603_04460_b200 import parallel
    n, hq, hkv = 1500, 8, 4
    q, k, v = qkv(n, hq, hkv, seed=23)
    p = _params(vsp, hkv, 5)
    budgets = [vsp.BudgetConfig(0.3 + 0.1 * g, 0.5, 1, None) for g in range(hkv)]
    o_ref, lse_ref, pat_ref = vsp.vs_prefill(q, k, v, p, budgets, head_major=True)
    vsp.sparse_attention(q, k, v, pat_ref, validate=False)  # the plan the counts are read from
    cost = vsp.sparse_tile_counts(n, hkv, n + 1, q.device)
    assert cost.shape == (hkv, (n + 127) // 128) and int(cost.sum()) > 0
    units = parallel.balanced_units(cost, world)
    o = torch.full_like(o_ref, float("nan"))
    lse = torch.full_like(lse_ref, float("nan"))
    for r in range(world):
        pat = vsp.vs_prefill_units(q, k, v, p, budgets, units[r], out=o, lse=lse)
        torch.cuda.synchronize()
        for g in {u[0] for u in units[r]}:
            assert pat.lists(g) == pat_ref.lists(g)
    assert torch.equal(o, o_ref) and torch.equal(lse, lse_ref)


def test_units_api_errors_and_empty_units(vsp):
    n, hq, hkv = 600, 4, 2
    q, k, v = qkv(n, hq, hkv, seed=24)
    p = _params(vsp, hkv, 6)
    budgets = [vsp.BudgetConfig(0.5, 0.5, 1, None)] * hkv
    o = torch.zeros(hq, n, 128, dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros(hq, n, device="cuda")
    with pytest.raises(vsp.VspError, match="unit out of range"):
        vsp.vs_prefill_units(q, k, v, p, budgets, [(hkv, 0, 1)], out=o, lse=lse)
    with pytest.raises(vsp.VspError, match="unit out of range"):
        vsp.vs_prefill_units(q, k, v, p, budgets, [(0, 3, 2)], out=o, lse=lse)
    with pytest.raises(vsp.VspError, match="head-major"):
        vsp.vs_prefill_units(q, k, v, p, budgets, [(0, 0, 1)], out=torch.empty_like(q), lse=lse)
    # no units: nothing written
    vsp.vs_prefill_units(q, k, v, p, budgets, [], out=o, lse=lse)
    torch.cuda.synchronize()
    assert not o.any() and not lse.any()
    # an empty block range is a no-op for that unit
    vsp.vs_prefill_units(q, k, v, p, budgets, [(1, 2, 2)], out=o, lse=lse)
    torch.cuda.synchronize()
    assert not o.any()
