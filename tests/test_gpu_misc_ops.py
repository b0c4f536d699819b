"""GPU parity of the standalone selection/merge operators (csrc/merge_topk.cu) against the
oracle, with the reference's own test bodies:

  * topk_indices (sparsity.hpp:83-97): TopK.HandValuesWithTies :93-104,
    DeterministicUnderPermutedTies :106-114, MatchesFullSortOracle :116-126 (coarse
    quantisation forces ties), RejectsBadK :128-131 — index sets bit-exact, plus negative
    values, -0.0 and long rows that the reference's normalised scores never have;
  * merge_row_columns (merge.hpp:18-56): MergeRowColumns.HandCases :274-283,
    RejectsUnsortedInput :285-288, MatchesSetUnionOracle :290-302 — bit-exact;
  * combine_scores (vsaggregate.hpp:133-157): CombineScores.MeanAndSum :144-155 at fp32
    (|d| <= 1e-7 instead of the reference's f64 1e-15), RejectsEmptyOrMismatched :157-162.
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vsp():
    import paper_2603_04460_b200 as m
    m.load_library()
    return m


def _topk(vsp, s, k):
    return vsp.topk_indices(torch.tensor(np.asarray(s, np.float32)).cuda(), k)[:k].cpu().tolist()


def test_topk_hand_values_with_ties(vsp):
    s = [0.2, 0.5, 0.2, 0.1]
    assert _topk(vsp, s, 1) == [1]
    assert _topk(vsp, s, 2) == [0, 1]
    assert _topk(vsp, s, 3) == [0, 1, 2]
    assert _topk(vsp, s, 4) == [0, 1, 2, 3]
    twin = [0.3, 0.2, 0.2, 0.3]
    assert _topk(vsp, twin, 2) == [0, 3]
    assert _topk(vsp, twin, 3) == [0, 1, 3]
    a, b = [0.4, 0.1, 0.1, 0.4], [0.1, 0.4, 0.4, 0.1]
    assert _topk(vsp, a, 2) == [0, 3] and _topk(vsp, b, 2) == [1, 2]
    assert all(_topk(vsp, a, 3) == _topk(vsp, a, 3) for _ in range(5))


def test_topk_matches_full_sort_oracle(vsp):
    rng = np.random.default_rng(93)
    port = oracle.port()
    for _ in range(200):
        n = 1 + int(rng.integers(50))
        s = rng.integers(0, 8, n) / 8.0
        k = 1 + int(rng.integers(n))
        assert _topk(vsp, s, k) == port.topk_indices(s, k).tolist()


@pytest.mark.parametrize("n", [1000, 131072, 300001])
def test_topk_general_values_batched(vsp, n):
    """Rows of mixed-sign values with -0.0/+0.0 and heavy ties, several rows and k per call."""
    rng = np.random.default_rng(n)
    rows = 3
    x = (rng.integers(-6, 6, size=(rows, n)) / 4.0).astype(np.float32)
    x[0, rng.choice(n, n // 10, replace=False)] = -0.0
    x[1] = rng.standard_normal(n).astype(np.float32)
    ks = [max(1, n // 7), 1 + n // 2, n]
    got = vsp.topk_indices(torch.tensor(x).cuda(), ks).cpu().numpy()
    port = oracle.port()
    for r in range(rows):
        want = port.topk_indices(x[r].astype(np.float64), ks[r])
        assert np.array_equal(got[r, : ks[r]], want), r


def test_topk_rejects_bad_k(vsp):
    s = torch.tensor([0.5, 0.5]).cuda()
    with pytest.raises(vsp.VspError, match="k must be >= 1"):
        vsp.topk_indices(s, 0)
    with pytest.raises(vsp.VspError, match="k exceeds score count"):
        vsp.topk_indices(s, 3)


def _lists(iv, is_):
    return (torch.tensor(iv, dtype=torch.int32).cuda(), torch.tensor(is_, dtype=torch.int32).cuda())


def test_merge_row_columns_hand_cases(vsp):
    for iv, is_, i, want in (([0, 5], [0, 2], 4, [0, 2, 4]), ([], [0], 7, [7]), ([1, 9], [], 3, [1]),
                             ([2], [3], 5, [2]), ([], [], 4, [])):
        assert vsp.merge_row_columns(*_lists(iv, is_), i).cpu().tolist() == want


def test_merge_row_columns_rejects_unsorted(vsp):
    with pytest.raises(vsp.VspError, match="^merge_row_columns: i_v not strictly ascending$"):
        vsp.merge_row_columns(*_lists([3, 1], []), 5)
    with pytest.raises(vsp.VspError, match="^merge_row_columns: i_s not strictly ascending$"):
        vsp.merge_row_columns(*_lists([], [2, 2]), 5)


def test_merge_row_columns_matches_union_oracle(vsp):
    rng = np.random.default_rng(44)
    port = oracle.port()
    for _ in range(300):
        n = 1 + int(rng.integers(40))
        iv = np.sort(rng.choice(n, 1 + int(rng.integers(n)), replace=False))
        is_ = np.sort(rng.choice(n, 1 + int(rng.integers(n)), replace=False))
        i = int(rng.integers(n))
        got = vsp.merge_row_columns(*_lists(iv.tolist(), is_.tolist()), i).cpu().tolist()
        assert got == port.merge_row_columns(iv, is_, i).tolist()


def test_merge_row_columns_long_lists_many_rows(vsp):
    """Thousands of entries per list: the rows' merges are split across 256 threads by merge
    path, with overlaps between verticals and slash columns collapsing at slice borders."""
    rng = np.random.default_rng(5)
    n = 50000
    iv = np.sort(rng.choice(n, 9000, replace=False))
    is_ = np.unique(np.concatenate([np.arange(0, 700), rng.choice(n, 3000, replace=False)]))
    rows = [0, 1, 699, 700, 12345, 31999, n - 1] + rng.integers(0, n, 25).tolist()
    got = vsp.merge_row_columns(*_lists(iv.tolist(), is_.tolist()), rows)
    port = oracle.port()
    for r, g in zip(rows, got):
        assert g.cpu().tolist() == port.merge_row_columns(iv, is_, r).tolist(), r


def test_combine_scores_mean_and_sum(vsp):
    v = torch.tensor([[0.6, 0.4], [0.2, 0.8]]).cuda()
    s = torch.tensor([[1.0, 0.0], [0.4, 0.6]]).cuda()
    mv, ms = vsp.combine_scores(v, s)
    assert abs(mv[0].item() - 0.4) <= 1e-7 and abs(ms[1].item() - 0.3) <= 1e-7
    sv, ss = vsp.combine_scores(v, s, reduce="sum")
    assert abs(sv[0].item() - 0.8) <= 1e-7 and abs(ss[0].item() - 1.4) <= 1e-7


def test_combine_scores_matches_oracle_random(vsp):
    rng = np.random.default_rng(3)
    heads, n = 4, 70001
    v = rng.random((heads, n)).astype(np.float32)
    s = rng.random((heads, n)).astype(np.float32)
    for mean in (True, False):
        gv, gs = vsp.combine_scores(torch.tensor(v).cuda(), torch.tensor(s).cuda(), "mean" if mean else "sum")
        wv, ws = oracle.port().combine_scores(v.astype(np.float64), s.astype(np.float64), mean=mean)
        assert np.allclose(gv.cpu().numpy(), wv, rtol=1e-7, atol=0) and np.allclose(gs.cpu().numpy(), ws, rtol=1e-7,
                                                                                    atol=0)


def test_combine_scores_rejects_empty_or_mismatched(vsp):
    with pytest.raises(vsp.VspError, match="combine_scores: no heads"):
        vsp.combine_scores(torch.zeros(0, 2).cuda(), torch.zeros(0, 2).cuda())
    with pytest.raises(vsp.VspError, match="combine_scores: length mismatch"):
        vsp.combine_scores(torch.zeros(2, 2).cuda(), torch.zeros(2, 1).cuda())
