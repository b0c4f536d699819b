"""CPU tests of the host side: the C-ABI library exports, loud failure without a GPU,
the bench's covered-pair arithmetic, the synthetic generator, the distillation objective,
and KV-head sharding + output assembly over a 2-rank gloo group."""
import ctypes
import math
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "vsp_gpu.h")).read()
    return sorted(set(re.findall(r"VSP_API\s+[\w\s\*]+?\b(vsp_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2603_04460_b200 as vsp
    lib = vsp.load_library()
    syms = _declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
    assert lib.vsp_version().decode().startswith("vsp-b200")


def test_no_cpu_fallback_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2603_04460_b200 as vsp
    lib = vsp.load_library()
    h = ctypes.c_void_p()
    rc = lib.vsp_create(ctypes.byref(h), 0)
    assert rc == vsp.VSP_ECUDA
    assert "no CPU fallback" in lib.vsp_last_error().decode()
    with pytest.raises(vsp.VspRuntimeError):
        vsp.blockwise_attention(torch.zeros(8, 2, 128), torch.zeros(8, 1, 128), torch.zeros(8, 1, 128))


def test_covered_pairs_formula_matches_bruteforce():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    from paper_2603_04460_b200 import SelectedIndices
    import oracle
    rng = np.random.default_rng(0)
    n = 97
    lists = []
    for _ in range(3):
        iv = sorted(rng.choice(n, size=17, replace=False).tolist())
        is_ = sorted(set(rng.choice(n, size=11, replace=False).tolist()) | {0})
        lists.append((iv, is_))
    cap = n + 1
    pat = SelectedIndices(torch.zeros(3, cap, dtype=torch.int32), torch.zeros(3, dtype=torch.int32),
                          torch.zeros(3, cap, dtype=torch.int32), torch.zeros(3, dtype=torch.int32))
    for g, (iv, is_) in enumerate(lists):
        pat.i_v[g, :len(iv)] = torch.tensor(iv)
        pat.i_s[g, :len(is_)] = torch.tensor(is_)
        pat.k_v[g] = len(iv)
        pat.k_s[g] = len(is_)
    got = bench.covered_pairs(pat, n, 3)
    port = oracle.port()
    for g, (iv, is_) in enumerate(lists):
        want = sum(len(port.merge_row_columns(iv, is_, i)) for i in range(n))
        assert got[g] == want


def test_synth_shapes_and_structure_cpu():
    from paper_2603_04460_b200.synth import planted_layer
    q, k, v, plants = planted_layer(256, 4, 2, seed=1, device="cpu")
    assert q.shape == (256, 4, 128) and k.shape == (256, 2, 128) and v.shape == (256, 2, 128)
    assert q.dtype == torch.bfloat16
    assert len(plants) == 2 and plants[0]["anchors"][0] == 0
    # the sink (token 0) outscores the typical causal key of every row
    s = (q[:, 0].float() @ k[:, 0].float().T) / math.sqrt(128)
    s = s.masked_fill(torch.triu(torch.ones(256, 256, dtype=torch.bool), 1), float("nan"))
    med = torch.nanmedian(s[64:], dim=1).values
    assert (s[64:, 0] > med + 3).all()


def test_distill_objective_decreases_and_matches_reference_kl():
    from paper_2603_04460_b200 import distill
    torch.manual_seed(0)
    n, hkv, d = 64, 2, 128
    k = torch.randn(n, hkv, d).to(torch.bfloat16)
    v = torch.randn(n, hkv, d).to(torch.bfloat16)
    tv = torch.softmax(torch.randn(hkv, n) * 2, dim=1)
    ts = torch.softmax(torch.randn(hkv, n) * 2, dim=1)
    # kl_loss (indexer.hpp:138-149) restated in numpy as the check
    lp = torch.log_softmax(torch.randn(hkv, n), dim=1)
    got = distill.kl_forward(lp, tv).numpy()
    p = lp.exp().double().numpy()
    want = (p * (np.log(p) - np.log(tv.double().numpy() + 1e-8))).sum(1)
    assert np.allclose(got, want, rtol=1e-5)
    params, losses = distill.distill_indexer_torch([(k, v, tv, ts)], d_h=256, steps=60, lr_peak=1e-2, warmup=5,
                                             log_every=1)
    assert losses[-1] < losses[0] * 0.8
    assert params.w_u.dtype == torch.bfloat16 and params.w_u.shape == (hkv, 2 * d, 256)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, hq, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_04460_b200 import parallel
    torch.manual_seed(0)
    o_full = torch.randn(n, hq, d)  # same on every rank
    mine = parallel.shard_heads(o_full, rank, world)
    full = parallel.assemble_heads(mine)
    ok = torch.equal(full, o_full.permute(1, 0, 2))
    t = parallel.max_over_ranks(float(rank + 1), "cpu")
    # the C-ABI path: the NCCL unique id made by rank 0 (vsp_comm_unique_id) reaches every rank
    import ctypes
    import paper_2603_04460_b200 as vsp
    lib = vsp.load_library()
    lib.vsp_comm_id_bytes.restype = ctypes.c_size_t

    def make_id():
        buf = ctypes.create_string_buffer(lib.vsp_comm_id_bytes())
        vsp._check(lib.vsp_comm_unique_id(buf))
        return buf.raw

    uid = parallel.exchange_unique_id(make_id)
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    ok_id = len(uid) == 128 and all(x == uid for x in ids)
    # head-major slabs: each rank fills only its slab, an in-place all-gather of the slabs
    # (vsp_allgather_heads semantics) gives the full head-major output
    buf = torch.zeros(hq, n, d)
    slab = parallel.head_slab(buf, rank, world)
    lo, hi = parallel.head_range(hq, rank, world)
    slab.copy_(o_full.permute(1, 0, 2)[lo:hi])
    parts = [torch.empty_like(slab) for _ in range(world)]
    dist.all_gather(parts, slab.contiguous())
    for r_, part in enumerate(parts):
        parallel.head_slab(buf, r_, world).copy_(part)
    ok = ok and ok_id and torch.equal(buf, o_full.permute(1, 0, 2)) and slab.data_ptr() == buf[lo].data_ptr()
    q.put((rank, ok, t, parallel.head_range(8, rank, world)))
    dist.destroy_process_group()


def test_head_sharding_and_assembly_gloo():
    world, n, hq, d = 2, 16, 8, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, hq, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    assert all(ok for _, ok, _, _ in res)
    assert all(t == 2.0 for _, _, t, _ in res)
    assert [r[3] for r in res] == [(0, 4), (4, 8)]


def test_balanced_units_cover_grid_once_and_balance():
    from paper_2603_04460_b200 import parallel
    rng = np.random.default_rng(3)
    hkv, nqb = 8, 100
    cost = rng.integers(0, 40, size=(hkv, nqb))
    cost[6] += np.arange(nqb) * 3  # one heavy, growing head (the adaptive-budget case)
    for world in (1, 2, 3, 4, 8):
        units = parallel.balanced_units(cost, world)
        seen = np.zeros((hkv, nqb), dtype=int)
        for r, us in enumerate(units):
            for g, lo, hi in us:
                assert 0 <= lo < hi <= nqb
                seen[g, lo:hi] += 1
        assert (seen == 1).all()
        assert len(units) == world
        costs = [parallel.units_cost(us, cost, head_overhead=2500.0) for us in units]
        worst_block = float(cost.max()) + 2.0
        ideal = (float(cost.sum()) + 2.0 * cost.size + 2500.0 * hkv) / world
        # min-max contiguous split: within one block and one extra head of the ideal share
        assert max(costs) <= ideal + worst_block + 2 * 2500.0
        # head sharding would put the heavy head's whole cost on one rank
        if world == 8:
            assert max(costs) < 0.5 * (float(cost[6].sum()) + 2.0 * nqb)


def test_balanced_units_float_costs_never_exceed_world():
    """Mean (non-integer) cost tables: the bisection's upper bound must fit in one run even
    when float summation order differs, so world=1 gets exactly one run."""
    from paper_2603_04460_b200 import parallel
    rng = np.random.default_rng(11)
    cost = rng.random((8, 1024)) * 97.3 + 0.1
    for world in (1, 2, 8):
        units = parallel.balanced_units(cost, world, cta_overhead=3.0, head_overhead=2000.0)
        assert len(units) == world
        assert sum(hi - lo for us in units for _, lo, hi in us) == cost.size
    assert len(parallel.balanced_units(cost, 1)[0]) == 8  # one unit per head, one rank


def test_spread_units_cover_every_head_evenly():
    from paper_2603_04460_b200 import parallel
    rng = np.random.default_rng(5)
    hkv, nqb = 8, 300
    cost = rng.integers(0, 50, size=(hkv, nqb)) + np.arange(nqb)[None, :] // 10
    for world in (1, 2, 3, 8):
        units = parallel.spread_units(cost, world)
        assert len(units) == world
        seen = np.zeros((hkv, nqb), dtype=int)
        for us in units:
            for g, lo, hi in us:
                seen[g, lo:hi] += 1
        assert (seen == 1).all()
        per_rank = [parallel.units_cost(us, cost) for us in units]
        worst_block = float(cost.max()) + 2.0
        assert max(per_rank) <= (float(cost.sum()) + 2.0 * cost.size) / world + hkv * worst_block


def _units_worker(rank, world, port, n, hq, hkv, d, split, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_04460_b200 import parallel
    g = torch.Generator().manual_seed(3)
    nqb = (n + 127) // 128
    cost = torch.randint(1, 50, (hkv, nqb), generator=g)
    all_units = (parallel.spread_units(cost, world) if split == "spread"
                 else parallel.balanced_units(cost, world, head_overhead=5.0))
    want_o = torch.randn(hq, n, d, generator=g)  # the assembled layer output, same everywhere
    want_l = torch.randn(hq, n, generator=g)
    # this rank writes only its units' (head, row) regions, as vs_prefill_units does
    o = torch.full((hq, n, d), float("nan"))
    lse = torch.full((hq, n), float("nan"))
    for own, h, lo, hi in parallel.unit_regions(all_units, n, hq, hkv):
        if own == rank:
            o[h, lo:hi] = want_o[h, lo:hi]
            lse[h, lo:hi] = want_l[h, lo:hi]
    parallel.assemble_units(o, lse, all_units, hkv)
    covered = torch.zeros(hq, n, dtype=torch.int32)
    for _, h, lo, hi in parallel.unit_regions(all_units, n, hq, hkv):
        covered[h, lo:hi] += 1
    q.put((rank, bool(torch.equal(o, want_o) and torch.equal(lse, want_l)), bool((covered == 1).all())))
    dist.destroy_process_group()


@pytest.mark.parametrize("split", ["balanced", "spread"])
def test_unit_split_assembly_gloo(split):
    """A unit split's output regions, written by their owners only, assemble bit-exactly on
    every rank (the torch.distributed form of vsp_assemble_units' broadcast schedule), and
    the regions tile the head-major output exactly once."""
    world, n, hq, hkv, d = 2, 1000, 8, 2, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_units_worker, args=(r, world, port, n, hq, hkv, d, split, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok and once for _, ok, once in res), res


def test_merge_path_partition_c_abi_matches_reference():
    """vsp_merge_path_partition (host part of the C ABI, merge.hpp:69-95): MergePath.HandCase
    (test_attention.cpp:328-337) and randomised cuts vs the pinned restatement, plus the
    per-slice merge property (concatenated slice merges reproduce the full merge)."""
    import oracle
    import paper_2603_04460_b200 as vsp
    assert vsp.merge_path_partition([1, 3, 5], [2, 4, 6], 2) == [(0, 0), (2, 1), (3, 3)]
    with pytest.raises(vsp.VspError, match="^merge_path_partition: p must be >= 1$"):
        vsp.merge_path_partition([1], [2], 0)
    rng = np.random.default_rng(45)
    port = oracle.port()
    for _ in range(200):
        a = np.sort(rng.integers(0, 60, int(rng.integers(0, 40))))
        b = np.sort(rng.integers(0, 60, int(rng.integers(0, 40))))
        p = 1 + int(rng.integers(8))
        cuts = vsp.merge_path_partition(a, b, p)
        assert cuts == port.merge_path_partition(a, b, p)
        merged = []
        for s in range(p):
            sa, sb = a[cuts[s][0]:cuts[s + 1][0]], b[cuts[s][1]:cuts[s + 1][1]]
            merged += sorted(list(sa) + list(sb), key=lambda x: x)  # equal keys: values identical
        assert merged == sorted(list(a) + list(b))


def test_balanced_head_sets_equal_counts_and_balance():
    """Cost-aware KV-head placement: equal counts per rank, every head once, and never a worse
    maximum than contiguous slabs on the round-2 bench costs (tiles per KV head)."""
    from paper_2603_04460_b200 import parallel
    costs = [12320, 3069, 3069, 5269, 3069, 38092, 73503, 13852]
    for world in (1, 2, 4, 8):
        sets = parallel.balanced_head_sets(costs, world)
        assert sorted(h for s_ in sets for h in s_) == list(range(8))
        assert all(len(s_) == 8 // world for s_ in sets)
        best = max(sum(costs[h] for h in s_) for s_ in sets)
        contig = max(sum(costs[r * (8 // world):(r + 1) * (8 // world)]) for r in range(world))
        assert best <= contig
    assert parallel.q_heads_of([1, 3], 4) == [4, 5, 6, 7, 12, 13, 14, 15]
