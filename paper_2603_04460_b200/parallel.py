"""KV-head sharding of the VS-prefill layer across the GPUs of one node.

Every hot-path step is per KV head (indexer, selection, and the sparse attention of the Q
heads in the group), so a layer splits into independent shards with NO collective on the
data path. Rank r owns KV heads [r*Hkv/N, (r+1)*Hkv/N) and their Q heads. The only
collective is the all-gather that assembles the full output. The sharded layer writes its
O head-major straight into its slab of the full [Hq, n, d] buffer (`head_slab`,
VSP_O_HEAD_MAJOR), so the slab IS the send buffer and `VspComm.allgather_heads` is one
in-place ncclAllGather over NVLink/NVSwitch through the C ABI (vsp_allgather_heads) — no
permute and no staging copy. `assemble_heads` is the torch.distributed equivalent for a
token-major shard.

Cost-aware head placement (`balanced_head_sets`): the heads split keeps whole KV heads and
equal head counts per rank, but places them by predicted cost instead of in contiguous
slabs; O is then all-gathered in the placement order and permuted once.

Balanced split (SURVEY.md §8e refinement, `balanced_units`): adaptive per-head budgets make
KV heads unequal — in the 128k bench one head carries ~40% of the tiles, so 8-way head
sharding would run at ~2.5x instead of 8x. With replicated Q/K/V, the (KV head, query
block) grid is cut into `world` contiguous runs of equal predicted cost (tile counts of a
calibration prompt + a per-CTA overhead); each rank scores/selects only the heads its run
touches and attends its units (`vs_prefill_units`). Still no collective on the data path.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist


def head_range(num_heads: int, rank: int, world: int) -> Tuple[int, int]:
    if num_heads % world:
        raise ValueError(f"{num_heads} heads do not split across {world} ranks")
    per = num_heads // world
    return rank * per, (rank + 1) * per


def shard_heads(x: torch.Tensor, rank: int, world: int, dim: int = 1) -> torch.Tensor:
    """Contiguous slice of the head dimension owned by `rank` (token-major [n, H, d] -> dim 1;
    per-head parameter tensors [H, ...] -> dim 0)."""
    lo, hi = head_range(x.shape[dim], rank, world)
    return x.narrow(dim, lo, hi - lo).contiguous()


def assemble_heads(o_shard: torch.Tensor, group=None) -> torch.Tensor:
    """[n, Hq/N, d] per rank -> [Hq, n, d] everywhere (head-major), one all-gather."""
    world = dist.get_world_size(group)
    oh = o_shard.permute(1, 0, 2).contiguous()
    full = torch.empty((world * oh.shape[0],) + tuple(oh.shape[1:]), dtype=oh.dtype, device=oh.device)
    dist.all_gather_into_tensor(full, oh, group=group)
    return full


def max_over_ranks(value: float, device) -> float:
    """Device-timed numbers are reported as the max over ranks."""
    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def head_slab(o_full: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """Rank `rank`'s contiguous slab [Hq/N, n, d] of a head-major output [Hq, n, d]: the
    `out=` of vs_prefill / sparse_attention with head_major=True, and the in-place send
    buffer of VspComm.allgather_heads."""
    lo, hi = head_range(o_full.shape[0], rank, world)
    return o_full[lo:hi]


def exchange_unique_id(make_id, group=None) -> bytes:
    """Rank 0 makes the NCCL unique id and every rank of `group` receives it (over whatever
    backend the group has: gloo on CPU, nccl on GPU)."""
    box = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return box[0]


class VspComm:
    """An NCCL communicator owned by the C ABI (vsp_comm_init) for vsp_allgather_heads."""

    def __init__(self, device: torch.device, group=None):
        from . import _check, load_library
        self._lib = lib = load_library()
        lib.vsp_comm_id_bytes.restype = ctypes.c_size_t
        lib.vsp_comm_unique_id.argtypes = [ctypes.c_char_p]
        lib.vsp_comm_init.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                      ctypes.c_int]
        lib.vsp_comm_destroy.argtypes = [ctypes.c_void_p]
        lib.vsp_allgather_heads.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        self._check = _check
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device

        def make_id():
            buf = ctypes.create_string_buffer(lib.vsp_comm_id_bytes())
            _check(lib.vsp_comm_unique_id(buf))
            return buf.raw

        uid = exchange_unique_id(make_id, group) if self.world > 1 else make_id()
        h = ctypes.c_void_p()
        _check(lib.vsp_comm_init(ctypes.byref(h), self.world, self.rank, uid, device.index or 0))
        self._h = h

    def allgather_heads(self, o_full: torch.Tensor, lse_full: Optional[torch.Tensor] = None) -> None:
        """In-place: this rank's slab of o_full [Hq, n, d] (and lse_full [Hq, n]) -> everywhere."""
        hq, n, d = o_full.shape
        st = ctypes.c_void_p(torch.cuda.current_stream(o_full.device).cuda_stream)
        self._check(self._lib.vsp_allgather_heads(self._h, ctypes.c_void_p(o_full.data_ptr()),
                                                  ctypes.c_void_p(lse_full.data_ptr() if lse_full is not None else 0),
                                                  n, hq, d, st))

    def assemble_units(self, o_full: torch.Tensor, lse_full: Optional[torch.Tensor], all_units, hkv: int) -> None:
        """In-place assembly of a unit split: all_units[r] = rank r's units (g, qb_lo, qb_hi);
        every region goes from its owner to every rank (vsp_assemble_units: one ncclBroadcast
        per (unit, Q head) in one NCCL group)."""
        hq, n, d = o_full.shape
        flat = [(r, g, lo, hi) for r, us in enumerate(all_units) for g, lo, hi in us]
        arr = (ctypes.c_int32 * (4 * max(len(flat), 1)))(*[x for u in flat for x in u])
        lib = self._lib
        lib.vsp_assemble_units.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                           ctypes.c_void_p]
        st = ctypes.c_void_p(torch.cuda.current_stream(o_full.device).cuda_stream)
        self._check(lib.vsp_assemble_units(self._h, ctypes.c_void_p(o_full.data_ptr()),
                                           ctypes.c_void_p(lse_full.data_ptr() if lse_full is not None else 0),
                                           n, hq, hkv, d, ctypes.cast(arr, ctypes.c_void_p), len(flat), st))

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._check(self._lib.vsp_comm_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unit_regions(all_units, n: int, hq: int, hkv: int) -> List[Tuple[int, int, int, int]]:
    """(owner rank, Q head, row_lo, row_hi) of every head-major output region a unit split
    writes: all_units[r] = rank r's units (g, qb_lo, qb_hi) over 128-row query blocks."""
    grp = hq // hkv
    return [(r, h, lo * 128, min(hi * 128, n)) for r, us in enumerate(all_units) for g, lo, hi in us
            for h in range(g * grp, (g + 1) * grp)]


def assemble_units(o_full: torch.Tensor, lse_full: Optional[torch.Tensor], all_units, hkv: int,
                   group=None) -> None:
    """torch.distributed form of VspComm.assemble_units (any backend; gloo on CPU in the
    tests): one broadcast per region from its owner, in place on every rank."""
    hq, n, _ = o_full.shape
    for r, h, lo, hi in unit_regions(all_units, n, hq, hkv):
        src = dist.get_global_rank(group, r) if group is not None else r
        reg = o_full[h, lo:hi]
        dist.broadcast(reg, src=src, group=group)  # contiguous: head-major rows of one head
        if lse_full is not None:
            dist.broadcast(lse_full[h, lo:hi], src=src, group=group)


def balanced_head_sets(head_cost, world: int) -> List[List[int]]:
    """KV-head sharding with cost-aware placement: every rank gets hkv / world WHOLE KV heads
    (the all-gather slabs stay equal), chosen so the most expensive rank is as cheap as the
    greedy longest-first rule makes it (heads by descending cost, each to the cheapest rank
    that still has room; ties to the lower rank). head_cost: predicted cost per KV head
    (e.g. tile counts of a calibration prompt plus a per-head overhead). Deterministic, so
    every rank computes the same sets. Returns per rank its heads, ascending."""
    costs = [float(c) for c in (head_cost.tolist() if hasattr(head_cost, "tolist") else head_cost)]
    hkv = len(costs)
    if hkv % world:
        raise ValueError(f"{hkv} KV heads do not split across {world} ranks")
    per = hkv // world
    load = [0.0] * world
    sets: List[List[int]] = [[] for _ in range(world)]
    for g in sorted(range(hkv), key=lambda h: (-costs[h], h)):
        r = min((r for r in range(world) if len(sets[r]) < per), key=lambda r: (load[r], r))
        sets[r].append(g)
        load[r] += costs[g]
    return [sorted(x) for x in sets]


def q_heads_of(kv_heads: List[int], grp: int) -> List[int]:
    """The Q heads (GQA groups of size grp) of the given KV heads, in order."""
    return [g * grp + j for g in kv_heads for j in range(grp)]


def balanced_units(cost, world: int, cta_overhead: float = 2.0, head_overhead: float = 2500.0
                   ) -> List[List[Tuple[int, int, int]]]:
    """Cut the (KV head, query block) grid, walked head-major, into `world` contiguous runs
    minimising the most expensive run. cost: [hkv, num_qb] predicted tiles per (head, block)
    (e.g. sparse_tile_counts on a calibration prompt); every block also pays `cta_overhead`
    tile-equivalents and every head a run touches pays `head_overhead` (its scoring,
    selection and planning). Smallest feasible bound by bisection with a greedy fill.
    Returns per rank a list of units (g, qb_lo, qb_hi)."""
    rows = [[float(x) + cta_overhead for x in r] for r in (cost.tolist() if hasattr(cost, "tolist") else cost)]
    hkv, nqb = len(rows), len(rows[0])
    flat = [(g, b, rows[g][b]) for g in range(hkv) for b in range(nqb)]

    def fill(bound: float):
        out: List[List[Tuple[int, int, int]]] = [[]]
        acc, cur_g = 0.0, -1
        for g, b, c in flat:
            add = c + (head_overhead if g != cur_g else 0.0)
            if out[-1] and acc + add > bound:
                out.append([])
                acc, cur_g = 0.0, -1
                add = c + head_overhead
            units = out[-1]
            if units and units[-1][0] == g and units[-1][2] == b:
                units[-1] = (g, units[-1][1], b + 1)
            else:
                units.append((g, b, b + 1))
            acc += add
            cur_g = g
        return out

    lo = max(c for _, _, c in flat) + head_overhead
    # a bound every fill() meets in one run, whatever the float summation order
    hi = (sum(c for _, _, c in flat) + head_overhead * hkv) * (1.0 + 1e-9) + 1.0
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if len(fill(mid)) <= world:
            hi = mid
        else:
            lo = mid
    out = fill(hi)
    assert len(out) <= world
    return out + [[] for _ in range(world - len(out))]


def spread_units(cost, world: int, cta_overhead: float = 2.0) -> List[List[Tuple[int, int, int]]]:
    """Split EVERY KV head's query blocks into `world` contiguous runs of equal predicted cost
    (tiles + per-block overhead) and give rank r the r-th run of each head. A rank's share is
    then ~1/world of every head, so it does not depend on how the cost splits across heads —
    the part of a static cost table that moves most from prompt to prompt — at the price of
    every rank scoring every head. Returns per rank a list of units (g, qb_lo, qb_hi)."""
    rows = [[float(x) + cta_overhead for x in r] for r in (cost.tolist() if hasattr(cost, "tolist") else cost)]
    out: List[List[Tuple[int, int, int]]] = [[] for _ in range(world)]
    for g, r in enumerate(rows):
        total = sum(r)
        bounds, acc, b = [0], 0.0, 0
        for k in range(1, world):
            target = total * k / world
            while b < len(r) and acc + r[b] <= target:
                acc += r[b]
                b += 1
            bounds.append(b)
        bounds.append(len(r))
        for k in range(world):
            if bounds[k + 1] > bounds[k]:
                out[k].append((g, bounds[k], bounds[k + 1]))
    return out


def units_cost(units, cost, cta_overhead: float = 2.0, head_overhead: float = 0.0) -> float:
    rows = cost.tolist() if hasattr(cost, "tolist") else cost
    heads = {g for g, _, _ in units}
    return (sum(float(rows[g][b]) + cta_overhead for g, lo, hi in units for b in range(lo, hi))
            + head_overhead * len(heads))
