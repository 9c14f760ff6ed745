"""Multi-GPU execution of the fused head-wise attention layer.

One process per GPU (torch.distributed, NCCL on GPUs / gloo in CPU tests).
Every (sample, head) is independent (/root/reference/proj/src/dispatch.cpp:62-83),
so no data-path collective is needed inside the layer:

* sample sharding (configs 4, weak scaling): rank r owns samples
  r, r + W, ... with their own cache slots; zero cross-GPU traffic.
* head sharding (configs 2/3, one sample on W GPUs, strong scaling): heads
  are assigned to ranks longest-processing-time-first on their plan cost
  (Full and Arrow heads carry very different FLOPs, Cached heads are copies),
  each rank runs ONE fused launch over the full layer plan with the heads it
  does not own marked DFA2C_SKIP, and the per-rank outputs are assembled
  with an all-gather over NVLink (all_gather_into_tensor on equal-size padded
  shards). Each rank owns the cache slots of its heads.

Outputs are bitwise identical for any W: a head's result depends only on
its own tile sequence and on scheduling decisions taken from the full layer
plan (DFA2C_SKIP keeps the plan whole), both fixed by the static schedule.

The gather can overlap the compute per head group
(pipelined_sharded_attention): each rank splits its heads into G groups,
launches group g (every other head DFA2C_SKIP), and all-gathers group g's
padded shard on a communication stream while group g+1 computes.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass
from typing import List, Optional, Sequence

from . import api


def head_costs(plan: api.LayerPlan, dims: api.AttentionDims, block_size: int) -> List[float]:
    """Relative cost per head: plan FLOPs of the head, Cached heads as their
    copy traffic expressed in FLOP-equivalents (bytes x 100)."""
    costs = []
    d1 = api.AttentionDims(1, dims.head_dim, dims.n_visual, dims.n_text, dims.order)
    for s in plan.strategies:
        one = api.LayerPlan([s])
        if s.kind == api.StrategyKind.cached:
            costs.append(float(2 * dims.seq_len() * dims.head_dim * 2) * 100.0)
        else:
            costs.append(float(api.plan_flops(one, d1, block_size)))
    return costs


def assign_heads(costs: Sequence[float], world: int) -> List[List[int]]:
    """LPT: heads in descending cost order, each to the least-loaded rank
    (ties to the lower rank); heads within a rank stay ascending."""
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    owner = [[] for _ in range(world)]
    for h in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        load, r = heapq.heappop(heap)
        owner[r].append(h)
        heapq.heappush(heap, (load + costs[h], r))
    return [sorted(o) for o in owner]


def shard_samples(batch: int, world: int, rank: int) -> List[int]:
    """Sample sharding: rank r owns samples r, r + world, ..."""
    return list(range(rank, batch, world))


@dataclass
class HeadShard:
    rank: int
    world: int
    heads: List[int]          # heads this rank computes / owns, ascending
    max_heads: int            # padding so every rank's shard has equal size
    all_heads: List[List[int]]


def make_head_shard(plan: api.LayerPlan, dims: api.AttentionDims, block_size: int, world: int,
                    rank: int) -> HeadShard:
    owner = assign_heads(head_costs(plan, dims, block_size), world)
    return HeadShard(rank, world, owner[rank], max(len(o) for o in owner), owner)


def sub_plan(plan: api.LayerPlan, heads: Sequence[int]) -> api.LayerPlan:
    return api.LayerPlan([plan.strategies[h] for h in heads])


def gather_heads(local_out, shard: HeadShard, full_out, group=None):
    """Assemble [H, N, d] from every rank's [len(heads), N, d] shard.

    All-gather of equal-size (padded to max_heads) shards, then a scatter
    into head order. Works on any torch.distributed backend (NCCL over
    NVLink on GPUs, gloo in CPU tests)."""
    import torch
    import torch.distributed as dist

    n, d = local_out.shape[-2], local_out.shape[-1]
    padded = local_out.new_zeros((shard.max_heads, n, d))
    if len(shard.heads):
        padded[: len(shard.heads)] = local_out
    gathered = local_out.new_empty((shard.world * shard.max_heads, n, d))
    if shard.world == 1:
        gathered.copy_(padded)
    elif dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(gathered, padded, group=group)
    else:  # gloo (CPU tests): list form
        parts = list(gathered.chunk(shard.world))
        dist.all_gather(parts, padded, group=group)
        gathered = torch.cat(parts)
    for r, hs in enumerate(shard.all_heads):
        for i, h in enumerate(hs):
            full_out[h].copy_(gathered[r * shard.max_heads + i])
    return full_out


def sharded_multi_strategy_attention(q, k, v, plan: api.LayerPlan, cache: Optional[api.HeadCache], layer: int,
                                     t: int, dims: api.AttentionDims, block_size: int, shard: HeadShard,
                                     gather: bool = True, out=None):
    """One sample on W GPUs: this rank runs ONE fused launch over the whole
    layer plan with every head it does not own marked DFA2C_SKIP, so the
    kernel's scheduling decisions (split-KV) follow the full plan and each
    head's result is bitwise what a single-GPU call gives. The rank's cache
    is the layer-shaped cache; only its own heads' slots are ever touched.
    Then the owned heads are all-gathered. q/k/v: the full [H, N, d] sample
    (replicated)."""
    import torch

    heads = shard.heads
    owned = set(heads)
    full = out if out is not None else torch.empty_like(q)
    if heads:
        api.multi_strategy_attention(q, k, v, plan, cache, layer, t, dims, block_size, out=full,
                                     skip_heads=[h for h in range(dims.n_heads) if h not in owned])
    idx = torch.tensor(heads, device=q.device, dtype=torch.long)
    local = full.index_select(0, idx) if heads else q.new_empty((0,) + tuple(q.shape[1:]))
    if not gather:
        return local
    return gather_heads(local, shard, full)


@dataclass
class HeadGroups:
    """Per rank, its heads split into G consecutive groups; sizes[g] = the
    largest group g over the ranks (the padded all-gather shard)."""

    per_rank: List[List[List[int]]]
    sizes: List[int]


def head_groups(shard: HeadShard, n_groups: int) -> HeadGroups:
    n_groups = max(1, n_groups)
    per_rank = []
    for hs in shard.all_heads:
        q, r = divmod(len(hs), n_groups)
        out, i = [], 0
        for g in range(n_groups):
            c = q + (1 if g < r else 0)
            out.append(list(hs[i:i + c]))
            i += c
        per_rank.append(out)
    sizes = [max(len(per_rank[r][g]) for r in range(shard.world)) for g in range(n_groups)]
    return HeadGroups(per_rank, sizes)


def pipelined_sharded_attention(compute_group, full_out, shard: HeadShard, n_groups: int, group=None,
                                comm_stream=None):
    """Compute + gather per head group. compute_group(heads) writes those
    heads of full_out (on the current stream); after each group its padded
    shard is all-gathered — on NCCL from `comm_stream` (which waits for the
    group's compute), so the transfer overlaps the next group's compute; on
    gloo (CPU tests) synchronously. Returns full_out with every rank's heads."""
    import torch
    import torch.distributed as dist

    hg = head_groups(shard, n_groups)
    mine = hg.per_rank[shard.rank]
    n, d = full_out.shape[-2], full_out.shape[-1]
    nccl = shard.world > 1 and dist.get_backend(group) == "nccl"
    pending = []
    for g in range(len(mine)):
        hs = mine[g]
        if hs:
            compute_group(hs)
        if shard.world == 1:
            continue
        padded = full_out.new_zeros((hg.sizes[g], n, d))
        if hs:
            padded[: len(hs)] = full_out[hs]
        gathered = full_out.new_empty((shard.world * hg.sizes[g], n, d))
        if nccl:
            ev = torch.cuda.current_stream().record_event()
            cs = comm_stream or torch.cuda.Stream()
            with torch.cuda.stream(cs):
                cs.wait_event(ev)
                work = dist.all_gather_into_tensor(gathered, padded, group=group, async_op=True)
            pending.append((g, gathered, padded, work))
        else:
            parts = list(gathered.chunk(shard.world))
            dist.all_gather(parts, padded, group=group)
            pending.append((g, torch.cat(parts), padded, None))
    for g, gathered, _padded, work in pending:
        if work is not None:
            work.wait()  # the current stream waits for the collective
        for r in range(shard.world):
            if r == shard.rank:
                continue
            for i, h in enumerate(hg.per_rank[r][g]):
                full_out[h].copy_(gathered[r * hg.sizes[g] + i])
    return full_out
