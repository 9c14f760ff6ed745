"""Multi-GPU execution of the fused head-wise attention layer.

One process per GPU. Every (sample, head, query block) is independent
(/root/reference/proj/src/dispatch.cpp:62-83, src/arrow.cpp:181-193), so
there is no data-path exchange inside the layer:

* sample sharding (config 4, weak scaling): rank r owns samples
  r, r + W, ... with their own cache slots; zero cross-GPU traffic.
* row sharding (configs 2/3: one sample on W GPUs, strong scaling): the
  C++ host (dfa2c_mha_forward_sharded) cuts the layer's (sample, head,
  query-tile pair) sequence into W contiguous ranges of near-equal plan
  cost; each rank's ONE fused launch computes its range over all 148 SMs,
  long pairs run as key chunks against a fixed 8-GPU reference (so every
  head's bits are the same for every W), and the ranges are all-gathered in
  place with one NCCL group of W broadcasts over NVLink / NVSwitch (the only
  collective). After the gather every rank commits all computed rows to
  its own cache, so caches stay complete whatever the next timestep's plan
  assigns to which rank (a Cached head never misses or goes stale).

This module is the Python face of that C++ path: it builds the library's
NCCL communicator from a torch.distributed group, and offers a
torch.distributed gather (gloo on CPU tests, or any backend) for callers
without NCCL.
"""
from __future__ import annotations

from typing import List, Optional

from . import api


def shard_samples(batch: int, world: int, rank: int) -> List[int]:
    """Sample sharding: rank r owns samples r, r + world, ..."""
    return list(range(rank, batch, world))


def gather_rows(out, bounds, rank: int, world: int, group=None):
    """In-place all-gather of the row ranges [bounds[r], bounds[r+1]) of the
    flattened [batch*H*N, d] view of `out` through torch.distributed (one
    broadcast per rank; CUDA tensors are staged through host memory on
    backends without CUDA support, e.g. gloo)."""
    import torch.distributed as dist

    if world == 1:
        return out
    flat = out.reshape(-1, out.shape[-1])
    host = dist.get_backend(group) != "nccl" and flat.is_cuda
    for r in range(world):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        if hi <= lo:
            continue
        part = flat[lo:hi]
        if host:
            buf = part.cpu()
            dist.broadcast(buf, src=r, group=group)
            if r != rank:
                part.copy_(buf)
        else:
            dist.broadcast(part, src=r, group=group)
    return out


class PeerOutputs:
    """Every rank's output buffer mapped into this process through CUDA IPC
    (dfa2c_ipc_handle / dfa2c_ipc_open; handles exchanged over the given
    torch.distributed group), for api.multi_strategy_attention_sharded_p2p:
    the fused kernel then writes each rank's rows into all ranks' buffers
    over NVLink, so the layer is assembled without a collective."""

    def __init__(self, out, rank: int, world: int, group=None):
        import ctypes

        import torch.distributed as dist

        lib = api.lib()
        h = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        api.check(lib.dfa2c_ipc_handle(ctypes.c_void_p(out.data_ptr()), h, ctypes.byref(off)))
        mine = (h.raw, off.value)
        allh = [None] * world
        if world > 1:
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        self.rank, self.world = rank, world
        self._opened = []  # (ptr, offset) this process mapped
        self.outs = []
        for r in range(world):
            if r == rank:
                self.outs.append(out)
                continue
            p = ctypes.c_void_p()
            api.check(lib.dfa2c_ipc_open(allh[r][0], allh[r][1], ctypes.byref(p)))
            self._opened.append((p.value, allh[r][1]))
            self.outs.append(p.value)

    def close(self):
        import ctypes

        for p, off in self._opened:
            api.check(api.lib().dfa2c_ipc_close(ctypes.c_void_p(p), off))
        self._opened = []


def sharded_multi_strategy_attention(q, k, v, plan: api.LayerPlan, cache: Optional[api.HeadCache], layer: int,
                                     t: int, dims: api.AttentionDims, block_size: int, rank: int, world: int,
                                     comm: Optional[api.NcclComm] = None, group=None, out=None, gather: bool = True):
    """One sample (or batch) on `world` GPUs: this rank's fused launch over
    its row range, then the assembly. With `comm` the library all-gathers and
    commits in C++ (NCCL); otherwise, if `gather`, the ranges are gathered
    through torch.distributed and the other ranks' computed rows committed
    with api.shard_commit. Returns (out, row_bounds)."""
    out, bounds = api.multi_strategy_attention_sharded(q, k, v, plan, cache, layer, t, dims, block_size, rank,
                                                       world, comm=comm, out=out)
    if comm is None and gather and world > 1:
        gather_rows(out, bounds, rank, world, group)
        if cache is not None:
            api.shard_commit(out, plan, cache, layer, dims, bounds, rank, world)
    return out, bounds
