"""Python mirror of the reference's `dfa2` operator API for the fused head-wise
attention path, on top of the C-ABI (include/dfa2c.h).

Names, argument meaning and error behaviour follow
/root/reference/proj/include/dfa2/{tensor,arrow,dispatch,cache,plan,calibrate}.hpp
so tests read like the reference's own (tests/test_*.cpp). Tensors are torch
CUDA tensors: bf16 is the compute type; f32 inputs are rounded to bf16 at the
boundary (the reference computes in f32; see DESIGN.md for the tolerance).
There is no CPU fallback: every attention / RSE value comes from the sm_100a
kernels of libdfa2_b200.so.
"""
from __future__ import annotations

import ctypes
import math
from ctypes import POINTER, byref, c_double, c_int32, c_int64, c_uint8, c_uint32, c_void_p
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (  # noqa: F401  (re-exported error taxonomy)
    CacheMissError,
    CudaError,
    DegenerateReferenceError,
    Dfa2Error,
    FullyMaskedRowError,
    IoError,
    NonFiniteError,
    OracleError,
    PlanValidationError,
    ShapeError,
    UnsupportedError,
    check,
    lib,
)

VISUAL_FIRST = "visual_first"
TEXT_FIRST = "text_first"


# --------------------------------------------------------------- geometry
@dataclass
class AttentionDims:
    """AttentionDims (inc/tensor.hpp:56-72)."""

    n_heads: int = 0
    head_dim: int = 0
    n_visual: int = 0
    n_text: int = 0
    order: str = VISUAL_FIRST

    def seq_len(self) -> int:
        return self.n_visual + self.n_text

    def text_begin(self) -> int:
        return self.n_visual if self.order == VISUAL_FIRST else 0

    def text_end(self) -> int:
        return self.seq_len() if self.order == VISUAL_FIRST else self.n_text

    def c(self) -> _lib.Dims:
        if self.order not in (VISUAL_FIRST, TEXT_FIRST):
            raise ShapeError(f"unknown token order {self.order!r}")
        return _lib.Dims(self.n_heads, self.head_dim, self.n_visual, self.n_text,
                         0 if self.order == VISUAL_FIRST else 1)

    def validate(self) -> None:
        if self.n_heads < 1 or self.head_dim < 1:
            raise ShapeError("n_heads and head_dim must be >= 1")
        if self.n_visual < 1 or self.n_text < 0:
            raise ShapeError("need n_visual >= 1 and n_text >= 0")


def _ceil_div(a: int, b: int) -> int:
    return (a + b - 1) // b


# --------------------------------------------------------------- masks
@dataclass
class BlockMask:
    """BlockMask (inc/arrow.hpp:12-34): row-major uint8 [nqb * nkb]."""

    block_size: int = 0
    seq_len: int = 0
    n_query_blocks: int = 0
    n_key_blocks: int = 0
    active: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    @staticmethod
    def all_active(seq_len: int, block_size: int) -> "BlockMask":
        if block_size < 1:
            raise ShapeError("block_size must be >= 1")
        if seq_len < 1:
            raise ShapeError("seq_len must be >= 1")
        nb = _ceil_div(seq_len, block_size)
        return BlockMask(block_size, seq_len, nb, nb, np.ones(nb * nb, np.uint8))

    def is_active(self, i: int, j: int) -> bool:
        return bool(self.active[i * self.n_key_blocks + j])

    def set(self, i: int, j: int, v: bool) -> None:
        self.active[i * self.n_key_blocks + j] = 1 if v else 0

    def block_begin(self, i: int) -> int:
        return i * self.block_size

    def block_len(self, i: int) -> int:
        return min(self.block_size, self.seq_len - i * self.block_size)

    def _stats(self, head_dim: int = 1):
        a = np.ascontiguousarray(self.active, dtype=np.uint8)
        ap, fl, sp = c_int64(), c_int64(), c_double()
        check(lib().dfa2c_mask_stats(a.ctypes.data_as(POINTER(c_uint8)), self.seq_len, self.block_size,
                                     head_dim, byref(ap), byref(fl), byref(sp)))
        return ap.value, fl.value, sp.value

    def active_positions(self) -> int:
        return self._stats()[0]

    def row_has_active(self, i: int) -> bool:
        return bool(self.active[i * self.n_key_blocks:(i + 1) * self.n_key_blocks].any())

    def grid(self) -> np.ndarray:
        return self.active.reshape(self.n_query_blocks, self.n_key_blocks)


@dataclass
class ArrowSpec:
    """ArrowSpec (inc/arrow.hpp:39-43)."""

    dims: AttentionDims
    block_size: int = 0
    window_blocks: int = 0


def build_arrow_mask(spec: ArrowSpec) -> BlockMask:
    """build_arrow_mask (inc/arrow.hpp:45; src/arrow.cpp:113-153), bit-exact."""
    d = spec.dims.c()
    nb = c_int64()
    check(lib().dfa2c_arrow_mask(byref(d), spec.block_size, spec.window_blocks, None, byref(nb)))
    active = np.zeros(nb.value * nb.value, np.uint8)
    check(lib().dfa2c_arrow_mask(byref(d), spec.block_size, spec.window_blocks,
                                 active.ctypes.data_as(POINTER(c_uint8)), byref(nb)))
    return BlockMask(spec.block_size, spec.dims.seq_len(), nb.value, nb.value, active)


def flops_count(mask: BlockMask, head_dim: int) -> int:
    """4*d per active (query, key) position (src/arrow.cpp:155-159)."""
    if head_dim < 1:
        raise ShapeError("head_dim must be >= 1")
    return mask._stats(head_dim)[1]


def dense_flops(seq_len: int, head_dim: int) -> int:
    return int(lib().dfa2c_dense_flops(seq_len, head_dim))


def sparsity_ratio(mask: BlockMask) -> float:
    return mask._stats()[2]


def tile_set(dims: AttentionDims, block_size: int, strategy: "HeadStrategy"):
    """The scheduler's KV tile list per 128-row query tile (CSR row_ptr, cols)."""
    d = dims.c()
    kind = {StrategyKind.full: 0, StrategyKind.arrow: 1}.get(strategy.kind)
    if kind is None:
        raise ShapeError("tile sets exist for Full and Arrow heads only")
    n = c_int64()
    check(lib().dfa2c_tile_set(byref(d), block_size, kind, strategy.window_blocks, None, None, byref(n)))
    nqt = _ceil_div(dims.seq_len(), 128)
    row_ptr = np.zeros(nqt + 1, np.int64)
    cols = np.zeros(max(n.value, 1), np.uint32)
    check(lib().dfa2c_tile_set(byref(d), block_size, kind, strategy.window_blocks,
                               row_ptr.ctypes.data_as(POINTER(c_int64)), cols.ctypes.data_as(POINTER(c_uint32)),
                               byref(n)))
    return row_ptr, cols[: n.value]


# --------------------------------------------------------------- plans
class StrategyKind:
    full = "full"
    arrow = "arrow"
    cached = "cached"


_KIND_CODE = {StrategyKind.full: 0, StrategyKind.arrow: 1, StrategyKind.cached: 2}


@dataclass(frozen=True)
class HeadStrategy:
    """HeadStrategy (inc/dispatch.hpp:14-25)."""

    kind: str = StrategyKind.full
    window_blocks: int = 0

    @staticmethod
    def Full() -> "HeadStrategy":
        return HeadStrategy(StrategyKind.full, 0)

    @staticmethod
    def Arrow(w: int) -> "HeadStrategy":
        return HeadStrategy(StrategyKind.arrow, int(w))

    @staticmethod
    def Cached() -> "HeadStrategy":
        return HeadStrategy(StrategyKind.cached, 0)


@dataclass
class LayerPlan:
    """LayerPlan (inc/dispatch.hpp:28-37)."""

    strategies: List[HeadStrategy] = field(default_factory=list)

    @staticmethod
    def all_full(n_heads: int) -> "LayerPlan":
        return LayerPlan([HeadStrategy.Full() for _ in range(n_heads)])

    def n_heads(self) -> int:
        return len(self.strategies)

    def __getstate__(self):  # the ctypes cache does not pickle (plans cross process groups)
        st = dict(self.__dict__)
        st.pop("_arr_cache", None)
        return st

    def _arrays_cached(self):
        # the per-call ctypes arrays of an unchanged plan (read-only use): a
        # layer call's host cost is otherwise dominated by rebuilding them
        key = tuple(self.strategies)
        c = self.__dict__.get("_arr_cache")
        if c is None or c[0] != key:
            c = (key, self.arrays())
            self.__dict__["_arr_cache"] = c
        return c[1]

    def arrays(self):
        kinds = (c_int32 * max(1, len(self.strategies)))(*[_KIND_CODE[s.kind] for s in self.strategies])
        wins = (c_int64 * max(1, len(self.strategies)))(*[s.window_blocks for s in self.strategies])
        return kinds, wins

    @staticmethod
    def parse(text: str) -> "LayerPlan":
        """'F A8 C A0' -> LayerPlan (bench / test shorthand)."""
        out = []
        for tok in text.split():
            if tok == "F":
                out.append(HeadStrategy.Full())
            elif tok == "C":
                out.append(HeadStrategy.Cached())
            elif tok.startswith("A"):
                out.append(HeadStrategy.Arrow(int(tok[1:])))
            else:
                raise ShapeError(f"bad plan token {tok!r}")
        return LayerPlan(out)


def plan_flops(plan: LayerPlan, dims: AttentionDims, block_size: int) -> int:
    """plan_flops (inc/dispatch.hpp:51-52; src/dispatch.cpp:93-120)."""
    d = dims.c()
    if plan.n_heads() != dims.n_heads:
        raise ShapeError("plan must assign exactly one strategy per head")
    kinds, wins = plan.arrays()
    out = c_int64()
    check(lib().dfa2c_plan_flops(byref(d), block_size, kinds, wins, byref(out)))
    return out.value


# --------------------------------------------------------------- tensors
def _torch():
    import torch

    return torch


def _stream_ptr(stream=None) -> Optional[int]:
    torch = _torch()
    if stream is not None:
        return stream.cuda_stream
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # the current stream without a Stream object
    if raw is not None:
        return raw(torch._C._cuda_getDevice())
    return torch.cuda.current_stream().cuda_stream


def _as_bf16_cuda(x, name: str):
    torch = _torch()
    if not isinstance(x, torch.Tensor):
        raise ShapeError(f"{name} must be a torch tensor")
    if not x.is_cuda:
        raise ShapeError(f"{name} must be a CUDA tensor (the path has no CPU implementation)")
    if x.dtype == torch.float32:
        x = x.to(torch.bfloat16)
    elif x.dtype != torch.bfloat16:
        raise ShapeError(f"{name} must be bf16 (or f32, rounded to bf16)")
    return x.contiguous()


# --------------------------------------------------------------- cache
def _device_out(out, like, shape_given, name="out"):
    """Validates a caller-supplied device output buffer (CUDA, bf16,
    contiguous, on q's device, shaped like the caller's q) and returns a view
    with `like`'s (4-D) shape; None -> a fresh buffer."""
    torch = _torch()
    if out is None:
        return torch.empty_like(like)
    if not isinstance(out, torch.Tensor) or not out.is_cuda or out.dtype != torch.bfloat16:
        raise ShapeError(f"{name} must be a CUDA bf16 tensor")
    if not out.is_contiguous():
        raise ShapeError(f"{name} must be contiguous")
    if out.get_device() != like.get_device():
        raise ShapeError(f"{name} must be on q's device")
    if out.shape != shape_given and tuple(out.shape) != tuple(shape_given):
        raise ShapeError(f"{name} must have q's shape {tuple(shape_given)} (got {tuple(out.shape)})")
    return out if out.shape == like.shape else out.view(like.shape)


class HeadCache:
    """HeadCache (inc/cache.hpp:15-32), device resident.

    One bf16 slot [batch, N, d] per (layer, head). store() deep-copies,
    fetch() returns a fresh tensor, produced_at/staleness follow
    src/cache.cpp:7-41 (CacheMissError on empty slots).
    """

    def __init__(self, n_layers: int, n_heads: int, seq_len: int, head_dim: int, batch: int = 1):
        self.n_layers, self.n_heads, self.seq_len, self.head_dim, self.batch = (
            n_layers, n_heads, seq_len, head_dim, batch)
        h = c_void_p()
        check(lib().dfa2c_cache_create(n_layers, n_heads, batch, seq_len, head_dim, byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().dfa2c_cache_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self) -> c_void_p:
        return self._h

    def store(self, layer: int, head: int, output, t: int) -> None:
        x = _as_bf16_cuda(output, "output")
        if x.dim() == 2:
            x = x.unsqueeze(0)
        if tuple(x.shape) != (self.batch, self.seq_len, self.head_dim):
            raise ShapeError("cache entries are per-head [N, d] tensors")
        check(lib().dfa2c_cache_store(self._h, layer, head, c_void_p(x.data_ptr()), t, c_void_p(_stream_ptr())))

    def fetch(self, layer: int, head: int):
        torch = _torch()
        out = torch.empty(self.batch, self.seq_len, self.head_dim, dtype=torch.bfloat16, device="cuda")
        check(lib().dfa2c_cache_fetch(self._h, layer, head, c_void_p(out.data_ptr()), c_void_p(_stream_ptr())))
        return out[0] if self.batch == 1 else out

    def has(self, layer: int, head: int) -> bool:
        v = c_int32()
        check(lib().dfa2c_cache_has(self._h, layer, head, byref(v)))
        return bool(v.value)

    def produced_at(self, layer: int, head: int) -> int:
        v = c_int64()
        check(lib().dfa2c_cache_produced_at(self._h, layer, head, byref(v)))
        return v.value

    def staleness(self, layer: int, head: int, t: int) -> int:
        v = c_int64()
        check(lib().dfa2c_cache_staleness(self._h, layer, head, t, byref(v)))
        return v.value

    def clear(self) -> None:
        check(lib().dfa2c_cache_clear(self._h))

    def size(self) -> int:
        v = c_int64()
        check(lib().dfa2c_cache_size(self._h, byref(v)))
        return v.value

    def nbytes(self) -> int:
        v = c_int64()
        check(lib().dfa2c_cache_bytes(self._h, byref(v)))
        return v.value


# --------------------------------------------------------------- attention
def _plan_kinds(plan: LayerPlan, skip_heads):
    if not skip_heads:
        return plan._arrays_cached()
    kinds, wins = plan.arrays()
    for h in skip_heads or ():
        if not 0 <= h < plan.n_heads():
            raise ShapeError(f"skip head {h} out of range")
        kinds[h] |= SKIP
    return kinds, wins


SKIP = 0x100  # DFA2C_SKIP


def set_split_kv(on: bool) -> None:
    """dfa2c_set_split_kv: split-KV scheduling for latency-bound layers
    (process-wide; default off, or DFA2_SPLIT_KV=1)."""
    check(lib().dfa2c_set_split_kv(1 if on else 0))


def set_influence_fused(on: bool) -> None:
    """dfa2c_set_influence_fused: influence_for_layer evaluates the original and
    every Arrow candidate in one fused launch (window-band snapshots; default
    on, or DFA2_INFLUENCE_FUSED=0). Off: one pass per candidate, outputs bitwise
    those of multi_strategy_attention."""
    check(lib().dfa2c_set_influence_fused(1 if on else 0))


def release_cached_memory() -> None:
    """dfa2c_release_cached_memory: drop cached work lists and trim the
    library's device memory pool (synchronises the device)."""
    check(lib().dfa2c_release_cached_memory())


def influence_fused_enabled() -> bool:
    return bool(lib().dfa2c_influence_fused_enabled())


def multi_strategy_attention(q, k, v, plan: LayerPlan, cache: Optional[HeadCache], layer: int, t: int,
                             dims: AttentionDims, block_size: int, out=None, stream=None, skip_heads=None):
    """multi_strategy_attention (inc/dispatch.hpp:44-47; src/dispatch.cpp:30-91).

    q/k/v: [H, N, d] or [batch, H, N, d] CUDA tensors. One fused sm_100a
    launch: Full/Arrow heads computed, Cached heads copied from `cache`,
    computed heads committed to `cache` (produced_at = t). skip_heads: heads
    of the layer this call leaves alone (DFA2C_SKIP; e.g. the heads another
    GPU owns); their output rows are not written.
    """
    q = _as_bf16_cuda(q, "q")
    k = _as_bf16_cuda(k, "k")
    v = _as_bf16_cuda(v, "v")
    squeeze = q.dim() == 3
    if squeeze:
        q, k, v = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
    if q.dim() != 4 or q.shape != k.shape or q.shape != v.shape:
        raise ShapeError("q/k/v must be identical [H, N, d] tensors")
    if tuple(q.shape[1:]) != (dims.n_heads, dims.seq_len(), dims.head_dim):
        raise ShapeError("tensor shape disagrees with dims")
    if plan.n_heads() != dims.n_heads:
        raise ShapeError("plan must assign exactly one strategy per head")
    given = out
    out4 = _device_out(out, q, q.shape[1:] if squeeze else q.shape)
    d = dims.c()
    kinds, wins = _plan_kinds(plan, skip_heads)
    check(lib().dfa2c_mha_forward(c_void_p(q.data_ptr()), c_void_p(k.data_ptr()), c_void_p(v.data_ptr()),
                                  q.shape[0], byref(d), block_size, kinds, wins,
                                  cache.handle if cache is not None else None, layer, t,
                                  c_void_p(out4.data_ptr()), c_void_p(_stream_ptr(stream))))
    if given is not None:
        return given  # the caller's buffer, in the caller's shape
    return out4[0] if squeeze else out4


def shard_rows(plan: LayerPlan, dims: AttentionDims, block_size: int, world: int, batch: int = 1) -> np.ndarray:
    """Row ranges [bounds[r], bounds[r+1]) of the flattened [batch*H*N] output
    that rank r of `world` computes in multi_strategy_attention_sharded
    (dfa2c_shard_rows; host only, no GPU)."""
    if plan.n_heads() != dims.n_heads:
        raise ShapeError("plan must assign exactly one strategy per head")
    kinds, wins = plan.arrays()
    out = (c_int64 * (world + 1))()
    d = dims.c()
    check(lib().dfa2c_shard_rows(batch, byref(d), block_size, kinds, wins, world, out))
    return np.array(list(out), dtype=np.int64)


def multi_strategy_attention_sharded(q, k, v, plan: LayerPlan, cache: Optional[HeadCache], layer: int, t: int,
                                     dims: AttentionDims, block_size: int, rank: int, world: int, comm=None,
                                     out=None, stream=None):
    """One layer on `world` GPUs (dfa2c_mha_forward_sharded).

    Every rank passes the same replicated q/k/v and plan; this rank's ONE
    fused launch computes its contiguous row range of the layer (near-equal
    cost per rank, long pairs split into key chunks against a fixed 8-GPU
    reference so each head's bits are independent of `world`). With `comm`
    (a NcclComm of `world` ranks) the ranges are all-gathered in place over
    NVLink and every rank's cache receives all computed rows; without it the
    caller gathers `out` (e.g. parallel.gather_rows) and calls shard_commit.
    Returns (out, row_bounds)."""
    q = _as_bf16_cuda(q, "q")
    k = _as_bf16_cuda(k, "k")
    v = _as_bf16_cuda(v, "v")
    squeeze = q.dim() == 3
    if squeeze:
        q, k, v = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
    if q.dim() != 4 or q.shape != k.shape or q.shape != v.shape:
        raise ShapeError("q/k/v must be identical [H, N, d] tensors")
    if tuple(q.shape[1:]) != (dims.n_heads, dims.seq_len(), dims.head_dim):
        raise ShapeError("tensor shape disagrees with dims")
    if plan.n_heads() != dims.n_heads:
        raise ShapeError("plan must assign exactly one strategy per head")
    given = out
    out4 = _device_out(out, q, q.shape[1:] if squeeze else q.shape)
    d = dims.c()
    kinds, wins = plan.arrays()
    bounds = (c_int64 * (world + 1))()
    check(lib().dfa2c_mha_forward_sharded(
        c_void_p(q.data_ptr()), c_void_p(k.data_ptr()), c_void_p(v.data_ptr()), q.shape[0], byref(d), block_size,
        kinds, wins, cache.handle if cache is not None else None, layer, t, c_void_p(out4.data_ptr()), rank, world,
        comm.handle if comm is not None else None, bounds, c_void_p(_stream_ptr(stream))))
    res = given if given is not None else (out4[0] if squeeze else out4)
    return res, np.array(list(bounds), dtype=np.int64)


def multi_strategy_attention_sharded_p2p(q, k, v, plan: LayerPlan, cache: Optional[HeadCache], layer: int, t: int,
                                         dims: AttentionDims, block_size: int, rank: int, world: int, outs,
                                         stream=None):
    """The sharded layer assembled over peer memory (dfa2c_mha_forward_sharded_p2p):
    `outs` lists every rank's output buffer as mapped in this process (a
    tensor for this rank; tensors or raw device pointers for the peers, e.g.
    from parallel.PeerOutputs). This rank's launch stores its rows into all
    of them from the kernel epilogue; after every rank's launch has completed
    (the caller's cross-rank sync) each out holds the whole layer. Returns
    the row bounds."""
    q = _as_bf16_cuda(q, "q")
    k = _as_bf16_cuda(k, "k")
    v = _as_bf16_cuda(v, "v")
    if q.dim() == 3:
        q, k, v = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
    if q.dim() != 4 or q.shape != k.shape or q.shape != v.shape:
        raise ShapeError("q/k/v must be identical [H, N, d] tensors")
    if tuple(q.shape[1:]) != (dims.n_heads, dims.seq_len(), dims.head_dim):
        raise ShapeError("tensor shape disagrees with dims")
    if plan.n_heads() != dims.n_heads or len(outs) != world:
        raise ShapeError("plan must cover every head and outs every rank")
    ptrs = []
    for r, o in enumerate(outs):
        if isinstance(o, int):
            ptrs.append(o)
            continue
        if o.dtype != _torch().bfloat16 or not o.is_cuda or not o.is_contiguous() or o.numel() != q.numel():
            raise ShapeError(f"outs[{r}] must be a contiguous bf16 CUDA tensor shaped like q")
        ptrs.append(o.data_ptr())
    arr = (c_void_p * world)(*ptrs)
    d = dims.c()
    kinds, wins = plan.arrays()
    bounds = (c_int64 * (world + 1))()
    check(lib().dfa2c_mha_forward_sharded_p2p(
        c_void_p(q.data_ptr()), c_void_p(k.data_ptr()), c_void_p(v.data_ptr()), q.shape[0], byref(d), block_size,
        kinds, wins, cache.handle if cache is not None else None, layer, t, arr, rank, world, bounds,
        c_void_p(_stream_ptr(stream))))
    return np.array(list(bounds), dtype=np.int64)


def shard_commit(out, plan: LayerPlan, cache: HeadCache, layer: int, dims: AttentionDims, bounds, rank: int,
                 world: int, stream=None) -> None:
    """After a caller-side gather of a sharded call's `out`: commit the
    computed heads' rows outside this rank's range into `cache`."""
    kinds, _ = plan.arrays()
    b = (c_int64 * (world + 1))(*[int(x) for x in bounds])
    d = dims.c()
    batch = 1 if out.dim() == 3 else out.shape[0]
    check(lib().dfa2c_shard_commit(batch, byref(d), kinds, cache.handle, layer, b, rank, world,
                                   c_void_p(out.data_ptr()), c_void_p(_stream_ptr(stream))))


class NcclComm:
    """An NCCL communicator owned by the library (dfa2c_nccl_comm_init; NCCL
    bound at run time). create() shares the unique id through the default
    torch.distributed group (any backend)."""

    def __init__(self, handle: c_void_p, rank: int, world: int):
        self._h, self.rank, self.world = handle, rank, world

    @staticmethod
    def available() -> bool:
        return bool(lib().dfa2c_nccl_available())

    @staticmethod
    def create(rank: int, world: int, group=None) -> "NcclComm":
        import torch.distributed as dist

        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            check(lib().dfa2c_nccl_unique_id(uid))
        if world > 1:
            obj = [uid.raw if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
        h = c_void_p()
        check(lib().dfa2c_nccl_comm_init(uid, world, rank, byref(h)))
        return NcclComm(h, rank, world)

    @property
    def handle(self) -> c_void_p:
        return self._h

    def allgather_rows(self, buf, bounds, row_bytes: int, stream=None) -> None:
        b = (c_int64 * (self.world + 1))(*[int(x) for x in bounds])
        check(lib().dfa2c_allgather_rows(self._h, c_void_p(buf.data_ptr()), b, self.world, row_bytes,
                                         c_void_p(_stream_ptr(stream))))

    def close(self) -> None:
        if self._h is not None and self._h.value:
            check(lib().dfa2c_nccl_comm_destroy(self._h))
        self._h = None


def multi_strategy_attention_host(q, k, v, plan: LayerPlan, cache: Optional[HeadCache], layer: int, t: int,
                                  dims: AttentionDims, block_size: int, out=None, stream=None, skip_heads=None):
    """multi_strategy_attention with HOST tensors (the reference's calling
    convention, inc/dispatch.hpp:44-47) through dfa2c_mha_forward_host:
    q/k/v are host bf16 [H, N, d] or [batch, H, N, d] (pin them for
    copy/compute overlap); only computed heads are uploaded, in head groups
    pipelined against their fused launches and the output download. Returns
    the host output tensor; it is final once `stream` (default: the current
    stream) is synchronized."""
    torch = _torch()
    for name, x in (("q", q), ("k", k), ("v", v)):
        if not isinstance(x, torch.Tensor) or x.is_cuda or x.dtype != torch.bfloat16 or not x.is_contiguous():
            raise ShapeError(f"{name} must be a contiguous host bf16 tensor")
    squeeze = q.dim() == 3
    if squeeze:
        q, k, v = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
    if q.dim() != 4 or q.shape != k.shape or q.shape != v.shape:
        raise ShapeError("q/k/v must be identical [H, N, d] tensors")
    if tuple(q.shape[1:]) != (dims.n_heads, dims.seq_len(), dims.head_dim):
        raise ShapeError("tensor shape disagrees with dims")
    if plan.n_heads() != dims.n_heads:
        raise ShapeError("plan must assign exactly one strategy per head")
    if out is None:
        out = torch.empty(q.shape, dtype=torch.bfloat16, pin_memory=True)
    elif out.is_cuda or out.dtype != torch.bfloat16 or out.shape != q.shape or not out.is_contiguous():
        raise ShapeError("out must be a contiguous host bf16 tensor shaped like q")
    d = dims.c()
    kinds, wins = _plan_kinds(plan, skip_heads)
    check(lib().dfa2c_mha_forward_host(c_void_p(q.data_ptr()), c_void_p(k.data_ptr()), c_void_p(v.data_ptr()),
                                       q.shape[0], byref(d), block_size, kinds, wins,
                                       cache.handle if cache is not None else None, layer, t,
                                       c_void_p(out.data_ptr()), c_void_p(_stream_ptr(stream))))
    return out[0] if squeeze else out


def sparse_attention_forward(q, k, v, mask: BlockMask, out=None, stream=None):
    """sparse_attention_forward (inc/arrow.hpp:59-63): [N, d] or [H, N, d] heads."""
    torch = _torch()
    q = _as_bf16_cuda(q, "q")
    k = _as_bf16_cuda(k, "k")
    v = _as_bf16_cuda(v, "v")
    if q.shape != k.shape or q.shape != v.shape or q.dim() not in (2, 3):
        raise ShapeError("sparse attention expects per-head [N, d] tensors")
    n, d = q.shape[-2], q.shape[-1]
    heads = 1 if q.dim() == 2 else q.shape[0]
    if mask.seq_len != n:
        raise ShapeError("mask sequence length disagrees with tensors")
    out = _device_out(out, q, q.shape)
    a = np.ascontiguousarray(mask.active, dtype=np.uint8)
    check(lib().dfa2c_sparse_attention_forward(
        c_void_p(q.data_ptr()), c_void_p(k.data_ptr()), c_void_p(v.data_ptr()), c_void_p(out.data_ptr()),
        heads, n, d, a.ctypes.data_as(POINTER(c_uint8)), mask.block_size, c_void_p(_stream_ptr(stream))))
    return out


def dense_tiled_attention(q, k, v, out=None, stream=None):
    """dense_tiled_attention (inc/arrow.hpp:67-69): unmasked [N, d] / [H, N, d]."""
    torch = _torch()
    q = _as_bf16_cuda(q, "q")
    k = _as_bf16_cuda(k, "k")
    v = _as_bf16_cuda(v, "v")
    if q.shape != k.shape or q.shape != v.shape or q.dim() not in (2, 3):
        raise ShapeError("dense attention expects per-head [N, d] tensors")
    n, d = q.shape[-2], q.shape[-1]
    heads = 1 if q.dim() == 2 else q.shape[0]
    out = _device_out(out, q, q.shape)
    check(lib().dfa2c_dense_attention_forward(c_void_p(q.data_ptr()), c_void_p(k.data_ptr()),
                                              c_void_p(v.data_ptr()), c_void_p(out.data_ptr()), heads, n, d,
                                              c_void_p(_stream_ptr(stream))))
    return out


def attention_reference(q, k, v, mask: Optional[BlockMask] = None, stream=None):
    """attention_reference (inc/tensor.hpp:86-93; src/tensor.cpp:73-114,
    268-295) at the operands' own precision: q/k/v CUDA float32 or float64
    [H, N, d] (or [N, d]); computed in that type by the SIMT reference kernel
    (dfa2c_attention_reference), never through the bf16 path. The drop-in's
    independent f32/f64 checker; agrees with the reference's sequential loops
    to rounding."""
    torch = _torch()
    if q.dtype not in (torch.float32, torch.float64):
        raise ShapeError("attention_reference computes in float32 or float64")
    for name, x in (("q", q), ("k", k), ("v", v)):
        if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != q.dtype:
            raise ShapeError(f"{name} must be a CUDA tensor of q's dtype")
    if q.shape != k.shape or q.shape != v.shape or q.dim() not in (2, 3):
        raise ShapeError("attention expects [H, N, d] tensors")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    n, d = q.shape[-2], q.shape[-1]
    heads = 1 if q.dim() == 2 else q.shape[0]
    out = torch.empty_like(q)
    a = None
    if mask is not None:
        if mask.seq_len != n:
            raise ShapeError("mask sequence length disagrees with tensors")
        a = np.ascontiguousarray(mask.active, dtype=np.uint8)
    check(lib().dfa2c_attention_reference(
        c_void_p(q.data_ptr()), c_void_p(k.data_ptr()), c_void_p(v.data_ptr()), c_void_p(out.data_ptr()),
        2 if q.dtype == torch.float64 else 1, heads, n, d,
        a.ctypes.data_as(POINTER(c_uint8)) if a is not None else None, mask.block_size if mask is not None else 0,
        c_void_p(_stream_ptr(stream))))
    return out


# --------------------------------------------------------------- RSE
class RseMode:
    standard = 0
    literal = 1


def _rse_operands(y_m, y_o):
    torch = _torch()
    if y_m.shape != y_o.shape or y_m.dtype != y_o.dtype:
        raise ShapeError("rse operands must share shape and dtype")
    if y_m.numel() == 0:
        raise ShapeError("rse needs at least one element")
    if not (y_m.is_cuda and y_o.is_cuda):
        raise ShapeError("rse operands must be CUDA tensors")
    if y_m.dtype == torch.bfloat16:
        dt = 0
    elif y_m.dtype == torch.float32:
        dt = 1
    else:
        raise ShapeError("rse operands must be bf16 or f32")
    return y_m.contiguous(), y_o.contiguous(), dt


def rse(y_m, y_o, mode: int = RseMode.standard, stream=None) -> float:
    """rse (inc/calibrate.hpp:18-20; src/calibrate.cpp:75-87) of one tensor pair."""
    return float(rse_per_head(y_m.reshape(1, -1), y_o.reshape(1, -1), mode, stream)[0])


def rse_per_head(y_m, y_o, mode: int = RseMode.standard, stream=None) -> np.ndarray:
    """RSE of every leading-axis slice ([H, ...] -> [H] doubles), one launch."""
    y_m, y_o, dt = _rse_operands(y_m, y_o)
    H = y_m.shape[0]
    numel = y_m.numel() // H
    out = np.zeros(H, np.float64)
    check(lib().dfa2c_rse(c_void_p(y_m.data_ptr()), c_void_p(y_o.data_ptr()), dt, H, numel, mode,
                          out.ctypes.data_as(POINTER(c_double)), c_void_p(_stream_ptr(stream))))
    return out


def rse_per_head_async(y_m, y_o, out, mode: int = RseMode.standard, stream=None):
    """RSE of every leading-axis slice into the DEVICE float64 tensor `out`
    ([H]), asynchronously on `stream` (dfa2c_rse_async): no host sync, and a
    zero-variance reference yields NaN instead of DegenerateReferenceError."""
    torch = _torch()
    y_m, y_o, dt = _rse_operands(y_m, y_o)
    H = y_m.shape[0]
    if not (out.is_cuda and out.dtype == torch.float64 and out.numel() == H and out.is_contiguous()):
        raise ShapeError("out must be a contiguous CUDA float64 tensor with one entry per head")
    check(lib().dfa2c_rse_async(c_void_p(y_m.data_ptr()), c_void_p(y_o.data_ptr()), dt, H, y_m.numel() // H, mode,
                                c_void_p(out.data_ptr()), c_void_p(_stream_ptr(stream))))
    return out


# --------------------------------------------------------------- calibration
@dataclass
class MethodCandidate:
    """MethodCandidate (inc/calibrate.hpp:24-28)."""

    id: str
    strategy: HeadStrategy


def method_id(s: HeadStrategy) -> str:
    """method_id (src/plan.cpp:86-96)."""
    if s.kind == StrategyKind.arrow:
        return f"arrow_w{s.window_blocks}"
    if s.kind == StrategyKind.cached:
        return "cached"
    return "full"


def make_candidates(windows: Sequence[int], include_cached: bool = True) -> List[MethodCandidate]:
    """make_candidates (src/calibrate.cpp:89-103)."""
    out = []
    for w in windows:
        if w < 0:
            raise ShapeError("window radii must be >= 0")
        s = HeadStrategy.Arrow(w)
        out.append(MethodCandidate(method_id(s), s))
    if include_cached:
        out.append(MethodCandidate("cached", HeadStrategy.Cached()))
    if not out:
        raise ShapeError("candidate set must be nonempty")
    return out


@dataclass
class CalibrationStats:
    attention_evals: int = 0


@dataclass
class LayerInfluence:
    """LayerInfluence (inc/calibrate.hpp:74-78)."""

    original: object
    method_outputs: object  # [M, H, N, d]
    influence: np.ndarray   # [H * M], h*M + m, +inf where ineligible


def influence_for_layer(q, k, v, methods: Sequence[MethodCandidate], cache: Optional[HeadCache], layer: int,
                        t: int, dims: AttentionDims, block_size: int, mode: int = RseMode.standard,
                        stats: Optional[CalibrationStats] = None, keep_outputs: bool = True,
                        stream=None) -> LayerInfluence:
    """influence_for_layer (inc/calibrate.hpp:80-86; src/calibrate.cpp:193-253).

    Candidates must be Arrow(w)* followed by at most one Cached, the order
    make_candidates produces."""
    torch = _torch()
    if not methods:
        raise ShapeError("candidate set must be nonempty")
    windows, include_cached = _candidate_windows(methods)
    q = _as_bf16_cuda(q, "q")
    k = _as_bf16_cuda(k, "k")
    v = _as_bf16_cuda(v, "v")
    M = len(methods)
    H, n, dd = dims.n_heads, dims.seq_len(), dims.head_dim
    original = torch.empty(H, n, dd, dtype=torch.bfloat16, device="cuda")
    # every Arrow candidate's output and (t > 0) the Cached candidate's are
    # fully written by the call; only an ineligible Cached slot (t == 0,
    # "unset" in the reference) needs clearing
    outs = torch.empty(M, H, n, dd, dtype=torch.bfloat16, device="cuda") if keep_outputs else None
    if outs is not None and include_cached and t == 0:
        outs[M - 1].zero_()
    infl = np.zeros(H * M, np.float64)
    evals = c_int64(0)
    d = dims.c()
    w_arr = (c_int64 * max(1, len(windows)))(*windows)
    check(lib().dfa2c_influence_for_layer(
        c_void_p(q.data_ptr()), c_void_p(k.data_ptr()), c_void_p(v.data_ptr()), byref(d), block_size,
        w_arr, len(windows), 1 if include_cached else 0, cache.handle if cache is not None else None,
        layer, t, mode, infl.ctypes.data_as(POINTER(c_double)), c_void_p(original.data_ptr()),
        c_void_p(outs.data_ptr()) if outs is not None else None, byref(evals), c_void_p(_stream_ptr(stream))))
    if stats is not None:
        stats.attention_evals += evals.value
    return LayerInfluence(original, outs, infl)


def _candidate_windows(methods: Sequence[MethodCandidate]):
    windows, include_cached = [], False
    for m in methods:
        if m.strategy.kind == StrategyKind.arrow:
            if include_cached:
                raise ShapeError("Cached must be the last candidate")
            windows.append(m.strategy.window_blocks)
        elif m.strategy.kind == StrategyKind.cached:
            include_cached = True
        else:
            raise ShapeError("Full is not a compression candidate")
    return windows, include_cached


@dataclass
class _PendingInfluence:
    """An influence_for_layer launched with dfa2c_influence_for_layer_async and
    not yet synchronised (the calibration driver's pipeline)."""

    original: object
    outs: object
    rse_host: object      # pinned float64 [M * H], m * H + h
    eligible: np.ndarray  # uint8 [M * H]
    event: object
    H: int
    M: int

    def finish(self) -> LayerInfluence:
        self.event.synchronize()
        infl = np.zeros(self.H * self.M, np.float64)
        check(lib().dfa2c_influence_finalize(
            ctypes.cast(self.rse_host.data_ptr(), POINTER(c_double)), self.eligible.ctypes.data_as(POINTER(c_uint8)),
            self.H, self.M, infl.ctypes.data_as(POINTER(c_double))))
        return LayerInfluence(self.original, self.outs, infl)


def _influence_launch(q, k, v, methods, cache, layer, t, dims, block_size, mode, stats, bufs) -> _PendingInfluence:
    torch = _torch()
    windows, include_cached = _candidate_windows(methods)
    q = _as_bf16_cuda(q, "q")
    k = _as_bf16_cuda(k, "k")
    v = _as_bf16_cuda(v, "v")
    M = len(methods)
    H, n, dd = dims.n_heads, dims.seq_len(), dims.head_dim
    if not bufs:
        bufs.extend([torch.empty(H, n, dd, dtype=torch.bfloat16, device="cuda"),
                     torch.empty(M, H, n, dd, dtype=torch.bfloat16, device="cuda"),
                     torch.empty(M * H, dtype=torch.float64, pin_memory=True)])
    original, outs, rse_host = bufs
    if include_cached and t == 0:
        outs[M - 1].zero_()
    eligible = np.zeros(M * H, np.uint8)
    evals = c_int64(0)
    d = dims.c()
    w_arr = (c_int64 * max(1, len(windows)))(*windows)
    check(lib().dfa2c_influence_for_layer_async(
        c_void_p(q.data_ptr()), c_void_p(k.data_ptr()), c_void_p(v.data_ptr()), byref(d), block_size,
        w_arr, len(windows), 1 if include_cached else 0, cache.handle if cache is not None else None,
        layer, t, mode, ctypes.cast(rse_host.data_ptr(), POINTER(c_double)),
        eligible.ctypes.data_as(POINTER(c_uint8)), c_void_p(original.data_ptr()), c_void_p(outs.data_ptr()),
        byref(evals), c_void_p(_stream_ptr(None))))
    if stats is not None:
        stats.attention_evals += evals.value
    ev = torch.cuda.Event()
    ev.record()
    return _PendingInfluence(original, outs, rse_host, eligible, ev, H, M)


# --------------------------------------------------------------- calibration driver
class InfluenceTable:
    """InfluenceTable (inc/calibrate.hpp:32-58; src/calibrate.cpp:105-191):
    measured I(t, layer, head, method), NaN where unmeasured (ineligible)."""

    HEADER = "t,layer,head,method,influence"

    def __init__(self, t: int, layers: int, heads: int, method_ids: Sequence[str]):
        self.method_ids = list(method_ids)
        self.values = np.full((t, layers, heads, len(self.method_ids)), np.nan)

    def _check(self, t, layer, head, m):
        T, L, H, M = self.values.shape
        if not (0 <= t < T and 0 <= layer < L and 0 <= head < H and 0 <= m < M):
            raise ShapeError("influence index out of range")

    def get(self, t: int, layer: int, head: int, m: int) -> float:
        self._check(t, layer, head, m)
        return float(self.values[t, layer, head, m])

    def set(self, t: int, layer: int, head: int, m: int, v: float) -> None:
        self._check(t, layer, head, m)
        self.values[t, layer, head, m] = v

    def measured(self, t: int, layer: int, head: int, m: int) -> bool:
        return not math.isnan(self.get(t, layer, head, m))

    def to_csv(self) -> str:
        """17 significant digits, so values round-trip exactly."""
        rows = [self.HEADER]
        T, L, H, M = self.values.shape
        for t in range(T):
            for l in range(L):
                for h in range(H):
                    for m in range(M):
                        v = self.values[t, l, h, m]
                        if not math.isnan(v):
                            rows.append(f"{t},{l},{h},{self.method_ids[m]},{v:.17g}")
        return "\n".join(rows) + "\n"

    @staticmethod
    def parse_csv(text: str, t: int, layers: int, heads: int, method_ids: Sequence[str]) -> "InfluenceTable":
        """parse_influence_csv (inc/calibrate.hpp:61-63); IoError on a bad header or unknown method."""
        table = InfluenceTable(t, layers, heads, method_ids)
        col = {m: i for i, m in enumerate(method_ids)}
        lines = text.split("\n")
        if not lines or lines[0] != InfluenceTable.HEADER:
            raise IoError("influence CSV header mismatch")
        for line in lines[1:]:
            if not line:
                continue
            f = line.split(",")
            if len(f) != 5 or f[3] not in col:
                raise IoError(f"bad influence CSV row: {line}")
            table.set(int(f[0]), int(f[1]), int(f[2]), col[f[3]], float(f[4]))
        return table


@dataclass
class CalibrationConfig:
    """CalibrationConfig (inc/calibrate.hpp:88-93)."""

    methods: List["MethodCandidate"] = field(default_factory=list)
    delta: float = 0.4
    coeff: float = 1.5
    rse_mode: int = 0


@dataclass
class CalibrationResult:
    """CalibrationResult (inc/calibrate.hpp:95-99)."""

    plan: "CompressionPlan"
    influences: InfluenceTable
    stats: "CalibrationStats"
    budget_spent: List[float] = field(default_factory=list)  # [T * L]
    objective: List[float] = field(default_factory=list)     # [T * L]
    wall_seconds: float = 0.0
    outputs: List[object] = field(default_factory=list)      # [T * L] spliced layer outputs (keep_outputs)


def calibrate_model(q_stream, k_stream, v_stream, dims: "AttentionDims", n_timesteps: int, n_layers: int,
                    block_size: int, config: CalibrationConfig, cache: Optional["HeadCache"] = None,
                    keep_outputs: bool = False) -> CalibrationResult:
    """calibrate_model (inc/calibrate.hpp:101-105; src/calibrate.cpp:255-348),
    GPU-resident: for each (t, layer) in forward order, influence_for_layer
    (one fused launch at block 128, else 1 + |M|, plus RSE kernels) on the
    already-compressed stream, enqueued before the previous layer's solve,
    the exact per-layer solve (host, microseconds), and the splice: each
    computed head commits the output of its chosen measurement pass to the
    device cache (no extra attention evaluation); Cached heads keep their
    slot. q_stream(t, l) etc. give the [H, N, d] device inputs. keep_outputs
    records each layer's spliced output (what the plan's run_pipeline must
    reproduce bit for bit)."""
    import time

    torch = _torch()
    if not config.methods:
        raise ShapeError("candidate set must be nonempty")
    if not (config.delta >= 0.0):
        raise ShapeError("delta must be >= 0")
    if not (config.coeff >= 1.0):
        raise ShapeError("coeff must be >= 1")
    t0 = time.perf_counter()
    H, M = dims.n_heads, len(config.methods)
    strategies = [m.strategy for m in config.methods]
    costs = analytic_costs(dims, block_size, strategies)
    plan = CompressionPlan(dims, n_timesteps, n_layers, block_size, config.delta, config.coeff,
                           [s.window_blocks for s in strategies if s.kind == StrategyKind.arrow],
                           [LayerPlan() for _ in range(n_timesteps * n_layers)])
    table = InfluenceTable(n_timesteps, n_layers, H, [m.id for m in config.methods])
    stats = CalibrationStats()
    res = CalibrationResult(plan, table, stats)
    if cache is None:
        cache = HeadCache(n_layers, H, dims.seq_len(), dims.head_dim)

    def finish(t, l, pending):
        li = pending.finish()
        grid = li.influence.reshape(H, M)
        finite = np.isfinite(grid)
        table.values[t, l][finite] = grid[finite]
        sol = solve(PlanProblem(H, M, li.influence, costs, config.delta, config.coeff))
        res.budget_spent.append(sol.total_influence)
        res.objective.append(sol.objective)
        plan.layers[t * n_layers + l] = to_layer_plan(sol, strategies)
        if keep_outputs:
            res.outputs.append(torch.stack([li.original[h] if c == kFullChoice else li.method_outputs[c][h]
                                            for h, c in enumerate(sol.choice)]))
        for h, c in enumerate(sol.choice):
            if c == kFullChoice:
                cache.store(l, h, li.original[h], t)
            elif strategies[c].kind == StrategyKind.arrow:
                cache.store(l, h, li.method_outputs[c][h], t)

    # Pipelined: (t, l)'s measurement passes are enqueued before (t, l-1)'s
    # solve and splice, so the GPU measures while the host solves. Only the
    # Cached candidate of (t, l) reads the cache, and only slot l (written at
    # t-1 or earlier); a splice into the same slot is finished first (L = 1).
    # Two output buffer sets alternate; the stream orders each splice before
    # the launch that reuses its buffers.
    bufs = ([], [])
    pending = None
    idx = 0
    for t in range(n_timesteps):
        for l in range(n_layers):
            if pending is not None and pending[1] == l:
                finish(*pending)
                pending = None
            cur = _influence_launch(q_stream(t, l), k_stream(t, l), v_stream(t, l), config.methods, cache, l, t,
                                    dims, block_size, config.rse_mode, stats, bufs[idx % 2])
            idx += 1
            if pending is not None:
                finish(*pending)
            pending = (t, l, cur)
    if pending is not None:
        finish(*pending)
    res.wall_seconds = time.perf_counter() - t0
    return res


def audit_plan_constraints(plan: "CompressionPlan", influences: InfluenceTable) -> int:
    """audit_plan_constraints (inc/calibrate.hpp:107-110; src/calibrate.cpp:350-382):
    number of budget / cap violations (0 for any plan calibrate_model emits)."""
    plan.validate()
    col = {m: i for i, m in enumerate(influences.method_ids)}
    cap = selection_cap(plan.coeff, plan.dims.n_heads, plan.delta)
    bad = 0
    for t in range(plan.n_timesteps):
        for l in range(plan.n_layers):
            spent = 0.0
            for h, s_ in enumerate(plan.at(t, l).strategies):
                if s_.kind == StrategyKind.full:
                    continue
                m = col.get(method_id(s_))
                if m is None or not influences.measured(t, l, h, m):
                    bad += 1
                    continue
                v = influences.get(t, l, h, m)
                spent += v
                bad += 1 if v > cap else 0
            bad += 1 if spent > plan.delta else 0
    return bad


# --------------------------------------------------------------- plan selection
kFullChoice = -1


@dataclass
class CostModel:
    """CostModel (inc/plansolver.hpp:12-17)."""

    full_cost: float = 1.0
    method_cost: List[float] = field(default_factory=list)


@dataclass
class PlanProblem:
    """PlanProblem (inc/plansolver.hpp:25-37): influence is [n_heads * n_methods], row-major by head."""

    n_heads: int = 0
    n_methods: int = 0
    influence: Sequence[float] = field(default_factory=list)
    costs: CostModel = field(default_factory=CostModel)
    delta: float = 0.0
    coeff: float = 1.5


@dataclass
class PlanSolution:
    """PlanSolution (inc/plansolver.hpp:43-48): choice[h] is kFullChoice or a method index."""

    choice: List[int] = field(default_factory=list)
    objective: float = 0.0
    total_influence: float = 0.0
    nodes: int = 0


def selection_cap(coeff: float, n_heads: int, delta: float) -> float:
    """Per-selection cap (coeff / n_heads) * delta (inc/plansolver.hpp:39-41)."""
    return float(lib().dfa2c_selection_cap(coeff, n_heads, delta))


def _problem_args(p: PlanProblem):
    infl = np.ascontiguousarray(np.asarray(p.influence, np.float64).reshape(-1))
    if infl.size != p.n_heads * p.n_methods or len(p.costs.method_cost) != p.n_methods:
        raise ShapeError("influence grid / cost model do not match H x M")
    mc = np.ascontiguousarray(np.asarray(p.costs.method_cost if p.n_methods else [0.0], np.float64))
    return infl, mc


def _solve(p: PlanProblem, exhaustive: bool) -> PlanSolution:
    infl, mc = _problem_args(p)
    choice = np.zeros(max(1, p.n_heads), np.int64)
    obj, tot, nodes = c_double(), c_double(), c_int64()
    check(lib().dfa2c_plan_solve(p.n_heads, p.n_methods, infl.ctypes.data_as(POINTER(c_double)), p.costs.full_cost,
                                 mc.ctypes.data_as(POINTER(c_double)), p.delta, p.coeff, 1 if exhaustive else 0,
                                 choice.ctypes.data_as(POINTER(c_int64)), byref(obj), byref(tot), byref(nodes)))
    return PlanSolution([int(c) for c in choice[:p.n_heads]], obj.value, tot.value, nodes.value)


def solve(problem: PlanProblem) -> PlanSolution:
    """solve (inc/plansolver.hpp:50-61): exact optimum with the reference's tie-break."""
    return _solve(problem, False)


def brute_force(problem: PlanProblem) -> PlanSolution:
    """brute_force (inc/plansolver.hpp:63-65): exhaustive enumeration, same tie-break."""
    return _solve(problem, True)


def lp_relaxation_bound(problem: PlanProblem) -> float:
    """lp_relaxation_bound (inc/plansolver.hpp:67-69)."""
    infl, mc = _problem_args(problem)
    b = c_double()
    check(lib().dfa2c_plan_lp_bound(problem.n_heads, problem.n_methods, infl.ctypes.data_as(POINTER(c_double)),
                                    problem.costs.full_cost, mc.ctypes.data_as(POINTER(c_double)), problem.delta,
                                    problem.coeff, byref(b)))
    return b.value


def analytic_costs(dims: AttentionDims, block_size: int, methods: Sequence[HeadStrategy]) -> CostModel:
    """analytic_costs (inc/plansolver.hpp:19-21): Arrow(w) = active fraction of its mask, Cached = 0."""
    M = len(methods)
    kinds = (c_int32 * max(1, M))(*[_KIND_CODE[m.kind] for m in methods])
    wins = (c_int64 * max(1, M))(*[m.window_blocks for m in methods])
    out = (c_double * max(1, M))()
    full = c_double()
    d = dims.c()
    check(lib().dfa2c_analytic_costs(byref(d), block_size, kinds, wins, M, byref(full), out))
    return CostModel(full.value, list(out[:M]))


def to_layer_plan(solution: PlanSolution, methods: Sequence[HeadStrategy]) -> LayerPlan:
    """to_layer_plan (inc/plansolver.hpp:74-76)."""
    return LayerPlan([HeadStrategy.Full() if c == kFullChoice else methods[c] for c in solution.choice])


# --------------------------------------------------------------- compression plan
@dataclass
class CompressionPlan:
    """CompressionPlan (inc/plan.hpp:14-42): layers[t*L + l], timestep-major."""

    dims: AttentionDims
    n_timesteps: int = 0
    n_layers: int = 0
    block_size: int = 0
    delta: float = 0.0
    coeff: float = 1.5
    window_set: List[int] = field(default_factory=list)
    layers: List[LayerPlan] = field(default_factory=list)
    influence_digest: str = ""

    @staticmethod
    def all_full(dims: AttentionDims, timesteps: int, layers: int, block_size: int) -> "CompressionPlan":
        return CompressionPlan(dims, timesteps, layers, block_size,
                               layers=[LayerPlan.all_full(dims.n_heads) for _ in range(timesteps * layers)])

    def at(self, t: int, layer: int) -> LayerPlan:
        return self.layers[t * self.n_layers + layer]

    def _arrays(self):
        H = self.dims.n_heads
        if len(self.layers) != self.n_timesteps * self.n_layers:
            raise PlanValidationError("plan must cover every (t, layer) exactly once")
        kinds, wins = [], []
        for lp in self.layers:
            if lp.n_heads() != H:
                raise PlanValidationError("head array length must equal H")
            kinds += [_KIND_CODE[s.kind] for s in lp.strategies]
            wins += [s.window_blocks for s in lp.strategies]
        n = max(1, len(kinds))
        return (c_int32 * n)(*kinds), (c_int64 * n)(*wins)

    def _aggregate(self):
        if not (self.delta >= 0.0):
            raise PlanValidationError("delta must be >= 0")
        if not (self.coeff >= 1.0):
            raise PlanValidationError("coeff must be >= 1")
        kinds, wins = self._arrays()
        d = self.dims.c()
        ft, fd, sp = c_int64(), c_int64(), c_double()
        check(lib().dfa2c_plan_aggregate(byref(d), self.n_timesteps, self.n_layers, self.block_size, kinds, wins,
                                         byref(ft), byref(fd), byref(sp)))
        return ft.value, fd.value, sp.value

    def validate(self) -> None:
        self.dims.validate()
        self._aggregate()

    def flops_total(self) -> int:
        return self._aggregate()[0]

    def flops_dense_total(self) -> int:
        return self._aggregate()[1]

    def aggregate_sparsity(self) -> float:
        return self._aggregate()[2]

    # ---- plan file (JSON v1, inc/plan.hpp:44-52), via dfa2c_plan_to/from_json
    def to_json(self) -> str:
        """plan_to_json (src/plan.cpp:109-143): the reference's file text."""
        H = self.dims.n_heads
        kinds, wins = [], []
        for lp in self.layers:
            if lp.n_heads() != H:
                raise ShapeError("head array length must equal H")
            kinds += [_KIND_CODE[s_.kind] for s_ in lp.strategies]
            wins += [s_.window_blocks for s_ in lp.strategies]
        n = max(1, len(kinds))
        k, w = (c_int32 * n)(*kinds), (c_int64 * n)(*wins)
        ws = (c_int64 * max(1, len(self.window_set)))(*self.window_set)
        hdr = _lib.PlanHeader(self.n_timesteps, self.n_layers, H, self.dims.head_dim, self.dims.n_visual,
                              self.dims.n_text, self.block_size, self.delta, self.coeff, len(self.window_set), 0)
        ln = c_int64()
        dig = self.influence_digest.encode()
        check(lib().dfa2c_plan_to_json(byref(hdr), k, w, ws, dig, None, 0, byref(ln)))
        buf = ctypes.create_string_buffer(ln.value + 1)
        check(lib().dfa2c_plan_to_json(byref(hdr), k, w, ws, dig, buf, ln.value + 1, byref(ln)))
        return buf.raw[:ln.value].decode()

    @staticmethod
    def from_json(text: str) -> "CompressionPlan":
        """plan_from_json (src/plan.cpp:145-209): parses and validates;
        PlanValidationError on malformed text or schema violations."""
        raw = text.encode()
        hdr = _lib.PlanHeader()
        check(lib().dfa2c_plan_from_json(raw, len(raw), byref(hdr), None, None, None, None, 0))
        T, L, H = hdr.n_timesteps, hdr.n_layers, hdr.n_heads
        k, w = (c_int32 * (T * L * H))(), (c_int64 * (T * L * H))()
        ws = (c_int64 * max(1, hdr.n_window_set))()
        dig = ctypes.create_string_buffer(hdr.digest_len + 1)
        check(lib().dfa2c_plan_from_json(raw, len(raw), byref(hdr), k, w, ws, dig, hdr.digest_len + 1))
        inv = {v: k_ for k_, v in _KIND_CODE.items()}
        layers = [LayerPlan([HeadStrategy(inv[k[i * H + h]], w[i * H + h] if k[i * H + h] == 1 else 0)
                             for h in range(H)]) for i in range(T * L)]
        dims = AttentionDims(H, hdr.head_dim, hdr.n_visual, hdr.n_text)
        return CompressionPlan(dims, T, L, hdr.block_size, hdr.delta, hdr.coeff, list(ws[:hdr.n_window_set]),
                               layers, dig.raw[:hdr.digest_len].decode())

    def save(self, path: str) -> None:
        """save_plan (inc/plan.hpp:51)."""
        try:
            with open(path, "w") as f:
                f.write(self.to_json())
        except OSError as e:
            raise IoError(f"cannot write {path}: {e}") from None

    @staticmethod
    def load(path: str) -> "CompressionPlan":
        """load_plan (inc/plan.hpp:52)."""
        try:
            with open(path) as f:
                text = f.read()
        except OSError as e:
            raise IoError(f"cannot open {path}: {e}") from None
        return CompressionPlan.from_json(text)


def plan_to_json(plan: CompressionPlan) -> str:
    return plan.to_json()


def plan_from_json(text: str) -> CompressionPlan:
    return CompressionPlan.from_json(text)


def fnv1a_hex(data) -> str:
    """fnv1a_hex (inc/plan.hpp:57-58): FNV-1a 64 as 16 hex chars."""
    raw = data.encode() if isinstance(data, str) else bytes(data)
    out = ctypes.create_string_buffer(17)
    check(lib().dfa2c_fnv1a_hex(raw, len(raw), out))
    return out.value.decode()


@dataclass
class RunStats:
    """RunStats (inc/workload.hpp:59-69)."""

    flops_total: int = 0
    flops_dense: int = 0
    sparsity: float = 0.0
    outputs: list = field(default_factory=list)

    def output(self, t: int, layer: int, n_layers: int):
        return self.outputs[t * n_layers + layer]


def run_pipeline(q_stream, k_stream, v_stream, plan: CompressionPlan, batch: int = 1, keep_outputs: bool = True,
                 cache: Optional[HeadCache] = None) -> RunStats:
    """run_pipeline (inc/workload.hpp:71; src/workload.cpp:230-262): t-major
    (t, l) loop over multi_strategy_attention with one shared device cache.
    q_stream(t, l) etc. return the [H, N, d] (or [batch, H, N, d]) inputs."""
    plan.validate()
    dims = plan.dims
    if cache is None:
        cache = HeadCache(plan.n_layers, dims.n_heads, dims.seq_len(), dims.head_dim, batch)
    stats = RunStats()
    dense = dims.n_heads * dense_flops(dims.seq_len(), dims.head_dim)
    for t in range(plan.n_timesteps):
        for l in range(plan.n_layers):
            lp = plan.at(t, l)
            o = multi_strategy_attention(q_stream(t, l), k_stream(t, l), v_stream(t, l), lp, cache, l, t, dims,
                                         plan.block_size)
            if keep_outputs:
                stats.outputs.append(o)
            stats.flops_total += plan_flops(lp, dims, plan.block_size)
            stats.flops_dense += dense
    stats.sparsity = 1.0 - stats.flops_total / stats.flops_dense
    return stats


class DeviceWorkload:
    """The reference's synthetic drifting Q/K/V stream (generate(),
    src/workload.cpp:120-228) produced on the GPU (dfa2c_workload_*):
    slot(t, layer) returns bf16 CUDA q, k, v [H, N, d]. Same model and
    profiles as the reference; per-element noise from a counter-based Philox
    stream (a pure function of (seed, t, layer)), so FLUX-scale schedules
    cost HBM time, not host time."""

    def __init__(self, dims: AttentionDims, n_layers: int, block_size: int, seed: int = 1234):
        self.dims, self.n_layers, self.block_size, self.seed = dims, n_layers, block_size, seed
        h = c_void_p()
        d = dims.c()
        check(lib().dfa2c_workload_create(byref(d), n_layers, block_size, seed, byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().dfa2c_workload_destroy(h)
            except Exception:
                pass
            self._h = None

    def profile(self, layer: int, head: int):
        loc, drift = c_double(), c_double()
        check(lib().dfa2c_workload_profile(self._h, layer, head, byref(loc), byref(drift)))
        return loc.value, drift.value

    def slot(self, t: int, layer: int, out=None, stream=None):
        torch = _torch()
        shape = (self.dims.n_heads, self.dims.seq_len(), self.dims.head_dim)
        q, k, v = out if out is not None else tuple(
            torch.empty(shape, dtype=torch.bfloat16, device="cuda") for _ in range(3))
        check(lib().dfa2c_workload_slot(self._h, t, layer, c_void_p(q.data_ptr()), c_void_p(k.data_ptr()),
                                        c_void_p(v.data_ptr()), c_void_p(_stream_ptr(stream))))
        return q, k, v


def flux68_plan(n_heads: int = 24) -> LayerPlan:
    """The survey's FLUX68 head pattern: head h,
    g = h // 4, r = h % 4 -> r0 Full, r1 Arrow(8), r2 Cached,
    r3 Arrow(0 if g % 3 != 1 else 8)."""
    out = []
    for h in range(n_heads):
        g, r = divmod(h, 4)
        if r == 0:
            out.append(HeadStrategy.Full())
        elif r == 1:
            out.append(HeadStrategy.Arrow(8))
        elif r == 2:
            out.append(HeadStrategy.Cached())
        else:
            out.append(HeadStrategy.Arrow(0 if g % 3 != 1 else 8))
    return LayerPlan(out)


def launch_count() -> int:
    return int(lib().dfa2c_launch_count())


__all__ = [n for n in dir() if not n.startswith("_")]
_ = (math, ctypes)
