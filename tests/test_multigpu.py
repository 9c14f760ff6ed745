"""Multi-GPU layer: row-range sharding through the C++ host
(dfa2c_mha_forward_sharded), its NCCL binding, and the world-2 process path.

CPU tests (no GPU): the host-only partition (dfa2c_shard_rows) is a cover of
the flattened rows by contiguous, cost-balanced, deterministic ranges; the
torch.distributed row gather works at world size 2 over gloo.

GPU tests: ranks emulated one after another on this GPU assemble, for every
W, bitwise the same layer (including Cached heads served from caches that
other ranks committed, over three timesteps whose plans move the row
ranges); two real processes on this GPU (gloo gather, real kernel per rank)
assemble the same bits; an NCCL communicator of one rank runs the in-library
all-gather path. (This image gives one GPU: NCCL across 2+ GPUs is exercised
only by bench.py --gpus N on a multi-GPU box.)
"""
import os
import socket

import numpy as np
import pytest

from paper_2503_22796_b200 import api
from paper_2503_22796_b200.api import AttentionDims, HeadCache, LayerPlan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FLUX68 = "F A8 C A0 F A8 C A8 F A8 C A0 F A8 C A0 F A8 C A8 F A8 C A0"


def _cost_of_rows(plan, dims, B, lo, hi):
    """Tile-units of the (head, pair) items whose rows fall in [lo, hi)."""
    n = dims.seq_len()
    nqt = (n + 127) // 128
    total = 0.0
    for h, s in enumerate(plan.strategies):
        if s.kind == "cached":
            per = [min(n, 256 * (p + 1)) / 128.0 - 2 * p for p in range((nqt + 1) // 2)]
        else:
            rp, _ = api.tile_set(AttentionDims(1, dims.head_dim, dims.n_visual, dims.n_text, dims.order), B, s)
            lens = np.diff(rp)
            per = [lens[2 * p] + (lens[2 * p + 1] if 2 * p + 1 < nqt else 0) + 1 for p in range((nqt + 1) // 2)]
        for p, c in enumerate(per):
            r = h * n + 256 * p
            if lo <= r < hi:
                total += c
    return total


@pytest.mark.parametrize("nv,nt,d,plan_text", [(16384, 512, 128, FLUX68), (4096, 333, 64, "F A0 C A2 A8 A16")])
def test_shard_rows_cover_and_balance(nv, nt, d, plan_text):
    plan = LayerPlan.parse(plan_text)
    H = plan.n_heads()
    dims = AttentionDims(H, d, nv, nt)
    n = dims.seq_len()
    total = _cost_of_rows(plan, dims, 128, 0, H * n)
    for W in (1, 2, 3, 4, 8):
        b = api.shard_rows(plan, dims, 128, W)
        assert b[0] == 0 and b[-1] == H * n and (np.diff(b) >= 0).all()
        # boundaries fall on pair boundaries (256-row pairs or head starts)
        for x in b:
            assert x % n == 0 or (x % n) % 256 == 0
        assert (b == api.shard_rows(plan, dims, 128, W)).all()  # deterministic
        loads = [_cost_of_rows(plan, dims, 128, b[r], b[r + 1]) for r in range(W)]
        # each part within one pair (<= 2 * 132 + 1 tile-units) of the ideal share
        assert max(loads) <= 1.02 * total / W + 300, (W, loads)


def test_sample_sharding():
    from paper_2503_22796_b200 import parallel

    assert parallel.shard_samples(8, 8, 3) == [3] and parallel.shard_samples(5, 2, 1) == [1, 3]


def test_shard_rows_batch_and_validation():
    plan = LayerPlan.parse("F A0 C")
    dims = AttentionDims(3, 64, 1024, 77)
    b1 = api.shard_rows(plan, dims, 128, 2, batch=1)
    b2 = api.shard_rows(plan, dims, 128, 2, batch=2)
    assert b2[-1] == 2 * 3 * 1101 and b1[-1] == 3 * 1101
    with pytest.raises(api.ShapeError):
        api.shard_rows(plan, dims, 128, 0)
    with pytest.raises(api.UnsupportedError):
        api.shard_rows(plan, AttentionDims(3, 40, 1024, 77), 128, 2)  # padded head dims are not sharded


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2503_22796_b200 import parallel

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = torch.full((2, 3, 40, 8), -1.0)
        bounds = [0, 100, 240]
        flat = out.reshape(-1, 8)
        lo, hi = bounds[rank], bounds[rank + 1]
        flat[lo:hi] = torch.arange(lo, hi, dtype=torch.float32)[:, None]
        parallel.gather_rows(out, bounds, rank, world)
        ok = bool((flat == torch.arange(240, dtype=torch.float32)[:, None]).all())
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gather_rows_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)


# ----------------------------------------------------------------- GPU
def _inputs(H, n, d, seed):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)


STEPS = ["F F F F F F F F F F F F", "F A0 C A2 F C A8 C F A1 C A0", "C A2 F C A0 F C C A8 F A0 C"]


def _emulated_ranks(W, q, k, v, dims, B):
    """Runs the STEPS timesteps with W ranks emulated sequentially on this
    GPU: every rank writes its rows into one shared buffer (the gather), then
    commits the others' rows into its own cache (dfa2c_shard_commit)."""
    import torch

    H, n, d = dims.n_heads, dims.seq_len(), dims.head_dim
    caches = [HeadCache(1, H, n, d) for _ in range(W)]
    outs = []
    for t, text in enumerate(STEPS):
        plan = LayerPlan.parse(text)
        out = torch.full_like(q, float("nan"))
        bounds = None
        for r in range(W):
            _, bounds = api.multi_strategy_attention_sharded(q, k, v, plan, caches[r], 0, t, dims, B, r, W, out=out)
        for r in range(W):
            api.shard_commit(out, plan, caches[r], 0, dims, bounds, r, W)
        torch.cuda.synchronize()
        outs.append(out.clone())
    return outs, caches


@pytest.mark.gpu
@pytest.mark.parametrize("nv,nt,d", [(2048, 77, 64), (2048, 256, 128)])
def test_sharded_layers_are_bitwise_identical_for_every_world(nv, nt, d):
    import torch

    H, B = 12, 128
    dims = AttentionDims(H, d, nv, nt)
    n = dims.seq_len()
    q, k, v = (_inputs(H, n, d, s) for s in (1, 2, 3))
    ref, ref_caches = _emulated_ranks(1, q, k, v, dims, B)
    for W in (2, 3, 4, 8):
        outs, caches = _emulated_ranks(W, q, k, v, dims, B)
        for t in range(len(STEPS)):
            assert torch.equal(outs[t], ref[t]), f"W={W} t={t}"
        for r in range(W):  # every rank's cache is complete and identical
            for h in range(H):
                assert torch.equal(caches[r].fetch(0, h), ref_caches[0].fetch(0, h)), (W, r, h)
                assert caches[r].produced_at(0, h) == ref_caches[0].produced_at(0, h)
    # the sharded layer against the single-call layer: Cached heads bitwise,
    # computed heads within the attention tolerance (long pairs run as key
    # chunks in the sharded schedule, which changes the fold's rounding)
    plain_cache = HeadCache(1, H, n, d)
    for t, text in enumerate(STEPS):
        plan = LayerPlan.parse(text)
        plain = api.multi_strategy_attention(q, k, v, plan, plain_cache, 0, t, dims, B)
        for h, s in enumerate(plan.strategies):
            a, b = ref[t][h].float(), plain[h].float()
            rel = (a - b).abs().max() / b.abs().max()
            assert rel <= 2e-2, (t, h, float(rel))


@pytest.mark.gpu
def test_nccl_single_rank_communicator_runs_the_library_gather():
    import torch

    if not api.NcclComm.available():
        pytest.skip("libnccl.so.2 not loadable")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    comm = api.NcclComm.create(0, 1)
    try:
        H, nv, nt, d, B = 6, 1024, 77, 64, 128
        dims = AttentionDims(H, d, nv, nt)
        n = dims.seq_len()
        q, k, v = (_inputs(H, n, d, s) for s in (4, 5, 6))
        cache = HeadCache(1, H, n, d)
        plan0, plan1 = LayerPlan.all_full(H), LayerPlan.parse("F A0 C A2 C F")
        o0, b = api.multi_strategy_attention_sharded(q, k, v, plan0, cache, 0, 0, dims, B, 0, 1, comm=comm)
        o1, _ = api.multi_strategy_attention_sharded(q, k, v, plan1, cache, 0, 1, dims, B, 0, 1, comm=comm)
        torch.cuda.synchronize()
        assert list(b) == [0, H * n]
        assert torch.equal(o1[2], o0[2]) and torch.equal(o1[4], o0[4])
        buf = o1.clone()
        comm.allgather_rows(buf, [0, H * n], d * 2)  # one rank: a no-op broadcast
        torch.cuda.synchronize()
        assert torch.equal(buf, o1)
    finally:
        comm.close()


def _process_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2503_22796_b200 import parallel

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)  # both ranks on the one GPU of this box
        H, nv, nt, d, B = 12, 2048, 77, 64, 128
        dims = AttentionDims(H, d, nv, nt)
        n = dims.seq_len()
        qq, kk, vv = (_inputs(H, n, d, s) for s in (1, 2, 3))
        cache = HeadCache(1, H, n, d)
        results = []
        for t, text in enumerate(STEPS):
            out, _ = parallel.sharded_multi_strategy_attention(qq, kk, vv, LayerPlan.parse(text), cache, 0, t, dims,
                                                               B, rank, world)
            torch.cuda.synchronize()
            results.append(out.cpu())
        q.put((rank, [r.view(torch.int16).numpy() for r in results]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_processes_assemble_the_single_rank_bits():
    """world_size 2, one process per rank (gloo gather through the host; the
    real fused kernel per rank), three timesteps with moving row ranges."""
    import torch
    import torch.multiprocessing as mp

    H, nv, nt, d, B = 12, 2048, 77, 64, 128
    dims = AttentionDims(H, d, nv, nt)
    n = dims.seq_len()
    q, k, v = (_inputs(H, n, d, s) for s in (1, 2, 3))
    ref, _ = _emulated_ranks(1, q, k, v, dims, B)
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_process_worker, args=(r, 2, port, qu)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(qu.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        for t in range(len(STEPS)):
            assert np.array_equal(res[r][t], ref[t].cpu().view(torch.int16).numpy()), (r, t)


# ------------------------------------------------ assembly over peer memory
def _p2p_emulated_ranks(W, q, k, v, dims, B):
    """The STEPS timesteps with W ranks emulated on this GPU, assembled over
    peer memory: each rank owns an output buffer, and its fused launch stores
    its rows into every rank's buffer from the epilogue
    (dfa2c_mha_forward_sharded_p2p); then each rank completes its cache."""
    import torch

    H, n, d = dims.n_heads, dims.seq_len(), dims.head_dim
    caches = [HeadCache(1, H, n, d) for _ in range(W)]
    per_t = []
    for t, text in enumerate(STEPS):
        plan = LayerPlan.parse(text)
        bufs = [torch.full_like(q.unsqueeze(0), float("nan")) for _ in range(W)]
        bounds = None
        for r in range(W):
            bounds = api.multi_strategy_attention_sharded_p2p(q, k, v, plan, caches[r], 0, t, dims, B, r, W, bufs)
        torch.cuda.synchronize()  # every "rank" has finished: every buffer holds the layer
        for r in range(W):
            api.shard_commit(bufs[r], plan, caches[r], 0, dims, bounds, r, W)
        torch.cuda.synchronize()
        per_t.append([b[0].clone() for b in bufs])
    return per_t, caches


@pytest.mark.gpu
@pytest.mark.parametrize("nv,nt,d", [(2048, 77, 64), (2048, 256, 128)])
def test_p2p_assembly_gives_every_rank_the_single_rank_bits(nv, nt, d):
    import torch

    H, B = 12, 128
    dims = AttentionDims(H, d, nv, nt)
    n = dims.seq_len()
    q, k, v = (_inputs(H, n, d, s) for s in (1, 2, 3))
    ref, ref_caches = _emulated_ranks(1, q, k, v, dims, B)
    for W in (2, 4, 8):
        per_t, caches = _p2p_emulated_ranks(W, q, k, v, dims, B)
        for t in range(len(STEPS)):
            for r in range(W):
                assert torch.equal(per_t[t][r], ref[t]), f"W={W} t={t} rank {r}"
        for r in range(W):
            for h in range(H):
                assert torch.equal(caches[r].fetch(0, h), ref_caches[0].fetch(0, h)), (W, r, h)
    with pytest.raises(api.ShapeError):  # every rank's buffer, distinct
        buf = torch.empty_like(q.unsqueeze(0))
        api.multi_strategy_attention_sharded_p2p(q, k, v, LayerPlan.all_full(H), None, 0, 0, dims, B, 0, 2,
                                                 [buf, buf])


@pytest.mark.gpu
def test_p2p_assembly_batched_without_cache():
    """Batch 2, no cache (no commits, no Cached heads): W = 3 emulated ranks
    assemble over their buffers to the single-rank sharded bits."""
    import torch

    Bt, H, nv, nt, d, B = 2, 6, 1024, 77, 128, 128
    dims = AttentionDims(H, d, nv, nt)
    n = dims.seq_len()
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn(Bt, H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    plan = LayerPlan.parse("F A0 A2 F A8 A1")
    ref, _ = api.multi_strategy_attention_sharded(q, k, v, plan, None, 0, 0, dims, B, 0, 1)
    W = 3
    bufs = [torch.full_like(q, float("nan")) for _ in range(W)]
    for r in range(W):
        api.multi_strategy_attention_sharded_p2p(q, k, v, plan, None, 0, 0, dims, B, r, W, bufs)
    torch.cuda.synchronize()
    for r in range(W):
        assert torch.equal(bufs[r], ref), r


def _p2p_process_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2503_22796_b200 import parallel

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)  # both ranks on the one GPU of this box (same-device CUDA IPC)
        H, nv, nt, d, B = 12, 2048, 77, 64, 128
        dims = AttentionDims(H, d, nv, nt)
        n = dims.seq_len()
        qq, kk, vv = (_inputs(H, n, d, s) for s in (1, 2, 3))
        cache = HeadCache(1, H, n, d)
        out = torch.empty(1, H, n, d, dtype=torch.bfloat16, device="cuda")
        peers = parallel.PeerOutputs(out, rank, world)
        results = []
        try:
            for t, text in enumerate(STEPS):
                plan = LayerPlan.parse(text)
                dist.barrier()  # nobody writes a buffer its owner is still reading
                bounds = api.multi_strategy_attention_sharded_p2p(qq, kk, vv, plan, cache, 0, t, dims, B, rank,
                                                                  world, peers.outs)
                torch.cuda.synchronize()
                dist.barrier()  # every rank's launch has completed: `out` holds the whole layer
                api.shard_commit(out, plan, cache, 0, dims, bounds, rank, world)
                torch.cuda.synchronize()
                results.append(out[0].cpu())
        finally:
            dist.barrier()
            peers.close()
        q.put((rank, [r.view(torch.int16).numpy() for r in results]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_processes_assemble_over_cuda_ipc():
    """world_size 2, one process per rank; each rank's fused kernel writes its
    rows into the other process's output buffer (CUDA IPC), no gather: both
    processes end with the single-rank bits, three timesteps."""
    import torch
    import torch.multiprocessing as mp

    H, nv, nt, d, B = 12, 2048, 77, 64, 128
    dims = AttentionDims(H, d, nv, nt)
    n = dims.seq_len()
    q, k, v = (_inputs(H, n, d, s) for s in (1, 2, 3))
    ref, _ = _emulated_ranks(1, q, k, v, dims, B)
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_process_worker, args=(r, 2, port, qu)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(qu.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        for t in range(len(STEPS)):
            assert np.array_equal(res[r][t], ref[t].cpu().view(torch.int16).numpy()), (r, t)
