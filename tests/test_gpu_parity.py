"""GPU parity of the sm_100a path against the oracle / the reference itself.

Stated tolerance for attention outputs (bf16 in, fp32 accumulate, bf16 out)
against the f64 two-pass oracle evaluated on the SAME bf16-rounded inputs
(attention_head_impl<double>, src/tensor.cpp:73-114, pinned bit-exact in
tests/test_oracle.py):
    max|gpu - ref| / max|ref| <= 1e-2   and   RSE(gpu, ref) <= 5e-5   per head.
Bit-exact: cached-head copies, cache commits, Full == Arrow(max window),
run-to-run determinism, head isolation, CacheMiss-before-compute.
"""
import ctypes
import os

import numpy as np
import pytest

import oracle
from paper_2503_22796_b200 import api
from paper_2503_22796_b200.api import (AttentionDims, ArrowSpec, BlockMask, CacheMissError, FullyMaskedRowError,
                                       HeadCache, HeadStrategy, LayerPlan, ShapeError)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MAX_REL = 1e-2
MAX_RSE = 5e-5


def torch():
    import torch as t

    return t


def bf16_inputs(shape, seed):
    """Seeded gaussian -> (bf16 CUDA tensor, the same values as f32 numpy)."""
    t = torch()
    x = oracle.round_bf16(oracle.gaussian(shape, seed))
    return t.from_numpy(x).to("cuda").to(t.bfloat16), x


def to_np(x):
    return x.float().cpu().numpy()


def head_mask(dims, B, s):
    n = dims.seq_len()
    nb = (n + B - 1) // B
    if s.kind == "full":
        return np.ones(nb * nb, np.uint8)
    return oracle.arrow_mask(dims.n_visual, dims.n_text, 1 if dims.order == api.TEXT_FIRST else 0, B,
                             s.window_blocks)


def check_close(got, want, what=""):
    got = np.asarray(got, np.float64)
    rel = np.abs(got - want).max() / np.abs(want).max()
    den = ((want - want.mean()) ** 2).sum()
    r = ((got - want) ** 2).sum() / den
    assert rel <= MAX_REL and r <= MAX_RSE, f"{what}: max-rel {rel:.3e} rse {r:.3e}"
    return rel, r


def oracle_head(qn, kn, vn, dims, B, s, rows=None):
    return oracle.attention_rows_f64(qn, kn, vn, head_mask(dims, B, s), B, rows)


CASES = [
    # (H, nv, nt, d, B, order, plan)
    (4, 1024, 77, 64, 128, 0, "F A0 A2 F"),     # cfg1 geometry (ragged 77-token tail)
    (4, 1024, 77, 64, 64, 0, "F A0 A2 A1"),     # cfg1 at B=64 (element masks inside 128 tiles)
    (3, 256, 32, 128, 32, 0, "A0 A1 F"),        # test_arrow.cpp:154-166 geometry, d=128
    (3, 300, 44, 64, 48, 1, "A0 A2 F"),         # text-first, B not dividing 128
    (2, 130, 17, 128, 16, 0, "A0 A3"),          # small ragged
    (2, 600, 50, 64, 200, 0, "A0 A1"),          # B > 128
    (2, 17, 3, 64, 8, 0, "A0 F"),               # N < one tile
    # head dims other than 64 / 128: direct TMA layout for
    # d % 8 == 0 above 64, zero-padded copies otherwise
    (2, 300, 20, 96, 64, 0, "F A1"),            # d=96 direct (partial second column box)
    (2, 200, 10, 100, 32, 1, "A0 F"),           # d=100 padded to 128
    (3, 256, 32, 32, 32, 0, "A0 A1 F"),         # d=32 padded to 64 (test_arrow.cpp geometry)
    (2, 130, 7, 8, 16, 0, "F A2"),              # d=8
    (2, 64, 16, 72, 16, 0, "A0 F"),             # d=72 direct
    (2, 512, 0, 128, 128, 0, "A0 A1"),          # no text band: block-diagonal (test_arrow.cpp:76-81)
    (1, 4096, 333, 64, 128, 1, "A8"),           # SD3 geometry, text-first, one head
]


@pytest.mark.parametrize("H,nv,nt,d,B,order,plan", CASES)
def test_multi_strategy_matches_oracle(H, nv, nt, d, B, order, plan):
    t = torch()
    dims = AttentionDims(H, d, nv, nt, api.TEXT_FIRST if order else api.VISUAL_FIRST)
    n = nv + nt
    q, qn = bf16_inputs((H, n, d), 11)
    k, kn = bf16_inputs((H, n, d), 12)
    v, vn = bf16_inputs((H, n, d), 13)
    lp = LayerPlan.parse(plan)
    out = api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B)
    t.cuda.synchronize()
    o = to_np(out)
    for h, s in enumerate(lp.strategies):
        check_close(o[h], oracle_head(qn[h], kn[h], vn[h], dims, B, s), f"head {h} {s}")


def test_cached_heads_and_cache_commit_semantics():
    """dispatch.cpp:62-88 + test_dispatch.cpp:63-88: cached heads splice the
    stored slot bit-exactly and keep produced_at; computed heads commit."""
    t = torch()
    H, nv, nt, d, B = 4, 1024, 77, 64, 128
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    cache = HeadCache(2, H, n, d)
    q0, _ = bf16_inputs((H, n, d), 21)
    k0, _ = bf16_inputs((H, n, d), 22)
    v0, _ = bf16_inputs((H, n, d), 23)
    o0 = api.multi_strategy_attention(q0, k0, v0, LayerPlan.all_full(H), cache, 1, 0, dims, B)
    t.cuda.synchronize()
    for h in range(H):
        assert cache.has(1, h) and cache.produced_at(1, h) == 0
        assert t.equal(cache.fetch(1, h), o0[h])
    assert not cache.has(0, 0)
    q1, q1n = bf16_inputs((H, n, d), 31)
    k1, k1n = bf16_inputs((H, n, d), 32)
    v1, v1n = bf16_inputs((H, n, d), 33)
    lp = LayerPlan.parse("F A0 A2 C")
    o1 = api.multi_strategy_attention(q1, k1, v1, lp, cache, 1, 1, dims, B)
    t.cuda.synchronize()
    assert t.equal(o1[3], o0[3])                      # spliced bit-exactly
    assert cache.produced_at(1, 3) == 0               # cached head keeps its slot
    assert [cache.produced_at(1, h) for h in range(3)] == [1, 1, 1]
    for h in range(3):
        assert t.equal(cache.fetch(1, h), o1[h])      # commit == output, bitwise
        check_close(to_np(o1[h]), oracle_head(q1n[h], k1n[h], v1n[h], dims, B, lp.strategies[h]))
    assert cache.staleness(1, 3, 5) == 5
    assert cache.size() == 4


@pytest.mark.parametrize("d,pinned", [(64, True), (128, True), (64, False)])
def test_host_buffer_path_matches_device_path(d, pinned):
    """dfa2c_mha_forward_host (head-group upload / compute / download
    pipeline, cached heads straight from their slots) is bitwise the device
    path: outputs, cache slots and produced_at, over two timesteps."""
    t = torch()
    Bt, H, nv, nt, B = 2, 7, 1024, 77, 128
    n = nv + nt
    dims = AttentionDims(H, d, nv, nt)
    dev_cache, host_cache = HeadCache(1, H, n, d, batch=Bt), HeadCache(1, H, n, d, batch=Bt)
    for step, plan in enumerate((LayerPlan.all_full(H), LayerPlan.parse("F C A0 A2 C C F"))):
        q, _ = bf16_inputs((Bt, H, n, d), 300 + 3 * step)
        k, _ = bf16_inputs((Bt, H, n, d), 301 + 3 * step)
        v, _ = bf16_inputs((Bt, H, n, d), 302 + 3 * step)
        od = api.multi_strategy_attention(q, k, v, plan, dev_cache, 0, step, dims, B)
        hq, hk, hv = (x.cpu() for x in (q, k, v))
        if pinned:
            hq, hk, hv = hq.pin_memory(), hk.pin_memory(), hv.pin_memory()
        oh = api.multi_strategy_attention_host(hq, hk, hv, plan, host_cache, 0, step, dims, B)
        t.cuda.synchronize()
        assert not oh.is_cuda and t.equal(oh.cuda(), od)
        for h in range(H):
            assert host_cache.produced_at(0, h) == dev_cache.produced_at(0, h)
            assert t.equal(host_cache.fetch(0, h), dev_cache.fetch(0, h))
    with pytest.raises(CacheMissError):  # validation before any transfer
        api.multi_strategy_attention_host(hq, hk, hv, LayerPlan.parse("C F F F F F F"), HeadCache(1, H, n, d, batch=Bt),
                                          0, 1, dims, B)


def test_padded_head_dim_cache_semantics():
    """The zero-padded path (d % 8 != 0) keeps the fused call's cache rules:
    cached heads are the stored slot bit for bit, computed heads commit."""
    t = torch()
    H, nv, nt, d, B = 4, 200, 20, 40, 32
    n = nv + nt
    dims = AttentionDims(H, d, nv, nt)
    cache = HeadCache(1, H, n, d)
    q, _ = bf16_inputs((H, n, d), 61)
    o0 = api.multi_strategy_attention(q, q, q, LayerPlan.all_full(H), cache, 0, 0, dims, B)
    q1, q1n = bf16_inputs((H, n, d), 62)
    lp = LayerPlan.parse("C A0 F C")
    o1 = api.multi_strategy_attention(q1, q1, q1, lp, cache, 0, 1, dims, B)
    t.cuda.synchronize()
    assert t.equal(o1[0], o0[0]) and t.equal(o1[3], o0[3])
    assert [cache.produced_at(0, h) for h in range(H)] == [0, 1, 1, 0]
    for h in (1, 2):
        assert t.equal(cache.fetch(0, h), o1[h])
        check_close(to_np(o1[h]), oracle_head(q1n[h], q1n[h], q1n[h], dims, B, lp.strategies[h]))


@pytest.mark.parametrize("d", [160, 256, 512])
def test_wide_head_dims_through_the_simt_path(d):
    """head_dim > 128 (the reference accepts any d >= 1, src/tensor.cpp:225-230)
    runs head by head through the SIMT attention kernel in f32 on the bf16
    inputs: same plan semantics (Full / Arrow / Cached, commits, FullyMasked)
    and the same tolerance against the f64 oracle."""
    t = torch()
    H, nv, nt, B = 3, 300, 40, 64
    n = nv + nt
    dims = AttentionDims(H, d, nv, nt)
    cache = HeadCache(1, H, n, d)
    q, qn = bf16_inputs((H, n, d), 71)
    k, kn = bf16_inputs((H, n, d), 72)
    v, vn = bf16_inputs((H, n, d), 73)
    o0 = api.multi_strategy_attention(q, k, v, LayerPlan.all_full(H), cache, 0, 0, dims, B)
    lp = LayerPlan.parse("A1 C F")
    o1 = api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B)
    t.cuda.synchronize()
    assert t.equal(o1[1], o0[1])                          # Cached: the stored slot, bitwise
    assert t.equal(o1[2], o0[2])                          # deterministic: Full again, same bits
    assert [cache.produced_at(0, h) for h in range(H)] == [1, 0, 1]
    assert t.equal(cache.fetch(0, 0), o1[0])              # commit == output
    for h in (0, 2):
        check_close(to_np(o1[h]), oracle_head(qn[h], kn[h], vn[h], dims, B, lp.strategies[h]), f"d={d} head {h}")
    # a mask with an empty block row fails before any compute
    nb = (n + B - 1) // B
    active = np.ones(nb * nb, np.uint8)
    active[nb:2 * nb] = 0
    with pytest.raises(FullyMaskedRowError):
        api.sparse_attention_forward(q[0], k[0], v[0], BlockMask(B, n, nb, nb, active))


def test_wide_head_dims_batched_and_through_the_host_path():
    """head_dim > 128 with batch 2 on the device path and through the
    host-buffer path (head groups, skipped heads): same bits both ways."""
    t = torch()
    Bt, H, nv, nt, d, B = 2, 3, 256, 30, 192, 64
    n = nv + nt
    dims = AttentionDims(H, d, nv, nt)
    q, qn = bf16_inputs((Bt, H, n, d), 81)
    k, kn = bf16_inputs((Bt, H, n, d), 82)
    v, vn = bf16_inputs((Bt, H, n, d), 83)
    lp = LayerPlan.parse("F A0 A2")
    dev = api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B)
    host = api.multi_strategy_attention_host(q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory(), lp,
                                             None, 0, 0, dims, B)
    t.cuda.synchronize()
    assert t.equal(host.to("cuda"), dev)
    for b in range(Bt):
        for h in range(H):
            check_close(to_np(dev[b, h]), oracle_head(qn[b, h], kn[b, h], vn[b, h], dims, B, lp.strategies[h]),
                        f"sample {b} head {h}")


def test_cache_miss_is_raised_before_any_compute():
    t = torch()
    H, n, d = 3, 300, 64
    dims = AttentionDims(H, d, 280, 20)
    cache = HeadCache(1, H, n, d)
    q, _ = bf16_inputs((H, n, d), 1)
    out = t.full((H, n, d), 7.0, dtype=t.bfloat16, device="cuda")
    with pytest.raises(CacheMissError):
        api.multi_strategy_attention(q, q, q, LayerPlan.parse("F C F"), cache, 0, 1, dims, 64, out=out)
    t.cuda.synchronize()
    assert bool((out == 7.0).all()) and cache.size() == 0
    with pytest.raises(ShapeError):
        api.multi_strategy_attention(q, q, q, LayerPlan.parse("F F"), cache, 0, 1, dims, 64)


def test_full_equals_max_window_arrow_bitwise_and_deterministic():
    t = torch()
    H, nv, nt, d, B = 3, 2048, 120, 128, 128
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, _ = bf16_inputs((H, n, d), 41)
    k, _ = bf16_inputs((H, n, d), 42)
    v, _ = bf16_inputs((H, n, d), 43)
    full = api.multi_strategy_attention(q, k, v, LayerPlan.all_full(H), None, 0, 0, dims, B)
    maxw = api.multi_strategy_attention(q, k, v, LayerPlan([HeadStrategy.Arrow(100)] * H), None, 0, 0, dims, B)
    again = api.multi_strategy_attention(q, k, v, LayerPlan.all_full(H), None, 0, 0, dims, B)
    t.cuda.synchronize()
    assert t.equal(full, maxw) and t.equal(full, again)
    # head isolation (test_dispatch.cpp:98-109)
    a = api.multi_strategy_attention(q, k, v, LayerPlan.parse("F F A1"), None, 0, 0, dims, B)
    b = api.multi_strategy_attention(q, k, v, LayerPlan.parse("F A0 A1"), None, 0, 0, dims, B)
    t.cuda.synchronize()
    assert t.equal(a[0], b[0]) and t.equal(a[2], b[2])


def test_batched_samples_match_single_sample_calls():
    t = torch()
    Bt, H, nv, nt, d, B = 3, 4, 1024, 77, 64, 128
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, _ = bf16_inputs((Bt, H, n, d), 51)
    k, _ = bf16_inputs((Bt, H, n, d), 52)
    v, _ = bf16_inputs((Bt, H, n, d), 53)
    lp = LayerPlan.parse("F A0 A2 A1")
    ob = api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B)
    for s in range(Bt):
        os_ = api.multi_strategy_attention(q[s], k[s], v[s], lp, None, 0, 0, dims, B)
        t.cuda.synchronize()
        assert t.equal(ob[s], os_)


def test_sparse_attention_forward_arbitrary_masks():
    t = torch()
    rng = np.random.default_rng(3)
    for n, d, B in ((300, 64, 16), (513, 128, 64), (1000, 64, 100)):
        nb = (n + B - 1) // B
        m = (rng.random((nb, nb)) < 0.3).astype(np.uint8)
        m[np.arange(nb), np.arange(nb)] = 1
        mask = BlockMask(B, n, nb, nb, m.ravel().copy())
        q, qn = bf16_inputs((2, n, d), 61)
        k, kn = bf16_inputs((2, n, d), 62)
        v, vn = bf16_inputs((2, n, d), 63)
        out = api.sparse_attention_forward(q, k, v, mask)
        t.cuda.synchronize()
        for h in range(2):
            check_close(to_np(out[h]), oracle.attention_rows_f64(qn[h], kn[h], vn[h], mask.active, B))
        dense = api.dense_tiled_attention(q, k, v)
        t.cuda.synchronize()
        check_close(to_np(dense[0]), oracle.attention_rows_f64(qn[0], kn[0], vn[0]))
    bad = BlockMask.all_active(64, 16)
    for j in range(4):
        bad.set(2, j, False)
    x, _ = bf16_inputs((64, 64), 1)
    with pytest.raises(FullyMaskedRowError):
        api.sparse_attention_forward(x, x, x, bad)


def test_against_reference_multi_strategy_golden():
    """The reference's own multi_strategy_attention outputs (golden, f32 on the
    same bf16-rounded inputs): t=0 all Full, t=1 [F, A0, A2, C] with its cache."""
    import os

    t = torch()
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))
    H, nv, nt, d, B = (int(x) for x in G["msa_geom"])
    n = nv + nt
    xs = [oracle.round_bf16(oracle.gaussian((H, n, d), 7000 + tt * 10 + j)) for tt in range(2) for j in range(3)]
    dev = [t.from_numpy(x).cuda().to(t.bfloat16) for x in xs]
    dims = AttentionDims(H, d, nv, nt)
    cache = HeadCache(1, H, n, d)
    o0 = api.multi_strategy_attention(dev[0], dev[1], dev[2], LayerPlan.all_full(H), cache, 0, 0, dims, B)
    o1 = api.multi_strategy_attention(dev[3], dev[4], dev[5], LayerPlan.parse("F A0 A2 C"), cache, 0, 1, dims, B)
    t.cuda.synchronize()
    for h in range(H):
        check_close(to_np(o0[h]), G["msa_out_t0"][h].astype(np.float64), f"t0 head {h}")
        check_close(to_np(o1[h]), G["msa_out_t1"][h].astype(np.float64), f"t1 head {h}")
    assert [cache.produced_at(0, h) for h in range(H)] == list(G["msa_produced_at"])


@pytest.mark.parametrize("plan_kind", ["flux68"])
def test_flux_2k_sampled_rows(plan_kind):
    """Config 3 at full size (16384+512, H=24, d=128, B=128, FLUX68 after an
    all-Full t=0): every head checked on sampled rows (incl. text rows) against
    the f64 oracle; cached heads bit-exact."""
    t = torch()
    H, nv, nt, d, B = 24, 16384, 512, 128, 128
    n = nv + nt
    dims = AttentionDims(H, d, nv, nt)
    cache = HeadCache(1, H, n, d)
    q, qn = bf16_inputs((H, n, d), 1)
    k, kn = bf16_inputs((H, n, d), 2)
    v, vn = bf16_inputs((H, n, d), 3)
    slots = {}
    for h in range(H):
        s, _ = bf16_inputs((n, d), 100 + h)
        cache.store(0, h, s, 0)
        slots[h] = s
    lp = api.flux68_plan(H)
    out = api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B)
    t.cuda.synchronize()
    rows = np.concatenate([np.arange(0, nv, 997), np.arange(nv, n, 61), [n - 1]]).astype(np.int64)
    o = out.float().cpu().numpy()
    for h, s in enumerate(lp.strategies):
        if s.kind == "cached":
            assert t.equal(out[h], slots[h])
            continue
        want = oracle_head(qn[h], kn[h], vn[h], dims, B, s, rows)
        check_close(o[h][rows], want, f"head {h} {s}")


@pytest.mark.parametrize("d,order", [(64, 0), (128, 1)])
def test_split_kv_text_rows(d, order):
    """Split-KV (opt-in): the text-row pairs of arrow heads
    run as key chunks combined in chunk order by the CTA that finishes last.
    Their rows match the f64 oracle, the committed cache slot equals the
    output, batched and repeated calls are bitwise identical."""
    t = torch()
    api.set_split_kv(True)
    try:
        _split_kv_text_rows(t, d, order)
    finally:
        api.set_split_kv(False)


def _split_kv_text_rows(t, d, order):
    Bt, H, nv, nt, B = 2, 3, 4096, 333, 128
    n = nv + nt
    dims = AttentionDims(H, d, nv, nt, api.TEXT_FIRST if order else api.VISUAL_FIRST)
    q, qn = bf16_inputs((Bt, H, n, d), 71)
    k, kn = bf16_inputs((Bt, H, n, d), 72)
    v, vn = bf16_inputs((Bt, H, n, d), 73)
    lp = LayerPlan.parse("A0 A2 A40")
    cache = HeadCache(1, H, n, d, batch=Bt)
    out = api.multi_strategy_attention(q, k, v, lp, cache, 0, 0, dims, B)
    again = api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B)
    single = api.multi_strategy_attention(q[1], k[1], v[1], lp, None, 0, 0, dims, B)
    t.cuda.synchronize()
    assert t.equal(out, again) and t.equal(out[1], single)
    lo, hi = dims.text_begin(), dims.text_end()
    rows = np.concatenate([np.arange(lo, hi, 7), np.arange(0, n, 503)]).astype(np.int64)
    o = to_np(out)
    for b in range(Bt):
        for h in range(2):
            want = oracle_head(qn[b, h], kn[b, h], vn[b, h], dims, B, lp.strategies[h], rows)
            check_close(o[b, h][rows], want, f"sample {b} head {h}")
            assert t.equal(cache.fetch(0, h)[b], out[b, h])


@pytest.mark.parametrize("split", [False, True])
def test_skip_heads_split_one_layer_bitwise(split):
    """DFA2C_SKIP: two calls over complementary head sets (as two GPUs would
    run) reproduce the single call bit for bit, leave skipped rows and
    skipped heads' cache bookkeeping untouched, and a skipped Cached head
    needs no slot."""
    t = torch()
    api.set_split_kv(split)
    try:
        _skip_heads(t)
    finally:
        api.set_split_kv(False)


def _skip_heads(t):
    H, nv, nt, d, B = 4, 4096, 333, 64, 128
    n = nv + nt
    dims = AttentionDims(H, d, nv, nt)
    q, _ = bf16_inputs((H, n, d), 81)
    k, _ = bf16_inputs((H, n, d), 82)
    v, _ = bf16_inputs((H, n, d), 83)
    ref_cache, a_cache = HeadCache(1, H, n, d), HeadCache(1, H, n, d)
    api.multi_strategy_attention(q, k, v, LayerPlan.all_full(H), ref_cache, 0, 0, dims, B)
    api.multi_strategy_attention(q, k, v, LayerPlan.all_full(H), a_cache, 0, 0, dims, B, skip_heads=[0, 3])
    plan = LayerPlan.parse("A0 C A2 F")
    ref = api.multi_strategy_attention(q, k, v, plan, ref_cache, 0, 1, dims, B)
    out = t.full_like(q, 7.0)
    api.multi_strategy_attention(q, k, v, plan, a_cache, 0, 1, dims, B, out=out, skip_heads=[0, 3])
    t.cuda.synchronize()
    assert bool((out[0] == 7.0).all()) and bool((out[3] == 7.0).all())  # skipped rows untouched
    assert not a_cache.has(0, 0) and not a_cache.has(0, 3)            # skipped heads never committed
    assert a_cache.produced_at(0, 2) == 1 and a_cache.produced_at(0, 1) == 0
    assert t.equal(out[1], ref[1]) and t.equal(out[2], ref[2])
    b_cache = HeadCache(1, H, n, d)
    api.multi_strategy_attention(q, k, v, plan, b_cache, 0, 0, dims, B, out=out, skip_heads=[1, 2])  # no slots
    t.cuda.synchronize()
    assert t.equal(out, ref)  # head 0 (split text rows) and head 3 from the other "GPU"


def test_rse_kernel_against_oracle_and_reference_semantics():
    t = torch()
    # f32 operands: fp64 accumulation, within 1e-9 of the reference's sequential rse
    for n, scale in ((2, 1.0), (1000, 0.1), (16896 * 128, 0.01), (12345, 3.0)):
        a = oracle.gaussian((n,), 7) + 2.5
        b = a + scale * oracle.gaussian((n,), 8)
        for mode in (0, 1):
            want = oracle.rse_f32(b, a, mode)
            got = api.rse(t.from_numpy(b).cuda(), t.from_numpy(a).cuda(), mode)
            assert abs(got - want) <= 1e-9 * abs(want), (n, mode, got, want)
    # bf16 operands, several heads in one launch
    H, n = 24, 16896 * 128
    a, an = bf16_inputs((H, n), 9)
    b, bn = bf16_inputs((H, n), 10)
    b = (a.float() + 0.05 * b.float()).to(t.bfloat16)
    bn = to_np(b)
    got = api.rse_per_head(b, a)
    for h in (0, 7, 23):
        want = oracle.rse_f32(bn[h], an[h])
        assert abs(got[h] - want) <= 1e-9 * want
    # hand values and the degenerate case (test_calibrate.cpp:48-72)
    y_o = t.tensor([1.0, 3.0], device="cuda")
    assert api.rse(t.tensor([2.0, 2.0], device="cuda"), y_o) == pytest.approx(1.0)
    assert api.rse(y_o, y_o) == 0.0
    assert api.rse(y_o, y_o, api.RseMode.literal) == pytest.approx(1.0)
    with pytest.raises(api.DegenerateReferenceError):
        api.rse(t.tensor([5.0, 6.0], device="cuda"), t.tensor([5.0, 5.0], device="cuda"))


@pytest.mark.parametrize("fused", [False, True], ids=["exact", "fused"])
def test_influence_for_layer_semantics(fused):
    """calibrate.cpp:193-253 + test_calibrate.cpp:85-146, with the
    per-candidate passes and with the fused band-snapshot pass."""
    before = api.influence_fused_enabled()
    api.set_influence_fused(fused)
    try:
        _influence_for_layer_semantics(fused)
    finally:
        api.set_influence_fused(before)


def _influence_for_layer_semantics(fused):
    t = torch()
    H, nv, nt, d, B = 4, 1024, 77, 64, 128
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, _ = bf16_inputs((H, n, d), 71)
    k, _ = bf16_inputs((H, n, d), 72)
    v, _ = bf16_inputs((H, n, d), 73)
    cache = HeadCache(1, H, n, d)
    stats = api.CalibrationStats()
    methods = api.make_candidates([0, 2, 100], include_cached=True)
    li = api.influence_for_layer(q, k, v, methods, cache, 0, 0, dims, B, stats=stats)
    M = len(methods)
    assert stats.attention_evals == 1 + M
    infl = li.influence.reshape(H, M)
    assert np.isinf(infl[:, 3]).all()          # Cached ineligible at t = 0
    assert (infl[:, 2] == 0.0).all()           # max window == Full, bitwise
    assert (infl[:, 0] >= infl[:, 1]).all()    # narrower window, larger error
    for h in range(H):                          # independent recomputation
        want = oracle.rse_f32(to_np(li.method_outputs[0][h]), to_np(li.original[h]))
        assert infl[h, 0] == pytest.approx(want, rel=1e-12)
    full = api.multi_strategy_attention(q, k, v, LayerPlan.all_full(H), None, 0, 0, dims, B)
    t.cuda.synchronize()
    if fused:  # key tiles folded in window-band order: equal up to bf16 rounding
        for h in range(H):
            check_close(to_np(li.original[h]), to_np(full[h]).astype(np.float64), f"original head {h}")
    else:
        assert t.equal(full, li.original)
    # Cached candidate against identical entries measures 0 (test_calibrate.cpp:97-109):
    # the slots hold the original of the same candidate set (in fused mode the
    # original is the band-order fold of that set's pass)
    for h in range(H):
        cache.store(0, h, li.original[h], 0)
    li2 = api.influence_for_layer(q, k, v, methods, cache, 0, 1, dims, B)
    assert (li2.influence.reshape(H, M)[:, 3] == 0.0).all()
    if not fused:
        li3 = api.influence_for_layer(q, k, v, api.make_candidates([], True), cache, 0, 1, dims, B)
        assert (li3.influence == 0.0).all()


def test_influence_matches_reference_values():
    """Same bf16-rounded inputs through the reference's influence_for_layer
    (f32) and ours (bf16): per-head influences agree to a few percent."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not available")
    from oracle import c_double, c_float, c_int64, ptr
    t = torch()
    H, nv, nt, d, B = 4, 512, 64, 64, 64
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, qn = bf16_inputs((H, n, d), 81)
    k, kn = bf16_inputs((H, n, d), 82)
    v, vn = bf16_inputs((H, n, d), 83)
    wins = np.array([0, 1, 3], np.int64)
    infl_ref = np.zeros(H * 3, np.float64)
    c = oracle.ref().ref_cache_create()
    oracle.ref_check(oracle.ref().ref_influence_for_layer(
        ptr(qn, c_float), ptr(kn, c_float), ptr(vn, c_float), H, d, nv, nt, 0, ptr(wins, c_int64), 3, 0, c, 0, 0,
        B, 0, ptr(infl_ref, c_double), None, None, None))
    oracle.ref().ref_cache_destroy(c)
    li = api.influence_for_layer(q, k, v, api.make_candidates([0, 1, 3], False), None, 0, 0, dims, B)
    np.testing.assert_allclose(li.influence, infl_ref, rtol=0.05)


def test_run_pipeline_on_reference_workload():
    """run_pipeline (workload.cpp:230-262) over the reference generator's
    drifting streams: every (t, l) within tolerance of the reference's own
    pipeline; cached heads replay their last computed output bitwise."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not available")
    from oracle import c_float, c_int32, c_int64, ptr
    t = torch()
    H, nv, nt, d, L, T, B = 4, 512, 64, 64, 2, 3, 64
    n = nv + nt
    per = H * n * d
    qs, ks, vs = (np.zeros((T * L, H, n, d), np.float32) for _ in range(3))
    oracle.ref_check(oracle.ref().ref_generate(H, d, nv, nt, 0, L, T, B, 1234, ptr(qs, c_float), ptr(ks, c_float),
                                               ptr(vs, c_float)))
    qs, ks, vs = (oracle.round_bf16(x).reshape(T * L, H, n, d) for x in (qs, ks, vs))
    dims = AttentionDims(H, d, nv, nt)
    plan = api.CompressionPlan.all_full(dims, T, L, B)
    plan.layers[1 * L + 0] = LayerPlan.parse("F A0 A2 C")
    plan.layers[2 * L + 1] = LayerPlan.parse("C A1 F C")
    plan.layers[2 * L + 0] = LayerPlan.parse("A0 C C F")
    dq, dk, dv = (t.from_numpy(x).cuda().to(t.bfloat16) for x in (qs, ks, vs))
    stats = api.run_pipeline(lambda tt, l: dq[tt * L + l], lambda tt, l: dk[tt * L + l],
                             lambda tt, l: dv[tt * L + l], plan)
    t.cuda.synchronize()
    assert stats.flops_total == plan.flops_total()
    assert stats.sparsity == pytest.approx(plan.aggregate_sparsity(), abs=1e-15)
    c = oracle.ref().ref_cache_create()
    for tt in range(T):
        for l in range(L):
            lp = plan.at(tt, l)
            kinds = np.array([api._KIND_CODE[s.kind] for s in lp.strategies], np.int32)
            wins = np.array([s.window_blocks for s in lp.strategies], np.int64)
            o = np.zeros((H, n, d), np.float32)
            s = tt * L + l
            oracle.ref_check(oracle.ref().ref_multi_strategy_attention(
                ptr(np.ascontiguousarray(qs[s]), c_float), ptr(np.ascontiguousarray(ks[s]), c_float),
                ptr(np.ascontiguousarray(vs[s]), c_float), H, d, nv, nt, 0, ptr(kinds, c_int32),
                ptr(wins, c_int64), c, l, tt, B, ptr(o, c_float)))
            got = to_np(stats.output(tt, l, L))
            for h in range(H):
                check_close(got[h], o[h].astype(np.float64), f"t{tt} l{l} h{h}")
    oracle.ref().ref_cache_destroy(c)
    # cached replay: (t=2, l=0) head 1 is Cached -> equals (t=1, l=0) head 1 output... which was A0 at t=1
    assert t.equal(stats.output(2, 0, L)[1], stats.output(1, 0, L)[1])
    assert t.equal(stats.output(2, 1, L)[0], stats.output(1, 1, L)[0])
    _ = (ctypes, per, ArrowSpec)


# ---- fused calibration pass (dfa2c_influence_for_layer at block 128):
# the original and every Arrow candidate from one launch, each candidate the
# snapshot of its query tiles after the candidate's window band.
FUSED_CASES = [
    # (H, nv, nt, d, order, windows)
    (2, 1024, 77, 64, 0, [0, 2, 5, 100]),                  # cfg1 geometry, ragged tail; 100 clamps to Full
    (2, 1024, 77, 128, 1, [3, 1, 1, 0]),                   # text-first; unsorted and duplicate windows
    (2, 768, 0, 128, 0, [0, 1]),                           # no text band (block diagonal)
    (1, 2048, 256, 128, 0, [0, 2, 4, 6, 8, 10, 12, 14]),   # eight bands, 15 (= Full) left to the original
    (3, 300, 20, 96, 0, [0, 1]),                           # d=96 in place; 3 query tiles (single-lane item)
]


@pytest.mark.parametrize("H,nv,nt,d,order,windows", FUSED_CASES)
def test_fused_influence_outputs_match_oracle(H, nv, nt, d, order, windows):
    t = torch()
    B = 128
    assert api.influence_fused_enabled()  # the default
    dims = AttentionDims(H, d, nv, nt, api.TEXT_FIRST if order else api.VISUAL_FIRST)
    n = nv + nt
    q, qn = bf16_inputs((H, n, d), 91)
    k, kn = bf16_inputs((H, n, d), 92)
    v, vn = bf16_inputs((H, n, d), 93)
    methods = api.make_candidates(windows, include_cached=False)
    launches = api.launch_count()
    li = api.influence_for_layer(q, k, v, methods, None, 0, 0, dims, B)
    t.cuda.synchronize()
    # one attention launch; the RSE grid (partial + finalize) per run of <= 8 candidates
    assert api.launch_count() - launches == 1 + 2 * ((len(windows) + 7) // 8)
    rows = None if n <= 1200 else np.arange(0, n, 5)
    for h in range(H):
        want = oracle_head(qn[h], kn[h], vn[h], dims, B, HeadStrategy.Full(), rows)
        got = to_np(li.original[h]) if rows is None else to_np(li.original[h])[rows]
        check_close(got, want, f"original head {h}")
        for m, w in enumerate(windows):
            want = oracle_head(qn[h], kn[h], vn[h], dims, B, HeadStrategy.Arrow(w), rows)
            got = to_np(li.method_outputs[m][h])
            check_close(got if rows is None else got[rows], want, f"Arrow({w}) head {h}")
    # equal effective windows share one snapshot; a window covering the row is the original
    nvb = (nv + B - 1) // B
    for m, w in enumerate(windows):
        weff = min(w, max(0, nvb - 1))
        for m2, w2 in enumerate(windows):
            if min(w2, max(0, nvb - 1)) == weff:
                assert t.equal(li.method_outputs[m], li.method_outputs[m2])
        if (head_mask(dims, B, HeadStrategy.Arrow(w)) == 1).all():
            assert t.equal(li.method_outputs[m], li.original)
            assert (li.influence.reshape(H, -1)[:, m] == 0.0).all()
    # deterministic: a second call is bitwise identical
    li2 = api.influence_for_layer(q, k, v, methods, None, 0, 0, dims, B)
    assert t.equal(li2.original, li.original) and t.equal(li2.method_outputs, li.method_outputs)
    assert np.array_equal(li2.influence, li.influence)


def test_fused_influence_agrees_with_per_candidate_passes():
    """Same influences as the per-candidate passes (the outputs differ only by
    the key-tile fold order); the per-candidate passes are bitwise the
    dispatcher's outputs."""
    t = torch()
    H, nv, nt, d, B = 4, 2048, 77, 128, 128
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, _ = bf16_inputs((H, n, d), 94)
    k, _ = bf16_inputs((H, n, d), 95)
    v, _ = bf16_inputs((H, n, d), 96)
    # sharpen the logits of two heads so the windows matter unequally
    q[:2] *= 3
    methods = api.make_candidates([0, 2, 8], include_cached=False)
    fused = api.influence_for_layer(q, k, v, methods, None, 0, 0, dims, B)
    api.set_influence_fused(False)
    try:
        exact = api.influence_for_layer(q, k, v, methods, None, 0, 0, dims, B)
    finally:
        api.set_influence_fused(True)
    np.testing.assert_allclose(fused.influence, exact.influence, rtol=2e-2, atol=1e-6)
    for m, w in enumerate([0, 2, 8]):
        lp = LayerPlan([HeadStrategy.Arrow(w)] * H)
        ref = api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B)
        t.cuda.synchronize()
        assert t.equal(exact.method_outputs[m], ref)
        for h in range(H):
            check_close(to_np(fused.method_outputs[m][h]), to_np(ref[h]).astype(np.float64), f"Arrow({w}) head {h}")


def test_fused_influence_falls_back_off_tile_blocks():
    """Mask blocks other than the 128-key tile take the per-candidate passes
    (outputs bitwise the dispatcher's)."""
    t = torch()
    H, nv, nt, d, B = 2, 512, 64, 64, 64
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, _ = bf16_inputs((H, n, d), 97)
    k, _ = bf16_inputs((H, n, d), 98)
    v, _ = bf16_inputs((H, n, d), 99)
    li = api.influence_for_layer(q, k, v, api.make_candidates([1], False), None, 0, 0, dims, B)
    full = api.multi_strategy_attention(q, k, v, LayerPlan.all_full(H), None, 0, 0, dims, B)
    t.cuda.synchronize()
    assert t.equal(full, li.original)


def test_async_influence_matches_sync_and_window_limit_falls_back():
    """dfa2c_influence_for_layer_async + dfa2c_influence_finalize give the
    synchronous call's influences bitwise; 16 windows (over the fused pass's
    15-candidate limit) take the per-candidate passes."""
    t = torch()
    H, nv, nt, d, B = 2, 1024, 77, 64, 128
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, _ = bf16_inputs((H, n, d), 101)
    k, _ = bf16_inputs((H, n, d), 102)
    v, _ = bf16_inputs((H, n, d), 103)
    cache = HeadCache(1, H, n, d)
    api.multi_strategy_attention(q, k, v, LayerPlan.all_full(H), cache, 0, 0, dims, B)
    methods = api.make_candidates([0, 1, 3], include_cached=True)
    sync = api.influence_for_layer(q, k, v, methods, cache, 0, 1, dims, B)
    bufs = []
    pend = api._influence_launch(q, k, v, methods, cache, 0, 1, dims, B, api.RseMode.standard, None, bufs)
    got = pend.finish()
    assert np.array_equal(got.influence, sync.influence)
    assert t.equal(got.original, sync.original) and t.equal(got.method_outputs, sync.method_outputs)
    # 16 windows: per-candidate passes, whose original is bitwise the dispatcher's Full output
    many = api.make_candidates(list(range(16)), include_cached=False)
    li = api.influence_for_layer(q, k, v, many, None, 0, 0, dims, B)
    full = api.multi_strategy_attention(q, k, v, LayerPlan.all_full(H), None, 0, 0, dims, B)
    t.cuda.synchronize()
    assert t.equal(li.original, full)
    assert np.isfinite(li.influence).all()


# 48 seeds over d in {64, 96, 128}, then head dims 40 (zero-padded) and 160
# (SIMT path) join the draw; DFA2_RANDOM_LAYERS=<n> runs a longer sweep
@pytest.mark.parametrize("seed", range(int(os.environ.get("DFA2_RANDOM_LAYERS", "64"))))
def test_random_plans_and_geometries_against_oracle(seed):
    """Seeded random layers: geometry (visual/text tokens, token order, mask
    block, head dim), a random F / A(w) / C plan with slots filled at t = 0,
    split-KV on or off. Sampled rows of every head against the f64 oracle;
    Cached heads bitwise their slot; every computed head's committed slot
    bitwise its output."""
    t = torch()
    rng = np.random.default_rng(1000 + seed)
    H = int(rng.integers(2, 6))
    d = int(rng.choice([64, 128, 96, 40, 160] if seed >= 48 else [64, 128, 96]))
    nv = int(rng.integers(200, 3000))
    nt = int(rng.choice([0, int(rng.integers(1, 400))]))
    order = int(rng.integers(0, 2))
    B = int(rng.choice([32, 64, 128, 128, 200]))
    split = bool(rng.integers(0, 2))
    dims = AttentionDims(H, d, nv, nt, api.TEXT_FIRST if order else api.VISUAL_FIRST)
    n = nv + nt
    nvb = (nv + B - 1) // B
    strategies = []
    for _ in range(H):
        r = rng.random()
        if r < 0.3:
            strategies.append(HeadStrategy.Full())
        elif r < 0.8:
            strategies.append(HeadStrategy.Arrow(int(rng.integers(0, max(1, nvb + 2)))))
        else:
            strategies.append(HeadStrategy.Cached())
    lp = LayerPlan(strategies)
    q, qn = bf16_inputs((H, n, d), 2000 + seed)
    k, kn = bf16_inputs((H, n, d), 3000 + seed)
    v, vn = bf16_inputs((H, n, d), 4000 + seed)
    cache = HeadCache(1, H, n, d)
    slots, _ = bf16_inputs((H, n, d), 5000 + seed)
    for h in range(H):
        cache.store(0, h, slots[h], 0)
    api.set_split_kv(split)
    try:
        out = api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B)
        t.cuda.synchronize()
    finally:
        api.set_split_kv(False)
    rows = np.unique(np.concatenate([np.arange(0, n, max(1, n // 97)), [n - 1],
                                     np.arange(dims.text_begin(), dims.text_end(), 11)])).astype(np.int64)
    o = to_np(out)
    for h, s_ in enumerate(strategies):
        if s_.kind == "cached":
            assert t.equal(out[h], slots[h]), f"head {h} cached copy"
            assert cache.produced_at(0, h) == 0
            continue
        want = oracle_head(qn[h], kn[h], vn[h], dims, B, s_, rows)
        check_close(o[h][rows], want, f"seed {seed} head {h} {s_} (d={d}, B={B}, order={order}, split={split})")
        assert t.equal(cache.fetch(0, h), out[h]) and cache.produced_at(0, h) == 1


@pytest.mark.parametrize("seed", range(8))
def test_random_fused_influence_against_oracle(seed):
    """Seeded random geometries through the fused calibration pass (block
    128): every candidate's sampled rows against the f64 oracle, influences
    against the per-candidate passes."""
    t = torch()
    rng = np.random.default_rng(7000 + seed)
    H = int(rng.integers(1, 4))
    d = int(rng.choice([64, 128, 96]))
    nv = int(rng.integers(300, 3000))
    nt = int(rng.choice([0, int(rng.integers(1, 400))]))
    order = int(rng.integers(0, 2))
    B = 128
    dims = AttentionDims(H, d, nv, nt, api.TEXT_FIRST if order else api.VISUAL_FIRST)
    n = nv + nt
    windows = [int(w) for w in rng.integers(0, (nv + B - 1) // B + 3, size=int(rng.integers(1, 7)))]
    q, qn = bf16_inputs((H, n, d), 8000 + seed)
    k, kn = bf16_inputs((H, n, d), 9000 + seed)
    v, vn = bf16_inputs((H, n, d), 10000 + seed)
    methods = api.make_candidates(windows, include_cached=False)
    li = api.influence_for_layer(q, k, v, methods, None, 0, 0, dims, B)
    api.set_influence_fused(False)
    try:
        exact = api.influence_for_layer(q, k, v, methods, None, 0, 0, dims, B)
    finally:
        api.set_influence_fused(True)
    t.cuda.synchronize()
    rows = np.unique(np.concatenate([np.arange(0, n, max(1, n // 61)), [n - 1]])).astype(np.int64)
    for h in range(H):
        check_close(to_np(li.original[h])[rows], oracle_head(qn[h], kn[h], vn[h], dims, B, HeadStrategy.Full(), rows),
                    f"seed {seed} original head {h}")
        for m, w in enumerate(windows):
            want = oracle_head(qn[h], kn[h], vn[h], dims, B, HeadStrategy.Arrow(w), rows)
            check_close(to_np(li.method_outputs[m][h])[rows], want, f"seed {seed} Arrow({w}) head {h}")
    np.testing.assert_allclose(li.influence, exact.influence, rtol=2e-2, atol=1e-6)


@pytest.mark.parametrize("mode", [0, 1], ids=["standard", "literal"])
def test_influence_rse_grid_matches_oracle_rse(mode):
    """The layer's RSE grid (one multi-candidate launch, original streamed
    once) against the oracle's rse on the same bf16 outputs, both numerator
    modes (src/calibrate.cpp:84-85), including more than 8 candidates (two
    launches) and the Cached candidate."""
    t = torch()
    H, nv, nt, d, B = 3, 1024, 77, 64, 128
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, _ = bf16_inputs((H, n, d), 111)
    k, _ = bf16_inputs((H, n, d), 112)
    v, _ = bf16_inputs((H, n, d), 113)
    cache = HeadCache(1, H, n, d)
    slots, _ = bf16_inputs((H, n, d), 114)
    for h in range(H - 1):  # the last head has no slot: Cached ineligible there
        cache.store(0, h, slots[h], 0)
    methods = api.make_candidates(list(range(9)), include_cached=True)
    li = api.influence_for_layer(q, k, v, methods, cache, 0, 1, dims, B, mode=mode)
    t.cuda.synchronize()
    M = len(methods)
    grid = li.influence.reshape(H, M)
    for h in range(H):
        o = to_np(li.original[h])
        for m in range(M):
            if m == M - 1 and h == H - 1:
                assert np.isinf(grid[h, m])
                continue
            ym = to_np(li.method_outputs[m][h])
            assert grid[h, m] == pytest.approx(oracle.rse_f32(ym, o, mode), rel=1e-10, abs=1e-15)


def test_plan_cache_eviction_keeps_results_bitwise(tmp_path):
    """Work lists are evicted (FIFO) and rebuilt while earlier launches that
    read them may still be in flight: with a 3-plan cache, 8 distinct plans
    cycled twice give bitwise the outputs of a fresh process's first pass."""
    import subprocess
    import sys as _sys

    script = tmp_path / "evict.py"
    script.write_text(r'''
import sys, hashlib
sys.path.insert(0, %r)
import torch
from paper_2503_22796_b200 import api
H, nv, nt, d, B = 6, 2048, 77, 128, 128
n = nv + nt
dims = api.AttentionDims(H, d, nv, nt)
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
plans = ["F A0 A2 F A8 A1", "A0 F F A3 A1 A2", "A2 A2 F A0 F A5", "F F F A0 A0 A0",
         "A1 A2 A3 A4 A5 A6", "A0 A0 A0 A0 A0 F", "F A4 A0 A1 F A9", "A7 F A0 F A2 F"]
outs = []
for rnd in range(2):
    for p in plans:
        outs.append(api.multi_strategy_attention(q, k, v, api.LayerPlan.parse(p), None, 0, 0, dims, B))
torch.cuda.synchronize()
h = [hashlib.sha256(o.view(torch.int16).cpu().numpy().tobytes()).hexdigest() for o in outs]
print(" ".join(h))
''' % ROOT)
    env = dict(os.environ)
    big = subprocess.run([_sys.executable, str(script)], capture_output=True, text=True, env=env, timeout=600)
    env["DFA2_PLAN_CACHE_MAX"] = "3"
    small = subprocess.run([_sys.executable, str(script)], capture_output=True, text=True, env=env, timeout=600)
    assert big.returncode == 0 and small.returncode == 0, big.stderr[-2000:] + small.stderr[-2000:]
    hb, hs = big.stdout.split(), small.stdout.split()
    assert len(hb) == 16 and hb == hs
    assert hb[:8] == hb[8:]  # second cycle (rebuilt plans) bitwise the first


def test_cache_layers_first_touched_on_a_side_stream():
    """A layer's slot buffer is created (pool allocation + zero fill) on the
    stream of the call that first touches it; calls on other streams order
    themselves after it. Fresh layers written from a non-default stream and
    read back from the default stream hold exactly the committed outputs."""
    t = torch()
    H, nv, nt, d, B = 4, 1024, 77, 64, 128
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, _ = bf16_inputs((H, n, d), 121)
    k, _ = bf16_inputs((H, n, d), 122)
    v, _ = bf16_inputs((H, n, d), 123)
    cache = HeadCache(8, H, n, d)
    side = t.cuda.Stream()
    outs = []
    with t.cuda.stream(side):
        for layer in range(8):
            outs.append(api.multi_strategy_attention(q, k, v, LayerPlan.parse("F A0 A2 F"), cache, layer, 0, dims, B,
                                                     stream=side))
    # default stream: fetch every committed slot (ordered after the side stream's creation + commits)
    t.cuda.current_stream().wait_stream(side)
    for layer in range(8):
        for h in range(H):
            assert t.equal(cache.fetch(layer, h), outs[layer][h])


def test_release_cached_memory_then_rebuild():
    """dfa2c_release_cached_memory drops the work lists and trims the pool;
    the next call rebuilds its plan and gives bitwise the same output."""
    t = torch()
    H, nv, nt, d, B = 4, 1024, 77, 128, 128
    dims = AttentionDims(H, d, nv, nt)
    n = nv + nt
    q, _ = bf16_inputs((H, n, d), 131)
    k, _ = bf16_inputs((H, n, d), 132)
    v, _ = bf16_inputs((H, n, d), 133)
    lp = LayerPlan.parse("F A0 A2 A5")
    a = api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B)
    api.release_cached_memory()
    b = api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B)
    t.cuda.synchronize()
    assert t.equal(a, b)


@pytest.mark.parametrize("order", [0, 1], ids=["visual_first", "text_first"])
def test_d64_text_rows_halved_across_lanes(order):
    """d = 64, narrow arrow windows: the text query tiles run on both lanes,
    each folding half of the key tiles, merged in the epilogue (HALVES).
    Rows against the f64 oracle; the rule depends on the head's own mask
    only, so a head's output does not change when another head's strategy
    does (test_dispatch.cpp:98-109), and it is deterministic."""
    t = torch()
    H, nv, nt, d, B = 3, 4096, 333, 64, 128
    dims = AttentionDims(H, d, nv, nt, api.TEXT_FIRST if order else api.VISUAL_FIRST)
    n = nv + nt
    q, qn = bf16_inputs((H, n, d), 141)
    k, kn = bf16_inputs((H, n, d), 142)
    v, vn = bf16_inputs((H, n, d), 143)
    a = api.multi_strategy_attention(q, k, v, LayerPlan.parse("A0 A0 F"), None, 0, 0, dims, B)
    b = api.multi_strategy_attention(q, k, v, LayerPlan.parse("A0 A8 A1"), None, 0, 0, dims, B)
    c = api.multi_strategy_attention(q, k, v, LayerPlan.parse("A0 A0 F"), None, 0, 0, dims, B)
    t.cuda.synchronize()
    assert t.equal(a[0], b[0]) and t.equal(a, c)
    lo, hi = dims.text_begin(), dims.text_end()
    rows = np.concatenate([np.arange(lo, hi, 5), np.arange(0, n, 97)]).astype(np.int64)
    o = to_np(a)
    for h, s_ in enumerate(LayerPlan.parse("A0 A0 F").strategies):
        check_close(o[h][rows], oracle_head(qn[h], kn[h], vn[h], dims, B, s_, rows), f"head {h} {s_}")


_COPY_MODES_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2503_22796_b200 import api
g = torch.Generator(device="cuda").manual_seed(3)
H, NV, NT, D = 8, 2048, 200, int(sys.argv[2])
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
cache = api.HeadCache(1, H, N, D)
out = torch.empty_like(q)
api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, 0, 0, dims, 128, out=out)
for plan in ("F C A2 C C A0 F C", "C C C C C C C C"):
    api.multi_strategy_attention(q, k, v, api.LayerPlan.parse(plan), cache, 0, 1, dims, 128, out=out)
    torch.cuda.synchronize()
    sys.stdout.buffer.write(out.view(torch.int16).cpu().numpy().tobytes())
"""


@pytest.mark.gpu
@pytest.mark.parametrize("D", [64, 128])
def test_copy_pool_and_per_cta_copies_give_the_same_bits(D, tmp_path):
    """The copy pool (default) and the per-CTA copy items (DFA2_COPY_POOL=0,
    with and without the copy tail) write the same layer."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"DFA2_COPY_POOL": "0"}, {"DFA2_COPY_POOL": "0", "DFA2_COPY_TAIL": "0"}):
        r = subprocess.run([sys.executable, "-c", _COPY_MODES_SCRIPT, root, str(D)], capture_output=True,
                           env={**os.environ, **env}, timeout=300)
        assert r.returncode == 0, r.stderr.decode()[-2000:]
        outs.append(r.stdout)
    assert len(outs[0]) > 0 and outs[0] == outs[1] == outs[2]
