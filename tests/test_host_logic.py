"""CPU tests of the product's host logic behind the C-ABI (no GPU calls):
bit-exact masks / FLOP accounting / plan aggregation against the reference
golden vectors and the oracle, and the per-head tile scheduler's tile sets."""
import os

import numpy as np
import pytest

import oracle
from paper_2503_22796_b200 import api
from paper_2503_22796_b200.api import (AttentionDims, ArrowSpec, BlockMask, CompressionPlan, HeadStrategy,
                                       LayerPlan, PlanValidationError, ShapeError)

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def dims(nv, nt, d=64, H=1, order=0):
    return AttentionDims(H, d, nv, nt, api.TEXT_FIRST if order else api.VISUAL_FIRST)


def test_masks_and_stats_bit_exact_against_reference_golden():
    for i in range(int(G["n_mask_cases"][0])):
        nv, nt, order, B, w = (int(x) for x in G[f"mask{i}_geom"])
        want = np.unpackbits(G[f"mask{i}_bits"])[: int(G[f"mask{i}_nbits"][0])]
        m = api.build_arrow_mask(ArrowSpec(dims(nv, nt, order=order), B, w))
        assert np.array_equal(m.active, want), (nv, nt, order, B, w)
        assert m.active_positions() == int(G[f"mask{i}_stats"][0])
        assert api.flops_count(m, 64) == int(G[f"mask{i}_stats"][1])
        assert api.sparsity_ratio(m) == float(G[f"mask{i}_sparsity"][0])


def test_reference_arrow_known_answers():
    m = api.build_arrow_mask(ArrowSpec(dims(512, 128), 128, 0))
    assert (m.n_query_blocks, m.n_key_blocks) == (5, 5)
    assert m.active.sum() == 13 and api.sparsity_ratio(m) == pytest.approx(0.48)
    assert all(m.is_active(4, j) and m.is_active(j, 4) for j in range(5)) and not m.is_active(0, 2)
    with pytest.raises(ShapeError):
        api.build_arrow_mask(ArrowSpec(dims(64, 8), 0, 0))
    with pytest.raises(ShapeError):
        api.build_arrow_mask(ArrowSpec(dims(64, 8), 8, -1))
    # ragged tails count true coverage (test_arrow.cpp:138-147)
    bm = BlockMask.all_active(5, 2)
    assert bm.n_query_blocks == 3 and bm.active_positions() == 25
    bm.set(2, 2, False)
    assert bm.active_positions() == 24
    bm.set(0, 2, False)
    assert bm.active_positions() == 22
    assert api.dense_flops(64, 8) == 4 * 8 * 64 * 64
    # monotone in w, dense at the max (test_arrow.cpp:149-152)
    prev = -1
    for w in range(10):
        f = api.flops_count(api.build_arrow_mask(ArrowSpec(dims(260, 30), 32, w)), 16)
        assert f >= prev
        prev = f
    assert prev == api.dense_flops(290, 16)


def test_plan_flops_against_reference_golden():
    for name in ("cfg1", "cfg1_b64", "flux68", "sd3_flux68"):
        H, d, nv, nt, order, B, f = (int(x) for x in G[f"plan_{name}"])
        kinds = G[f"plan_{name}_kinds"]
        wins = G[f"plan_{name}_windows"]
        plan = LayerPlan([HeadStrategy.Full() if k == 0 else HeadStrategy.Arrow(int(w)) if k == 1
                          else HeadStrategy.Cached() for k, w in zip(kinds, wins)])
        assert api.plan_flops(plan, AttentionDims(H, d, nv, nt), B) == f, name
    assert api.flux68_plan() == LayerPlan.parse("F A8 C A0 F A8 C A8 F A8 C A0 F A8 C A0 F A8 C A8 F A8 C A0")
    # dispatch tests (test_dispatch.cpp:133-162)
    dd = AttentionDims(2, 8, 56, 8)
    dense = api.dense_flops(64, 8)
    assert api.plan_flops(LayerPlan.all_full(2), dd, 8) == 2 * dense
    assert api.plan_flops(LayerPlan([HeadStrategy.Cached()] * 2), dd, 8) == 0
    assert api.plan_flops(LayerPlan([HeadStrategy.Full(), HeadStrategy.Cached()]), dd, 8) * 2 == 2 * dense
    with pytest.raises(ShapeError):
        api.plan_flops(LayerPlan([HeadStrategy.Full()]), dd, 8)


def test_plan_aggregate_and_validate():
    d = AttentionDims(4, 64, 1024, 77)
    p = CompressionPlan.all_full(d, 3, 2, 128)
    assert p.aggregate_sparsity() == 0.0
    p.layers[2 * 1 + 0] = LayerPlan.parse("F A0 A2 C")  # (t=1, l=0)
    ft = p.flops_total()
    assert ft == 5 * api.plan_flops(LayerPlan.all_full(4), d, 128) + api.plan_flops(p.at(1, 0), d, 128)
    assert p.flops_dense_total() == 6 * 4 * api.dense_flops(1101, 64)
    bad = CompressionPlan.all_full(d, 2, 1, 128)
    bad.layers[0] = LayerPlan.parse("F F F C")  # Cached at t = 0 (plan.cpp:46-48)
    with pytest.raises(PlanValidationError):
        bad.validate()
    bad.layers = bad.layers[:1]
    with pytest.raises(PlanValidationError):
        bad.validate()


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_plan_aggregate_matches_live_reference():
    import ctypes
    from oracle import c_double, c_int32, c_int64, ptr
    rng = np.random.default_rng(5)
    d = AttentionDims(6, 64, 900, 100)
    T, L = 4, 3
    plan = CompressionPlan.all_full(d, T, L, 64)
    for t in range(T):
        for l in range(L):
            toks = []
            for h in range(6):
                k = int(rng.integers(3 if t > 0 else 2))
                toks.append("F" if k == 0 else f"A{int(rng.integers(6))}" if k == 1 else "C")
            plan.layers[t * L + l] = LayerPlan.parse(" ".join(toks))
    kinds = np.array([api._KIND_CODE[s.kind] for lp in plan.layers for s in lp.strategies], np.int32)
    wins = np.array([s.window_blocks for lp in plan.layers for s in lp.strategies], np.int64)
    ft, fd, sp = c_int64(), c_int64(), c_double()
    oracle.ref_check(oracle.ref().ref_plan_aggregate(6, 64, 900, 100, 0, T, L, 64, ptr(kinds, c_int32),
                                                     ptr(wins, c_int64), ctypes.byref(ft), ctypes.byref(fd),
                                                     ctypes.byref(sp)))
    assert plan.flops_total() == ft.value
    assert plan.flops_dense_total() == fd.value
    assert plan.aggregate_sparsity() == sp.value


def kv_tile():
    return int(api.lib().dfa2c_kv_tile_keys())


def _expand(row_ptr, cols, n):
    """Token-pair coverage of a tile set: bool [n, n] of pairs inside listed tiles."""
    kt = kv_tile()
    cov = np.zeros((n, n), bool)
    part = np.zeros((n, n), bool)
    for i in range(len(row_ptr) - 1):
        for c in cols[row_ptr[i]:row_ptr[i + 1]]:
            t = int(c) & 0x7FFFFFFF
            cov[i * 128:(i + 1) * 128, t * kt:(t + 1) * kt] = True
            if int(c) >> 31:
                part[i * 128:(i + 1) * 128, t * kt:(t + 1) * kt] = True
    return cov, part


@pytest.mark.parametrize("nv,nt,order,B,w", [
    (1024, 77, 0, 128, 0), (1024, 77, 0, 64, 2), (300, 44, 1, 48, 1), (256, 44, 0, 16, 0), (4096, 333, 0, 128, 8),
    (200, 0, 0, 128, 0), (130, 5, 0, 7, 3), (1000, 300, 1, 200, 1)])
def test_tile_set_covers_exactly_the_active_token_pairs(nv, nt, order, B, w):
    d = dims(nv, nt, order=order)
    n = nv + nt
    m = oracle.arrow_mask(nv, nt, order, B, w)
    nb = (n + B - 1) // B
    blk = np.arange(n) // B
    active = m.reshape(nb, nb)[blk[:, None], blk[None, :]].astype(bool)  # token-level predicate
    row_ptr, cols = api.tile_set(d, B, HeadStrategy.Arrow(w))
    kt = kv_tile()
    cov, part = _expand(row_ptr, cols, n)
    assert not (active & ~cov).any(), "an active pair lies outside every scheduled tile"
    # every scheduled tile holds >= 1 active pair; non-partial tiles hold only active pairs
    for i in range(len(row_ptr) - 1):
        for c in cols[row_ptr[i]:row_ptr[i + 1]]:
            t = int(c) & 0x7FFFFFFF
            blk_act = active[i * 128:(i + 1) * 128, t * kt:(t + 1) * kt]
            assert blk_act.any()
            full_tile = blk_act.shape[1] == kt and blk_act.all()  # rows past n are never stored
            assert bool(int(c) >> 31) == (not full_tile)
        ts = [int(c) & 0x7FFFFFFF for c in cols[row_ptr[i]:row_ptr[i + 1]]]
        assert ts == sorted(ts)  # ascending key order (arrow.cpp:184-186)


def test_flux68_tile_counts():
    d = AttentionDims(24, 128, 16384, 512)
    total = 0
    for s in api.flux68_plan().strategies:
        if s.kind == "cached":
            continue
        rp, cols = api.tile_set(d, 128, s)
        total += len(cols)
        assert not any(int(c) >> 31 for c in cols)  # block-aligned: no element masking at FLUX 2K
    # 134,368 computed 128x128 tiles of 418,176 dense
    assert total * kv_tile() == 134368 * 128 and 24 * 132 * 132 == 418176


def _schedule(costs, m, refine):
    import ctypes

    from paper_2503_22796_b200 import _lib
    c = np.ascontiguousarray(costs, dtype=np.float64)
    cta = np.full(len(c), -1, dtype=np.int32)
    mx = ctypes.c_double()
    _lib.check(_lib.lib().dfa2c_debug_schedule(c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(c), m,
                                               int(refine), cta.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                               ctypes.byref(mx)))
    return cta, mx.value


def _sd3_arrow_costs(w, H=24):
    # the scheduler's cost model for an SD3 Arrow(w) layer (32 visual + 3 text
    # query tiles): pairs 2 x union + 1, the trailing text tile as HALVES
    out = []
    for _ in range(H):
        for p in range(16):
            lo, hi = max(0, 2 * p - w), min(31, 2 * p + 1 + w)
            out.append(2 * (hi - lo + 1 + 3) + 1)
        out += [2 * 35 + 1, 1.2 * 35 + 1]
    return out


def test_schedule_refinement_lowers_the_costliest_cta_and_keeps_every_item():
    # SD3 Arrow(8): LPT leaves the costliest CTA 17% above the mean; the
    # move / swap refinement brings it under 8% (late round 2)
    costs = _sd3_arrow_costs(8)
    mean = sum(costs) / 148
    cta0, lpt = _schedule(costs, 148, False)
    cta1, ref = _schedule(costs, 148, True)
    assert lpt / mean > 1.15 and ref / mean < 1.08 and ref <= lpt
    for cta in (cta0, cta1):
        assert cta.min() >= 0 and cta.max() < 148  # every item placed exactly once
        loads = np.bincount(cta, weights=costs, minlength=148)
        assert loads.sum() == pytest.approx(sum(costs))
    assert np.bincount(cta1, weights=costs, minlength=148).max() == pytest.approx(ref)
    # deterministic, and never worse than LPT on random cost mixes
    assert np.array_equal(_schedule(costs, 148, True)[0], cta1)
    rng = np.random.default_rng(5)
    for _ in range(20):
        c = rng.choice([3.0, 15.0, 43.0, 71.0, 265.0], size=int(rng.integers(1, 900)))
        m = int(rng.integers(1, 160))
        assert _schedule(c, m, True)[1] <= _schedule(c, m, False)[1] + 1e-9
        assert _schedule(c, m, True)[1] >= max(c.max(), c.sum() / min(m, len(c))) - 1e-9


def test_schedule_hook_rejects_bad_arguments():
    with pytest.raises(ShapeError):
        _schedule([1.0, -2.0], 4, True)
    with pytest.raises(ShapeError):
        _schedule([1.0], 0, True)
