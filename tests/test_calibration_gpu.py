"""The GPU-resident calibration driver (api.calibrate_model, contract of
/root/reference/proj/src/calibrate.cpp:255-382) on a drifting multi-layer
stream: the properties the reference's test_calibrate.cpp / test_workload.cpp
assert, at d=128 and a ragged text block, plus the replay of the
calibration stream by run_pipeline: bitwise with the per-candidate
influence passes (dfa2c_set_influence_fused(0)), within the bf16 output
tolerance with the fused band-snapshot pass (the default at block 128)."""
import math

import numpy as np
import pytest

from paper_2503_22796_b200 import api

pytestmark = pytest.mark.gpu

H, NV, NT, D, B, L, T = 6, 1024, 77, 128, 128, 2, 3


def streams():
    import torch

    g = torch.Generator(device="cuda").manual_seed(5)
    base = [[torch.randn(H, NV + NT, D, device="cuda", generator=g) for _ in range(3)] for _ in range(L)]
    cache = {}

    def get(t, l, which):
        key = (t, l, which)
        if key not in cache:  # random walk over timesteps (head 0 frozen: full temporal redundancy)
            x = base[l][which].clone()
            for s in range(1, t + 1):
                gs = torch.Generator(device="cuda").manual_seed(1000 * s + 10 * l + which)
                step = 0.15 * torch.randn(x.shape, device="cuda", generator=gs)
                step[0] = 0
                x = x + step
            cache[key] = x.to(torch.bfloat16)
        return cache[key]

    return (lambda t, l: get(t, l, 0)), (lambda t, l: get(t, l, 1)), (lambda t, l: get(t, l, 2))


@pytest.fixture(params=[False, True], ids=["exact", "fused"])
def fused(request):
    before = api.influence_fused_enabled()
    api.set_influence_fused(request.param)
    yield request.param
    api.set_influence_fused(before)


def same_stream(a, b, fused):
    """Bitwise for the per-candidate passes; the fused pass folds key tiles
    in window-band order, so its spliced outputs differ from the executed
    plan's by bf16 rounding only (tests/test_gpu_parity.py tolerance)."""
    import torch

    if not fused:
        return torch.equal(a, b)
    x, y = a.double(), b.double()
    return bool((x - y).abs().max() <= 1e-2 * y.abs().max())


def calibrate(delta, keep=True):
    q, k, v = streams()
    cfg = api.CalibrationConfig(api.make_candidates([0, 2], include_cached=True), delta, 1.5)
    dims = api.AttentionDims(H, D, NV, NT)
    return api.calibrate_model(q, k, v, dims, T, L, B, cfg, keep_outputs=keep), (q, k, v), cfg, dims


def test_zero_budget_is_all_full_and_replays_the_baseline(fused):
    import torch

    r, (q, k, v), cfg, dims = calibrate(0.0)
    assert all(s_.kind == "full" for lp in r.plan.layers for s_ in lp.strategies)
    assert r.stats.attention_evals == T * L * (1 + len(cfg.methods))
    base = api.run_pipeline(q, k, v, api.CompressionPlan.all_full(dims, T, L, B))
    torch.cuda.synchronize()
    assert all(same_stream(a, b, fused) for a, b in zip(r.outputs, base.outputs))


def test_calibrated_plan_constraints_and_csv():
    r, _, cfg, _ = calibrate(0.4, keep=False)
    assert api.audit_plan_constraints(r.plan, r.influences) == 0
    assert all(s_ <= 0.4 for s_ in r.budget_spent)
    # temporal redundancy is exploited: frozen head 0 is Cached after t = 0
    assert any(r.plan.at(t, l).strategies[0].kind == "cached" for t in range(1, T) for l in range(L))
    assert not any(s_.kind == "cached" for l in range(L) for s_ in r.plan.at(0, l).strategies)
    back = api.InfluenceTable.parse_csv(r.influences.to_csv(), T, L, H, r.influences.method_ids)
    assert np.array_equal(np.isnan(back.values), np.isnan(r.influences.values))
    assert np.array_equal(np.nan_to_num(back.values), np.nan_to_num(r.influences.values))
    # the cached candidate is never measured at t = 0
    assert not any(r.influences.measured(0, l, h, len(cfg.methods) - 1) for l in range(L) for h in range(H))


def test_executing_the_plan_reproduces_the_calibration_stream(fused):
    import torch

    r, (q, k, v), _, _ = calibrate(0.4)
    run = api.run_pipeline(q, k, v, r.plan)
    torch.cuda.synchronize()
    assert run.sparsity == pytest.approx(r.plan.aggregate_sparsity(), abs=0)
    for i, (a, b) in enumerate(zip(r.outputs, run.outputs)):
        assert same_stream(a, b, fused), f"layer slot {i}"


def test_remeasuring_under_the_plan_reproduces_the_influences(fused):
    r, (q, k, v), cfg, dims = calibrate(0.4, keep=False)
    cache = api.HeadCache(L, H, NV + NT, D)
    M = len(cfg.methods)
    for t in range(T):
        for l in range(L):
            li = api.influence_for_layer(q(t, l), k(t, l), v(t, l), cfg.methods, cache, l, t, dims, B)
            for h in range(H):
                for m in range(M):
                    val = li.influence[h * M + m]
                    if math.isfinite(val):
                        assert val == r.influences.get(t, l, h, m)
                    else:
                        assert not r.influences.measured(t, l, h, m)
            for h, s_ in enumerate(r.plan.at(t, l).strategies):
                if s_.kind == "full":
                    cache.store(l, h, li.original[h], t)
                elif s_.kind == "arrow":
                    m = [c.strategy for c in cfg.methods].index(s_)
                    cache.store(l, h, li.method_outputs[m][h], t)


def test_single_layer_schedule_orders_splice_before_next_measurement():
    """L = 1: every (t, 0) measurement reads the slot the previous timestep's
    splice wrote, so the pipelined driver must finish that splice first.
    Re-measuring under the plan (splicing as the driver does) reproduces
    every influence bitwise."""
    import torch

    q, k, v = streams()
    cfg = api.CalibrationConfig(api.make_candidates([0, 2], include_cached=True), 0.4, 1.5)
    dims = api.AttentionDims(H, D, NV, NT)
    r = api.calibrate_model(q, k, v, dims, T, 1, B, cfg)
    assert api.audit_plan_constraints(r.plan, r.influences) == 0
    cache = api.HeadCache(1, H, NV + NT, D)
    M = len(cfg.methods)
    for t in range(T):
        li = api.influence_for_layer(q(t, 0), k(t, 0), v(t, 0), cfg.methods, cache, 0, t, dims, B)
        for h in range(H):
            for m in range(M):
                val = li.influence[h * M + m]
                if math.isfinite(val):
                    assert val == r.influences.get(t, 0, h, m)
        for h, s_ in enumerate(r.plan.at(t, 0).strategies):
            if s_.kind == "full":
                cache.store(0, h, li.original[h], t)
            elif s_.kind == "arrow":
                cache.store(0, h, li.method_outputs[[c.strategy for c in cfg.methods].index(s_)][h], t)
    torch.cuda.synchronize()
