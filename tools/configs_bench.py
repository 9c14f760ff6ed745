"""BASELINE.json configs 1-5 on one B200 (config 3, the headline, is bench.py;
here it is repeated in both token orders).

    python tools/configs_bench.py [--out gpurun_out/configs.json]

  cfg1  1024+77 tok, H=4, d=64, plan [F, A0, A2, C] at t=1 (B=128 and 64)
  cfg2  SD3 4096+333, H=24, d=64: all-Arrow(w) window sweep + all Full
  cfg4  FLUX 2K 28-step x 57-layer schedule with one shared device cache
        (5 F, 9 A8, 4 A0, 6 C per layer for t >= 1, rotated per (t, l);
        all Full at t = 0), one sample per GPU (batch 8 over 8 GPUs = 8x this),
        every (t, l) slot a drifting input from the device generator
  cfg5  FLUX-shaped progressive calibration (calibrate_model) over 57 layers
        x 2 timesteps, candidates Arrow {0, 2, 8, 16, 32} + Cached, plus the
        RSE kernel alone
All timings: CUDA events, warm-up first; inputs resident in HBM.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/configs.json")
ap.add_argument("--only", default="1,2,3,4,5")
args = ap.parse_args()
only = set(args.only.split(","))
res = {}
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def randn(seed, *shape):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(*shape, device="cuda", generator=g).to(torch.bfloat16)


def time_calls(fn, steps=20, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


if "1" in only:
    out = {}
    for B in (128, 64):
        H, nv, nt, d = 4, 1024, 77, 64
        n = nv + nt
        dims = api.AttentionDims(H, d, nv, nt)
        q, k, v = (randn(s, H, n, d) for s in (1, 2, 3))
        cache = api.HeadCache(1, H, n, d)
        api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, 0, 0, dims, B)
        lp = api.LayerPlan.parse("F A0 A2 C")
        o = torch.empty_like(q)
        ms = time_calls(lambda: api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=o), 50)
        # the layer is one pair's 9-tile chain long: split-KV (opt-in) spreads it
        api.set_split_kv(True)
        ms_split = time_calls(lambda: api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=o), 50)
        api.set_split_kv(False)
        fl = api.plan_flops(lp, dims, B)
        out[f"B{B}"] = {"ms": ms, "ms_split_kv": ms_split, "plan_gflop": fl / 1e9, "computed_tflops": fl / ms / 1e9,
                        "reduction": 1 - fl / (H * api.dense_flops(n, d))}
    res["cfg1"] = out
    print("cfg1", json.dumps(out))

if "2" in only:
    H, nv, nt, d, B = 24, 4096, 333, 64, 128
    n = nv + nt
    dims = api.AttentionDims(H, d, nv, nt)
    q, k, v = (randn(s, H, n, d) for s in (1, 2, 3))
    o = torch.empty_like(q)
    dense = H * api.dense_flops(n, d)
    full_ms = time_calls(lambda: api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), None, 0, 0, dims,
                                                              B, out=o))
    rows = [{"plan": "all Full", "ms": full_ms, "sparsity": 0.0, "computed_tflops": dense / full_ms / 1e9,
             "effective_tflops": dense / full_ms / 1e9, "speedup_vs_full": 1.0}]
    for w in (0, 1, 2, 4, 8, 16, 31):
        lp = api.LayerPlan([api.HeadStrategy.Arrow(w)] * H)
        fl = api.plan_flops(lp, dims, B)
        ms = time_calls(lambda: api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B, out=o))
        rows.append({"plan": f"all Arrow({w})", "ms": ms, "sparsity": 1 - fl / dense,
                     "computed_tflops": fl / ms / 1e9, "effective_tflops": dense / ms / 1e9,
                     "speedup_vs_full": full_ms / ms, "ideal_speedup": dense / fl})
    res["cfg2_sd3_window_sweep"] = rows
    for r in rows:
        print("cfg2", json.dumps(r))

if "3" in only:
    # config 3 in both token orders (bench.py measures visual-first; FLUX
    # concatenates text first): FLUX68 and all-Full, layer time per order
    H, nv, nt, d, B = 24, 16384, 512, 128, 128
    n = nv + nt
    q, k, v = (randn(s, 1, H, n, d) for s in (11, 12, 13))
    out3 = {}
    orders = ((api.VISUAL_FIRST, "visual_first"), (api.TEXT_FIRST, "text_first"))
    caches = {}
    for order, name in orders:
        dims = api.AttentionDims(H, d, nv, nt, order)
        caches[name] = api.HeadCache(1, H, n, d)
        api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), caches[name], 0, 0, dims, B)
        out3[name] = {}
    # orders alternate over 3 rounds (the clock drifts as the GPU heats); best of 3
    for _ in range(3):
        for pname, lp in (("FLUX68", api.flux68_plan()), ("all Full", api.LayerPlan.all_full(H))):
            for order, name in orders:
                dims = api.AttentionDims(H, d, nv, nt, order)
                ms = time_calls(lambda: api.multi_strategy_attention(q, k, v, lp, caches[name], 0, 1, dims, B))
                best = out3[name].get(pname)
                if best is None or ms < best["ms"]:
                    out3[name][pname] = {"ms": ms, "computed_tflops": api.plan_flops(lp, dims, B) / ms / 1e9}
    res["cfg3_token_orders"] = out3
    print("cfg3", json.dumps(out3))
    del q, k, v

if "4" in only:
    T, L, H, nv, nt, d, B = 28, 57, 24, 16384, 512, 128, 128
    n = nv + nt
    dims = api.AttentionDims(H, d, nv, nt)
    base = api.LayerPlan.parse(" ".join(["F"] * 5 + ["A8"] * 9 + ["A0"] * 4 + ["C"] * 6)).strategies
    plan = api.CompressionPlan.all_full(dims, T, L, B)
    for t in range(1, T):
        for l in range(L):
            r = (7 * t + 3 * l) % H
            plan.layers[t * L + l] = api.LayerPlan(base[r:] + base[:r])
    agg = plan.aggregate_sparsity()
    # the per-(t, l) activations are the reference's drifting stream model
    # produced on the device (dfa2c_workload_*); each slot is generated into
    # the input buffers right before its layer, and only the layer is timed
    wl = api.DeviceWorkload(dims, L, B, seed=2503)
    q, k, v = (torch.empty(H, n, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    cache = api.HeadCache(L, H, n, d)
    evs = [(ev(), ev()) for _ in range(T * L)]

    def run_schedule(p):
        for t in range(T):
            for l in range(L):
                wl.slot(t, l, out=(q, k, v))
                e0, e1 = evs[t * L + l]
                e0.record()
                api.multi_strategy_attention(q, k, v, p.at(t, l), cache, l, t, dims, B, out=o)
                e1.record()
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs)

    run_schedule(plan)  # warm-up (also fills every slot)
    ms = run_schedule(plan)
    full_ms = run_schedule(api.CompressionPlan.all_full(dims, T, L, B))
    # a calibrated schedule has its own plan in every slot: the same head mix,
    # shuffled per (t, l) (1,539 distinct plans) - the first pass builds every
    # work list (plan-cache misses), later passes (images) reuse them
    import numpy as np
    rng = np.random.default_rng(4)
    distinct = api.CompressionPlan.all_full(dims, T, L, B)
    for t in range(1, T):
        for l in range(L):
            distinct.layers[t * L + l] = api.LayerPlan([base[i] for i in rng.permutation(H)])
    first_ms = run_schedule(distinct)
    steady_ms = run_schedule(distinct)
    out = {"T": T, "L": L, "aggregate_sparsity": agg, "schedule_ms": ms, "per_layer_ms": ms / (T * L),
           "distinct_plans_first_pass_ms": first_ms, "distinct_plans_steady_ms": steady_ms,
           "all_full_schedule_ms": full_ms, "speedup_vs_full": full_ms / ms,
           "effective_tflops": plan.flops_dense_total() / ms / 1e9,
           "computed_tflops": plan.flops_total() / ms / 1e9, "cache_gb": cache.nbytes() / 1e9,
           "inputs": "device generator: the reference's drifting stream model per (t, layer) slot "
                     "(DeviceWorkload, seed 2503); layer time only (CUDA events per layer, summed)",
           "note": "one sample per GPU; batch 8 on 8 GPUs shards samples (no inter-GPU traffic)"}
    res["cfg4_flux_schedule"] = out
    print("cfg4", json.dumps(out))
    del q, k, v, cache, wl

if "5" in only:
    # the progressive calibration driver at FLUX 2K scale: every layer of a
    # 57-layer model at t = 0 (Cached ineligible) and t = 1 (Cached measured
    # against the t = 0 commits), candidates Arrow {0, 2, 8, 16, 32} + Cached;
    # per layer one fused launch (original + 5 Arrow candidates), 6 RSE launches, the exact solve and the
    # device-side splice into the cache
    L, H, nv, nt, d, B, T = 57, 24, 16384, 512, 128, 128, 2
    n = nv + nt
    dims = api.AttentionDims(H, d, nv, nt)
    # inputs: the reference's drifting stream model on the device (per-layer
    # locality and drift profiles, so the Arrow / Cached choices differ by
    # layer and timestep); one slot at a time, memoised for the three streams
    # every (t, layer) slot generated up front (114 x 311 MB = 35 GB of HBM),
    # so the timed sweep is the calibration alone
    wl = api.DeviceWorkload(dims, L, B, seed=2503)
    memo = {(t, l): wl.slot(t, l) for t in range(T) for l in range(L)}
    torch.cuda.synchronize()

    def slot(t, l, i):
        return memo[(t, l)][i]

    cfg = api.CalibrationConfig(api.make_candidates([0, 2, 8, 16, 32], include_cached=True), 0.4, 1.5)
    # the per-candidate passes first (1 + 5 attention launches per layer),
    # then the default fused band-snapshot pass (1 launch per layer)
    api.set_influence_fused(False)
    warm = api.calibrate_model(lambda t, l: slot(t, l, 0), lambda t, l: slot(t, l, 1), lambda t, l: slot(t, l, 2), dims, 2, 1, B, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = api.calibrate_model(lambda t, l: slot(t, l, 0), lambda t, l: slot(t, l, 1), lambda t, l: slot(t, l, 2), dims, T, L, B, cfg)
    torch.cuda.synchronize()
    per_candidate_s = time.perf_counter() - t0
    per_candidate_sparsity = r.plan.aggregate_sparsity()
    api.set_influence_fused(True)
    warm = api.calibrate_model(lambda t, l: slot(t, l, 0), lambda t, l: slot(t, l, 1), lambda t, l: slot(t, l, 2), dims, 2, 1, B, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = api.calibrate_model(lambda t, l: slot(t, l, 0), lambda t, l: slot(t, l, 1), lambda t, l: slot(t, l, 2), dims, T, L, B, cfg)
    torch.cuda.synchronize()
    sweep_s = time.perf_counter() - t0
    kinds = {}
    for lp in r.plan.layers[L:]:
        for s_ in lp.strategies:
            kinds[api.method_id(s_)] = kinds.get(api.method_id(s_), 0) + 1
    # the RSE kernel alone: 24 heads x [N, d] bf16, 2 operands
    a, b = randn(7, H, n, d), randn(8, H, n, d)
    dev = torch.empty(H, device="cuda", dtype=torch.float64)
    ms = time_calls(lambda: api.rse_per_head_async(a, b, dev), 20)
    bytes_ = 2 * a.numel() * 2
    out = {"layers": L, "timesteps": T, "candidates": [m.id for m in cfg.methods], "calibration_s": sweep_s,
           "per_layer_ms": 1e3 * sweep_s / (T * L), "attention_evals": r.stats.attention_evals,
           "influence_pass": "fused (original + 5 arrow candidates in one launch)",
           "per_candidate_calibration_s": per_candidate_s,
           "per_candidate_per_layer_ms": 1e3 * per_candidate_s / (T * L),
           "per_candidate_aggregate_sparsity": per_candidate_sparsity,
           "aggregate_sparsity": r.plan.aggregate_sparsity(), "t1_choices": kinds,
           "audit_violations": api.audit_plan_constraints(r.plan, r.influences),
           "inputs": "device generator (DeviceWorkload, seed 2503): the reference's drifting stream model",
           "rse_ms": ms, "rse_bytes": bytes_, "rse_gbs": bytes_ / ms / 1e6}
    res["cfg5_calibration"] = out
    print("cfg5", json.dumps(out))

os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
with open(args.out, "w") as f:
    json.dump(res, f, indent=1)
