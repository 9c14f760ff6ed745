"""Cost of a plan-cache miss: FLUX 2K layers where every call has a plan never
seen before (a calibrated schedule: one plan per (t, layer)) vs one plan
repeated. CUDA events around the whole sequence (host work included)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_22796_b200 import api

H, NV, NT, D, B = 24, 16384, 512, 128, 128
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
cache = api.HeadCache(1, H, N, D)
api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, 0, 0, dims, B, out=out)
rng = np.random.default_rng(0)
kinds = ["F", "A0", "A2", "A8", "A16", "C"]


def random_plan():
    return api.LayerPlan.parse(" ".join(rng.choice(kinds, size=H, p=[0.25, 0.15, 0.1, 0.2, 0.1, 0.2])))


warm = [random_plan() for _ in range(20)]  # first misses also create the staging ring
plans = [random_plan() for _ in range(60)]
same = [plans[0]] * 60
for name, seq in (("warm-up misses", warm), ("distinct plans", plans), ("one plan", same),
                  ("distinct plans (cached now)", plans)):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for lp in seq:
        api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)
    e1.record()
    torch.cuda.synchronize()
    fl = sum(api.plan_flops(lp, dims, B) for lp in seq)
    ms = e0.elapsed_time(e1)
    import time as _t
    print(f"{name:28s} {ms / len(seq):.3f} ms/layer  computed {fl / ms / 1e9:.0f} TF")
