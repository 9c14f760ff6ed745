"""Computed-TFLOPS of the fused kernel per plan kind at the FLUX 2K shape
(or SD3 with --sd3): where does efficiency go (item length, copies, commits)?"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

ap = argparse.ArgumentParser()
ap.add_argument("--sd3", action="store_true")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--out", default="")
a = ap.parse_args()
H, NV, NT, D, B = (24, 4096, 333, 64, 128) if a.sd3 else (24, 16384, 512, 128, 128)
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, torch.randn(N, D, device="cuda").to(torch.bfloat16), 0)
plans = {
    "all_F": " ".join(["F"] * H),
    "all_A16": " ".join(["A16"] * H),
    "all_A8": " ".join(["A8"] * H),
    "all_A2": " ".join(["A2"] * H),
    "all_A0": " ".join(["A0"] * H),
    "FLUX68": "F A8 C A0 F A8 C A8 F A8 C A0 F A8 C A0 F A8 C A8 F A8 C A0",
    "FLUX68_noC": "F A8 F A0 F A8 F A8 F A8 F A0 F A8 F A0 F A8 F A8 F A8 F A0",
    "all_C": " ".join(["C"] * H),
}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
rows = []
for name, p in plans.items():
    lp = api.LayerPlan.parse(p)
    fl = api.plan_flops(lp, dims, B)
    for use_cache in (True, False):
        if not use_cache and "C" in p.split():
            continue
        c = cache if use_cache else None
        for _ in range(5):
            api.multi_strategy_attention(q, k, v, lp, c, 0, 1, dims, B, out=out)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.steps):
            api.multi_strategy_attention(q, k, v, lp, c, 0, 1, dims, B, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        print(f"{name:11s} commit={int(use_cache)} {ms:8.4f} ms  computed {fl / ms / 1e9:7.1f} TF  "
              f"(plan {fl / 1e9:7.1f} GFLOP)")
        rows.append({"plan": name, "commit": use_cache, "ms": ms, "plan_gflop": fl / 1e9,
                     "computed_tflops": fl / ms / 1e9})
if a.out:
    import json

    json.dump({"shape": "SD3" if a.sd3 else "FLUX 2K", "rows": rows}, open(a.out, "w"), indent=1)
