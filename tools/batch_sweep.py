"""FLUX68 layer throughput vs samples per call on one GPU (batch 1, 2, 4, 8):
one fused launch over batch x 24 heads; CUDA events, best of 3 (alternating)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

H, NV, NT, D, B = 24, 16384, 512, 128, 128
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
lp = api.flux68_plan()
res = {}
bufs = {}
for bt in (1, 2, 4, 8):
    q, k, v = (torch.randn(bt, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
    cache = api.HeadCache(1, H, N, D, batch=bt)
    api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, 0, 0, dims, B)
    bufs[bt] = (q, k, v, torch.empty_like(q), cache)
fl = api.plan_flops(lp, dims, B)
for _ in range(3):
    for bt, (q, k, v, o, cache) in bufs.items():
        for _ in range(3):
            api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=o)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=o)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        if bt not in res or ms < res[bt]["ms"]:
            res[bt] = {"ms": ms, "ms_per_sample": ms / bt, "computed_tflops": bt * fl / ms / 1e9}
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/batch_sweep.json", "w"), indent=1)
