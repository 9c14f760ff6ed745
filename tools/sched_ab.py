"""Same FLUX68 layer through dfa2c_mha_forward (plain LPT list) and through
dfa2c_mha_forward_sharded with world = 1 (whole-layer-load key chunking),
alternated in one process so clocks are comparable."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

H, NV, NT, D, B = 24, 16384, 512, 128, 128
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = (torch.randn(1, H, N, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, torch.randn(N, D, device="cuda", generator=g).to(torch.bfloat16), 0)
plans = {"FLUX68": "F A8 C A0 F A8 C A8 F A8 C A0 F A8 C A0 F A8 C A8 F A8 C A0", "all_F": " ".join(["F"] * H),
         "all_A8": " ".join(["A8"] * H)}
out = torch.empty_like(q)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for name, p in plans.items():
    lp = api.LayerPlan.parse(p)
    a, b = [], []
    for _ in range(5):
        a.append(t(lambda: api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)))
        b.append(t(lambda: api.multi_strategy_attention_sharded(q, k, v, lp, cache, 0, 1, dims, B, 0, 1, out=out)))
    print(f"{name:7s} plain {statistics.median(a):.4f} ms  sharded(W=1) {statistics.median(b):.4f} ms", flush=True)
