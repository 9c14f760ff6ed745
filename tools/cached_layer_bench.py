"""A heavily cached FLUX 2K layer (20 Cached + 4 Arrow(0) heads), the
latency-bound case of late timesteps: fused-launch time (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

H, NV, NT, D, B = 24, 16384, 512, 128, 128
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, torch.randn(N, D, device="cuda").to(torch.bfloat16), 0)
lp = api.LayerPlan.parse(" ".join(["C"] * 5 + ["A0"] + ["C"] * 5 + ["A0"] + ["C"] * 5 + ["A0"] + ["C"] * 5 + ["A0"]))
for _ in range(5):
    api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30):
    api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)
e1.record()
torch.cuda.synchronize()
t_off = e0.elapsed_time(e1) / 30 * 1e3
api.set_split_kv(True)
for _ in range(5):
    api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)
torch.cuda.synchronize()
e0.record()
for _ in range(30):
    api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)
e1.record()
torch.cuda.synchronize()
print(f"cached20+A0x4 {t_off:.0f} us (split-KV on: {e0.elapsed_time(e1) / 30 * 1e3:.0f} us)")
