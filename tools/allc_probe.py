import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2503_22796_b200 import api
shape = sys.argv[1] if len(sys.argv) > 1 else "flux"
H, NV, NT, D = (24, 16384, 512, 128) if shape == "flux" else (24, 4096, 333, 64)
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, torch.randn(N, D, device="cuda").to(torch.bfloat16), 0)
lp = api.LayerPlan.parse(" ".join(["C"] * H))
for _ in range(5):
    api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, 128, out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, 128, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"{shape} all-C: host {1e6*(t1-t0)/50:.1f} us/call, wall incl. drain {1e6*(t2-t0)/50:.1f} us/call")
