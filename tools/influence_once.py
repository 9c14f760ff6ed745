import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2503_22796_b200 import api
H, nv, nt, d, B = 24, 16384, 512, 128, 128
n = nv + nt
dims = api.AttentionDims(H, d, nv, nt)
q, k, v = (torch.randn(H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
cache = api.HeadCache(1, H, n, d)
api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, 0, 0, dims, B)
methods = api.make_candidates([0, 2, 8, 16, 32], include_cached=True)
for _ in range(2):
    api.influence_for_layer(q, k, v, methods, cache, 0, 1, dims, B, keep_outputs=True)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
for _ in range(5):
    api.influence_for_layer(q, k, v, methods, cache, 0, 1, dims, B, keep_outputs=True)
torch.cuda.synchronize()
print(f"influence: {(time.perf_counter()-t0)/5*1e3:.2f} ms")
