"""influence_for_layer at FLUX 2K (24 heads, 16384+512, d=128, B=128),
candidates Arrow {0, 2, 8, 16, 32} + Cached: the fused band-snapshot pass
against the per-candidate passes (wall time per layer, CUDA-synchronised)."""
import sys
import time

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
res = {}
for fused in (True, False):
    api.set_influence_fused(fused)
    for _ in range(2):
        api.influence_for_layer(q, k, v, methods, cache, 0, 1, dims, B, keep_outputs=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        li = api.influence_for_layer(q, k, v, methods, cache, 0, 1, dims, B, keep_outputs=True)
    torch.cuda.synchronize()
    res[fused] = li
    print(f"influence ({'fused' if fused else 'per-candidate'}): {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms")
api.set_influence_fused(True)
import numpy as np

a, b = res[True].influence.reshape(H, -1), res[False].influence.reshape(H, -1)
fin = np.isfinite(b) & (b > 0)
print("max rel influence diff (fused vs per-candidate, nonzero entries):",
      float(np.max(np.abs(a[fin] - b[fin]) / b[fin])))
