"""Host-side cost of one fused-layer call vs its GPU time (FLUX68 shape, or
the cfg1 layer with --cfg1)."""
import time
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

H, NV, NT, D, B = (4, 1024, 77, 64, 128) if "--cfg1" in sys.argv else (24, 16384, 512, 128, 128)
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, torch.randn(N, D, device="cuda").to(torch.bfloat16), 0)
lp = api.LayerPlan.parse("F A0 A2 C") if "--cfg1" in sys.argv else api.flux68_plan()
for _ in range(5):
    api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6 * (t1 - t0) / n:.1f} us/call; wall incl. drain {1e3 * (t2 - t0) / n:.3f} ms/call")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)
e1.record()
torch.cuda.synchronize()
print(f"events back-to-back {e0.elapsed_time(e1) / n:.4f} ms/call")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(20):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"cuda graph (10 calls/graph) {e0.elapsed_time(e1) / 200:.4f} ms/call")
