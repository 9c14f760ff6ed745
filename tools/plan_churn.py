import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch, time
from paper_2503_22796_b200 import api
H, NV, NT, D, B = 24, 4096, 333, 64, 128
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
cache = api.HeadCache(1, H, N, D)
api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, 0, 0, dims, B, out=out)
rng = np.random.default_rng(1)
kinds = ["F", "A0", "A2", "A8", "C"]
side = torch.cuda.Stream()
free0 = torch.cuda.mem_get_info()[0]
t0 = time.time()
for i in range(3000):
    lp = api.LayerPlan.parse(" ".join(rng.choice(kinds, size=H)))
    s = side if i % 3 == 0 else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, B, out=out, stream=s)
    if i % 500 == 499:
        torch.cuda.synchronize()
        print(i + 1, "calls", f"{time.time() - t0:.1f}s", "free GB", round(torch.cuda.mem_get_info()[0] / 1e9, 2), flush=True)
torch.cuda.synchronize()
print("ok; free GB before/after", round(free0 / 1e9, 2), round(torch.cuda.mem_get_info()[0] / 1e9, 2))
