import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2503_22796_b200 import api
H, nv, nt, d, B = 24, 16384, 512, 128, 128
n = nv + nt
dims = api.AttentionDims(H, d, nv, nt)
q, k, v = (torch.randn(H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
tot = 0
for plan in ["F", "A0", "A2", "A8", "A16", "A32"]:
    lp = api.LayerPlan.parse(" ".join([plan] * H))
    for _ in range(3):
        api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    fl = api.plan_flops(lp, dims, B)
    tot += ms
    print(f"{plan:4s} {ms*1e3:7.0f} us  {fl/ms/1e9:6.0f} TFLOP/s")
print(f"sum {tot:.3f} ms")
