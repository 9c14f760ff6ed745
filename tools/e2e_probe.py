"""bench.py's e2e leg alone: the FLUX68 layer through the host-buffer entry
(pinned bf16 q/k/v in, pinned out), CUDA events over `--steps` calls.

    [DFA2_HOST_STREAMS=1] python tools/e2e_probe.py [--steps 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--plan", default="FLUX68")
a = ap.parse_args()
H, NV, NT, D = 24, 16384, 512, 128
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
g = torch.Generator().manual_seed(1)
q, k, v = (torch.randn(1, H, N, D, generator=g).to(torch.bfloat16).pin_memory() for _ in range(3))
out = torch.empty(1, H, N, D, dtype=torch.bfloat16).pin_memory()
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, torch.randn(N, D, generator=g).to(torch.bfloat16).cuda(), 0)
lp = api.flux68_plan() if a.plan == "FLUX68" else api.LayerPlan.parse(a.plan)
for _ in range(3):
    api.multi_strategy_attention_host(q, k, v, lp, cache, 0, 1, dims, 128, out=out)
torch.cuda.synchronize()
ref = out.clone()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    api.multi_strategy_attention_host(q, k, v, lp, cache, 0, 1, dims, 128, out=out)
e1.record()
torch.cuda.synchronize()
print(f"{a.plan[:24]:24s} host streams {'1' if os.environ.get('DFA2_HOST_STREAMS') == '1' else '2'}: "
      f"{e0.elapsed_time(e1) / a.steps:.3f} ms per layer; same output: {torch.equal(out, ref)}")
