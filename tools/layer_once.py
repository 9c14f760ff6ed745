"""Runs one joint-attention layer a few times (for ncu captures).
    python tools/layer_once.py sd3|flux "<plan>" [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

shape = sys.argv[1]
H, NV, NT, D = (24, 4096, 333, 64) if shape == "sd3" else (24, 16384, 512, 128)
N = NV + NT
plan = api.LayerPlan.parse(sys.argv[2] if len(sys.argv[2].split()) > 1 else " ".join([sys.argv[2]] * H))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
cache = api.HeadCache(1, H, N, D)
api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, 0, 0, dims, 128)
for _ in range(reps):
    api.multi_strategy_attention(q, k, v, plan, cache, 0, 1, dims, 128)
torch.cuda.synchronize()
