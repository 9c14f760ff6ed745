"""Per-CTA start / end of one fused launch (-DDFA2_TRACE=4 build): the
schedule's tail (how long the last CTAs run past the average), per plan.

    DFA2_LIB=build/lt4.so python tools/cta_tail.py [plan ...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_22796_b200 import _lib, api

H, NV, NT, D, B = 24, 16384, 512, 128, 128
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, torch.randn(N, D, device="cuda").to(torch.bfloat16), 0)
plans = sys.argv[1:] or ["FLUX68", "F", "A8", "A0"]
for name in plans:
    p = api.flux68_plan() if name == "FLUX68" else api.LayerPlan.parse(" ".join([name] * H))
    trace = torch.zeros(148 * 4, dtype=torch.int64, device="cuda")
    for _ in range(3):
        api.multi_strategy_attention(q, k, v, p, cache, 0, 1, dims, B, out=out)
    torch.cuda.synchronize()
    _lib.lib().dfa2c_debug_set_trace(ctypes.c_void_p(trace.data_ptr()))
    api.multi_strategy_attention(q, k, v, p, cache, 0, 1, dims, B, out=out)
    torch.cuda.synchronize()
    _lib.lib().dfa2c_debug_set_trace(None)
    t = trace.view(148, 4).cpu().numpy().astype(np.float64)
    t = t[t[:, 0] > 0]  # launched CTAs
    t0 = t[:, 0].min()
    start, la, lb, end = (t[:, i] - t0 for i in range(4))
    print(f"{name:7s} launch span {end.max() / 1e3:.1f} us | CTA start max {start.max() / 1e3:.1f} us | "
          f"CTA end: mean {end.mean() / 1e3:.1f} p10 {np.percentile(end, 10) / 1e3:.1f} "
          f"p50 {np.median(end) / 1e3:.1f} p90 {np.percentile(end, 90) / 1e3:.1f} max {end.max() / 1e3:.1f} us | "
          f"tail (max - mean) {(end.max() - end.mean()) / end.max() * 100:.1f}%", flush=True)
