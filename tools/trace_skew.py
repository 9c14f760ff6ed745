"""Softmax-warp skew within a lane (a -DDFA2_TRACE=5 build): P is complete
for the MMA warp only when the slowest of the lane's 4 softmax warps (one
per SMSP) arrives; per tile, each warp's end relative to the earliest.

    DFA2_LIB=build/lt5.so python tools/trace_skew.py [plan] [--sd3]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_22796_b200 import _lib, api

plan = next((a for a in sys.argv[1:] if not a.startswith("--")), "F")
sd3 = "--sd3" in sys.argv
H, NV, NT, D = (24, 4096, 333, 64) if sd3 else (24, 16384, 512, 128)
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
lp = api.LayerPlan.parse(" ".join([plan] * H))
trace = torch.zeros(2 * 4096 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, 128, out=out)
_lib.lib().dfa2c_debug_set_trace(ctypes.c_void_p(trace.data_ptr()))
api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, 128, out=out)
torch.cuda.synchronize()
_lib.lib().dfa2c_debug_set_trace(None)
t = trace.view(2, 4096, 8).cpu().numpy().astype(np.float64)
for L in range(2):
    ends = t[L, :, 4:8]
    ok = (ends > 0).all(axis=1)
    e = ends[ok][5:-5]
    rel = e - e.min(axis=1, keepdims=True)
    sready = t[L, ok, 1][5:-5]
    soft = e.max(axis=1) - sready
    print(f"lane {'AB'[L]}: tiles {len(e)}  softmax (S ready -> last warp) median {np.median(soft):.0f} clk; "
          f"per-warp end after the earliest, median by SMSP 0..3: "
          + " ".join(f"{np.median(rel[:, w]):.0f}" for w in range(4))
          + f"; skew (last - first) median {np.median(rel.max(axis=1)):.0f} p90 {np.percentile(rel.max(axis=1), 90):.0f}")
