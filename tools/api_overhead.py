"""Host cost of one Python API call (multi_strategy_attention) broken into
its steps, at a small layer where the host can bound the launch rate.

    python tools/api_overhead.py
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import _lib, api

H, NV, NT, D = 24, 4096, 333, 64
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, torch.randn(N, D, device="cuda").to(torch.bfloat16), 0)
lp = api.LayerPlan.parse(" ".join(["C"] * H))
R = 2000


def per_call(fn):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(R):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return 1e6 * (t1 - t0) / R


L = _lib.lib()
kinds, wins = lp.arrays()
dc = dims.c()
args = (ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()), 1,
        ctypes.byref(dc), 128, kinds, wins, cache.handle, 0, 1, ctypes.c_void_p(out.data_ptr()), None)
rows = {
    "api.multi_strategy_attention": lambda: api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, 128, out=out),
    "raw dfa2c_mha_forward (prebuilt ctypes args)": lambda: L.dfa2c_mha_forward(*args),
    "plan.arrays()": lambda: lp.arrays(),
    "dims.c()": lambda: dims.c(),
    "torch.cuda.current_stream().cuda_stream": lambda: torch.cuda.current_stream().cuda_stream,
    "api._stream_ptr()": lambda: api._stream_ptr(),
    "api._plan_kinds(plan, None)": lambda: api._plan_kinds(lp, None),
    "api._device_out(out, q, shape)": lambda: api._device_out(out, q, q.shape),
    "api._as_bf16_cuda(q) x3": lambda: (api._as_bf16_cuda(q, "q"), api._as_bf16_cuda(k, "k"), api._as_bf16_cuda(v, "v")),
    "x.contiguous() x3": lambda: (q.contiguous(), k.contiguous(), v.contiguous()),
}
for name, fn in rows.items():
    print(f"{name:48s} {per_call(fn):7.2f} us/call", flush=True)
