"""One 4096+512-token d=64 head (the reference's run_bench / acceptance
criterion 7 workload): device time per call (CUDA events over back-to-back
calls) vs host time per call, dense vs Arrow at the 25/50/75% windows, with
and without split-KV — is the single-head call host- or device-bound?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

NV, NT, D, B = 4096, 512, 64, 128
N = NV + NT
dims = api.AttentionDims(1, D, NV, NT)
q, k, v = (torch.randn(N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3, (h1 - h0) / n * 1e6


for split in (True, False):
    api.set_split_kv(split)
    d_us, dh = t(lambda: api.dense_tiled_attention(q, k, v, out=out))
    print(f"split={split} dense: device {d_us:.1f} us/call, host {dh:.1f} us/call", flush=True)
    for w in (13, 6, 0):
        m = api.build_arrow_mask(api.ArrowSpec(dims, B, w))
        s_us, sh = t(lambda: api.sparse_attention_forward(q, k, v, m, out=out))
        print(f"   w={w:2d} sparsity {api.sparsity_ratio(m):.3f}: device {s_us:.1f} us, host {sh:.1f} us, "
              f"speedup {d_us / s_us:.2f}", flush=True)
api.set_split_kv(False)
