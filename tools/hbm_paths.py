"""HBM-bound paths on one B200: the calibration RSE kernel and the
cached-head copy-back, timed alone (CUDA events, back-to-back launches,
inputs >> L2).

    python tools/hbm_paths.py [--out gpurun_out/hbm.json] [--ncu]

  rse   dfa2c_rse_async over a FLUX layer (24 heads x [16896, 128]) for
        bf16 and f32 operands, standard and literal numerators.
        Algorithmic bytes = 2 operands x H x N x d x elem.
  copy  dfa2c_mha_forward with every head Cached (FLUX shape): the fused
        kernel's copy items alone. Algorithmic bytes = 2 x H x N x d x 2
        (slot read + out write).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/hbm.json")
ap.add_argument("--ncu", action="store_true", help="few launches, for profiler captures")
args = ap.parse_args()

H, NV, NT, D, B = 24, 16384, 512, 128, 128
N = NV + NT
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    peak = 6460.5
steps, warm = (3, 2) if args.ncu else (30, 5)


def randn(seed, *shape, dtype=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(*shape, device="cuda", generator=g).to(dtype)


def timed(fn):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


res = {"hbm_peak_gbs": peak}
for dt, name in ((torch.bfloat16, "bf16"), (torch.float32, "f32")):
    a, b = randn(7, H, N, D, dtype=dt), randn(8, H, N, D, dtype=dt)
    out = torch.empty(H, device="cuda", dtype=torch.float64)
    for mode, mname in ((api.RseMode.standard, "standard"), (api.RseMode.literal, "literal")):
        ms = timed(lambda: api.rse_per_head_async(a, b, out, mode))
        nbytes = 2 * a.numel() * a.element_size()
        res[f"rse_{name}_{mname}"] = {"ms": ms, "bytes": nbytes, "gbs": nbytes / ms / 1e6,
                                      "frac": nbytes / ms / 1e6 / peak}
        print(f"rse {name} {mname}: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s", flush=True)
    del a, b

dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (randn(s, 1, H, N, D) for s in (1, 2, 3))
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, randn(100 + h, N, D), 0)
o = torch.empty_like(q)
plan = api.LayerPlan.parse(" ".join(["C"] * H))
ms = timed(lambda: api.multi_strategy_attention(q, k, v, plan, cache, 0, 1, dims, B, out=o))
nbytes = 2 * H * N * D * 2
res["cached_copy_layer"] = {"ms": ms, "bytes": nbytes, "gbs": nbytes / ms / 1e6, "frac": nbytes / ms / 1e6 / peak}
print(f"all-Cached layer: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s", flush=True)
ms = timed(lambda: o.copy_(q))
res["torch_copy_same_bytes"] = {"ms": ms, "gbs": nbytes / ms / 1e6}
print(f"torch copy (same bytes): {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s", flush=True)

os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
with open(args.out, "w") as f:
    json.dump(res, f, indent=1)
