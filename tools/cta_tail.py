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

SD3 = "--sd3" in sys.argv
H, NV, NT, D, B = (24, 4096, 333, 64, 128) if SD3 else (24, 16384, 512, 128, 128)
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
cache = api.HeadCache(1, H, N, D)
for h in range(H):
    cache.store(0, h, torch.randn(N, D, device="cuda").to(torch.bfloat16), 0)
plans = [a for a in sys.argv[1:] if not a.startswith("--")] or ["FLUX68", "F", "A8", "A0"]
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
    print(f"{'SD3 ' if SD3 else ''}{name:7s} launch span {end.max() / 1e3:.1f} us | CTA start max {start.max() / 1e3:.1f} us | "
          f"CTA end: mean {end.mean() / 1e3:.1f} p10 {np.percentile(end, 10) / 1e3:.1f} "
          f"p50 {np.median(end) / 1e3:.1f} p90 {np.percentile(end, 90) / 1e3:.1f} max {end.max() / 1e3:.1f} us | "
          f"tail (max - mean) {(end.max() - end.mean()) / end.max() * 100:.1f}%", flush=True)

if "--items" in sys.argv:
    # per-item durations on the latest plan: lane A's start of item i to its
    # start of the next item on the same CTA (the last item: to the CTA end)
    name = plans[-1]
    p = api.flux68_plan() if name == "FLUX68" else api.LayerPlan.parse(" ".join([name] * H))
    trace = torch.zeros(148 * 4 + 8192 * 4, dtype=torch.int64, device="cuda")
    _lib.lib().dfa2c_debug_set_trace(ctypes.c_void_p(trace.data_ptr()))
    api.multi_strategy_attention(q, k, v, p, cache, 0, 1, dims, B, out=out)
    torch.cuda.synchronize()
    _lib.lib().dfa2c_debug_set_trace(None)
    t = trace.cpu().numpy()
    cta = t[:148 * 4].reshape(148, 4)
    it = t[148 * 4:].reshape(8192, 4)
    n_items = int((it[:, 0] > 0).sum())
    it = it[:n_items]
    rows = []
    for c in range(148):
        idx = np.where(it[:, 2] == c)[0]
        idx = idx[np.argsort(it[idx, 0])]
        for j, i in enumerate(idx):
            end = it[idx[j + 1], 0] if j + 1 < len(idx) else cta[c, 3]
            info = int(it[i, 1])
            rows.append((c, int(info & 0xFFFF), (info >> 16) & 0x3FFF, bool(info >> 30 & 1), (end - it[i, 0]) / 1e3))
    import collections
    kinds = collections.defaultdict(list)
    for c, nt, fl, single, us in rows:
        kinds[(nt, fl, single)].append(us)
    print(f"{name}: item kinds (n_tiles, flags, single-lane): count, mean us, max us, us per union tile")
    for key in sorted(kinds, key=lambda x: -x[0]):
        v_ = kinds[key]
        print(f"  {key}: {len(v_):4d}  {np.mean(v_):7.2f}  {np.max(v_):7.2f}  {np.mean(v_) / max(key[0], 1):6.3f}")
    ends = cta[:, 3] - cta[cta[:, 0] > 0, 0].min()
    worst = int(np.argmax(np.where(cta[:, 0] > 0, ends, 0)))
    print(f"  slowest CTA {worst}: " + ", ".join(f"{nt}t/f{fl}{'/1' if sg else ''}:{us:.1f}"
                                                 for c, nt, fl, sg, us in rows if c == worst))
