"""Where a FLUX-layer calibration step's time goes: calibrate_model wall time
per layer vs the GPU time of its work enqueued back to back (the fused
influence pass + RSE grid per layer), and the host time of each driver phase."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

L, T, H, nv, nt, d, B = 12, 2, 24, 16384, 512, 128, 128
dims = api.AttentionDims(H, d, nv, nt)
wl = api.DeviceWorkload(dims, L, B, seed=2503)
memo = {(t, l): wl.slot(t, l) for t in range(T) for l in range(L)}
torch.cuda.synchronize()
cfg = api.CalibrationConfig(api.make_candidates([0, 2, 8, 16, 32], include_cached=True), 0.4, 1.5)
sl = lambda i: (lambda t, l: memo[(t, l)][i])  # noqa: E731
api.calibrate_model(sl(0), sl(1), sl(2), dims, 1, 2, B, cfg)  # warm-up (plans, buffers)
torch.cuda.synchronize()
t0 = time.perf_counter()
r = api.calibrate_model(sl(0), sl(1), sl(2), dims, T, L, B, cfg)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / (T * L)
# the same GPU work back to back: one influence launch per (t, l) with a cache
cache = api.HeadCache(L, H, nv + nt, d)
for l in range(L):
    for h in range(H):
        cache.store(l, h, memo[(0, l)][0][h], 0)
stats = api.CalibrationStats()
bufs = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
pend = [api._influence_launch(*memo[(1, 0)], cfg.methods, cache, 0, 1, dims, B, cfg.rse_mode, stats, bufs)]
torch.cuda.synchronize()
h0 = time.perf_counter()
e0.record()
host_launch = 0.0
for l in range(L):
    a = time.perf_counter()
    p = api._influence_launch(*memo[(1, l)], cfg.methods, cache, l, 1, dims, B, cfg.rse_mode, stats, bufs)
    host_launch += time.perf_counter() - a
e1.record()
torch.cuda.synchronize()
gpu = e0.elapsed_time(e1) / L
print(f"calibrate_model: {wall * 1e3:.3f} ms per layer (T={T}, L={L}); GPU work alone: {gpu:.3f} ms per layer; "
      f"host enqueue of one influence step: {host_launch / L * 1e3:.3f} ms", flush=True)
# host solve + splice time
t1 = time.perf_counter()
for _ in range(20):
    li = p.finish()
    sol = api.solve(api.PlanProblem(H, len(cfg.methods), li.influence,
                                    api.analytic_costs(dims, B, [m.strategy for m in cfg.methods]), 0.4, 1.5))
solve_ms = (time.perf_counter() - t1) / 20 * 1e3
t2 = time.perf_counter()
for _ in range(5):
    for h in range(H):
        cache.store(0, h, li.original[h], 1)
torch.cuda.synchronize()
splice_ms = (time.perf_counter() - t2) / 5 * 1e3
print(f"host: finish + solve {solve_ms:.3f} ms, splice (24 cache.store + sync) {splice_ms:.3f} ms", flush=True)
