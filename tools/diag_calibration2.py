"""Phase timing of api.calibrate_model at FLUX scale (57 layers x 2 timesteps)."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

from paper_2503_22796_b200 import api

L, H, nv, nt, d, B, T = 57, 24, 16384, 512, 128, 128, 2
n = nv + nt
dims = api.AttentionDims(H, d, nv, nt)
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
qs = [q, (q.float() + 0.05 * torch.randn(H, n, d, device="cuda", generator=g)).to(torch.bfloat16)]
cfg = api.CalibrationConfig(api.make_candidates([0, 2, 8, 16, 32], include_cached=True), 0.4, 1.5)
import subprocess


def clocks():
    q_ = ("clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.hw_slowdown,"
          "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")
    return subprocess.run(["nvidia-smi", f"--query-gpu={q_}", "--format=csv,noheader"], capture_output=True,
                          text=True).stdout.strip()


for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = api.calibrate_model(lambda t, l: qs[t], lambda t, l: k, lambda t, l: v, dims, T, L, B, cfg)
    mid = clocks()
    torch.cuda.synchronize()
    print(f"calibrate_model rep {rep}: {(time.perf_counter() - t0) / (T * L) * 1e3:.2f} ms/layer | {mid}", flush=True)
    del r
# phases, by hand
cache = api.HeadCache(L, H, n, d)
strategies = [m.strategy for m in cfg.methods]
costs = api.analytic_costs(dims, B, strategies)
tp = {"influence": 0.0, "solve": 0.0, "splice": 0.0}
for t in range(T):
    for l in range(L):
        torch.cuda.synchronize(); a = time.perf_counter()
        li = api.influence_for_layer(qs[t], k, v, cfg.methods, cache, l, t, dims, B, keep_outputs=True)
        torch.cuda.synchronize(); b = time.perf_counter()
        sol = api.solve(api.PlanProblem(H, len(cfg.methods), li.influence, costs, 0.4, 1.5))
        c = time.perf_counter()
        for h, ch in enumerate(sol.choice):
            if ch == api.kFullChoice:
                cache.store(l, h, li.original[h], t)
            elif strategies[ch].kind == "arrow":
                cache.store(l, h, li.method_outputs[ch][h], t)
        torch.cuda.synchronize(); e = time.perf_counter()
        tp["influence"] += b - a; tp["solve"] += c - b; tp["splice"] += e - c
print({k_: f"{v_ / (T * L) * 1e3:.2f} ms/layer" for k_, v_ in tp.items()})
