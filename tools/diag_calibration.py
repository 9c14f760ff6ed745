import time, sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2503_22796_b200 import api
L, H, nv, nt, d, B = 57, 24, 16384, 512, 128, 128
n = nv + nt
dims = api.AttentionDims(H, d, nv, nt)
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
methods = api.make_candidates([0, 2, 8, 16, 32], include_cached=True)
cache = api.HeadCache(L, H, n, d)
for l in range(L):
    api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, l, 0, dims, B)
torch.cuda.synchronize()
for keep in (False, True):
    for rep in range(2):
        t0 = time.perf_counter()
        for l in range(L):
            li = api.influence_for_layer(q, k, v, methods, cache, l, 1, dims, B, keep_outputs=keep)
        torch.cuda.synchronize()
        print(f"influence x57 keep_outputs={keep}: {(time.perf_counter()-t0)/L*1e3:.2f} ms/layer", flush=True)
t0 = time.perf_counter()
for l in range(L):
    for h in range(H):
        cache.store(l, h, q[h], 1)
torch.cuda.synchronize()
print(f"cache.store x24 per layer: {(time.perf_counter()-t0)/L*1e3:.2f} ms/layer")
# the solve step on the measured grids of t = 1
costs = api.analytic_costs(dims, B, [m.strategy for m in methods])
tot_nodes, t_solve = 0, 0.0
for l in range(L):
    li = api.influence_for_layer(q, k, v, methods, cache, l, 1, dims, B, keep_outputs=False)
    t0 = time.perf_counter()
    sol = api.solve(api.PlanProblem(H, len(methods), li.influence, costs, 0.4, 1.5))
    t_solve += time.perf_counter() - t0
    tot_nodes += sol.nodes
print(f"solve: {t_solve / L * 1e3:.2f} ms/layer, {tot_nodes / L:.0f} nodes/layer")
