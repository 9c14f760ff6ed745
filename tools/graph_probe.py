"""CUDA-graph capture of layer calls (after one plain call built each work
list): replay bits vs direct calls, and per-layer time direct vs replayed for
a host-bound layer (SD3 all-Cached: 27 MB of copies) and a GPU-bound one.

    python tools/graph_probe.py [global|thread_local|relaxed]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

mode = sys.argv[1] if len(sys.argv) > 1 else "global"


def case(name, H, NV, NT, D, plan, n_layers=8):
    N = NV + NT
    dims = api.AttentionDims(H, D, NV, NT)
    q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
    outs = [torch.empty_like(q) for _ in range(n_layers)]
    cache = api.HeadCache(n_layers, H, N, D)
    full = api.LayerPlan.all_full(H)
    lp = api.LayerPlan.parse(plan)
    for l in range(n_layers):  # t = 0 fills every layer's cache; t = 1 builds the plan
        api.multi_strategy_attention(q, k, v, full, cache, l, 0, dims, 128, out=outs[l])
        api.multi_strategy_attention(q, k, v, lp, cache, l, 1, dims, 128, out=outs[l])
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs]

    def step():
        for l in range(n_layers):
            api.multi_strategy_attention(q, k, v, lp, cache, l, 1, dims, 128, out=outs[l])

    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream(), capture_error_mode=mode):
        step()
    for o in outs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(outs, ref))
    times = {}
    for tag, fn in (("direct", step), ("graph", g.replay)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        torch.cuda.synchronize()
        times[tag] = e0.elapsed_time(e1) / 50 / n_layers * 1e3
    print(f"{name:28s} replay bitwise equal: {same}; per layer: direct {times['direct']:.1f} us, "
          f"graph {times['graph']:.1f} us", flush=True)


case("cfg1 [F A0 A2 C]", 4, 1024, 77, 64, "F A0 A2 C")
case("SD3 all-Cached", 24, 4096, 333, 64, " ".join(["C"] * 24))
case("SD3 all-Arrow(0)", 24, 4096, 333, 64, " ".join(["A0"] * 24))
