"""Strong-scaling compute of the row-sharded FLUX68 layer, emulated on ONE GPU.

Every rank r of `world` runs exactly the launch dfa2c_mha_forward_sharded
issues on its own GPU (same plan, same row range, comm = None so no gather);
timing each rank's launch alone on this device gives the per-GPU compute time
at world = 1, 2, 4, 8 (max over ranks), against the ideal t(1)/world.

    python tools/shard_emulation.py [--out gpurun_out/shard_emulation.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

H, NV, NT, D, B = 24, 16384, 512, 128, 128
N = NV + NT
PLAN = "F A8 C A0 F A8 C A8 F A8 C A0 F A8 C A0 F A8 C A8 F A8 C A0"


def run(worlds=(1, 2, 4, 8), steps=20, warm=5):
    dims = api.AttentionDims(H, D, NV, NT)
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v = (torch.randn(1, H, N, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    cache = api.HeadCache(1, H, N, D)
    for h in range(H):
        cache.store(0, h, torch.randn(N, D, device="cuda", generator=g).to(torch.bfloat16), 0)
    plan = api.LayerPlan.parse(PLAN)
    out = torch.empty_like(q)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {"workload": "FLUX68 layer (BASELINE configs[2]) row-sharded, each rank's launch timed alone on one B200",
           "ideal": "t(world=1) / world", "worlds": {}}
    t1 = None
    for world in worlds:
        per_rank = []
        for r in range(world):
            call = lambda: api.multi_strategy_attention_sharded(q, k, v, plan, cache, 0, 1, dims, B, r, world,
                                                                out=out)
            for _ in range(warm):
                call()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(steps):
                call()
            e1.record()
            torch.cuda.synchronize()
            per_rank.append(e0.elapsed_time(e1) / steps)
        mx = max(per_rank)
        if world == 1:
            t1 = mx
        res["worlds"][str(world)] = {"per_rank_ms": per_rank, "max_ms": mx, "ideal_ms": t1 / world,
                                     "ratio_to_ideal": mx / (t1 / world)}
        print(f"world {world}: per-rank compute max {mx:.4f} ms (ideal {t1 / world:.4f}, "
              f"x{mx / (t1 / world):.2f}); ranks {[round(x, 4) for x in per_rank]}", flush=True)
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/shard_emulation.json")
    a = ap.parse_args()
    r = run()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(r, open(a.out, "w"), indent=1)
