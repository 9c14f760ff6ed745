"""Interleaved A/B of prebuilt library variants in ONE process: every
variant's launches alternate round by round on the same inputs, so the
power-capped clock's drift hits all of them alike (separate bench runs on
these boxes scatter by +-2-4%, more than most kernel changes).

    python tools/ab_interleaved.py build/ab_base.so build/ab_x.so ... [--rounds 12] [--steps 10]

Prints, per plan, each variant's median ms over the rounds and its ratio to
the first variant.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_22796_b200 import _lib, api

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--rounds", type=int, default=12)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--plans", default="FLUX68,flux_F,flux_A8,sd3_F,sd3_A8,sd3_A2,sd3_A0")
a = ap.parse_args()

FLUX68 = "F A8 C A0 F A8 C A8 F A8 C A0 F A8 C A0 F A8 C A8 F A8 C A0"
SHAPES = {"flux": (24, 16384, 512, 128), "sd3": (24, 4096, 333, 64)}
B = 128


MIXED = {  # a late-timestep layer: most heads Cached, a few narrow arrows (latency-bound)
    "LATE": " ".join((["C"] * 5 + ["A0"]) * 4),
}


def plan_of(name, H):
    if name == "FLUX68":
        return "flux", FLUX68
    if name in MIXED:
        return "flux", MIXED[name]
    shape, kind = name.split("_")
    return shape, " ".join([kind] * H)


variants = []
for path in a.libs:
    _lib._lib = None
    _lib.LIB_PATH = os.path.abspath(path)
    L = _lib.lib()
    caches = {}
    for shape, (H, NV, NT, D) in SHAPES.items():
        c = api.HeadCache(1, H, NV + NT, D)
        g = torch.Generator(device="cuda").manual_seed(7)
        for h in range(H):
            c.store(0, h, torch.randn(NV + NT, D, device="cuda", generator=g).to(torch.bfloat16), 0)
        caches[shape] = c
    variants.append((os.path.basename(path), L, caches))

inputs = {}
for shape, (H, NV, NT, D) in SHAPES.items():
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v = (torch.randn(1, H, NV + NT, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    inputs[shape] = (q, k, v, torch.empty_like(q), api.AttentionDims(H, D, NV, NT))

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for pname in a.plans.split(","):
    shape, pstr = plan_of(pname, 24)
    q, k, v, out, dims = inputs[shape]
    lp = api.LayerPlan.parse(pstr)
    fl = api.plan_flops(lp, dims, B)
    times = {name: [] for name, _, _ in variants}
    outs = {}
    for rnd in range(a.rounds + 1):
        for name, L, caches in variants:
            _lib._lib = L
            for _ in range(2):
                api.multi_strategy_attention(q, k, v, lp, caches[shape], 0, 1, dims, B, out=out)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.steps):
                api.multi_strategy_attention(q, k, v, lp, caches[shape], 0, 1, dims, B, out=out)
            e1.record()
            torch.cuda.synchronize()
            if rnd > 0:  # round 0 warms every variant up
                times[name].append(e0.elapsed_time(e1) / a.steps)
            if rnd == a.rounds:
                outs[name] = out.clone()
    ref = None
    line = []
    for name, _, _ in variants:
        med = float(np.median(times[name]))
        ref = ref or med
        same = torch.equal(outs[name], outs[variants[0][0]])
        line.append(f"{name} {med * 1e3:7.1f} us ({med / ref:5.3f}{'' if same else ' DIFF'})")
    print(f"{pname:8s} {fl / 1e9:7.1f} GF | " + " | ".join(line), flush=True)
