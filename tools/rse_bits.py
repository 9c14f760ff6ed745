"""Prints per-head RSE values (bf16 operands) with full precision for
cases that exercise the bf16 fast path's exactness guard: ordinary values,
zeros, denormals, huge exponent gaps. Run under two builds and diff."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_22796_b200 import api

g = torch.Generator(device="cuda").manual_seed(5)
H, n = 6, 16896 * 128
yo = torch.randn(H, n, device="cuda", generator=g)
ym = yo + 0.03 * torch.randn(H, n, device="cuda", generator=g)
yo[1, ::97] = 0.0                       # zeros
ym[2, ::89] = 1e-39                     # bf16 denormals
ym[3, ::101] *= 2.0 ** 20               # exponent gaps > 15
yo[4, ::103] = 2.0 ** -60               # tiny references
yo[5, 0] = 3.0e-39                      # a denormal shift K
yo, ym = yo.to(torch.bfloat16), ym.to(torch.bfloat16)
for mode in (api.RseMode.standard, api.RseMode.literal):
    v = api.rse_per_head(ym.view(H, -1), yo.view(H, -1), mode)
    print(mode, " ".join(repr(float(x)) for x in v))
