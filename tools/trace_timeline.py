"""Absolute per-tile event timeline of CTA 0, both lanes interleaved, from a
-DDFA2_TRACE=1 build (see trace_tiles.py): shows the lanes' phase relation.

    DFA2_LIB=build/lt1.so python tools/trace_timeline.py [plan] [first_tile] [count]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_22796_b200 import _lib, api

plan = sys.argv[1] if len(sys.argv) > 1 else "F"
j0 = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cnt = int(sys.argv[3]) if len(sys.argv) > 3 else 6
sd3 = "--sd3" in sys.argv
H, NV, NT, D, B = (24, 4096, 333, 64, 128) if sd3 else (24, 16384, 512, 128, 128)
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
lp = api.LayerPlan.parse(" ".join([plan] * H) if len(plan.split()) == 1 else plan)
trace = torch.zeros(4 * 4096 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B, out=out)
_lib.lib().dfa2c_debug_set_trace(ctypes.c_void_p(trace.data_ptr()))
api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B, out=out)
torch.cuda.synchronize()
_lib.lib().dfa2c_debug_set_trace(None)
t = trace.view(4, 4096, 8).cpu().numpy().astype(np.int64)
names = {0: "sm.wait", 1: "S ready", 2: "sm.end(P)", 3: "mma:Phalf", 4: "mma:PVissued", 5: "mma:Sissued",
         6: "mma:Kready", 7: "mma:Vready"}
ev = []
base = t[0, j0, 1]
for L in range(2):
    for j in range(j0, j0 + cnt):
        for s, nm in names.items():
            if t[L, j, s] > 0:
                ev.append((int(t[L, j, s] - base), "AB"[L], j, nm))
pn = {0: "prod:Kwait", 1: "prod:Kissue", 2: "prod:Vwait", 3: "prod:Vissue"}
for j in range(j0, j0 + cnt):
    for s_, nm in pn.items():
        if t[2, j, s_] > 0:
            ev.append((int(t[2, j, s_] - base), "P", j, nm))
mn = {0: "mma:Vwait(A)", 1: "mma:step commits", 2: "mma:step done"}
for j in range(j0, j0 + cnt):
    for s_, nm in mn.items():
        if t[3, j, s_] > 0:
            ev.append((int(t[3, j, s_] - base), "M", j, nm))
ev.sort()
for e in ev:
    print(f"{e[0]:8d}  {e[1]}{e[2]:<5d} {e[3]}")
