"""Per-tile timeline of CTA 0 from a -DDFA2_TRACE=1 build (cycles, medians).

    python -m paper_2503_22796_b200.build --out /tmp/libtrace.so -DDFA2_TRACE=1
    DFA2_LIB=/tmp/libtrace.so python tools/trace_tiles.py [plan]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_22796_b200 import _lib, api

plan = sys.argv[1] if len(sys.argv) > 1 else "F"
sd3 = "--sd3" in sys.argv
H, NV, NT, D, B = (24, 4096, 333, 64, 128) if sd3 else (24, 16384, 512, 128, 128)
N = NV + NT
dims = api.AttentionDims(H, D, NV, NT)
q, k, v = (torch.randn(1, H, N, D, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
lp = api.LayerPlan.parse(" ".join([plan] * H) if len(plan.split()) == 1 else plan)
trace = torch.zeros(2 * 4096 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B, out=out)
_lib.lib().dfa2c_debug_set_trace(ctypes_ptr := __import__("ctypes").c_void_p(trace.data_ptr()))
api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B, out=out)
torch.cuda.synchronize()
_lib.lib().dfa2c_debug_set_trace(None)
t = trace.view(2, 4096, 8).cpu().numpy()
for L in range(2):
    n = int((t[L, :, 1] > 0).sum())
    x = t[L, :n].astype(np.float64)
    if n < 3:
        continue
    wait = x[:, 1] - x[:, 0]
    soft = x[:, 2] - x[:, 1]
    pseen = x[:, 3] - x[:, 2]                    # P(j) arrive -> MMA warp sees it
    period = np.diff(x[:, 1])
    med = lambda a: float(np.median(a))
    extra = ""
    if (x[:, 4] > 0).all() and (x[:, 5] > 0).all():
        extra = (f"  PV issue {med(x[:, 4] - x[:, 3]):.0f}  PV->S issue {med(x[1:, 5] - x[:-1, 4]):.0f}  "
                 f"S issue->ready {med(x[1:, 1] - x[1:, 5]):.0f}")
    if os.environ.get("DFA2_TRACE_MODE") == "2":
        d = lambda a_, b_: med(x[:, b_] - x[:, a_])
        extra = (f"\n   softmax detail: ld+wait {d(1, 3):.0f}  max+decide {d(3, 4):.0f}  P(hi) {d(4, 5):.0f}  "
                 f"st.wait+arrive {d(5, 6):.0f}  reload lo {d(6, 7):.0f}  P(lo)+st+arrive {d(7, 2):.0f}")
    elif (x[:, 6] > 0).sum() > 3 and (x[:, 7] > 0).sum() > 3:
        # MMA warp (TRACE=1), per lane tile j: 7 = V(j) ready, 3 = P(j) half seen, 4 = PV(j) issued,
        # 6 = K(j) ready (before S(j) issue), 5 = S(j) issued
        extra += (f"\n   MMA warp: V ready->P seen {med(x[:, 3] - x[:, 7]):.0f}  "
                  f"PV(j-1) issued->K(j) ready {med(x[1:, 6] - x[:-1, 4]):.0f}  K ready->S issued {med(x[:, 5] - x[:, 6]):.0f}")
    if os.environ.get("DFA2_TRACE_PCT"):
        pct = lambda a: "/".join(f"{np.percentile(a, p_):.0f}" for p_ in (50, 90, 99))
        extra += f"\n   p50/p90/p99: wait_S {pct(wait)}  softmax {pct(soft)}  period {pct(period)}  total {x[-1, 2] - x[0, 0]:.0f} clk"
    print(f"lane {L}: tiles {n}  period {med(period):.0f}  softmax {med(soft):.0f}  wait_S {med(wait):.0f}  "
          f"P->MMA {med(pseen):.0f}" + extra)
