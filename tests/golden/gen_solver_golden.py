"""Generates tests/golden/solver_golden.json from the REFERENCE ITSELF:
seeded per-layer selection problems (H heads x M methods; +inf ineligible
entries, quantised values so cost/influence ties occur, delta = 0 and
binding per-selection caps) with the reference's solve() / brute_force() /
lp_relaxation_bound() answers (/root/reference/proj/src/plansolver.cpp via
oracle/ref_capi.cpp).

    make -C oracle all ref && python tests/golden/gen_solver_golden.py
"""
import ctypes
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402
from oracle import c_double, c_int64, ptr, ref  # noqa: E402


def ref_solve(H, M, infl, full, mcost, delta, coeff, brute):
    choice = np.zeros(H, np.int64)
    obj, tot, lp = c_double(), c_double(), c_double()
    a = np.ascontiguousarray(infl, np.float64)
    c = np.ascontiguousarray(mcost if M else [0.0], np.float64)
    oracle.ref_check(ref().ref_plan_solve(H, M, ptr(a, c_double), full, ptr(c, c_double), delta, coeff, brute,
                                          ptr(choice, c_int64), ctypes.byref(obj), ctypes.byref(tot),
                                          ctypes.byref(lp)))
    return choice.tolist(), obj.value, tot.value, lp.value


def main():
    rng = np.random.default_rng(96)
    cases = []
    for i in range(160):
        H = int(rng.integers(1, 25 if i >= 40 else 7))
        M = int(rng.integers(0, 8))
        quant = i % 3 == 0
        mcost = np.sort(rng.random(M))[::-1] if M else np.zeros(0)
        if quant:
            mcost = np.round(mcost * 4) / 4
        if M and i % 5 == 0:
            mcost[-1] = 0.0  # a Cached-like free method
        infl = rng.gamma(0.7, 0.08, size=(H, M)) * (np.arange(M) + 1) / max(M, 1)
        if quant:
            infl = np.round(infl * 20) / 20
        infl[rng.random((H, M)) < 0.12] = math.inf
        delta = [0.0, 0.05, 0.1, 0.4, 1.0, 3.0][i % 6]
        coeff = [1.0, 1.5, 2.0, 8.0][(i // 6) % 4]
        brute_ok = (M + 1) ** H <= 200000
        sol = ref_solve(H, M, infl.ravel(), 1.0, mcost, delta, coeff, 0)
        case = {"H": H, "M": M, "influence": [x if math.isfinite(x) else "inf" for x in infl.ravel().tolist()],
                "full_cost": 1.0, "method_cost": mcost.tolist(), "delta": delta, "coeff": coeff,
                "choice": sol[0], "objective": sol[1], "total_influence": sol[2], "lp_bound": sol[3]}
        if brute_ok:
            b = ref_solve(H, M, infl.ravel(), 1.0, mcost, delta, coeff, 1)
            case["brute_choice"] = b[0]
        cases.append(case)
    with open(os.path.join(HERE, "solver_golden.json"), "w") as f:
        json.dump(cases, f)
    print(len(cases), "cases;", sum("brute_choice" in c for c in cases), "with brute force")


if __name__ == "__main__":
    main()
